mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -15 gpurun_out/gputest.log
python tools/prefill_bench.py --variant 3 2>&1 | tail -6
python bench.py --skip-failure-states --skip-mixed --skip-recovery --skip-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['launch_ms'])"
