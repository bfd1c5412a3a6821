mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu/bench_full.sh
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 python tools/step_trace.py --world 8 > gpurun_out/step_trace_c3n8.txt 2>&1; echo trace rc=$?
timeout 600 python tools/step_trace.py --model 8b --world 1 --layers-shown 1 > gpurun_out/step_trace_c2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_bench.csv python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu --skip-mixed > gpurun_out/launches_bench.log 2>&1; echo launches rc=$?
