mkdir -p gpurun_out
python -m pytest tests/test_config_parity_gpu.py -x -q > gpurun_out/cfg_parity.log 2>&1; tail -3 gpurun_out/cfg_parity.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
compute-sanitizer --tool synccheck python -m pytest -x -q -p no:cacheprovider tests/test_prefill_gpu.py::test_prefill_splits > gpurun_out/synccheck_prefill.log 2>&1; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/synccheck_prefill.log
python bench.py --skip-failure-states --skip-mixed --skip-recovery --cpu-layers 2 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -c 3000 gpurun_out/bench_quick.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -c 1500 gpurun_out/bench_ref.json
free -g; df -h /dev/shm; nproc
