mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 tools/ubench/stream_probe > gpurun_out/stream_probe.csv 2>&1; echo probe rc=$?
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
bash tools/gpu/bench_full.sh
