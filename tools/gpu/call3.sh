mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cluster_gpu.py -x -q > gpurun_out/cluster.log 2>&1; tail -60 gpurun_out/cluster.log
