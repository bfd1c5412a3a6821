python -m pytest tests/test_failover_gpu.py tests/test_cluster_gpu.py tests/test_serving_gpu.py -x -q 2>&1 | tail -25
