for i in 1 2 3; do python -m pytest tests/test_cluster_gpu.py -x -q 2>&1 | tail -2; done
python -m pytest tests/test_recovery_gpu.py tests/test_config_parity_gpu.py -q --durations=8 2>&1 | tail -14
