timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_config_parity_gpu.py tests/test_exchange_gpu.py tests/test_failover_gpu.py tests/test_cluster_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
