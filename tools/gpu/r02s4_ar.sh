timeout 1200 python -m pytest tests/test_exchange_gpu.py tests/test_cluster_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for w in 2 4; do FS_BENCH_SHARED_GPU=1 timeout 300 torchrun --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2961$w tools/ar_bench.py 2>/dev/null | tail -2; done
