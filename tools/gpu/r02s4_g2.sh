timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_cluster_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
FS_BENCH_SHARED_GPU=1 timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29527 bench.py --gpus 2 --steps 5 --warmup 3 --failures 1 --chain-layers 8 > gpurun_out/chain2.json 2> gpurun_out/chain2.err; echo chain2 rc=$?
tail -c 1500 gpurun_out/chain2.json
