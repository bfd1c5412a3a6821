mkdir -p gpurun_out
FS_BENCH_SHARED_GPU=1 timeout 900 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 4 --steps 5 --warmup 3 --failures 3,1 --chain-layers 8 > gpurun_out/chain4.json 2> gpurun_out/chain4.err; echo chain rc=$?
tail -c 3000 gpurun_out/chain4.json; tail -5 gpurun_out/chain4.err
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
