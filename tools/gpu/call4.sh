mkdir -p gpurun_out
python tools/shm_register_bench.py 8 2>&1 | tail -2
FS_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 --failures 3,1 --chain-layers 2 > gpurun_out/chain4.json 2> gpurun_out/chain4.err; echo rc=$?
tail -c 4000 gpurun_out/chain4.json; tail -20 gpurun_out/chain4.err
