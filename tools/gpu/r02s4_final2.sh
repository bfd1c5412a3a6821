mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
bash tools/gpu/bench_full.sh
FS_BENCH_SHARED_GPU=1 timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29527 bench.py --gpus 2 --steps 5 --warmup 3 --failures 1 --chain-layers 8 > gpurun_out/chain2.json 2> gpurun_out/chain2.err; echo chain2 rc=$?
tail -c 400 gpurun_out/chain2.json
