mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cluster_gpu.py -x -q > gpurun_out/cluster.log 2>&1; tail -5 gpurun_out/cluster.log
FS_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 --failures 3,1 --chain-layers 8 > gpurun_out/chain4.json 2> gpurun_out/chain4.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/chain4.json').read().strip().splitlines()[-1]); c=d['failure_chain']
print(json.dumps(c.get('recoveries', c), indent=0)); print([ (s['world'], s['max_rank_step_ms']) for s in c.get('states',[])])"
tail -5 gpurun_out/chain4.err
