ls /dev/shm | head; df -h /dev/shm | tail -1
FS_BENCH_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 --failures 3,1 --chain-layers 8 > gpurun_out/chain4.json 2> gpurun_out/chain4.err; echo rc=$?
grep -v "^\s*$" gpurun_out/chain4.err | grep -B5 -A25 Traceback | head -60
python -c "
import json; d=json.loads(open('gpurun_out/chain4.json').read().strip().splitlines()[-1]); c=d['failure_chain']
print(json.dumps(c.get('recoveries', c), indent=0)); print([ (s['world'], s['max_rank_step_ms']) for s in c.get('states',[])], c.get('setup_s'))"
ls /dev/shm | head
