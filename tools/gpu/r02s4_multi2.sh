# N>1 bench path on one GPU (2 processes sharing cuda:0): C2 line + a 2 -> 1 failure chain (8 layers)
mkdir -p gpurun_out
FS_BENCH_SHARED_GPU=1 timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 5 --warmup 3 --failures 1 --chain-layers 8 > gpurun_out/chain2.json 2> gpurun_out/chain2.err; echo chain rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/chain2.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'launches', d['gpu_launches'])
fc=d.get('failure_chain',{}); print(json.dumps(fc)[:1500])
"
tail -3 gpurun_out/chain2.err
