mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
tail -c 600 gpurun_out/bench_full.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])
fs=d.get('failure_states',{}); print([(s['world'], s['tok_s'], s['attn_frac_min'], s['step_frac_max_rank'], s.get('vs_8_scaled')) for s in fs.get('states',[])])
print('mixed', d.get('mixed_trace',{}).get('tok_s'))
print(json.dumps(d.get('cost_calibration'), indent=0)[:3000])
print(json.dumps(d.get('recovery'), indent=0)[:2000])
print(json.dumps(d.get('cpu_baseline')))
"
