for cfg in "65536 32" "60293 32" "60293 64" "55705 64" "55705 128"; do
set -- $cfg
FS_DECODE_TAIL_STATIC=$1 FS_DECODE_TAIL_CHUNK=$2 python bench.py --skip-mixed --skip-recovery --skip-cpu --steps 10 > gpurun_out/b_t.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b_t.json').read().strip().splitlines()[-1])
fs=d['failure_states']
print('$1 $2', d['value'], d['roofline']['frac'], [(s['world'], s['tok_s'], s['attn_frac_min']) for s in fs['states']])"
done
