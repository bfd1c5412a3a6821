python -m pytest tests/test_decode_gpu.py tests/test_config_parity_gpu.py tests/test_exchange_gpu.py -x -q 2>&1 | tail -3
for st in 65536 49152 40000; do
FS_DECODE_TAIL_STATIC=$st python bench.py --skip-mixed --skip-recovery --skip-cpu > gpurun_out/b_$st.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b_$st.json').read().strip().splitlines()[-1])
fs=d['failure_states']
print('$st', d['value'], d['roofline']['frac'], [(s['world'], s['tok_s'], s['attn_frac_min']) for s in fs['states']])"
done
