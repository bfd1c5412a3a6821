timeout 900 python -m pytest tests/test_decode_gpu.py -x -q -p no:cacheprovider -k "qkv_partials or engine or skew or ragged" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_exchange_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 1 0; do echo "== FS_QKV_PARTIALS=$v"
for w in 8 5; do FS_QKV_PARTIALS=$v timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_QKV_PARTIALS=$v timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
