timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_config_parity_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for d in 0 8 16 24 32; do echo "== FS_K1_HEAD_PAGES=$d"
for w in 8 5; do FS_K1_HEAD_PAGES=$d timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_K1_HEAD_PAGES=$d timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
