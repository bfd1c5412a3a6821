# K1: L2 prefetch of each warp's next pages before griddepcontrol.wait (A/B on one box)
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do
for d in 0 4 8 14 28; do echo "== FS_K1_L2_PREFETCH=$d"
for w in 8 5; do FS_K1_L2_PREFETCH=$d timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_K1_L2_PREFETCH=$d timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done; done
