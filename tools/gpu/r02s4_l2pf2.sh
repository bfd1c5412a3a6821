# K1: L2 prefetch before the wait (FS_K1_L2_PREFETCH) and a continuous L2 prefetch distance (FS_K1_L2_AHEAD)
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_K1_L2_PREFETCH=0 FS_K1_L2_PREFETCH=2 FS_K1_L2_PREFETCH=3 FS_K1_L2_PREFETCH=4 FS_K1_L2_PREFETCH=6 \
         FS_K1_L2_AHEAD=2 FS_K1_L2_AHEAD=4 FS_K1_L2_AHEAD=6 FS_K1_L2_AHEAD=10 FS_K1_L2_PREFETCH=0; do run $v; done
