# K1: each CTA sends its slice of the O projection's weights to L2 once its pages are done
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_config_parity_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_K1_L2_NEXT=0 FS_K1_L2_NEXT=1 FS_K1_L2_NEXT=0 FS_K1_L2_NEXT=1; do run "$v"; done
