# GEMM: packed-W stages sent to L2 before griddepcontrol.wait (FS_GEMM_L2_PREFETCH); K1 L2 prefetch default 2
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_K1_L2_PREFETCH=0 FS_GEMM_L2_PREFETCH=0 FS_GEMM_L2_PREFETCH=1 FS_GEMM_L2_PREFETCH=2 FS_GEMM_L2_PREFETCH=4 \
         FS_GEMM_L2_PREFETCH=8 FS_GEMM_L2_PREFETCH=0; do run $v; done
