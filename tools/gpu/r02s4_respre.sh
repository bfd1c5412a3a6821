# GEMM residual epilogue: first round's residual loaded before the accumulator is ready (FS_GEMM_RES_PRELOAD)
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_knobs_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_config_parity_gpu.py -x -q -p no:cacheprovider -k "full_layer or whole" 2>&1 | tail -1
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_GEMM_RES_PRELOAD=0 FS_GEMM_RES_PRELOAD=1 FS_GEMM_RES_PRELOAD=0 FS_GEMM_RES_PRELOAD=1; do run "$v"; done
