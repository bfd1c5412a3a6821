# GEMM split cap (FS_GEMM_MAX_SPLITS), optionally only for launches with < FS_GEMM_CAP_GROUPS column groups
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_GEMM_MAX_SPLITS=8 FS_GEMM_MAX_SPLITS=6 FS_GEMM_MAX_SPLITS=4 "FS_GEMM_MAX_SPLITS=4 FS_GEMM_CAP_GROUPS=16" \
         "FS_GEMM_MAX_SPLITS=5 FS_GEMM_CAP_GROUPS=16" "FS_GEMM_MAX_SPLITS=2 FS_GEMM_CAP_GROUPS=16" FS_GEMM_MAX_SPLITS=8; do run "$v"; done
