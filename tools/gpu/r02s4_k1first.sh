# K1: deeper pre-wait L2 prefetch for the first CTAs (those that land on SMs the QKV GEMM leaves free)
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done; }
for v in "FS_K1_L2_FIRST_CTAS=0" "FS_K1_L2_FIRST_CTAS=68 FS_K1_L2_FIRST_PAGES=4" "FS_K1_L2_FIRST_CTAS=68 FS_K1_L2_FIRST_PAGES=8" \
         "FS_K1_L2_FIRST_CTAS=68 FS_K1_L2_FIRST_PAGES=14" "FS_K1_L2_FIRST_CTAS=68 FS_K1_L2_FIRST_PAGES=0" \
         "FS_K1_L2_FIRST_CTAS=148 FS_K1_L2_FIRST_PAGES=0" "FS_K1_L2_FIRST_CTAS=0"; do run "$v"; done
