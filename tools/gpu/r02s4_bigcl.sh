# GEMM: non-portable clusters (split counts above 8) via FS_GEMM_MAX_SPLITS
FS_GEMM_MAX_SPLITS=16 timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
FS_GEMM_MAX_SPLITS=16 python -c "
import torch
from paper_2511_14116_b200 import _native as N
for K, n in [(8192, 1280), (8192, 2560), (4096, 6144), (8192, 1536), (1024, 8192), (8192, 7168)]:
    print(K, n, 'splits', N.lib.fs_gemm_plan(0, K, n, 1))
"
run() { echo "== $1"; for w in 8 7 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_GEMM_MAX_SPLITS=8 FS_GEMM_MAX_SPLITS=10 FS_GEMM_MAX_SPLITS=12 FS_GEMM_MAX_SPLITS=14 FS_GEMM_MAX_SPLITS=16 FS_GEMM_MAX_SPLITS=8; do run "$v"; done
