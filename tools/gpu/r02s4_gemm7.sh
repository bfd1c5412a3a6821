timeout 300 python tools/gemm_tl.py 1024 8192 3584 8192 2>&1
