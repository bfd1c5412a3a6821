timeout 300 python tools/gemm_tl.py 1024 8192 4096 28672 2>&1
