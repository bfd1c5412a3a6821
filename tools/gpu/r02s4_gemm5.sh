timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/gemm_tl.py 1024 8192 8192 1280 3584 8192 2>&1
timeout 600 python tools/gemm_bw.py all 2>&1 | grep -v "^$"
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --model 8b --world 1 --gemm tcgen05 --time 2>&1 | tail -1
