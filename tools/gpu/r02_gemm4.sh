python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/gemm_coresidence.py 3584 8192; python tools/gemm_coresidence.py 8192 1280
timeout 300 python tools/gemm_bw.py 2>&1 | grep -v "^$"
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
