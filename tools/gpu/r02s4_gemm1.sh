mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 600 python tools/gemm_bw.py all 2>&1 | grep -v "^$"
for w in 8 5; do for b in tcgen05 cublas; do timeout 300 python tools/c3_step.py --world $w --gemm $b --time 2>&1 | tail -1; done; done
for b in tcgen05 cublas; do timeout 300 python tools/c3_step.py --model 8b --world 1 --gemm $b --time 2>&1 | tail -1; done
