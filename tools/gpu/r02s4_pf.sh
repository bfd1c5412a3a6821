timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_failover_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 0 1; do echo "== FS_GEMM_NO_L2_PREFETCH=$v"
for w in 8 5; do FS_GEMM_NO_L2_PREFETCH=$v timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_GEMM_NO_L2_PREFETCH=$v timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
for v in 0 1; do FS_GEMM_NO_L2_PREFETCH=$v timeout 300 python tools/c3_step.py --world 8 --time 2>&1 | tail -1; done
