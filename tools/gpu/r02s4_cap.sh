for cap in 0 6 4 3; do
for w in 8 5; do FS_GEMM_MAX_SPLITS=$cap timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_GEMM_MAX_SPLITS=$cap timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
