for cap in 0 60 48; do echo "== FS_GEMM_MIN_GROUPS_NOSPLIT=$cap"
FS_GEMM_MIN_GROUPS_NOSPLIT=$cap timeout 600 python tools/gemm_bw.py all 2>&1 | grep -v "^$"
for w in 8 5; do FS_GEMM_MIN_GROUPS_NOSPLIT=$cap timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_GEMM_MIN_GROUPS_NOSPLIT=$cap timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
