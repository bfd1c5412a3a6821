for r in default max_ctas prefer2; do echo "== $r"
for w in 8 5; do FS_GEMM_GROUP_RULE=$r timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
FS_GEMM_GROUP_RULE=$r timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
done
