for pm in 1000000 32 48; do
echo "== panel_min $pm"
FS_GEMM_PANEL_MIN=$pm python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
FS_GEMM_PANEL_MIN=$pm timeout 300 python tools/gemm_bw.py 2>&1 | grep -v "^$"
for w in 8 5; do FS_GEMM_PANEL_MIN=$pm timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
done
