FS_GEMM_OCC_DEBUG=1 python -c "
import paper_2511_14116_b200._native as N
N.lib.fs_gemm_set_tuning(4, -1); print('stages 4 ctas/SM', N.lib.fs_gemm_ctas_per_sm(0))" 2>&1 | head -3
python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/gemm_bw.py 2>&1 | grep -v "^$"
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
