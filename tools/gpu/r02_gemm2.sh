mkdir -p gpurun_out
python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
python -c "
import paper_2511_14116_b200._native as N
for s in (4,6,8):
    N.lib.fs_gemm_set_tuning(s, -1); print('stages', s, 'ctas/SM', N.lib.fs_gemm_ctas_per_sm(0))"
for st in 4 6 8; do
  echo "== stages $st"
  FS_GEMM_STAGES=$st timeout 300 python tools/gemm_bw.py 2>&1 | grep -v "^$"
  for w in 8 5; do FS_GEMM_STAGES=$st timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
done
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --gemm cublas --time 2>&1 | tail -1; done
