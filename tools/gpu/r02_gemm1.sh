mkdir -p gpurun_out
python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for cfg in "4 4" "4 1000" "4 0" "8 4"; do set -- $cfg
  echo "== stages $1 in_grid_max $2"
  FS_GEMM_STAGES=$1 FS_GEMM_IN_GRID_MAX=$2 timeout 300 python tools/gemm_bw.py 2>&1 | grep -v "^$"
  for w in 8 5; do FS_GEMM_STAGES=$1 FS_GEMM_IN_GRID_MAX=$2 timeout 300 python tools/c3_step.py --world $w --gemm tcgen05 --time 2>&1 | tail -1; done
done
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --gemm cublas --time 2>&1 | tail -1; done
