mkdir -p gpurun_out/sanitize_gemm
CS="compute-sanitizer --print-limit 50 --target-processes all"
for tool in racecheck synccheck memcheck; do
for t in tests/test_gemm_gpu.py::test_split_reduction_rows tests/test_gemm_gpu.py::test_store; do
  name=$(echo $t | sed 's/.*:://')
  timeout 1200 $CS --tool $tool python -m pytest -x -q -p no:cacheprovider "$t" > gpurun_out/sanitize_gemm/${tool}_${name}.log 2>&1
  echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_gemm/${tool}_${name}.log | tail -3 | tr '\n' ' ')"
done; done
