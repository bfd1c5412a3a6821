mkdir -p gpurun_out/sanitize_gemm
CS="compute-sanitizer --print-limit 50 --target-processes all"
for tool in memcheck racecheck synccheck; do
  for t in tests/test_gemm_gpu.py::test_split_reduction_rows tests/test_gemm_gpu.py::test_packed_panels_match_row_major tests/test_gemm_gpu.py::test_store; do
    name=$(echo $t | sed 's/.*:://')
    timeout 1200 $CS --tool $tool python -m pytest -x -q -p no:cacheprovider "$t" > gpurun_out/sanitize_gemm/${tool}_${name}.log 2>&1
    echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_gemm/${tool}_${name}.log | tail -3 | tr '\n' ' ')"
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_bench.csv python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu --skip-mixed > gpurun_out/launches_bench.log 2>&1; echo launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_c3n8.csv python tools/c3_step.py --world 8 --rank 0 --steps 2 > gpurun_out/launches_c3.log 2>&1; echo c3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 200 -c 4 -o gpurun_out/r02s4_gemm_c3 python tools/c3_step.py --world 8 --rank 0 --steps 2 > gpurun_out/ncu_gc3.log 2>&1; echo gc3 rc=$?
