mkdir -p gpurun_out/sanitize_gemm
CS="compute-sanitizer --print-limit 50 --target-processes all"
for t in tests/test_gemm_gpu.py::test_split_reduction_rows tests/test_gemm_gpu.py::test_store; do
  name=$(echo $t | sed 's/.*:://')
  timeout 1200 $CS --tool racecheck python -m pytest -x -q -p no:cacheprovider "$t" > gpurun_out/sanitize_gemm/racecheck_${name}.log 2>&1
  echo "racecheck $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_gemm/racecheck_${name}.log | tail -3 | tr '\n' ' ')"
done
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_c3n8.csv python tools/c3_step.py --world 8 --rank 0 --steps 2 > gpurun_out/launches_c3.log 2>&1; echo c3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 200 -c 4 -o gpurun_out/r02s4_gemm_c3 python tools/c3_step.py --world 8 --rank 0 --steps 2 > gpurun_out/ncu_gc3.log 2>&1; echo gc3 rc=$?
