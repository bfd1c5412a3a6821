#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over smoke() and one
# decode, prefill, exchange and backup test each.  Logs -> gpurun_out/sanitize/.
# Usage (on the GPU box): bash tools/sanitize.sh
set -u
OUT=gpurun_out/sanitize
rm -rf $OUT; mkdir -p $OUT
CS="compute-sanitizer --print-limit 50 --target-processes all"
SMOKE="python -c 'import __graft_entry__ as g; g.smoke()'"
TESTS=(
  "tests/test_decode_gpu.py::test_fused_append_then_decode"
  "tests/test_decode_gpu.py::test_decode_hybrid_rank_ragged"
  "tests/test_prefill_gpu.py::test_prefill_splits"
  "tests/test_exchange_gpu.py::test_fused_exchange_ordered_sum"
  "tests/test_recovery_gpu.py::test_backup_then_restore_is_bitexact"
  "tests/test_recovery_gpu.py::test_restore_failed_rank_onto_survivor_per_plan"
  "tests/test_gemm_gpu.py::test_store"
  "tests/test_gemm_gpu.py::test_split_reduction_rows"
  "tests/test_gemm_gpu.py::test_packed_panels_match_row_major"
  "tests/test_exchange_gpu.py::test_fused_exchange_decode_step_matches_emulation"
  "tests/test_exchange_gpu.py::test_fused_exchange_two_shot"
)
for tool in memcheck racecheck synccheck; do
  echo "== $tool smoke" | tee -a $OUT/summary.txt
  timeout 900 bash -c "$CS --tool $tool $SMOKE" > $OUT/${tool}_smoke.log 2>&1
  echo "rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${tool}_smoke.log | tail -2 | tr '\n' ' ')" | tee -a $OUT/summary.txt
  for t in "${TESTS[@]}"; do
    name=$(echo $t | sed 's/.*:://')
    echo "== $tool $t" | tee -a $OUT/summary.txt
    timeout 1200 $CS --tool $tool python -m pytest -x -q -p no:cacheprovider "$t" > $OUT/${tool}_${name}.log 2>&1
    echo "rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $OUT/${tool}_${name}.log | tail -3 | tr '\n' ' ')" | tee -a $OUT/summary.txt
  done
done
