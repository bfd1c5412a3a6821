#!/bin/bash
# Profiling pass for the bench command (run under gpurun on one B200).
#  1. launch list of the bench command (cold-cache, serialised durations)
#  2. one `--set full` capture of the top kernel (decode_kernel) in the same command
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $BENCH > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel \
    -s 40 -c 1 -o $OUT/decode_full $BENCH > $OUT/full_bench.log 2>&1
ls -la $OUT
