# session-2 profiling pass: full bench line, launch list, ncu captures of the
# decode kernel (C2 bench config) and the chunked-prefill kernel (C5-like)
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
BENCH="python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu --skip-mixed"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $BENCH > $OUT/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode \
    -s 40 -c 1 -o $OUT/decode_full $BENCH > $OUT/full_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc \
    -s 3 -c 1 -o $OUT/prefill_full python tools/prefill_bench.py --variant 3 --cases 1x2048@8192 --iters 2 > $OUT/full_prefill.log 2>&1
ls -la $OUT
