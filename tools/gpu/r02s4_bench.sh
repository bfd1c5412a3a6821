mkdir -p gpurun_out
bash tools/gpu/bench_full.sh
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
tail -c 800 gpurun_out/bench_ref.json
