mkdir -p gpurun_out
for w in 2 4 8; do FS_BENCH_SHARED_GPU=1 timeout 300 torchrun --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2951$w tools/ar_bench.py 2>/dev/null | tail -1; done
# ncu: K5/K6 page copies (backup / restore test), tcgen05 GEMM (C3 QKV + down shapes)
python tools/pagecopy_prof.py; timeout 600 ncu --set full --clock-control none --import-source on -k regex:page_copy -s 6 -c 2 -o gpurun_out/r02_pagecopy python tools/pagecopy_prof.py > gpurun_out/ncu_pc.log 2>&1; echo pc rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 1 -o gpurun_out/r02_gemm_qkv python tools/gemm_prof.py 8192 1280 > gpurun_out/ncu_g1.log 2>&1; echo g1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 1 -o gpurun_out/r02_gemm_down python tools/gemm_prof.py 3584 8192 > gpurun_out/ncu_g2.log 2>&1; echo g2 rc=$?
# C2 bench launch list + one ncu --set full of K1 in the bench command (the bench line's traffic)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu --skip-mixed > gpurun_out/launches_bench.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 40 -c 1 -o gpurun_out/r02_decode_c2 python bench.py --steps 3 --warmup 3 --skip-failure-states --skip-recovery --skip-cpu --skip-mixed > gpurun_out/full_bench.log 2>&1; echo full rc=$?
ls -la gpurun_out | tail -20
