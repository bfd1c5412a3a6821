# round-2 profiling pass 1: C3 K1 ncu, GEMM shapes, step breakdown, K5/K6, sanitizers
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 100 -c 1 -o gpurun_out/r02_decode70_n8 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0 --iters 2 > gpurun_out/ncu70.log 2>&1; echo ncu70 rc=$?
timeout 600 python tools/gemm_bw.py > gpurun_out/gemm_bw.txt 2>&1; cat gpurun_out/gemm_bw.txt
timeout 600 python tools/step_cmp.py > gpurun_out/step_cmp.txt 2>&1; cat gpurun_out/step_cmp.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3n8.csv python tools/c3_step.py --world 8 --rank 0 --steps 2 > gpurun_out/c3_step_ncu.log 2>&1; echo c3launch rc=$?
timeout 900 bash tools/sanitize.sh > gpurun_out/sanitize_run.log 2>&1; echo sanitize rc=$?
cat gpurun_out/sanitize/summary.txt
