mkdir -p gpurun_out
timeout 300 python tools/gemm_tl.py 1024 8192 4096 28672 3584 8192 2>&1
timeout 600 python tools/gemm_bw.py c3 2>&1 | grep -v "^$"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 1 -o gpurun_out/s4_gemm_o python tools/gemm_prof.py 1024 8192 > gpurun_out/ncu_g1.log 2>&1; echo g1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 4 -c 1 -o gpurun_out/s4_gemm_gu8b python tools/gemm_prof.py 4096 28672 > gpurun_out/ncu_g2.log 2>&1; echo g2 rc=$?
