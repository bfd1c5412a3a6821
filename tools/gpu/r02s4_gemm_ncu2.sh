# ncu --set full of one layer's four projection GEMMs at C2 (8b, N=1) and C3 N=5
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 64 -c 4 -o gpurun_out/r02s4_gemm_c2 python tools/c3_step.py --model 8b --world 1 --rank 0 --steps 2 > gpurun_out/ncu_gc2.log 2>&1; echo gc2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 200 -c 4 -o gpurun_out/r02s4_gemm_c3n5 python tools/c3_step.py --world 5 --rank 0 --steps 2 > gpurun_out/ncu_gc3n5.log 2>&1; echo gc3n5 rc=$?
ls -la gpurun_out/*.ncu-rep
