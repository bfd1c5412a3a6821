# ncu --set full of one K1 launch at C3 N=8 and N=5 (rank 0), final tree
mkdir -p gpurun_out
for w in 8 5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_cta -s 50 -c 1 -o gpurun_out/r02s4_k1_c3n$w python tools/c3_step.py --world $w --rank 0 --steps 2 > gpurun_out/ncu_k1_$w.log 2>&1; echo k1 $w rc=$?
done
