set -x
mkdir -p gpurun_out
python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0,1,2,3,4,5,6,7,8,9,10 --graph --iters 10 > gpurun_out/kb70_n8.txt 2>&1
python tools/kbench.py --layers 80 --world 5 --qpk 8 --configs 0,1,2,5,7 --graph --iters 10 > gpurun_out/kb70_n5.txt 2>&1
python tools/kbench.py --layers 32 --world 1 --qpk 4 --configs 0,1,2,7 --graph --iters 5 > gpurun_out/kb8_n1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 100 -c 1 -o gpurun_out/decode70_n8 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0 --iters 2 > gpurun_out/ncu70.log 2>&1
timeout 300 python tools/step_cmp.py > gpurun_out/step_cmp.txt 2>&1
cat gpurun_out/kb70_n8.txt gpurun_out/kb70_n5.txt gpurun_out/kb8_n1.txt gpurun_out/step_cmp.txt
