echo "== C3 N=8"; timeout 300 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0,1,2,3,4,5 --graph --iters 10
echo "== C2"; timeout 300 python tools/kbench.py --layers 32 --world 1 --qpk 4 --configs 0,2,3,4,5 --graph --iters 5
