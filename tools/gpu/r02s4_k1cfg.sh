timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -p no:cacheprovider -k "ragged" 2>&1 | tail -2
echo "== C3 N=8 (70B, qpk 8, 80 layers)"
timeout 300 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0,6,11,12,13,14,15 --graph --iters 10
echo "== C3 N=5"
timeout 300 python tools/kbench.py --layers 80 --world 5 --qpk 8 --configs 0,6,11,12,13,14,15 --graph --iters 10
echo "== C2 N=1"
timeout 300 python tools/kbench.py --layers 32 --world 1 --qpk 4 --configs 0,6,11,12,13,14,15 --graph --iters 5
