for t in . oldtree .; do echo "== $t"
(cd $t && timeout 300 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0 --graph --iters 10 2>&1 | tail -1)
done
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_config_parity_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
