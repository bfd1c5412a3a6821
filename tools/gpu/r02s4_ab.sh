for t in . oldtree . oldtree; do echo "== $t"
(cd $t && timeout 300 python tools/kbench.py --layers 80 --world 8 --qpk 8 --configs 0 --graph --iters 10 2>&1 | tail -1)
(cd $t && timeout 300 python tools/c3_step.py --world 8 --time 2>&1 | tail -1)
done
