for rep in 1 2 3; do for d in 0 16; do timeout 300 python tools/c3_step.py --world 8 --time --head-pages $d 2>&1 | tail -1; done; done
for rep in 1 2; do for d in 0 16; do timeout 300 python tools/c3_step.py --world 7 --time --head-pages $d 2>&1 | tail -1; done; done
