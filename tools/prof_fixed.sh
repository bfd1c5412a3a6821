# per-launch time vs launch size for the C3 decode shape (fixed-cost fit)
for b in 1 16 64 256; do
  python tools/kbench.py --layers 80 --world 8 --qpk 8 --batch $b --ctx 4096 --configs 0 --graph --iters 10 | tail -1 | sed "s/^/batch $b ctx 4096 /"
done
python tools/kbench.py --layers 80 --world 8 --qpk 8 --batch 1 --ctx 16 --configs 0 --graph --iters 10 | tail -1 | sed "s/^/batch 1 ctx 16 /"
python tools/kbench.py --layers 80 --world 8 --qpk 8 --batch 1 --ctx 16 --configs 0 --iters 10 | tail -1 | sed "s/^/nograph batch 1 ctx 16 /"
