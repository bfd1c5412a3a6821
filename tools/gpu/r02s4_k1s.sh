for c in 0 2 1 5 6; do
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time --config $c 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --model 8b --world 1 --time --config $c 2>&1 | tail -1
done
