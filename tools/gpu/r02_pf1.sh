for pf in "" o d q od odq; do for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time --pf "$pf" 2>&1 | tail -1; done; done
for pf in "" od odq; do timeout 300 python tools/c3_step.py --model 8b --world 1 --time --pf "$pf" 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --world 8 --time --pf od --pf-ctas 4 2>&1 | tail -1
timeout 300 python tools/c3_step.py --world 8 --time --pf od --pf-ctas 64 2>&1 | tail -1
