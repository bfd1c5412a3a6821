timeout 600 python tools/step_trace.py --world 8 2>&1 | tail -30
timeout 600 python tools/step_trace.py --model 8b --world 1 --layers-shown 1 2>&1 | tail -20
