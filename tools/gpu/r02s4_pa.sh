timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for w in 8 5; do timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1
timeout 600 python tools/step_trace.py --world 8 2>&1 | tail -14
