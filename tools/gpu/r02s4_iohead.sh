# step_io split into a short head graph (H2D + first layers) and the rest: graph start latency
for h in 0 1 2 4 0 1 2; do echo "== FS_IO_HEAD_LAYERS=$h"; FS_IO_HEAD_LAYERS=$h timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "step_io|back to back|replay \+ sync per step:"; done
FS_IO_HEAD_LAYERS=2 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q -p no:cacheprovider -k graph 2>&1 | tail -1
