# step_io: input / result copies as PDL kernels (fs_io_copy) vs graph memcpy nodes
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_knobs_gpu.py tests/test_boundary*.py -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for v in kernel memcpy; do echo "== FS_IO_COPY=$v"; FS_IO_COPY=$v timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "step_io \+ sync|back to back|replay \+ sync per step:"; done; done
