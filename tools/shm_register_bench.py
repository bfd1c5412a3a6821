"""Cost of mapping + page-locking a populated /dev/shm region (the KV mirror
of a dead rank) and of K6 / H2D reads from it.  Usage: python tools/shm_register_bench.py GB"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14116_b200.hostmirror import SharedHostRegion, SegmentCopy  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gb * (1 << 30))
name = f"fs_regbench_{os.getpid()}"
t0 = time.perf_counter()
r = SharedHostRegion(name, n, create=True, register=False)
r.host.view(torch.int64)[:: 512].fill_(1)  # touch every page
t1 = time.perf_counter()
r.close()
t2 = time.perf_counter()
r2 = SharedHostRegion(name, register=True)
t3 = time.perf_counter()
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for _ in range(2):
    seg = SegmentCopy()
    seg.add_bytes(dev.data_ptr(), r2.dev_ptr, n)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    seg.run(dev.device)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
t6 = time.perf_counter()
dev.copy_(r2.host, non_blocking=True)
torch.cuda.synchronize()
t7 = time.perf_counter()
print(f"create+touch {gb} GB: {t1 - t0:.2f}s; open+register: {t3 - t2:.2f}s "
      f"({gb / (t3 - t2):.1f} GB/s); zero-copy H2D kernel: {(t5 - t4) * 1e3:.1f} ms "
      f"({n / (t5 - t4) / 1e9:.1f} GB/s); cudaMemcpy H2D: {(t7 - t6) * 1e3:.1f} ms "
      f"({n / (t7 - t6) / 1e9:.1f} GB/s)")
r2.close()
r2.unlink()
