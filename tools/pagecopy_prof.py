"""K5 / K6 page copies at C3 sizes for ncu: gather 320 pages (one C3 N=8
decode step's new KV, 2.6 MB) device -> pinned host, and scatter 16384 pages
(128 MiB, a slice of an 8->7 host restore) pinned host -> device.
python tools/pagecopy_prof.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.recovery_exec import restore_pages

pool = torch.zeros((65536, 8192), dtype=torch.uint8, device="cuda")
host = torch.zeros((65536, 8192), dtype=torch.uint8).pin_memory()
host.view(torch.int32).random_()
s = torch.cuda.current_stream()
for _ in range(3):
    ids = torch.arange(0, 65536, 204, dtype=torch.int32, device="cuda")[:320]
    N.check(N.lib.fs_pages_gather(N.ptr(pool), N.ptr(ids), ids.numel(), N.ptr(host), N.ptr(ids), 16,
                                  N.C.c_void_p(s.cuda_stream)), "fs_pages_gather")
    restore_pages(pool, np.arange(16384) * 3 % 65536, host, np.arange(16384))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
restore_pages(pool, np.arange(16384) * 3 % 65536, host, np.arange(16384))
e1.record()
torch.cuda.synchronize()
print(f"K6 scatter 128 MiB: {e0.elapsed_time(e1):.2f} ms ({16384 * 8192 / e0.elapsed_time(e1) / 1e6:.1f} GB/s)")
