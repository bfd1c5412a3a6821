"""Probe host-memory settings that decide how fast a /dev/shm region can be
mapped and page-locked (THP for shmem, hugetlb) and time the variants."""
import mmap
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14116_b200 import _native as N  # noqa: E402
import ctypes as C  # noqa: E402

for f in ["/sys/kernel/mm/transparent_hugepage/shmem_enabled",
          "/sys/kernel/mm/transparent_hugepage/enabled"]:
    try:
        print(f, open(f).read().strip())
    except OSError as e:
        print(f, e)
print([ln.strip() for ln in open("/proc/meminfo") if "Huge" in ln])
os.system("mount | grep -E 'shm|huge'")
gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(gb * (1 << 30))
for variant in ("plain", "thp", "populate"):
    path = f"/dev/shm/fs_probe_{variant}"
    fd = os.open(path, os.O_RDWR | os.O_CREAT, 0o600)
    os.ftruncate(fd, n)
    mm = mmap.mmap(fd, n, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
    if variant == "thp":
        mm.madvise(mmap.MADV_HUGEPAGE)
    t0 = time.perf_counter()
    t = torch.frombuffer(mm, dtype=torch.uint8)
    t.view(torch.int64)[::512].fill_(1)
    t1 = time.perf_counter()
    del t
    mm.close()
    # a second process-like mapping: map + register
    flags = mmap.MAP_SHARED | (mmap.MAP_POPULATE if variant == "populate" else 0)
    t2 = time.perf_counter()
    mm2 = mmap.mmap(fd, n, flags, mmap.PROT_READ | mmap.PROT_WRITE)
    if variant == "thp":
        mm2.madvise(mmap.MADV_HUGEPAGE)
    t3 = time.perf_counter()
    t = torch.frombuffer(mm2, dtype=torch.uint8)
    p = C.c_void_p()
    N.check(N.lib.fs_host_register(C.c_void_p(t.data_ptr()), n, C.byref(p)), "reg")
    t4 = time.perf_counter()
    N.lib.fs_host_unregister(C.c_void_p(t.data_ptr()))
    print(f"{variant}: first touch {gb / (t1 - t0):.1f} GB/s; map {t3 - t2:.2f}s; "
          f"register {gb / (t4 - t3):.1f} GB/s")
    del t
    mm2.close()
    os.close(fd)
    os.unlink(path)
