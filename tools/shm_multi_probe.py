"""Can several processes page-lock the same /dev/shm region?  Usage:
python tools/shm_multi_probe.py GB NPROC POPULATE(0/1)"""
import ctypes as C
import mmap
import multiprocessing as mp
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(path, n, populate, q):
    import torch
    from paper_2511_14116_b200 import _native as N
    fd = os.open(path, os.O_RDWR)
    flags = mmap.MAP_SHARED | (mmap.MAP_POPULATE if populate else 0)
    mm = mmap.mmap(fd, n, flags, mmap.PROT_READ | mmap.PROT_WRITE)
    t = torch.frombuffer(mm, dtype=torch.uint8)
    p = C.c_void_p()
    t0 = time.perf_counter()
    rc = N.lib.fs_host_register(C.c_void_p(t.data_ptr()), n, C.byref(p))
    q.put((os.getpid(), rc, N.lib.fs_last_error().decode() if rc else "", time.perf_counter() - t0))
    time.sleep(3)


if __name__ == "__main__":
    gb, nproc, populate = float(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    n = int(gb * (1 << 30))
    os.system("ulimit -l; cat /proc/sys/vm/max_map_count; grep -i -E 'memlock|locked' /proc/self/limits")
    path = "/dev/shm/fs_multi_probe"
    fd = os.open(path, os.O_RDWR | os.O_CREAT, 0o600)
    os.ftruncate(fd, n)
    mm = mmap.mmap(fd, n, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
    import numpy as np
    if os.environ.get("PROBE_TOUCH", "1") == "1":
        a = np.frombuffer(mm, dtype=np.int64)
        a[::512] = 1
        del a
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(path, n, populate, q)) for _ in range(nproc)]
    for p in ps:
        p.start()
    for _ in ps:
        print(q.get())
    for p in ps:
        p.join()
    os.unlink(path)
