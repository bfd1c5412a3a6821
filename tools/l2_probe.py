"""Is a skinny decode GEMM capped by HBM or by per-SM ingest?  cuBLAS on the
C3 per-rank shapes with cold weights (rotating copies > L2) vs hot weights
(one copy, L2-resident after the first launch).  python tools/l2_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

M = 64
shapes = {"qkv 1 slot": (8192, 1280), "o 1 slot": (1024, 8192), "down tp8": (3584, 8192),
          "o 4 slots": (4096, 8192), "gate/up tp8": (8192, 7168)}


def timeit(fn, n):
    for i in range(n):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            fn(i)
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (5 * n)


for name, (K, N) in shapes.items():
    reps = max(2, int(1.2e9 // (K * N * 2)))
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(reps)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cold = timeit(lambda i: torch.matmul(x, ws[i], out=out), reps)
    hot = timeit(lambda i: torch.matmul(x, ws[0], out=out), reps)
    mb = K * N * 2 / 1e6
    print(f"{name:12s} {mb:6.1f} MB: cold {cold:6.1f} us ({mb/cold:5.2f} TB/s)  "
          f"hot {hot:6.1f} us ({mb/hot:5.2f} TB/s)", flush=True)
    del ws
    torch.cuda.empty_cache()
