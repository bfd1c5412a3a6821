"""Skinny decode GEMMs at the C3 (70B, per rank) and C2 (8B) shapes: cuBLAS
vs the in-tree tcgen05 kernel, HBM GB/s of the weight stream (rotating
weight copies so nothing is L2-resident between launches, CUDA graph of
back-to-back launches).  python tools/gemm_bw.py [c3|c2|all]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight

M = 64
C3 = {  # name: (K, N) per rank, C3 Llama-3-70B, N=8 (1 TP head) / N=5 (1 TP + 3 DP)
    "qkv 1 slot": (8192, 1280), "qkv 4 slots": (8192, 5120),
    "o 1 slot": (1024, 8192), "o 4 slots": (4096, 8192),
    "gate/up tp8": (8192, 7168), "down tp8": (3584, 8192),
    "gate/up tp5": (8192, 11520), "down tp5": (5760, 8192),
}
C2 = {"qkv 8b": (4096, 6144), "o 8b": (4096, 4096), "gate/up 8b": (4096, 28672),
      "down 8b": (14336, 4096)}
which = sys.argv[1] if len(sys.argv) > 1 else "all"
shapes = {**(C3 if which in ("c3", "all") else {}), **(C2 if which in ("c2", "all") else {})}
sk = SkinnyGemm(28672)
for name, (K, N) in shapes.items():
    reps = max(2, int(1.2e9 // (K * N * 2)))  # > L2 of distinct weights
    ws = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(reps)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {}
    for impl in ("cublas", "tcgen05"):
        if impl == "tcgen05":
            if N % 128 or K % 64:
                continue
            pw = [PackedWeight(w) for w in ws]
            f = lambda i: sk(x, pw[i], out, STORE)
        else:
            f = lambda i: torch.matmul(x, ws[i], out=out)
        for i in range(reps):
            f(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                f(i)
        g.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            g.replay()
        e.record(); torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / (5 * reps)
        res[impl] = (us, K * N * 2 / us / 1e3)
        del g
        if impl == "tcgen05":
            del pw
    print(f"{name:14s} K {K:5d} N {N:5d}: " + "  ".join(
        f"{k} {v[0]:6.1f} us {v[1]:6.0f} GB/s" for k, v in res.items()), flush=True)
    del ws
    torch.cuda.empty_cache()
