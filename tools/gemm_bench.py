"""Skinny (M=64) GEMM timings: NN (x @ W[K,N]) vs TN (F.linear with W[N,K])."""
import torch, torch.nn.functional as F
shapes = {"8b_qkv": (4096, 6144), "8b_o": (4096, 4096), "8b_gu": (4096, 28672), "8b_d": (14336, 4096),
          "70b8_qkv": (8192, 1280), "70b8_o": (1024, 8192), "70b8_gu": (8192, 7168), "70b8_d": (3584, 8192),
          "70b5_qkv": (8192, 5120), "70b5_o": (4096, 8192), "70b5_gu": (8192, 11520), "70b5_d": (5760, 8192)}
M = 64
def t(fn, it=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it): fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3
for name, (K, N) in shapes.items():
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    # rotate through several weight copies so L2 never holds W
    reps = max(1, int(400e6 // (K * N * 2)))
    Ws = [torch.randn(K, N, device="cuda", dtype=torch.bfloat16) for _ in range(reps)]
    Wt = [w.t().contiguous() for w in Ws]
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    i = [0]
    def nn():
        i[0] = (i[0] + 1) % reps; torch.matmul(x, Ws[i[0]], out=out)
    def tn():
        i[0] = (i[0] + 1) % reps; torch.nn.functional.linear(x, Wt[i[0]], out=out) if False else torch.matmul(x, Wt[i[0]].t(), out=out)
    a, b = t(nn), t(tn)
    gb = K * N * 2 / 1e9
    print(f"{name:10s} K={K:6d} N={N:6d} W={gb*1e3:7.1f}MB  NN {a:7.2f}us {gb/a*1e6:6.0f}GB/s   TN {b:7.2f}us {gb/b*1e6:6.0f}GB/s")
    del Ws, Wt
