"""fs_gemm_skinny vs cuBLAS on the decode-step shapes (M=64), graph-timed."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
shapes = {"8b_qkv": (4096, 6144), "8b_o": (4096, 4096), "8b_gu": (4096, 28672), "8b_d": (14336, 4096),
          "70b8_qkv": (8192, 1280), "70b8_o": (1024, 8192), "70b8_gu": (8192, 7168), "70b8_d": (3584, 8192),
          "70b5_qkv": (8192, 5120), "70b5_o": (4096, 8192), "70b5_gu": (8192, 11520), "70b5_d": (5760, 8192)}
def t(fn, it=40):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it): fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3
for name, (K, N) in shapes.items():
    x = torch.randn(64, K, device="cuda", dtype=torch.bfloat16)
    reps = max(1, int(400e6 // (K * N * 2)))
    Ws = [torch.randn(K, N, device="cuda", dtype=torch.bfloat16) for _ in range(reps)]
    out = torch.empty(64, N, device="cuda", dtype=torch.bfloat16)
    gm = SkinnyGemm(N); Ps = [PackedWeight(w) for w in Ws]
    i = [0]
    def cub():
        i[0] = (i[0] + 1) % reps; torch.matmul(x, Ws[i[0]], out=out)
    def ours():
        i[0] = (i[0] + 1) % reps; gm(x, Ps[i[0]], out, STORE)
    a, b = t(cub), t(ours)
    gb = K * N * 2 / 1e9
    print(f"{name:10s} W={gb*1e3:7.1f}MB  cuBLAS {a:7.2f}us {gb/a*1e6:6.0f}GB/s   tcgen05 {b:7.2f}us {gb/b*1e6:6.0f}GB/s", flush=True)
    del Ws
