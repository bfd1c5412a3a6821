"""One skinny GEMM shape (packed weights) for ncu: python tools/gemm_prof.py K N"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
K, N = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn(64, K, device="cuda", dtype=torch.bfloat16)
w = PackedWeight(torch.randn(K, N, device="cuda", dtype=torch.bfloat16))
out = torch.empty(64, N, device="cuda", dtype=torch.bfloat16)
g = SkinnyGemm(N)
for _ in range(5):
    g(x, w, out, STORE)
torch.cuda.synchronize()
