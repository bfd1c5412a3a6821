import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE
K, N = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn(64, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
out = torch.empty(64, N, device="cuda", dtype=torch.bfloat16)
g = SkinnyGemm(N)
for _ in range(3): g(x, w, out, STORE)
torch.cuda.synchronize()
