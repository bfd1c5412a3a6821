"""Do consecutive skinny-GEMM launches co-reside on an SM under PDL?
Per-CTA start / end (%globaltimer) and %smid of two back-to-back launches:
python tools/gemm_coresidence.py K N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
K, Nc = int(sys.argv[1]), int(sys.argv[2])
ws = [PackedWeight(torch.randn(K, Nc, device="cuda").to(torch.bfloat16)) for _ in range(3)]
x = torch.randn(64, K, device="cuda").to(torch.bfloat16)
out = torch.empty(64, Nc, device="cuda", dtype=torch.bfloat16)
sk = SkinnyGemm(Nc)
dbg = [torch.zeros(148 * 8, dtype=torch.int64, device="cuda") for _ in range(3)]
for i in range(3):
    sk(x, ws[i], out, STORE)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):  # back to back in one graph (no host gaps)
    for i in range(3):
        N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(dbg[i].data_ptr()))
        sk(x, ws[i], out, STORE)
N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(0))
g.replay()
torch.cuda.synchronize()
d = [b.view(148, 8).cpu().numpy().astype(np.int64) for b in dbg]
t0 = min(a[:, 0].min() for a in d)
for i, a in enumerate(d):
    print(f"launch {i}: start {(a[:,0].min()-t0)/1e3:6.2f}..{(a[:,0].max()-t0)/1e3:6.2f} us  "
          f"first stage med {np.median(a[:,1]-a[:,0])/1e3:5.2f}  pdl wait done med {(np.median(a[:,6])-t0)/1e3:6.2f}  "
          f"end {(a[:,4].min()-t0)/1e3:6.2f}..{(a[:,4].max()-t0)/1e3:6.2f} us")
for i in (1, 2):
    prev, cur = d[i - 1], d[i]
    end_by_sm = {int(s): e for s, e in zip(prev[:, 7], prev[:, 4])}
    overlap = [(end_by_sm[int(s)] - st) / 1e3 for s, st in zip(cur[:, 7], cur[:, 0]) if int(s) in end_by_sm]
    ov = np.array(overlap)
    print(f"launch {i} CTAs starting before launch {i-1}'s CTA on the same SM ended: "
          f"{(ov > 0).sum()}/{len(ov)} (median lead {np.median(ov):.2f} us)")
