"""Per-CTA phase timeline of the skinny tcgen05 GEMM (fs_gemm_debug_timestamps).
python tools/gemm_tl.py K N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
K, Nc = int(sys.argv[1]), int(sys.argv[2])
reps = max(2, int(1.2e9 // (K * Nc * 2)))
ws = [PackedWeight(torch.randn(K, Nc, device="cuda").to(torch.bfloat16)) for _ in range(reps)]
x = torch.randn(64, K, device="cuda").to(torch.bfloat16)
out = torch.empty(64, Nc, device="cuda", dtype=torch.bfloat16)
sk = SkinnyGemm(Nc)
dbg = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
for i in range(reps):
    sk(x, ws[i], out, STORE)
torch.cuda.synchronize()
N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(dbg.data_ptr()))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); sk(x, ws[0], out, STORE); e.record(); torch.cuda.synchronize()
N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(0))
d = dbg.view(148, 16).cpu().numpy().astype(np.int64)
t0 = d[:, 0].min()
print(f"K {K} N {Nc}: event {s.elapsed_time(e)*1e3:.1f} us; span {(d[:, 4].max() - t0)/1e3:.1f} us")
for name, a, b in (("start spread", None, 0), ("start->first stage", 0, 1), ("first stage->MMA done", 1, 2),
                   ("MMA done->epilogue/reduce done", 2, 3), ("->CTA end", 3, 4), ("PDL wait", 5, 6)):
    v = (d[:, b] - (t0 if a is None else d[:, a])) / 1e3
    print(f"  {name:32s} median {np.median(v):6.2f} max {v.max():6.2f} us")
if d[:, 8].any():
    m2 = d[:, 2]
    for name, i in (("acc0 read", 8), ("acc1 read", 9), ("pub0 done", 10), ("pub1 done", 11),
                    ("wait0 done", 12), ("wait1 done", 13), ("red0 landed", 14), ("red1 landed", 15)):
        v = d[:, i]; ok = v > 0
        if ok.any():
            print(f"  {name:12s} after MMA done: median {np.median((v[ok] - m2[ok]) / 1e3):6.2f} max {((v[ok] - m2[ok]) / 1e3).max():6.2f} us  (n={ok.sum()})")
