"""Per-CTA phase timestamps of fs_gemm_skinny (testing hook)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
K, Nn = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn(64, K, device="cuda", dtype=torch.bfloat16)
w = PackedWeight(torch.randn(K, Nn, device="cuda", dtype=torch.bfloat16))
out = torch.empty(64, Nn, device="cuda", dtype=torch.bfloat16)
g = SkinnyGemm(Nn)
dbg = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
N.lib.fs_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
for mode in ("single", "back2back"):
    for _ in range(3): g(x, w, out, STORE)
    torch.cuda.synchronize()
    N.lib.fs_gemm_debug_timestamps(dbg.data_ptr())
    dbg.zero_()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g(x, w, out, STORE); e.record(); torch.cuda.synchronize()
    N.lib.fs_gemm_debug_timestamps(None)
    d = dbg.view(148, 8).cpu().numpy().astype(np.float64)
    t0 = d[:, 0].min()
    rel = (d[:, :7] - t0) / 1e3
    print(f"{K}x{Nn} event {s.elapsed_time(e)*1e3:.1f}us | start {rel[:,0].min():.1f}-{rel[:,0].max():.1f} first-data {rel[:,1].min():.1f}-{rel[:,1].max():.1f} mma-done {rel[:,2].min():.1f}-{rel[:,2].max():.1f} epi-done {rel[:,3].min():.1f}-{rel[:,3].max():.1f} exit {rel[:,4].min():.1f}-{rel[:,4].max():.1f} A-issued {rel[:,5].min():.1f}-{rel[:,5].max():.1f} pdl-wait-done {rel[:,6].min():.1f}-{rel[:,6].max():.1f}")
    break
