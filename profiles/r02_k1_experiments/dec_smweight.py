"""K1 experiment: partition the page space over SMs weighted by each SM's
measured streaming speed (per-SM speed is a stable property of the SM:
tools/dec_smvar.py).  Calibrate from per-CTA stamps of uniform launches,
then time the 80-layer attention graph uniform vs weighted.
DEC_SHAPE=world,layers,heads,qpk,batch,ctx (default C3 N=8)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
from oracle.placement import owner_table
world, layers, heads, qpk, batch, ctx = [int(v) for v in os.environ.get("DEC_SHAPE", "8,80,8,8,64,4096").split(",")]
owner = np.array(owner_table("hybrid", layers, heads, range(world)), dtype=np.int32)
work = RankWork.build(owner, 0, {r: r % world for r in range(batch)}, batch)
cache = PagedKVCache(work, ctx, qpk)
cache.pool.view(torch.bfloat16).normal_()
cache.set_lengths([ctx] * batch)
rows = batch * work.n_slots
q = torch.randn((rows, qpk, 128), device="cuda").to(torch.bfloat16)
out = torch.zeros((rows, qpk, 128), device="cuda", dtype=torch.bfloat16)
C = 148
stamps = torch.zeros(C * 4, dtype=torch.int64, device="cuda")
for l in range(layers):
    cache.decode_layer(l, q, out)
torch.cuda.synchronize()
lib = N.lib
lib.fs_decode_debug_stamps.argtypes = [N.C.c_void_p]
lib.fs_decode_sm_weights.argtypes = [N.C.c_void_p]


def calibrate(n=24):
    durs = np.zeros((n, C))
    lib.fs_decode_debug_stamps(N.C.c_void_p(stamps.data_ptr()))
    for it in range(n):
        stamps.zero_()
        cache.decode_layer(it % layers, q, out)
        torch.cuda.synchronize()
        d = stamps.view(C, 4).cpu().numpy()
        durs[it] = (d[:, 2] - d[:, 1]) / 1e3
    lib.fs_decode_debug_stamps(None)
    return durs


def graph_ms(iters=10):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for l in range(layers):
            cache.decode_layer(l, q, out)
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        g.replay()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


kvb = sum(cache.layer_kv_bytes(l) for l in range(layers))
base = graph_ms()
ref = out.clone()
for l in range(layers):
    cache.decode_layer(l, q, out)
ref = out.clone()
durs = calibrate()
speed = 1.0 / durs.mean(0)            # uniform partition: equal pages per SM (stamp slot = blockIdx)
print(f"uniform: graph {base:.3f} ms ({kvb / base / 1e6:.0f} GB/s); per-CTA duration "
      f"{durs.mean():.2f} us, spread {np.mean(durs.max(1) - durs.min(1)):.2f} us")
# stamps are indexed by blockIdx under the uniform partition: map to smid
lib.fs_decode_debug_stamps(N.C.c_void_p(stamps.data_ptr()))
per_sm = np.zeros((24, C))
for it in range(24):
    stamps.zero_()
    cache.decode_layer(it % layers, q, out)
    torch.cuda.synchronize()
    d = stamps.view(C, 4).cpu().numpy()
    per_sm[it, d[:, 3].astype(int)] = (d[:, 2] - d[:, 1]) / 1e3
lib.fs_decode_debug_stamps(None)
speed = 1.0 / per_sm.mean(0)
for label, w in (("weighted", speed), ("weighted^2", speed ** 2), ("uniform-by-smid", np.ones(C))):
    cw = torch.tensor(np.concatenate([[0.0], np.cumsum(w / w.sum())]), dtype=torch.float64, device="cuda")
    lib.fs_decode_sm_weights(N.C.c_void_p(cw.data_ptr()))
    ms = graph_ms()
    out.zero_()
    for l in range(layers):
        cache.decode_layer(l, q, out)
    torch.cuda.synchronize()
    diff = (out.float() - ref.float()).abs().max().item()
    # per-SM durations under this partition
    lib.fs_decode_debug_stamps(N.C.c_void_p(stamps.data_ptr()))
    dd = []
    for it in range(12):
        stamps.zero_()
        cache.decode_layer(it % layers, q, out)
        torch.cuda.synchronize()
        d = stamps.view(C, 4).cpu().numpy()
        dd.append((d[:, 2] - d[:, 1]) / 1e3)
    lib.fs_decode_debug_stamps(None)
    dd = np.array(dd)
    print(f"{label}: graph {ms:.3f} ms ({kvb / ms / 1e6:.0f} GB/s, {base / ms:.3f}x); per-CTA "
          f"{dd.mean():.2f} us, spread {np.mean(dd.max(1) - dd.min(1)):.2f} us; max |out - uniform| {diff:.2e}")
    lib.fs_decode_sm_weights(None)
    del cw
