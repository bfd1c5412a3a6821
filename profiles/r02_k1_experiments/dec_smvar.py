"""Is K1's per-CTA streaming time a fixed property of the SM?  Needs the
instrumented build (tools/dec_instrument.py).  Runs one layer's decode
launch N times (graph of back-to-back launches excluded: eager, synced),
records (smid, first-page -> end) per CTA and reports the correlation of
per-SM durations between launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
big = torch.zeros((1 << 24) + 2 * 148 * 16 * 4 * 2, device="cuda")
cache.part_lse = big
for l in range(layers):
    cache.decode_layer(l, q, out)
torch.cuda.synchronize()
W = 148
runs = []
maps = []
graph = os.environ.get("DEC_GRAPH") == "1"
if graph:  # every layer's launch back to back (PDL), stamps of the LAST launch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for l in range(layers):
            cache.decode_layer(l, q, out)
for it in range(12):
    big[1 << 24:].zero_()
    if graph:
        g.replay()
    else:
        cache.decode_layer(it % layers, q, out)
    torch.cuda.synchronize()
    d = big[1 << 24:].view(torch.int64)[:W * 4].view(W, 4).cpu().numpy()
    maps.append(d[:, 3].copy())
    per_sm = np.full(160, np.nan)
    for row in d:
        if row[2] > 0:
            per_sm[int(row[3])] = (row[2] - row[1]) / 1e3
    t0 = d[:, 0][d[:, 0] > 0].min()
    runs.append((per_sm, (d[:, 2].max() - t0) / 1e3))
M = np.array([r[0] for r in runs])
ok = ~np.isnan(M).any(axis=0)
M = M[:, ok]
mp = np.array(maps)
print(f"blockIdx -> smid identical to launch 0 for {np.mean([(m == mp[0]).mean() for m in mp[1:]]) * 100:.0f}% of CTAs")
print(f"launches {len(runs)}, SMs {ok.sum()}, end-to-end us: {[round(r[1], 1) for r in runs]}")
print(f"per-CTA duration: mean {M.mean():.2f} us, spread within a launch (max-min) "
      f"{np.mean(M.max(1) - M.min(1)):.2f} us, std {np.mean(M.std(1)):.2f}")
c = np.corrcoef(M)
print(f"correlation of per-SM durations between launches: mean off-diagonal "
      f"{(c.sum() - len(c)) / (len(c) ** 2 - len(c)):.3f}")
avg = M.mean(0)
resid = M - avg
print(f"per-SM mean duration range {avg.min():.2f}..{avg.max():.2f} us; "
      f"residual std after removing the per-SM mean {resid.std():.2f} us")
sms = np.nonzero(ok)[0]
order = np.argsort(avg)
print("fastest SMs:", [(int(sms[i]), round(avg[i], 1)) for i in order[:10]])
print("slowest SMs:", [(int(sms[i]), round(avg[i], 1)) for i in order[-10:]])
