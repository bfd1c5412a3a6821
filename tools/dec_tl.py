"""Per-warp decode timeline (build with tools/dec_instrument.py).  Same args as kbench."""
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
big.zero_()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); cache.decode_layer(5, q, out); e.record(); torch.cuda.synchronize()
W = 148
d = big[1 << 24:].view(torch.int64)[:W * 4].view(W, 4).cpu().numpy()
ok = d[:, 2] > 0
t0 = d[:, 0][d[:, 0] > 0].min()
print(f"event {s.elapsed_time(e)*1e3:.1f} us; warps {ok.sum()}")
for nm, a, b in (("start spread", None, 0), ("start->first page", 0, 1), ("first page->end", 1, 2)):
    v = (d[ok, b] - (t0 if a is None else d[ok, a])) / 1e3
    print(f"  {nm:20s} min {v.min():6.2f} median {np.median(v):6.2f} max {v.max():6.2f} us")
print(f"  last warp end {(d[ok, 2].max() - t0)/1e3:.2f} us")

dur = (d[ok, 2] - d[ok, 1]) / 1e3
sm = d[ok, 3]
order = np.argsort(dur)
print("fastest (us, sm):", [(round(dur[i], 1), int(sm[i])) for i in order[:8]])
print("slowest (us, sm):", [(round(dur[i], 1), int(sm[i])) for i in order[-12:]])
import collections
print("sm parity of slowest 30:", collections.Counter(int(sm[i]) % 2 for i in order[-30:]), " fastest 30:", collections.Counter(int(sm[i]) % 2 for i in order[:30]))
print("sm < 74 among slowest 30:", sum(int(sm[i]) < 74 for i in order[-30:]), " fastest 30:", sum(int(sm[i]) < 74 for i in order[:30]))
