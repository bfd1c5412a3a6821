"""Quick K1 timing: one rank of a hybrid plan, all layers, CUDA events."""
import argparse, math, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
from oracle.placement import owner_table

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--heads", type=int, default=8)
ap.add_argument("--world", type=int, default=1)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--qpk", type=int, default=4)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--configs", default="0,1,2,3,7")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--order", default="contiguous", help="page order: contiguous | shuffled | interleaved")
a = ap.parse_args()
owner = np.array(owner_table("hybrid", a.layers, a.heads, range(a.world)), dtype=np.int32)
routing = {r: r % a.world for r in range(a.batch)}
work = RankWork.build(owner, a.rank, routing, a.batch)
cache = PagedKVCache(work, a.ctx, a.qpk, page_order=a.order)
cache.pool.view(torch.bfloat16).normal_()
cache.set_lengths([a.ctx] * a.batch)
rows = a.batch * work.n_slots
q = torch.randn((rows, a.qpk, 128), device="cuda").to(torch.bfloat16)
out = torch.zeros((rows, a.qpk, 128), device="cuda", dtype=torch.bfloat16)
kvb = sum(cache.layer_kv_bytes(l) for l in range(a.layers))
print(f"items={work.n_items} KV bytes/step={kvb/1e9:.3f} GB pages={cache.n_pages}")
for cfg in [int(c) for c in a.configs.split(",")]:
    cache.config = cfg
    try:
        for _ in range(2):
            for l in range(a.layers): cache.decode_layer(l, q, out)
        torch.cuda.synchronize()
    except Exception as exc:
        print(f"config {cfg}: {exc}"); continue
    run = lambda: [cache.decode_layer(l, q, out) for l in range(a.layers)]
    if a.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        run = g.replay
        run(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        run()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    print(f"config {cfg}: {ms:.3f} ms/step  {kvb/ms/1e6:.1f} GB/s  ({kvb/ms/1e6/6543.4*100:.1f}% of 6543 GB/s)")
