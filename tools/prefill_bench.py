"""K8 timing: chunked-prefill attention TFLOP/s on C5-like chunks."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
from paper_2511_14116_b200.prefill import PrefillLaunch

ap = argparse.ArgumentParser()
ap.add_argument("--qpk", type=int, default=8)
ap.add_argument("--cases", default="1x2048@0,1x2048@8192,8x256@4096,1x512@30000,64x32@2000")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--target", type=int, default=None, help="target_units of the tile planner")
a = ap.parse_args()
for case in a.cases.split(","):
    cnt, rest = case.split("x")
    ln, st = rest.split("@")
    cnt, ln, st = int(cnt), int(ln), int(st)
    work = RankWork.build(np.zeros((1, 1), np.int32), 0, {r: 0 for r in range(cnt)}, cnt)
    cache = PagedKVCache(work, st + ln, a.qpk)
    cache.pool.view(torch.bfloat16).normal_()
    stride = (a.qpk + 2) * 128
    q = torch.randn((cnt * ln, stride), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    row0 = np.arange(cnt) * ln * stride
    L = PrefillLaunch(cache, np.arange(cnt), [st] * cnt, [ln] * cnt, row0, row0,
                      variant=a.variant, target_units=a.target)
    for _ in range(3):
        L(q, stride, out, stride)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        L(q, stride, out, stride)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    print(f"{case:16s} v{a.variant} qpk {a.qpk}: {ms*1e3:8.1f} us  {L.flops/ms/1e9:7.1f} TFLOP/s  "
          f"tiles {L.n_tiles} splits {L.n_comb}")
