import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
from paper_2511_14116_b200.prefill import PrefillLaunch
starts, lens = [2392, 750, 3052], [563, 1013, 472]
cnt = 3
work = RankWork.build(np.zeros((1, 1), np.int32), 0, {r: 0 for r in range(cnt)}, cnt)
cache = PagedKVCache(work, max(s + l for s, l in zip(starts, lens)), 8)
cache.pool.view(torch.bfloat16).normal_()
stride = 10 * 128
T = sum(lens)
q = torch.randn((T, stride), device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
row0 = np.concatenate([[0], np.cumsum(lens)[:-1]]) * stride
variant = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L = PrefillLaunch(cache, np.arange(cnt), starts, lens, row0, row0, variant=variant)
for _ in range(5): L(q, stride, out, stride)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): L(q, stride, out, stride)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"C5-like chunk v{variant}: {ms*1e3:.1f} us  {L.flops/ms/1e9:.1f} TFLOP/s tiles {L.n_tiles} comb {L.n_comb}")
