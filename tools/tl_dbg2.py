import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
from paper_2511_14116_b200.prefill import PrefillLaunch
cnt, ln, st = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (1, 2048, 8192)
variant = int(sys.argv[4]) if len(sys.argv) > 4 else 0
work = RankWork.build(np.zeros((1, 1), np.int32), 0, {r: 0 for r in range(cnt)}, cnt)
cache = PagedKVCache(work, st + ln, 8)
cache.pool.view(torch.bfloat16).normal_()
stride = 10 * 128
q = torch.randn((cnt * ln, stride), device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
row0 = np.arange(cnt) * ln * stride
L = PrefillLaunch(cache, np.arange(cnt), [st] * cnt, [ln] * cnt, row0, row0, variant=variant)
L.part_lse = torch.zeros(max(4_000_000, L.part_lse.numel() if L.part_lse is not None else 0), device="cuda")
for _ in range(3): L(q, stride, out, stride)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); L(q, stride, out, stride); e.record(); torch.cuda.synchronize()
print("launch ms", s.elapsed_time(e))
n = L.n_tiles
d = L.part_lse.view(torch.int64)[1000000:1000000 + n * 8].view(n, 8).cpu().numpy()
np.save("gpurun_out/qload.npy", d)
e = L.part_lse.view(torch.int64)[1000000 + n * 8:1000000 + n * 8 + n * 16].view(n, 2, 8).cpu().numpy()
if e[:, :, 5].any():
    nbk = np.maximum(e[:, :, 5], 1)
    for i, nm in enumerate(("wait S", "tcgen05.ld", "max", "exp+P store", "rest (rescale, arrive)")):
        print(f"softmax per block {nm:24s} half0 {np.median(e[:, 0, i] / nbk[:, 0]):7.0f}  half1 {np.median(e[:, 1, i] / nbk[:, 1]):7.0f} cycles")
t0 = d[:, 0].min()
st_, mma0, mma1, end, sm, nb = [d[:, i] for i in range(6)]
cyc = nb >> 16; nb = nb & 0xffff
if cyc.any():
    print("MMA warp per block: loop cycles %.0f, k_full wait %.0f, v_full wait %.0f, p_full wait %.0f" % (
        np.median(cyc / nb), np.median((d[:, 6] & 0xffffffff) / nb), np.median((d[:, 6] >> 32) / nb),
        np.median(d[:, 7] / nb)))
if not cyc.any() and d[:, 6].any():
    print("setup us %.2f, Q stored us %.2f (from CTA start)" % (np.median(d[:, 6] - st_) / 1e3, np.median(d[:, 7] - st_) / 1e3))
print("tiles", n, "kernel span us", (end.max() - t0) / 1e3)
print("start spread us", (st_.max() - t0) / 1e3)
pro = (mma0 - st_) / 1e3; loop = (mma1 - mma0) / 1e3; epi = (end - mma1) / 1e3
print("prologue us mean/max", pro.mean(), pro.max(), " loop us mean/max", loop.mean(), loop.max(), " epi mean/max", epi.mean(), epi.max())
print("loop ns per block", np.median((mma1 - mma0) / nb))
# per-SM busy
busy = {}
for i in range(n):
    busy.setdefault(int(sm[i]), []).append((st_[i] - t0, end[i] - t0, nb[i]))
fin = sorted((max(e for _, e, _ in v) / 1e3, k, len(v), sum(b for *_, b in v)) for k, v in busy.items())
print("SM finish us min/median/max", fin[0][0], fin[len(fin) // 2][0], fin[-1][0])
print("slowest SMs", fin[-5:])
print("fastest SMs", fin[:5])
print("nb hist", np.bincount(nb.astype(int))[np.bincount(nb.astype(int)) > 0], np.unique(nb))
