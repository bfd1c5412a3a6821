"""Per-CTA phase timeline of the skinny tcgen05 GEMM (fs_gemm_debug_timestamps):
one eager launch after warm-up, stamps (globaltimer ns) per CTA:
0 start (TMEM allocated), 5/6 producer before/after the PDL wait, 1 first
stage landed (MMA warp), 2 last MMA committed, 3 tile in shared memory, 7 cluster
barrier passed, 10 slice reduced + written, 4 end.   python tools/gemm_tl.py K N [K N ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14116_b200 import _native as N
from paper_2511_14116_b200.gemm import SkinnyGemm, STORE, PackedWeight
args = [int(a) for a in sys.argv[1:]]
for K, Nc in zip(args[0::2], args[1::2]):
    reps = max(2, int(1.2e9 // (K * Nc * 2)))
    ws = [PackedWeight(torch.randn(K, Nc, device="cuda").to(torch.bfloat16)) for _ in range(reps)]
    x = torch.randn(64, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(64, Nc, device="cuda", dtype=torch.bfloat16)
    sk = SkinnyGemm(Nc)
    dbg = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
    for i in range(reps):
        sk(x, ws[i], out, STORE)
    torch.cuda.synchronize()
    N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(dbg.data_ptr()))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); sk(x, ws[1], out, STORE); e.record(); torch.cuda.synchronize()
    N.lib.fs_gemm_debug_timestamps(N.C.c_void_p(0))
    d = dbg.view(1024, 16).cpu().numpy().astype(np.int64)
    d = d[d[:, 0] > 0]
    t0 = d[:, 0].min()
    sm = d[:, 12]
    print(f"  distinct SMs {len(set(sm.tolist()))} for {len(d)} CTAs (max CTAs on one SM "
          f"{max(np.bincount(sm)) if len(sm) else 0})")
    print(f"K {K} N {Nc}: {len(d)} CTAs, event {s.elapsed_time(e)*1e3:.1f} us; span {(d[:, 4].max() - t0)/1e3:.1f} us")
    for name, a, b in (("start spread", None, 0), ("start->pdl wait", 0, 5), ("pdl wait", 5, 6),
                       ("start->first stage", 0, 1), ("first stage->MMA done", 1, 2),
                       ("MMA done->partials stored", 2, 3), ("tile stored->cluster barrier", 3, 7),
                       ("MMA issued->acc ready", 2, 8), ("cluster barrier->received", 7, 9),
                       ("received->arrived", 9, 11), ("arrived->reduced", 11, 10),
                       ("write: enter->1st chunk", 13, 14), ("write: 1st chunk->done", 14, 15),
                       ("arrived->write enter", 11, 13), ("write done->stamp10", 15, 10),
                       ("reduced->end", 10, 4), ("->CTA end", 3, 4), ("start->end", 0, 4), ("t0->end", None, 4)):
        v = (d[:, b] - (t0 if a is None else d[:, a])) / 1e3
        ok = (d[:, b] > 0) & ((d[:, a] > 0) if a is not None else True)
        if ok.any():
            v = v[ok]
            print(f"  {name:28s} min {v.min():6.2f} median {np.median(v):6.2f} max {v.max():6.2f} us")
