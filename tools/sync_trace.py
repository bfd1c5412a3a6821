"""CUPTI timeline of C2 decode steps replayed back to back vs each after a
host sync: per-layer span of each step (where does the post-sync step lose
its ~85 us?).  python tools/sync_trace.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2511_14116_b200.placement import make_placement  # noqa: E402

model = bench.llama8b()
plan = make_placement("hybrid", model, [0])
eng = bench.build_rank(model, plan, 0, {r: 0 for r in range(64)}, 64, 4096, None, 0)
bench.time_graph(eng.step, 3, 3)
L = model.num_layers


def steps(sync):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(4):
            eng.step()
            if sync:
                torch.cuda.current_stream().synchronize()
        torch.cuda.synchronize()
    path = f"/tmp/sync_trace_{int(sync)}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    per = len(ev) // 4
    out = []
    for k in range(1, 4):
        st = ev[k * per:(k + 1) * per]
        t0 = st[0]["ts"]
        lay = []
        for l in range(L):
            a = st[l * (per // L)]["ts"]
            b = max(e["ts"] + e["dur"] for e in st[l * (per // L):(l + 1) * (per // L)])
            lay.append((a - t0, b - a))
        span = max(e["ts"] + e["dur"] for e in st) - t0
        gap = st[0]["ts"] - (ev[k * per - 1]["ts"] + ev[k * per - 1]["dur"])
        out.append((span, gap, lay))
    return out


for sync in (False, True):
    res = steps(sync)
    print(f"== {'sync per step' if sync else 'back to back'}")
    for span, gap, lay in res:
        first = " ".join(f"{d:.1f}" for _, d in lay[:4])
        last = " ".join(f"{d:.1f}" for _, d in lay[-4:])
        kinds = {}
        print(f"  step span {span:.1f} us, gap before {gap:.1f} us; layer spans first 4: {first}; "
              f"last 4: {last}; mean {sum(d for _, d in lay) / L:.1f}")
