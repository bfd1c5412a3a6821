"""In-graph kernel timeline of one decode step (CUPTI via torch.profiler):
per-kernel durations, gaps and overlaps of a CUDA-graph replay.
python tools/step_trace.py [--model 70b|8b] [--world 8] [--rank 0] [--layers-shown 2]"""
import argparse, json, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2511_14116_b200.placement import make_placement
from paper_2511_14116_b200.recovery import plan_weight_recovery

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--model", default="70b")
ap.add_argument("--layers-shown", type=int, default=2)
a = ap.parse_args()
model = bench.llama70b() if a.model == "70b" else bench.llama8b()
base = 8 if a.model == "70b" else a.world
plan = make_placement("hybrid", model, range(base))
alive = list(range(base))
for f in (7, 3, 5)[:base - a.world]:
    alive = [g for g in alive if g != f]
    plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
routing = bench.route(64, alive, 4096)
eng = bench.build_rank(model, plan, a.rank, routing, 64, 4096, None, 0)
bench.time_graph(eng.step, 3, 3)  # capture + warm
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        eng.step()
    torch.cuda.synchronize()
path = "/tmp/step_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# keep the second step
L = model.num_layers
per_step = len(ev) // 2
ev = ev[per_step:]
t0 = ev[0]["ts"]
def short(n):
    for k in ("gemm_skinny", "decode_cta", "ar_residual", "swiglu", "plan_pages", "nvjet", "backup"):
        if k in n:
            return k
    return n[:30]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in ev:
    tot[short(e["name"])] += e["dur"]; cnt[short(e["name"])] += 1
span = ev[-1]["ts"] + ev[-1]["dur"] - t0
print(f"step span {span:.1f} us, {len(ev)} kernels")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {k:14s} {cnt[k]:5d} launches  {v:9.1f} us  avg {v / cnt[k]:7.2f}")
busy = 0.0
end = t0
for e in ev:
    s, f = e["ts"], e["ts"] + e["dur"]
    if f > end:
        busy += f - max(s, end)
        end = f
print(f"  union of kernel intervals {busy:.1f} us (idle {span - busy:.1f} us)")
print("first layers (start offset us, duration us, gap to previous end):")
prev_end = t0
shown = ev[: (len(ev) // L) * a.layers_shown]
for e in shown:
    print(f"  {e['ts'] - t0:9.2f} {e['dur']:7.2f} {e['ts'] - prev_end:+7.2f}  {short(e['name'])}")
    prev_end = e["ts"] + e["dur"]
