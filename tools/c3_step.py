"""One C3 (Llama-3-70B-shaped, B=64, ctx 4096) decode step of one rank of a
hybrid(8) / on-demand-shrunk world, for ncu launch lists and graph timing:
python tools/c3_step.py --world 8 --rank 0 [--gemm tcgen05|cublas] [--steps 2]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2511_14116_b200.placement import make_placement
from paper_2511_14116_b200.recovery import plan_weight_recovery

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--gemm", default="tcgen05")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--time", action="store_true", help="graph-time the step instead")
ap.add_argument("--model", default="70b")
ap.add_argument("--config", type=int, default=0, help="K1 kernel config")
a = ap.parse_args()
model = bench.llama70b() if a.model == "70b" else bench.llama8b()
base = 8 if a.model == "70b" else a.world
plan = make_placement("hybrid", model, range(base))
alive = list(range(base))
for f in (7, 3, 5)[:base - a.world]:
    alive = [g for g in alive if g != f]
    plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
routing = bench.route(64, alive, 4096)
bench.GEMM_BACKEND = a.gemm
eng = bench.build_rank(model, plan, a.rank, routing, 64, 4096, None, a.config)
if a.time:
    ms = bench.time_graph(eng.step, 10, 3)
    wb, kb = eng.weight_bytes(), bench.step_kv_bytes(eng)
    print(f"{a.model} world {a.world} rank {a.rank} {a.gemm} K1 config {a.config}: step {ms:.3f} ms, weights {wb/1e9:.2f} GB "
          f"kv {kb/1e9:.2f} GB, {(wb+kb)/ms/1e6:.0f} GB/s")
else:
    for _ in range(a.steps):
        eng.step()
    torch.cuda.synchronize()
