"""Full decode step: cuBLAS vs tcgen05 projections (graph-timed)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2511_14116_b200.placement import make_placement
from paper_2511_14116_b200.recovery import plan_weight_recovery
for label, model, world, rank in (("8B N=1", bench.llama8b(), 1, 0), ("70B N=8 r0", bench.llama70b(), 8, 0),
                                   ("70B N=5 r0", bench.llama70b(), 5, 0)):
    plan = make_placement("hybrid", model, range(8 if world < 8 else world))
    alive = list(range(8))
    for f in (7, 3, 5)[:8 - world]:
        alive = [g for g in alive if g != f]
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
    routing = bench.route(64, alive, 4096)
    for be in ("cublas", "tcgen05"):
        bench.GEMM_BACKEND = be
        eng = bench.build_rank(model, plan, rank, routing, 64, 4096, None, 0)
        ms = bench.time_graph(eng.step, 10, 3)
        print(f"{label:12s} {be:8s} step {ms:.3f} ms", flush=True)
        del eng; torch.cuda.empty_cache()
