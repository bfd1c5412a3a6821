"""Host cost of HybridServingRank.plan (StepPlan) on the C5 trace: cProfile of
one rank's plans.  python tools/plan_prof.py"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2511_14116_b200.placement import make_placement, owner_array
from paper_2511_14116_b200.recovery import plan_weight_recovery
from paper_2511_14116_b200.serving import HybridServingRank
model = bench.llama70b()
plan = make_placement("hybrid", model, range(8))
alive = [g for g in range(8) if g != 7]
plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
owner = owner_array(plan, model.num_kv_heads)
shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
routing, steps, caps = bench.mixed_iterations(bench.sharegpt_trace(), alive, 2048, 24, 3)
eng = HybridServingRank(model, owner, 0, routing, caps, max(s.num_tokens for s in steps),
                        seed=0, shard_owner=shards)
eng.plan(steps[0])
t0 = time.perf_counter()
for s in steps:
    eng.plan(s)
print("plan ms", (time.perf_counter() - t0) * 1e3 / len(steps))
pr = cProfile.Profile()
pr.enable()
for s in steps:
    eng.plan(s)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
