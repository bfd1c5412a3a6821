"""One C5 mixed iteration on one rank (bench.mixed_trace shapes) for an ncu
launch list: ncu --metrics gpu__time_duration.sum python tools/c5_launches.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
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
routing, steps, caps = bench.mixed_iterations(bench.sharegpt_trace(), alive, 2048, 24, 2)
eng = HybridServingRank(model, owner, 1, routing, caps, max(s.num_tokens for s in steps),
                        seed=0, shard_owner=shards)
eng.fill_random_kv(101)
plans = [eng.plan(s) for s in steps]
xs = [torch.randn((s.num_tokens, model.hidden_dim), device="cuda").to(torch.bfloat16) for s in steps]
eng.serve(plans[0], xs[0])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
eng.serve(plans[1], xs[1])
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
