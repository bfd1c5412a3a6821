"""CPU tests of the drop-in API (routing, backup, recovery planners) against
golden vectors produced by the live reference."""

import numpy as np
import pytest

from paper_2511_14116_b200.core import ClusterSpec, ModelSpec, Request
from paper_2511_14116_b200.placement import plan_from_tables, owner_array
from paper_2511_14116_b200.recovery import (BackupState, advance_backup, plan_kv_recovery,
                                            plan_weight_recovery, validate_weight_plan)
from paper_2511_14116_b200.scheduler import SchedulerState, route_request


def _ikeys(d):
    return {int(k): v for k, v in d.items()}


def _toy(L, H, shards):
    return ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H, head_dim=8, hidden_dim=32,
                     ffn_intermediate_dim=96, ffn_num_shards=shards)


def test_routing_golden(golden):
    g = golden("routing")
    for c in g["cases"]:
        st = SchedulerState(token_budget=2048, rank_set=tuple(range(c["n"])),
                            include_decode_in_workload=c["include_decode"])
        ranks = [route_request(st, Request(id=i, arrival_time=0.0, input_len=a, output_len=b))
                 for i, (a, b) in enumerate(c["requests"])]
        assert ranks == c["ranks"]
        assert [st.workload[r] for r in range(c["n"])] == c["workload"]
    inter = g["interleaved"]
    st = SchedulerState(token_budget=64, rank_set=(0, 1, 2))
    reqs = [Request(id=i, arrival_time=0.0, input_len=a, output_len=b)
            for i, (a, b) in enumerate(inter["requests"])]
    for kind, rid, rank in inter["events"]:
        if kind == "route":
            assert route_request(st, reqs[rid]) == rank
        else:
            reqs[rid].tokens_decoded += 1
            st.note_decode_token(reqs[rid], rank)
    assert [st.workload[r] for r in range(3)] == inter["workload"]


def test_weight_recovery_golden(golden):
    for c in golden("recovery")["weight"]:
        m = _toy(c["L"], c["H"], c["num_shards"])
        old = plan_from_tables(c["mode"], np.array(c["owner"]), c["shard_owner"], range(c["n"]))
        rp = plan_weight_recovery(m, old, c["new_alive"], c["wmode"])
        got = [[t.dest_gpu, t.num_bytes, t.medium, t.content, list(t.detail)]
               for t in rp.transfers]
        assert got == c["transfers"]
        tgt = rp.target_plan(c["mode"], m)
        assert owner_array(tgt, c["H"]).tolist() == c["target_owner"]
        assert [tgt.ffn.owner[s] for s in range(c["num_shards"])] == c["target_shards"]
        validate_weight_plan(old, rp, m)


def test_kv_recovery_golden(golden):
    for c in golden("recovery")["kv"]:
        m = _toy(c["L"], c["H"], 12)
        old = plan_from_tables("x", np.array(c["old_owner"]), [0] * 12, range(c["n"]))
        new = plan_from_tables("x", np.array(c["new_owner"]), [c["surv"][0]] * 12, c["surv"])
        b = BackupState(host_memory_bytes=10 ** 12, kv_bytes_per_token=m.kv_bytes_per_token())
        for r, w in _ikeys(c["backed"]).items():
            b.register(r)
            b.backed[r] = w
        rp = plan_kv_recovery(b, old, new, m, _ikeys(c["contexts"]), _ikeys(c["old_routing"]),
                              _ikeys(c["new_routing"]), c["mode"])
        got = [[t.dest_gpu, t.num_bytes, t.medium, t.content, list(t.detail)]
               for t in rp.transfers]
        assert got == c["transfers"]
        assert rp.recompute_tokens == _ikeys(c["recompute_tokens"])
        assert rp.recompute_start == _ikeys(c["recompute_start"])


def test_backup_golden(golden):
    for c in golden("recovery")["backup"]:
        b = BackupState(host_memory_bytes=c["host"], kv_bytes_per_token=c["unit"])
        cl = ClusterSpec(num_gpus=8, hbm_bytes_per_gpu=10 ** 9, pcie_bw_per_gpu=c["pcie"],
                         nvlink_bw_per_gpu=1e12, allreduce_alpha=0.0, allreduce_beta=0.0,
                         host_memory_bytes=c["host"])
        for step in c["steps"]:
            for r in step["finish"]:
                b.mark_finished(r)
            advance_backup(b, step["elapsed"], _ikeys(step["new"]), cl, c["frac"])
            assert b.backed == _ikeys(step["backed"])
            assert b.lag == _ikeys(step["lag"])
            assert b.host_bytes_used == step["used"]
            assert b.carry_bytes == step["carry"]
            assert b.evictions == step["evictions"]


def test_llama70b_chain_via_api(golden):
    from paper_2511_14116_b200.core import load_config
    from paper_2511_14116_b200.placement import make_placement
    import os
    from conftest import ROOT
    m = load_config(os.path.join(ROOT, "paper_2511_14116_b200", "data", "llama70b.toml"))[0]
    for chain in golden("placement")["chains"]:
        plan = make_placement(chain["mode"], m, range(8))
        alive = list(range(8))
        for step in chain["steps"]:
            alive = [g for g in alive if g != step["fail"]]
            rp = plan_weight_recovery(m, plan, alive, "on_demand")
            assert rp.total_pcie_bytes() == step["total_pcie"]
            assert {str(k): v for k, v in rp.pcie_bytes_by_gpu().items()} == step["pcie_by_gpu"]
            assert {str(k): v for k, v in rp.nvlink_bytes_by_gpu().items()} == \
                step["nvlink_by_gpu"]
            plan = rp.target_plan(chain["mode"], m)
            assert owner_array(plan, 8).tolist() == step["owner"]
