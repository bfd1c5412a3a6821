"""The host controller's reconfiguration decisions (controller.WorldController)
against the live reference's serving loop (tests/golden/reconfig.json,
oracle/gen_golden.py gen_reconfig): a Llama-3-70B world losing GPU 7, then
GPU 3, then GPU 7 rejoining -- on-demand shrink targets, the fresh expansion
plan, re-routing, router rebuild, capacities, reservations and (small-HBM
scenario) the preempted residents and the waiting line.  Bit-exact."""

import os
from collections import deque

import numpy as np
import pytest

from conftest import ROOT


def _controller(scn, ev):
    import dataclasses
    from paper_2511_14116_b200.controller import WorldController
    from paper_2511_14116_b200.core import Request, load_config
    from paper_2511_14116_b200.placement import plan_from_tables
    model, cluster = load_config(os.path.join(ROOT, "paper_2511_14116_b200", "data",
                                              "llama70b.toml"))
    cluster = dataclasses.replace(cluster, hbm_bytes_per_gpu=scn["hbm_bytes_per_gpu"],
                                  switch_latency=scn["switch_latency"])
    c = WorldController(model, cluster)
    c.alive = set(ev["alive"])
    c.serving = list(ev["serving"])
    c.plan = plan_from_tables(ev["plan_mode"], np.array(ev["owner"], np.int32), ev["shards"],
                              ev["serving"])
    c.tp_total, c.dp_total = c.plan_arrays(c.plan)
    for rid, arr, inp, out, pre, dec in ev["residents"]:
        r = Request(id=rid, arrival_time=arr, input_len=inp, output_len=out,
                    tokens_prefilled=pre, tokens_decoded=dec)
        c.requests[rid] = r
        c.residents.append(rid)
    c.routing = {rid: g for rid, g in ev["routing"]}
    for rid, b in ev["backed"]:
        c.backup.register(rid)
        c.backup.backed[rid] = b
    return c


def _owner(plan, H=8):
    from paper_2511_14116_b200.placement import owner_array
    return owner_array(plan, H).tolist()


@pytest.mark.parametrize("name", ["expand", "preempt"])
def test_reconfiguration_matches_reference(golden, name):
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.scheduler import request_pending_cost
    scn = [s for s in golden("reconfig")["scenarios"] if s["name"] == name][0]
    assert scn["events"]
    if name == "preempt":
        assert scn["reference_stopped"] and "KeyError" in scn["reference_stopped"]
    for ev in scn["events"]:
        c = _controller(scn, ev)
        d = c.plan_reconfigure()
        assert d is not None and d.desired == ev["desired"]
        assert _owner(d.new_plan) == ev["new_owner"]
        assert [d.new_plan.ffn.owner[s] for s in range(d.new_plan.ffn.num_shards)] == \
            ev["new_shards"]
        assert sorted([r, g] for r, g in d.new_routing.items()) == ev["new_routing"]
        assert sorted([r, n] for r, n in d.merged.recompute_tokens.items()) == ev["recompute"]
        assert d.merged.total_pcie_bytes() == ev["pcie_bytes"]
        after = ev["after"]
        # the waiting line at reconfig_done, before the preemptions
        for rid, arr, inp, out, pre, dec in after["waiting_state"]:
            if rid not in c.requests:
                c.requests[rid] = Request(id=rid, arrival_time=arr, input_len=inp,
                                          output_len=out, tokens_prefilled=pre,
                                          tokens_decoded=dec)
        pending = {rid: request_pending_cost(c.requests[rid], c.kappa) for rid in c.residents}
        c.waiting = deque(w for w in after["waiting"] if w not in after["preempted"])
        pre = c.apply(d)
        assert pre == after["preempted"]
        assert c.serving == after["serving"]
        assert sorted([r, g] for r, g in c.routing.items()) == after["routing"]
        assert c.residents == after["residents"]
        assert list(c.waiting) == after["waiting"]
        assert sorted([g, v] for g, v in c.capacity.items()) == after["capacity"]
        assert sorted([g, v] for g, v in c.reserved.items()) == after["reserved"]
        # router workload: the reference keeps a preempted request's pending
        # cost queued (its next iteration then fails); we withdraw it
        want = dict(after["workload"])
        for rid in pre:
            rank = d.new_routing.get(rid)
            want[rank] = max(0.0, want[rank] - pending[rid])
        assert {g: v for g, v in c.sched.workload.items()} == pytest.approx(want, rel=0, abs=1e-9)
        if name == "expand":
            assert {g: v for g, v in c.sched.workload.items()} == dict(after["workload"])
