"""The multi-process failure path (cluster.ClusterRank): real processes (all
on cuda:0 here -- one process per GPU on a node), the fused exchange over
IPC-mapped peer buffers, K5 token backup into per-rank /dev/shm mirrors, a
rank that EXITS, survivors that regroup over the store, pull the plan's
weight slices from the node's host weight store (pcie_host) and from each
other (nvlink_peer), adopt the on-demand target in place, restore the lost
KV from the dead rank's mirror (K6) and resume.

Checked against a single-process emulation: the same model / KV history /
inputs stepped on hybrid(4), then FRESH engines built on each on-demand
target placement (with the emulated world's KV copied in) stepped once --
the survivors' first step after every recovery must be bit-identical.
"""

import json
import os
import socket
import subprocess
import sys
from datetime import timedelta

import numpy as np
import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(ROOT, "tests"))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulated(world, fails, steps_before, batch, ctx):
    """Expected x after `steps_before` steps and after each failure's first
    step (single process, fresh engines per placement)."""
    from _cluster_worker import fill_kv, tiny_model, x0
    from paper_2511_14116_b200.hybrid import HybridDecodeRank, emulated_parallel_step
    from paper_2511_14116_b200.kvcache import item_keys
    from paper_2511_14116_b200.failover import route_for
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    from paper_2511_14116_b200.cluster import _decode_requests
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.scheduler import SchedulerState, route_request
    model = tiny_model()
    plan = make_placement("hybrid", model, range(world))
    st = SchedulerState(token_budget=2048, rank_set=tuple(range(world)))
    routing = {i: route_request(st, Request(id=i, arrival_time=0.0, input_len=ctx - 1,
                                            output_len=1)) for i in range(batch)}

    def build(plan, routing):
        owner = owner_array(plan, model.num_kv_heads)
        shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
        out = []
        for g in plan.alive:
            e = HybridDecodeRank(model, owner, g, routing, batch, ctx, seed=3, mlp=True,
                                 shard_owner=shards, page_order="shuffled")
            e.set_lengths([ctx] * batch)
            out.append(e)
        return out

    ranks = build(plan, routing)
    for e in ranks:
        fill_kv(e, ctx)
    x = x0(batch, model.hidden_dim).cuda()
    for _ in range(steps_before):
        x = emulated_parallel_step(ranks, x)
    outs = [x.cpu()]
    alive = list(range(world))
    requests = _decode_requests(batch, ctx, 1024)
    for f in fails:
        alive = [g for g in alive if g != f]
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
        routing = route_for(sorted(requests), requests, routing, alive)
        new = build(plan, routing)
        # KV of every (layer, head, request) from whichever old engine held it
        src = {}
        for e in ranks:
            bt = e.cache.block_table.cpu().numpy()
            for i, k in enumerate(item_keys(e.work).tolist()):
                src[k] = (e, bt[i])
        for e in new:
            bt = e.cache.block_table.cpu().numpy()
            for i, k in enumerate(item_keys(e.work).tolist()):
                old, row = src[k]
                n = (ctx + 15) // 16
                e.cache.pool[torch.from_numpy(bt[i, :n].astype(np.int64)).cuda()] = \
                    old.cache.pool[torch.from_numpy(row[:n].astype(np.int64)).cuda()]
        ranks = new
        x = emulated_parallel_step(ranks, x)
        outs.append(x.cpu())
    return outs


@pytest.mark.parametrize("world,fails", [(4, (3, 1))])
def test_processes_lose_ranks_and_resume_bit_exact(tmp_path, world, fails):
    batch, ctx, steps_before, reserve = 6, 40, 2, 256
    port = _port()
    store = torch.distributed.TCPStore("127.0.0.1", port, None, True,
                                       timeout=timedelta(seconds=120))
    job = f"fst{os.getpid()}"
    worker = os.path.join(ROOT, "tests", "_cluster_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), str(port), job,
                               str(tmp_path), str(steps_before), ",".join(map(str, fails)),
                               str(batch), str(ctx), str(reserve)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=600)
            logs.append(out.decode(errors="replace"))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
        from paper_2511_14116_b200.cluster import shm_cleanup
        shm_cleanup(job)
    bad = [r for r, p in enumerate(procs) if p.returncode != 0]
    assert not bad, "\n".join(f"rank {r} (rc {procs[r].returncode}):\n{logs[r][-2500:]}"
                               for r in bad)
    del store
    exp = _emulated(world, fails, steps_before, batch, ctx)
    alive = list(range(world))
    for r in alive:
        assert torch.equal(torch.load(tmp_path / f"x_pre_r{r}.pt"), exp[0]), r
    for k, f in enumerate(fails):
        alive = [g for g in alive if g != f]
        for r in alive:
            got = torch.load(tmp_path / f"x_fail{k}_r{r}.pt")
            assert torch.equal(got, exp[k + 1]), (k, r, float((got.float() - exp[k + 1].float())
                                                             .abs().max()))
            rep = json.load(open(tmp_path / f"rep_fail{k}_r{r}.json"))
            # executed bytes == the reference plans' bytes for this GPU
            assert rep["weight_pcie_bytes"] == rep["planned_weight_pcie_bytes"], rep
            assert rep["weight_nvlink_bytes"] == rep["planned_weight_nvlink_bytes"], rep
            assert rep["kv_restore_bytes"] >= rep["planned_kv_pcie_bytes"], rep
            assert rep["recovery_ms"] > 0
