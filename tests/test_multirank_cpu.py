"""Multi-process (gloo, CPU) tests of the N>1 host path: every rank builds
its work tables from the shared plan + routing, computes its partial of the
hybrid attention (oracle math on CPU), and the all-reduce reproduces the
single-device result -- the exchange structure of refexec.parallel_forward
(refexec.py:283-298) with the rank partition of RankWork."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(L, H, qpk, B, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 40, size=B)
    kv = {(l, h, r): (rng.standard_normal((lens[r], 16)), rng.standard_normal((lens[r], 16)))
          for l in range(L) for h in range(H) for r in range(B)}
    q = rng.standard_normal((L, B, H, qpk, 16))
    wo = rng.standard_normal((L, H, qpk * 16, 8))
    return lens, kv, q, wo


def _partial(owner, rank, routing, L, H, qpk, B, prob):
    from oracle.attention import head_decode
    from paper_2511_14116_b200.kvcache import RankWork
    lens, kv, q, wo = prob
    work = RankWork.build(owner, rank, routing, B)
    out = np.zeros((L, B, 8))
    for i in range(work.n_items):
        layer = int(np.searchsorted(work.seg_items, i, side="right") - 1)
        r, h = int(work.item_req[i]), int(work.item_head[i])
        k, v = kv[(layer, h, r)]
        o = head_decode(q[layer, r, h], k, v, 0.25).reshape(-1)
        out[layer, r] += o @ wo[layer, h]
    return out, work


def _worker(rank, world, port, mode, L, H, qpk, B, seed, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_14116_b200.core import ModelSpec, Request
        from paper_2511_14116_b200.placement import make_placement, owner_array
        from paper_2511_14116_b200.scheduler import SchedulerState, route_request
        m = ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H * qpk, head_dim=16,
                      hidden_dim=8, ffn_intermediate_dim=160)
        plan = make_placement(mode, m, range(world))
        owner = owner_array(plan, H)
        prob = _problem(L, H, qpk, B, seed)
        st = SchedulerState(token_budget=64, rank_set=tuple(range(world)))
        routing = {r: route_request(st, Request(id=r, arrival_time=0.0,
                                                input_len=int(prob[0][r]), output_len=4))
                   for r in range(B)}
        part, work = _partial(owner, rank, routing, L, H, qpk, B, prob)
        t = torch.from_numpy(part)
        dist.all_reduce(t)
        n = torch.tensor([work.n_items], dtype=torch.int64)
        dist.all_reduce(n)
        results[rank] = (t.numpy(), int(n.item()), routing)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("hybrid", 2), ("hybrid", 3), ("cyclic", 3),
                                        ("hybrid", 5)])
def test_allreduce_of_rank_partials_matches_single_device(mode, world):
    L, H, qpk, B, seed = 3, 8, 2, 7, 11
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, mode, L, H, qpk, B, seed, results), nprocs=world,
             join=True)
    owner1 = np.zeros((L, H), dtype=np.int32)
    prob = _problem(L, H, qpk, B, seed)
    ref, _ = _partial(owner1, 0, {r: 0 for r in range(B)}, L, H, qpk, B, prob)
    routing = results[0][2]
    for g in range(world):
        got, n_items, rt = results[g]
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
        assert rt == routing                      # every rank routed identically
        assert n_items == L * H * B               # each (layer, head, request) exactly once
