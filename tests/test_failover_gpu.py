"""A GPU failure handled end to end on the emulated world (failover.py):
serve with incremental KV backup, lose a GPU, adopt the on-demand target,
restore the lost GPU's KV from its pinned-host mirror (K6), recompute the
tails past the backup watermark, resume -- and the served outputs keep
matching a world-1 run of the same iterations that never failed.  Restored
pages are checked byte for byte against the lost GPU's pages."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _model():
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=2, num_kv_heads=8, num_q_heads=32, head_dim=128,
                     hidden_dim=512, ffn_intermediate_dim=1024, ffn_num_shards=16)


def _close(got, ref, tol=3e-2):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    assert err.max().item() <= tol * max(1.0, ref.abs().max().item()), err.max().item()
    assert (err.mean() / ref.abs().mean()).item() <= 1e-2


@pytest.mark.parametrize("world,fails", [(4, [3]), (8, [7, 3])])
def test_failover_resumes_with_identical_outputs(world, fails):
    from paper_2511_14116_b200.failover import EmulatedCluster
    model = _model()
    inputs = [(40, 8), (100, 6), (17, 10), (64, 7), (33, 9), (90, 5)]
    cl = EmulatedCluster(model, world, inputs, token_budget=64, seed=5)
    ref = EmulatedCluster(model, 1, inputs, token_budget=64, seed=5)
    gen = torch.Generator().manual_seed(1)

    def run(n):
        for _ in range(n):
            b = cl.next_batch()
            if not b.num_tokens:
                return
            x = torch.randn((b.num_tokens, model.hidden_dim), generator=gen).to(torch.bfloat16)
            _close(cl.step(b, x), ref.step(b, x))

    run(3)
    for g in fails:
        rep = cl.fail(g)
        assert rep.world_after == len(cl.alive)
        assert rep.restored_exact
        assert rep.kv_restore_bytes > 0
        # the lost GPU's slices that were not yet on the host (partial pages)
        # are recomputed, everything else restored
        assert rep.recompute_tokens >= 0
        run(3)
    # every request finishes on the shrunk world
    run(40)
    assert all(r.tokens_decoded == r.output_len for r in cl.requests)
    # the measured run in the reference's metrics wire format
    from paper_2511_14116_b200.metrics import summarize
    log = cl.metrics()
    kinds = [r["kind"] for r in log.records]
    assert kinds.count("request") == len(inputs) and kinds.count("failure") == len(fails)
    assert kinds.count("reconfig_done") == len(fails) and kinds[-1] == "run_summary"
    s = summarize(log)
    assert s["requests_completed"] == len(inputs)
    assert s["prefill_tokens"] == sum(a for a, _ in inputs)
    assert s["decode_tokens"] == sum(o for _, o in inputs)
    assert s["ttft"]["max"] > 0 and s["tbt"]["max"] > 0


def _run_pair(cl, ref, model, gen, n):
    """n iterations of cl's batches on both worlds; stops when idle."""
    for _ in range(n):
        b = cl.next_batch()
        if not b.num_tokens:
            return False
        x = torch.randn((b.num_tokens, model.hidden_dim), generator=gen).to(torch.bfloat16)
        _close(cl.step(b, x), ref.step(b, x))
    return True


def test_rejoin_reloads_fresh_and_resumes():
    """GPU 3 fails, then rejoins: the expanded world's fresh placement is
    adopted in place by the survivors (KV of re-placed heads moved between
    GPUs, new slots' weights reloaded from the host store), the rejoined GPU
    reloads its whole assignment -- outputs keep matching world 1."""
    from paper_2511_14116_b200.failover import EmulatedCluster
    from paper_2511_14116_b200.placement import make_placement, owner_array
    model = _model()
    inputs = [(40, 12), (100, 10), (17, 14), (64, 11), (33, 13), (90, 9)]
    cl = EmulatedCluster(model, 4, inputs, token_budget=64, seed=5)
    ref = EmulatedCluster(model, 1, inputs, token_budget=64, seed=5)
    gen = torch.Generator().manual_seed(2)
    _run_pair(cl, ref, model, gen, 3)
    rep = cl.fail(3)
    assert rep.restored_exact and rep.world_after == 3
    _run_pair(cl, ref, model, gen, 2)
    rep = cl.rejoin(3)
    assert cl.alive == [0, 1, 2, 3]
    assert rep.weight_pcie_bytes > 0 and rep.kv_move_bytes > 0
    # the expanded world runs the fresh hybrid(4) placement again
    fresh = make_placement("hybrid", model, range(4))
    assert np.array_equal(owner_array(cl.plan, 8), owner_array(fresh, 8))
    while _run_pair(cl, ref, model, gen, 5):
        pass
    assert all(r.tokens_decoded == r.output_len for r in cl.requests)
    kinds = [r["kind"] for r in cl.metrics().records]
    assert kinds.count("recovery") == 1 and kinds.count("reconfig_done") == 2


def _tight_cluster(model, world, inputs, fail):
    """HBM per GPU such that every request fits the full world but the
    shrink after losing ``fail`` forces preemption (controller only)."""
    import dataclasses
    from paper_2511_14116_b200.controller import WorldController
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.failover import default_cluster
    from paper_2511_14116_b200.placement import make_placement, weight_bytes_per_gpu
    base = default_cluster(world)

    def trial(hbm):
        c = WorldController(model, dataclasses.replace(base, hbm_bytes_per_gpu=hbm))
        for i, (a, o) in enumerate(inputs):
            c.add_request(Request(id=i, arrival_time=0.0, input_len=a, output_len=o))
        c.start()
        c.admit()
        if c.waiting:
            return None
        d = c.fail(fail)
        return len(c.apply(d))

    w = max(weight_bytes_per_gpu(make_placement("hybrid", model, [g for g in range(world)
                                                                  if g != fail]),
                                 model).values())
    best = None
    for extra in range(1 << 13, 1 << 24, 1 << 13):
        n = trial(w + extra)
        if n is not None and n >= 1 and (best is None or n <= best[1]):
            best = (w + extra, n)
        if n == 0:
            break
    assert best is not None, "no preempting capacity found"
    return dataclasses.replace(base, hbm_bytes_per_gpu=best[0]), best[1]


def test_shrink_preempts_over_capacity_and_readmits():
    """After the shrink the survivors' KV reservations exceed HBM: the
    latest arrivals are preempted (simulation.py:273-310: progress reset,
    back to the waiting line), re-admitted once capacity frees, re-prefilled
    and finished; the survivors' outputs keep matching world 1."""
    from paper_2511_14116_b200.failover import EmulatedCluster
    model = _model()
    inputs = [(40, 6), (100, 5), (17, 8), (64, 7), (33, 9), (90, 5), (50, 6), (20, 7)]
    cluster, _ = _tight_cluster(model, 4, inputs, 3)
    cl = EmulatedCluster(model, 4, inputs, token_budget=64, seed=5, cluster=cluster)
    ref = EmulatedCluster(model, 1, inputs, token_budget=64, seed=5)
    assert len(cl.residents) == len(inputs)
    gen = torch.Generator().manual_seed(3)
    _run_pair(cl, ref, model, gen, 3)
    rep = cl.fail(3)
    n_pre = len(rep.preempted)
    assert n_pre >= 1
    # latest arrivals first (equal arrival times: highest ids first)
    assert rep.preempted == list(range(len(inputs) - 1, len(inputs) - 1 - n_pre, -1))
    for rid in rep.preempted:
        r = cl.requests[rid]
        assert r.tokens_prefilled == 0 and r.tokens_decoded == 0 and rid not in cl.residents
    while _run_pair(cl, ref, model, gen, 5):
        pass
    assert all(r.tokens_decoded == r.output_len for r in cl.requests)
    log = cl.metrics()
    assert len(log.of_kind("preemption")) == n_pre
    assert log.of_kind("run_summary")[-1]["preempted"] == n_pre
