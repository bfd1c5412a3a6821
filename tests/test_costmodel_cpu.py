"""The restated iteration-time model (costmodel.py of the reference) against
the live reference's numbers (tests/golden/costmodel.json), and the
calibration fit recovering known constants."""

import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2511_14116_b200.core import load_config
from paper_2511_14116_b200.costmodel import (BatchWork, ChunkWork, CostParams, PlanCost,
                                             calibrate)
from paper_2511_14116_b200.placement import make_placement
from paper_2511_14116_b200.recovery import plan_weight_recovery


def _llama70b():
    return load_config(os.path.join(ROOT, "paper_2511_14116_b200", "data", "llama70b.toml"))


def _plan(model, mode, world, fail):
    plan = make_placement(mode, model, range(world))
    if fail is not None:
        alive = [g for g in range(world) if g != fail]
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan(mode, model)
    return plan


def _work(chunks):
    return BatchWork([ChunkWork.prefill(*c[1:]) if c[0] == "prefill" else ChunkWork.decode(*c[1:])
                      for c in chunks])


def test_matches_reference_golden(golden):
    import dataclasses
    g = golden("costmodel")
    model, cluster = _llama70b()
    # the reference's node (H100-class) all-reduce constants
    cluster = dataclasses.replace(cluster, allreduce_alpha=g["allreduce"][0],
                                  allreduce_beta=g["allreduce"][1])
    p = CostParams.from_model(model)
    assert [p.attn_flop_per_head_token, p.attn_flop_per_head_ctx_token,
            p.ffn_flop_per_token_per_shard, p.gpu_throughput] == g["params"]
    for c in g["cases"]:
        pc = PlanCost(_plan(model, c["mode"], c["world"], c["fail"]), model, p, cluster)
        work = _work(c["chunks"])
        assert pc.iteration_time(work) == pytest.approx(c["iteration_time"], rel=1e-12)
        got = pc.per_gpu_compute_time(work)
        for gpu, t in c["per_gpu"].items():
            assert got[int(gpu)] == pytest.approx(t, rel=1e-12)


def test_features_reproduce_compute_time():
    model, cluster = _llama70b()
    p = CostParams.from_model(model)
    pc = PlanCost(_plan(model, "hybrid", 8, 7), model, p, cluster)
    work = _work([["decode", r, r % 7, 4095] for r in range(64)] +
                 [["prefill", 64, 3, 100, 300]])
    f = pc.features(work)
    want = pc.per_gpu_compute_time(work)
    coef = np.array([p.attn_flop_per_head_token, p.attn_flop_per_head_ctx_token,
                     p.ffn_flop_per_token_per_shard]) / p.gpu_throughput
    for i, g in enumerate(pc.ranks):
        assert f[i] @ coef == pytest.approx(want[g], rel=1e-12)


def test_calibration_recovers_constants():
    model, cluster = _llama70b()
    true = CostParams(attn_flop_per_head_token=2e-9, attn_flop_per_head_ctx_token=3e-12,
                      ffn_flop_per_token_per_shard=5e-9, gpu_throughput=1.0)
    rng = np.random.default_rng(0)
    samples = []
    for world, fail in ((8, None), (8, 7), (6, None)):
        pc_true = PlanCost(_plan(model, "hybrid", world, fail), model, true, cluster)
        for _ in range(3):
            ranks = pc_true.ranks
            work = _work([["decode", r, ranks[r % len(ranks)], int(rng.integers(100, 8000))]
                          for r in range(64)] +
                         [["prefill", 64 + i, ranks[i % len(ranks)], 0, int(rng.integers(1, 500))]
                          for i in range(3)])
            samples.append((pc_true, work, pc_true.per_gpu_compute_time(work)))
    fit, err = calibrate(samples)
    assert err < 1e-6
    assert fit.attn_flop_per_head_token == pytest.approx(2e-9, rel=1e-5)
    assert fit.attn_flop_per_head_ctx_token == pytest.approx(3e-12, rel=1e-5)
    assert fit.ffn_flop_per_token_per_shard == pytest.approx(5e-9, rel=1e-5)


def test_b200_calibration_recovers_weight_and_fixed_terms():
    """The extended model (reference features + weight bytes + fixed) is
    recovered from synthetic measurements and predicts HELD-OUT worlds."""
    from paper_2511_14116_b200.costmodel import CalibratedCost, calibrate_b200, rms_error
    model, cluster = _llama70b()
    true = CalibratedCost([2e-9, 3e-12, 5e-9, 1.6e-13, 4e-4])
    ref = CostParams.from_model(model)
    rng = np.random.default_rng(1)

    def samples(worlds):
        out = []
        for world, fail in worlds:
            pc = PlanCost(_plan(model, "hybrid", world, fail), model, ref, cluster)
            for _ in range(3):
                ranks = pc.ranks
                work = _work([["decode", r, ranks[r % len(ranks)], int(rng.integers(100, 8000))]
                              for r in range(64)] +
                             [["prefill", 64 + i, ranks[i % len(ranks)], 0,
                               int(rng.integers(1, 500))] for i in range(3)])
                out.append((pc, work, true.per_gpu_time(pc, work)))
        return out
    train, test = samples([(8, None), (8, 7)]), samples([(6, None), (5, None)])
    fit, err = calibrate_b200(train)
    assert err < 1e-6
    assert rms_error(fit.per_gpu_time, test) < 1e-6
