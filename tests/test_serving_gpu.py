"""The mixed prefill/decode serving iteration (BASELINE config 5) on the GPU:
Alg. 1 batches from the router/batcher (scheduler.py:160-245) executed by
HybridServingRank (K3 append + K8 chunked prefill + K1 decode + projections
+ TP MLP), checked against

* an independent dense torch fp32 reference of the same iterations (same
  bf16 rounding points: projections, attention output, residual), and
* the hybrid partition itself: the N-rank emulation (ordered sum of the
  per-rank partials, refexec.py:283-307) equals the 1-rank result, for the
  hybrid placement and an on-demand shrink target.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _model(qpk=4, L=2):
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=L, num_kv_heads=8, num_q_heads=8 * qpk, head_dim=128,
                     hidden_dim=512, ffn_intermediate_dim=1024, ffn_num_shards=16)


def _iterations(model, ranks, inputs, budget, n_iter):
    """Drive the reference's router + Alg. 1 batcher: returns routing and a
    list of StepBatch (prefill entries + one decode token per request whose
    prefill finished, as simulation.py:413-443)."""
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.scheduler import (SchedulerState, build_prefill_batch,
                                                 route_request)
    from paper_2511_14116_b200.serving import StepBatch
    st = SchedulerState(token_budget=budget, rank_set=tuple(ranks))
    reqs = [Request(id=i, arrival_time=0.0, input_len=a, output_len=o)
            for i, (a, o) in enumerate(inputs)]
    routing = {r.id: route_request(st, r) for r in reqs}
    steps = []
    for _ in range(n_iter):
        b = build_prefill_batch(st)
        dec = [(r.id, r.input_len + r.tokens_decoded - 1) for r in reqs
               if r.tokens_prefilled == r.input_len and 1 <= r.tokens_decoded < r.output_len]
        steps.append(StepBatch(prefill=list(b.entries), decode=dec))
        for r_id, s, n in b.entries:
            reqs[r_id].tokens_prefilled += n
        for r_id, _ in dec:
            reqs[r_id].tokens_decoded += 1
            st.note_decode_token(reqs[r_id], routing[r_id])
        for r in reqs:  # prefill completion emits the first token
            if r.tokens_prefilled == r.input_len and r.tokens_decoded == 0:
                r.tokens_decoded = 1
    caps = [a + o - 1 for a, o in inputs]
    return routing, steps, caps


def _engine(model, owner, rank, routing, caps, shards, max_tokens):
    from paper_2511_14116_b200.serving import HybridServingRank
    return HybridServingRank(model, owner, rank, routing, caps, max_tokens, seed=3,
                             shard_owner=shards, page_order="shuffled")


def _dense_reference(eng, steps, xs):
    """fp32 torch restatement on the 1-rank engine's weights: per layer
    q/k/v = bf16(x W), causal attention over the request's dense K/V
    history, o (bf16) @ Wo, residual, SwiGLU MLP, residual."""
    m = eng.model
    L, H, qpk, hd = m.num_layers, m.num_kv_heads, eng.qpk, m.head_dim
    qw = eng.n_slots * qpk * hd
    hist = {}
    outs = []
    bf = (lambda t: t.to(torch.bfloat16).float())
    C = len(eng.ffn_cols)
    for step, x in zip(steps, xs):
        x = bf(x.float().cuda())
        rows = []  # (request, position) per token row
        for r, s, n in step.prefill:
            rows += [(r, s + j) for j in range(n)]
        rows += list(step.decode)
        for layer in range(L):
            W = eng.wqkv[layer].float()
            qkv = bf(x @ W)
            o = torch.zeros((len(rows), qw), device=x.device)
            for h in range(H):
                q = qkv[:, h * qpk * hd:(h + 1) * qpk * hd].view(-1, qpk, hd)
                k = qkv[:, qw + h * hd: qw + (h + 1) * hd]
                v = qkv[:, qw + (H + h) * hd: qw + (H + h + 1) * hd]
                for t, (r, pos) in enumerate(rows):
                    K, V = hist.setdefault((layer, h, r), ({}, {}))
                    K[pos], V[pos] = k[t], v[t]
                for t, (r, pos) in enumerate(rows):
                    K, V = hist[(layer, h, r)]
                    Kt = torch.stack([K[p] for p in range(pos + 1)])
                    Vt = torch.stack([V[p] for p in range(pos + 1)])
                    s = (q[t] @ Kt.T) / math.sqrt(hd)
                    o[t, h * qpk * hd:(h + 1) * qpk * hd] = (torch.softmax(s, -1) @ Vt).reshape(-1)
            x = bf(x + bf(bf(o) @ eng.wo[layer].float()))
            g = bf(x @ eng.w_gu[layer].float())
            act = bf(torch.nn.functional.silu(g[:, :C]) * g[:, C:])
            x = bf(x + bf(act @ eng.w_d[layer].float()))
        outs.append(x)
    return outs


def _close(got, ref, tol=3e-2):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    scale = ref.abs().max().item()
    assert err.max().item() <= tol * max(1.0, scale), (err.max().item(), scale)
    assert (err.mean() / ref.abs().mean()).item() <= 1e-2


@pytest.mark.parametrize("qpk", [4, 8])
def test_serving_matches_dense_reference(qpk):
    from paper_2511_14116_b200.placement import make_placement, owner_array
    model = _model(qpk)
    inputs = [(40, 5), (17, 3), (100, 4), (3, 6), (64, 2)]
    routing, steps, caps = _iterations(model, [0], inputs, budget=48, n_iter=6)
    assert any(s.prefill and s.decode for s in steps)  # mixed iterations occur
    plan = make_placement("hybrid", model, [0])
    owner = owner_array(plan, 8)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    eng = _engine(model, owner, 0, routing, caps, shards, 64)
    gen = torch.Generator().manual_seed(7)
    xs = [torch.randn((s.num_tokens, 512), generator=gen).to(torch.bfloat16) for s in steps]
    got = []
    for s, x in zip(steps, xs):
        got.append(eng.serve(eng.plan(s), x.cuda()).clone())
    ref = _dense_reference(eng, steps, xs)
    for g, r in zip(got, ref):
        _close(g, r)


@pytest.mark.parametrize("qpk", [4, 8])
def test_serving_matches_float64_oracle(qpk):
    """The same mixed prefill/decode iterations against the float64 oracle
    (``oracle.decode_step.MixedIterationF64``) on the engine's bf16 weights
    and inputs: the engine rounds qkv, attention output, x and the MLP
    activation to bf16 and the oracle carries float64, so the bound is on
    each iteration's output relative to the scale of its update."""
    from oracle.decode_step import MixedIterationF64
    from paper_2511_14116_b200.placement import make_placement, owner_array
    model = _model(qpk)
    inputs = [(40, 5), (17, 3), (100, 4), (3, 6), (64, 2)]
    routing, steps, caps = _iterations(model, [0], inputs, budget=48, n_iter=6)
    plan = make_placement("hybrid", model, [0])
    owner = owner_array(plan, 8)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    eng = _engine(model, owner, 0, routing, caps, shards, 64)
    assert list(eng.work.slot_heads[0]) == list(range(8))  # slot j is head j at world 1
    f64 = (lambda t: t.double().cpu().numpy())
    ora = MixedIterationF64(8, qpk, 128, [(f64(eng.wqkv[l]), f64(eng.wo[l]), f64(eng.w_gu[l]),
                                          f64(eng.w_d[l])) for l in range(model.num_layers)])
    gen = torch.Generator().manual_seed(7)
    worst = 0.0
    for s in steps:
        x = torch.randn((s.num_tokens, 512), generator=gen).to(torch.bfloat16)
        got = f64(eng.serve(eng.plan(s), x.cuda()))
        rows = [(r, p0 + j) for r, p0, n in s.prefill for j in range(n)] + list(s.decode)
        xd = f64(x)
        ref = ora.step(rows, xd)
        upd = np.abs(ref - xd).mean()
        err = np.abs(got - ref)
        assert err.max() <= 4e-2, (err.max(), upd)
        assert err.mean() <= 2e-2 * upd, (err.mean(), upd)
        worst = max(worst, err.mean() / upd)
    print(f"serving vs float64 (qpk {qpk}): worst mean-abs / mean |update| {worst:.3e}")


@pytest.mark.parametrize("world,fail", [(3, None), (8, 7), (6, None)])
def test_serving_partition_matches_single_rank(world, fail):
    """Hybrid partition (and the on-demand target after losing GPU 7 of 8):
    the ordered sum of the per-rank partials == the 1-rank iteration."""
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    from paper_2511_14116_b200.serving import emulated_serving_step
    model = _model(4)
    plan = make_placement("hybrid", model, range(world))
    alive = list(range(world))
    if fail is not None:
        alive.remove(fail)
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
    inputs = [(40, 5), (17, 3), (100, 4), (3, 6), (64, 2), (9, 9), (33, 2)]
    routing, steps, caps = _iterations(model, alive, inputs, budget=64, n_iter=5)
    owner = owner_array(plan, 8)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    ranks = [_engine(model, owner, g, routing, caps, shards, 96) for g in alive]
    p1 = make_placement("hybrid", model, [0])
    one = _engine(model, owner_array(p1, 8), 0, {r: 0 for r in routing}, caps,
                  [0] * p1.ffn.num_shards, 96)
    gen = torch.Generator().manual_seed(11)
    for s in steps:
        x = torch.randn((s.num_tokens, 512), generator=gen).to(torch.bfloat16).cuda()
        plans = [e.plan(s) for e in ranks]
        got = emulated_serving_step(ranks, plans, x)
        ref = one.serve(one.plan(s), x).clone()
        _close(got, ref)
