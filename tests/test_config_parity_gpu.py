"""Oracle parity of the engine's decode attention (K1 with the fused K3
append, inside ``HybridDecodeRank``) at BASELINE.json's exact shapes.

* C1: toy GQA decoder -- 4 layers, 32 q / 8 KV heads, head_dim 128,
  hidden 4096, batch 16, context 1024 -- on cyclic(8), hybrid(8) and the
  on-demand 7-survivor target of hybrid(8) after GPU 7 fails, EVERY rank;
* C2: one layer of the Llama-3-8B shape (qpk 4), batch 64, context 4096, N=1;
* C3: one layer of the Llama-3-70B shape (hidden 8192, qpk 8), batch 64,
  context 4096, ranks of hybrid(8) and of the N=5 on-demand target
  (8 -> 7 -> 6 -> 5 after GPUs 7, 3, 5 fail).

Placement tables come from the oracle (``oracle.placement``), routing from
the oracle router (``oracle.routing``), expected outputs from
``oracle.attention.head_decode`` (float64, refexec.py:85-103) on the same
bf16 inputs: the item's K/V history, the new token's K/V from the engine's
own projection output and its q.  Tolerance PER ITEM (north star): max-abs
<= 2e-2 and mean-rel <= 1e-3.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MEAN_REL = 1e-3


def _item_close(got, ref, what):
    err = np.abs(got - ref)
    max_abs = float(err.max())
    mean_rel = float(err.mean() / max(np.abs(ref).mean(), 1e-30))
    assert max_abs <= MAX_ABS and mean_rel <= MEAN_REL, (what, max_abs, mean_rel)
    return max_abs, mean_rel


def _model(L, hidden, qheads, ffn):
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=L, num_kv_heads=8, num_q_heads=qheads, head_dim=128,
                     hidden_dim=hidden, ffn_intermediate_dim=ffn)


def _plans(mode, world, fails, L, H=8):
    """Oracle owner table after the on-demand shrink chain ``fails``."""
    from oracle.placement import on_demand_target, owner_table, shard_owner_table
    owner = owner_table(mode, L, H, range(world))
    shards = shard_owner_table(224, range(world))
    alive = list(range(world))
    for f in fails:
        alive = [g for g in alive if g != f]
        owner, shards = on_demand_target(owner, shards, alive)
    return np.array(owner, dtype=np.int32), alive


def _check_rank(model, owner, rank, routing, batch, ctx, seed, layers=None):
    """Build ``rank``'s engine, write a random K/V history of ctx-1 tokens
    per item, run each layer's QKV GEMM + fused K1 and compare every item
    against the oracle.  Returns (items checked, worst max-abs, worst
    mean-rel)."""
    from oracle.attention import head_decode
    from paper_2511_14116_b200.hybrid import HybridDecodeRank
    eng = HybridDecodeRank(model, owner, rank, routing, batch, ctx, seed=seed,
                           page_order="shuffled")
    w, cache = eng.work, eng.cache
    eng.set_lengths([ctx] * batch)
    gen = torch.Generator(device="cuda").manual_seed(seed * 131 + rank)
    n_hist = ctx - 1
    hist_k = torch.randn((w.n_items, n_hist, 128), generator=gen, device="cuda").to(torch.bfloat16)
    hist_v = torch.randn((w.n_items, n_hist, 128), generator=gen, device="cuda").to(torch.bfloat16)
    seq = np.repeat(np.arange(w.n_items), n_hist)
    pos = np.tile(np.arange(n_hist), w.n_items)
    cache.write_tokens(seq, pos, hist_k.view(-1, 128), hist_v.view(-1, 128))
    S, qpk, hd = eng.n_slots, eng.qpk, 128
    scale = 1.0 / math.sqrt(hd)
    worst = [0, 0.0, 0.0]
    for layer in (range(model.num_layers) if layers is None else layers):
        eng.x.copy_(torch.randn((batch, model.hidden_dim), generator=gen, device="cuda")
                    .to(torch.bfloat16))
        eng.attention_partial(layer)
        torch.cuda.synchronize()
        qkv = eng.qkv.double().cpu().numpy()
        o = eng.o.float().cpu().numpy()
        a, b = int(w.seg_items[layer]), int(w.seg_items[layer + 1])
        for i in range(a, b):
            r, j = int(w.item_req[i]), int(w.item_slot[i])
            q = qkv[r, j * qpk * hd:(j + 1) * qpk * hd].reshape(qpk, hd)
            kn = qkv[r, S * qpk * hd + j * hd:S * qpk * hd + (j + 1) * hd]
            vn = qkv[r, S * (qpk + 1) * hd + j * hd:S * (qpk + 1) * hd + (j + 1) * hd]
            k = np.concatenate([hist_k[i].double().cpu().numpy(), kn[None]])
            v = np.concatenate([hist_v[i].double().cpu().numpy(), vn[None]])
            ref = head_decode(q, k, v, scale)
            # the engine's attention output is bf16 (it feeds the O GEMM):
            # compare against the bf16 rounding of the oracle, plus the
            # fp32-accumulation tolerance
            ref_b = torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
            ma, mr = _item_close(o[r * S + j], ref_b, (rank, layer, i))
            worst = [worst[0] + 1, max(worst[1], ma), max(worst[2], mr)]
        # every (layer, head, request) the oracle placement assigns to this
        # rank was attended exactly once
        heads = [h for h in range(8) if owner[layer][h] == rank]
        dp = [h for h in range(8) if owner[layer][h] < 0]
        want = len(heads) * batch + len(dp) * sum(1 for r in range(batch) if routing[r] == rank)
        assert b - a == want
    del eng
    torch.cuda.empty_cache()
    return tuple(worst)


def _routing(batch, ctx, alive):
    from oracle.routing import route_sequence
    ranks, _ = route_sequence([(ctx - 1, 1)] * batch, alive)
    return {r: g for r, g in enumerate(ranks)}


@pytest.mark.parametrize("mode,fails", [("cyclic", ()), ("hybrid", ()), ("hybrid", (7,))])
def test_c1_every_rank_every_layer(mode, fails):
    """BASELINE config 1 exactly: 4 L, 32q/8kv, hd 128, B=16, ctx 1024."""
    model = _model(4, 4096, 32, 14336)
    owner, alive = _plans(mode, 8, fails, 4)
    routing = _routing(16, 1024, alive)
    total = 0
    for g in alive:
        n, _, _ = _check_rank(model, owner, g, routing, 16, 1024, seed=1 + g)
        total += n
    # every (layer, head, request) served once over the world: 4 * 8 * 16
    assert total == 4 * 8 * 16


def test_c2_one_layer_n1():
    """BASELINE config 2 shape, one layer: B=64, ctx 4096, qpk 4, N=1."""
    model = _model(1, 4096, 32, 14336)
    owner, alive = _plans("hybrid", 1, (), 1)
    n, _, _ = _check_rank(model, owner, 0, {r: 0 for r in range(64)}, 64, 4096, seed=5)
    assert n == 8 * 64


@pytest.mark.parametrize("fails,ranks", [((), (0, 7)), ((7, 3, 5), (0, 4, 6))])
def test_c3_one_layer(fails, ranks):
    """BASELINE config 3 shape, one layer: hidden 8192, qpk 8, B=64,
    ctx 4096; hybrid(8) and the N=5 on-demand target (1 TP + 3 DP heads
    per rank)."""
    model = _model(1, 8192, 64, 28672)
    owner, alive = _plans("hybrid", 8, fails, 1)
    routing = _routing(64, 4096, alive)
    for g in ranks:
        n, _, _ = _check_rank(model, owner, g, routing, 64, 4096, seed=9 + g)
        tp = int((owner[0] == g).sum())
        dp = int((owner[0] < 0).sum())
        assert n == tp * 64 + dp * sum(1 for r in range(64) if routing[r] == g)
