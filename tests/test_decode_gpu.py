"""GPU parity of K1/K2 (paged GQA decode + combine), K3 (KV write) and K4
(page planner) against the CPU oracle and the reference golden vectors.

Tolerance (north star): bf16 K/V, fp32 accumulation -> max-abs <= 2e-2 and
mean-rel <= 1e-3 vs the float64 oracle on the same bf16 inputs, where
mean-rel = mean|gpu - ref| / mean|ref|.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MEAN_REL = 1e-3


def _close(gpu, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(gpu - ref)
    max_abs = float(err.max()) if err.size else 0.0
    mean_rel = float(err.mean() / max(np.abs(ref).mean(), 1e-30)) if err.size else 0.0
    assert max_abs <= MAX_ABS, (max_abs, mean_rel)
    assert mean_rel <= MEAN_REL, (max_abs, mean_rel)
    return max_abs, mean_rel


def _bf16(t):
    return t.to(torch.bfloat16)


def _build(owner, rank, routing, lens, qpk, order="shuffled", seed=0, config=0):
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    work = RankWork.build(np.asarray(owner, dtype=np.int32), rank, routing, len(lens))
    cache = PagedKVCache(work, max(max(lens), 1), qpk, device="cuda", page_order=order,
                         seed=seed, config=config)
    cache.set_lengths(lens)
    return work, cache


def _fill(cache, work, lens, gen):
    """Random bf16 K/V for every (item, position); returns dense copies."""
    kv = {}
    seqs, poss, ks, vs = [], [], [], []
    for i in range(work.n_items):
        n = lens[work.item_req[i]]
        k = _bf16(torch.randn((n, 128), generator=gen))
        v = _bf16(torch.randn((n, 128), generator=gen))
        kv[i] = (k.double().numpy(), v.double().numpy())
        seqs.append(np.full(n, i))
        poss.append(np.arange(n))
        ks.append(k)
        vs.append(v)
    cache.write_tokens(np.concatenate(seqs), np.concatenate(poss),
                       torch.cat(ks).cuda(), torch.cat(vs).cuda())
    return kv


def _expected(work, kv, q, lens, n_rows):
    from oracle.attention import head_decode
    out = np.zeros((n_rows,) + q.shape[1:])
    for i in range(work.n_items):
        r, j = work.item_req[i], work.item_slot[i]
        row = r * work.n_slots + j
        k, v = kv[i]
        out[row] = head_decode(q[row], k[:lens[r]], v[:lens[r]], 1.0 / math.sqrt(128))
    return out


@pytest.mark.parametrize("qpk", [1, 3, 4, 6, 8])
@pytest.mark.parametrize("config", [0, 3, 7, 9])
def test_decode_hybrid_rank_ragged(qpk, config):
    """Hybrid N=7 rank: 1 TP head for all requests + 1 DP head for routed
    requests; ragged lengths incl. 1, page edges and multi-warp items."""
    from oracle.placement import owner_table
    owner = owner_table("hybrid", 2, 8, range(7))
    lens = [1, 15, 16, 17, 33, 300, 1000, 4097, 2]
    routing = {r: r % 7 for r in range(len(lens))}
    from oracle.attention import head_decode
    gen = torch.Generator().manual_seed(qpk * 10 + config)
    for rank in (0, 3):
        work, cache = _build(owner, rank, routing, lens, qpk, config=config)
        kv = _fill(cache, work, lens, gen)
        n_rows = len(lens) * work.n_slots
        q = _bf16(torch.randn((n_rows, qpk, 128), generator=gen))
        qn = q.double().numpy()
        out = torch.zeros((n_rows, qpk, 128), dtype=torch.float32, device="cuda")
        q_dev = q.cuda()
        ref = np.zeros((n_rows, qpk, 128))
        for layer in range(2):
            out.zero_()
            cache.decode_layer(layer, q_dev, out)
            torch.cuda.synchronize()
            a, b = work.seg_items[layer], work.seg_items[layer + 1]
            exp = np.zeros_like(ref)
            for i in range(a, b):
                r, j = work.item_req[i], work.item_slot[i]
                row = r * work.n_slots + j
                k, v = kv[i]
                exp[row] = head_decode(qn[row], k[:lens[r]], v[:lens[r]], 1 / math.sqrt(128))
            _close(out.cpu().numpy(), exp)


def test_decode_bf16_output_and_determinism():
    from oracle.placement import owner_table
    owner = owner_table("cyclic", 1, 8, range(2))
    lens = [4096, 777, 64]
    routing = {r: 0 for r in range(3)}
    work, cache = _build(owner, 1, routing, lens, 4)
    gen = torch.Generator().manual_seed(3)
    kv = _fill(cache, work, lens, gen)
    n_rows = 3 * work.n_slots
    q = _bf16(torch.randn((n_rows, 4, 128), generator=gen))
    o1 = torch.zeros((n_rows, 4, 128), dtype=torch.bfloat16, device="cuda")
    o2 = torch.zeros_like(o1)
    cache.decode_layer(0, q.cuda(), o1)
    cache.decode_layer(0, q.cuda(), o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    exp = _expected(work, kv, q.double().numpy(), lens, n_rows)
    # bf16 output rounding adds <= 2^-9 relative; check max-abs only
    assert float(np.abs(o1.float().cpu().numpy() - exp).max()) <= MAX_ABS


def test_decode_reference_golden(golden):
    """Decode rows of the reference _head_attention (bf16-exact inputs)."""
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    g = golden("decode")
    for case in g["cases"]:
        qpk, seq_lens = case["qpk"], case["seq_lens"]
        x = torch.tensor(case["x"], dtype=torch.float64)
        owner = np.zeros((1, 1), dtype=np.int32)  # one KV head owned by rank 0
        work = RankWork.build(owner, 0, {r: 0 for r in range(len(seq_lens))}, len(seq_lens))
        cache = PagedKVCache(work, max(seq_lens), qpk, page_order="shuffled", seed=1)
        cache.set_lengths(seq_lens)
        seqs, poss = [], []
        start = 0
        q = torch.zeros((len(seq_lens), qpk, 128), dtype=torch.float64)
        diag = torch.tensor(case["diag"], dtype=torch.float64)
        for r, n in enumerate(seq_lens):
            seqs.append(np.full(n, r))
            poss.append(np.arange(n))
            q[r] = x[start + n - 1][None, :] * diag
            start += n
        xb = x.to(torch.bfloat16).cuda()
        assert torch.equal(xb.double().cpu(), x)  # inputs are bf16-exact
        cache.write_tokens(np.concatenate(seqs), np.concatenate(poss), xb, xb)
        out = torch.zeros((len(seq_lens), qpk, 128), dtype=torch.float32, device="cuda")
        cache.decode_layer(0, q.to(torch.bfloat16).cuda(), out)
        torch.cuda.synchronize()
        _close(out.cpu().numpy(), np.array(case["out"]))


def test_kv_write_read_roundtrip_bitexact():
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    owner = np.zeros((1, 2), dtype=np.int32)
    work = RankWork.build(owner, 0, {0: 0, 1: 0}, 2)
    cache = PagedKVCache(work, 100, 1, page_order="shuffled", seed=5)
    n = 4 * 100
    seq = np.repeat(np.arange(4), 100)
    pos = np.tile(np.arange(100), 4)
    k = torch.randn((n, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((n, 128), device="cuda").to(torch.bfloat16)
    cache.write_tokens(seq, pos, k, v)
    k2, v2 = cache.read_tokens(seq, pos)
    # K and V pages hold the bf16 values exactly
    assert torch.equal(k, k2) and torch.equal(v, v2)
    # the page format: K half = 2 atoms (dims 0-63, 64-127) x 16 rows x 8
    # chunks, chunk c of row r at (c & 7) ^ (r & 7) of atom c >> 3
    page = cache.block_table[0, 0].item()
    raw = cache.pool[page].view(torch.bfloat16)[: 16 * 128].view(2, 16, 8, 8)
    for r in (0, 5, 9):
        for c in (0, 3, 9, 15):
            assert torch.equal(raw[c >> 3, r, (c & 7) ^ (r & 7)], k[r, c * 8:(c + 1) * 8])


def test_kv_write_runs_matches_token_writes():
    """fs_kv_write_runs (runs of consecutive tokens, strided source rows, a
    slice of a prefix sum) leaves the pool bit-identical to fs_kv_write of
    the same tokens listed one by one."""
    from paper_2511_14116_b200 import _native as N
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    owner = np.zeros((1, 3), dtype=np.int32)
    work = RankWork.build(owner, 0, {0: 0, 1: 0}, 2)
    step, rows = 3, 400  # source rows: run r's token i at run_src[r] + i * step
    src_k = torch.randn((rows * step, 128), device="cuda").to(torch.bfloat16)
    src_v = torch.randn((rows * step, 128), device="cuda").to(torch.bfloat16)
    # runs: (seq, pos0, src0, len); a leading dummy run is skipped via the slice
    runs = [(0, 0, 0, 1), (1, 5, 1, 37), (3, 0, 2, 1), (4, 17, 40, 100), (2, 99, 9, 1),
            (5, 0, 300, 16)]
    seq = np.array([r[0] for r in runs], np.int32)
    pos = np.array([r[1] for r in runs], np.int32)
    src = np.array([r[2] for r in runs], np.int32)
    off = np.concatenate([[7], 7 + np.cumsum([r[3] for r in runs])]).astype(np.int32)
    t_seq = np.concatenate([[s] * n for s, _, _, n in runs[1:]]).astype(np.int32)
    t_pos = np.concatenate([np.arange(p, p + n) for _, p, _, n in runs[1:]]).astype(np.int32)
    t_src = np.concatenate([s + step * np.arange(n) for _, _, s, n in runs[1:]]).astype(np.int32)
    pools = []
    for mode in ("runs", "tokens"):
        cache = PagedKVCache(work, 200, 1, page_order="shuffled", seed=3)
        st = N.C.c_void_p(torch.cuda.current_stream().cuda_stream)
        if mode == "runs":
            dev = [torch.from_numpy(a).cuda() for a in (seq, pos, src, off)]
            N.check(N.lib.fs_kv_write_runs(
                N.ptr(cache.pool), N.ptr(cache.block_table), cache.pages_per_seq,
                N.C.c_void_p(dev[0].data_ptr() + 4), N.C.c_void_p(dev[1].data_ptr() + 4),
                N.C.c_void_p(dev[2].data_ptr() + 4), N.C.c_void_p(dev[3].data_ptr() + 4),
                len(runs) - 1, int(off[-1] - off[1]), step, N.ptr(src_k), N.ptr(src_v), 128, st),
                "fs_kv_write_runs")
        else:
            dev = [torch.from_numpy(a).cuda() for a in (t_seq, t_pos, t_src)]
            N.check(N.lib.fs_kv_write(N.ptr(cache.pool), N.ptr(cache.block_table),
                                      cache.pages_per_seq, N.ptr(dev[0]), N.ptr(dev[1]),
                                      N.ptr(dev[2]), t_seq.size, N.ptr(src_k), N.ptr(src_v), 128,
                                      st), "fs_kv_write")
        torch.cuda.synchronize()
        pools.append(cache.pool.clone())
    assert torch.equal(pools[0], pools[1])


def test_plan_pages_matches_host_prefix():
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    rng = np.random.default_rng(0)
    owner = np.array([[0, 0, -1], [0, -1, 0], [-1, -1, -1]], dtype=np.int32)
    B = 2500
    lens = rng.integers(0, 70, size=B)
    routing = {r: int(rng.integers(0, 2)) for r in range(B)}
    work = RankWork.build(owner, 0, routing, B)
    cache = PagedKVCache(work, 70, 1)
    cache.set_lengths(lens)
    torch.cuda.synchronize()
    got = cache.page_off.cpu().numpy()
    for layer in range(3):
        a, b = work.seg_items[layer], work.seg_items[layer + 1]
        pages = (lens[work.item_req[a:b]] + 15) // 16
        exp = np.concatenate([[0], np.cumsum(pages)])
        assert np.array_equal(got[a + layer:b + layer + 1], exp)


def test_decode_errors_map_to_reference_exceptions():
    from paper_2511_14116_b200 import ValidationError
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    work = RankWork.build(np.zeros((1, 1), np.int32), 0, {0: 0}, 1)
    with pytest.raises(ValidationError):
        PagedKVCache(work, 16, 9)
    cache = PagedKVCache(work, 16, 2)
    cache.qpk = 9
    cache.set_lengths([3])
    with pytest.raises(ValidationError):
        cache.decode_layer(0, torch.zeros((1, 9, 128), dtype=torch.bfloat16, device="cuda"),
                           torch.zeros((1, 9, 128), dtype=torch.bfloat16, device="cuda"))


@pytest.mark.parametrize("config", [0, 7])
def test_fused_append_then_decode(config):
    """Fused K3: the token at len-1 comes from the projection row and is
    both attended and persisted into its page by the decode launch."""
    from oracle.attention import head_decode
    from oracle.placement import owner_table
    owner = owner_table("hybrid", 1, 8, range(3))
    lens = [1, 16, 17, 40, 513, 2]
    B = len(lens)
    routing = {r: r % 3 for r in range(B)}
    qpk = 4
    work, cache = _build(owner, 1, routing, lens, qpk, config=config)
    rw = cache.set_fused_layout()
    gen = torch.Generator().manual_seed(11)
    S = work.n_slots
    kv = {}
    seqs, poss, ks, vs = [], [], [], []
    for i in range(work.n_items):
        n = lens[work.item_req[i]]
        k = _bf16(torch.randn((n, 128), generator=gen))
        v = _bf16(torch.randn((n, 128), generator=gen))
        kv[i] = (k, v)
        if n > 1:
            seqs.append(np.full(n - 1, i))
            poss.append(np.arange(n - 1))
            ks.append(k[:-1])
            vs.append(v[:-1])
    cache.write_tokens(np.concatenate(seqs), np.concatenate(poss), torch.cat(ks).cuda(),
                       torch.cat(vs).cuda())
    qkv = _bf16(torch.randn((B, rw), generator=gen))
    for i in range(work.n_items):
        r, j = work.item_req[i], work.item_slot[i]
        qkv[r, S * qpk * 128 + j * 128:S * qpk * 128 + (j + 1) * 128] = kv[i][0][-1]
        qkv[r, S * (qpk + 1) * 128 + j * 128:S * (qpk + 1) * 128 + (j + 1) * 128] = kv[i][1][-1]
    out = torch.zeros((B * S, qpk, 128), dtype=torch.float32, device="cuda")
    cache.decode_layer_fused(0, qkv.cuda(), out)
    torch.cuda.synchronize()
    exp = np.zeros(out.shape)
    for i in range(work.n_items):
        r, j = work.item_req[i], work.item_slot[i]
        q = qkv[r, j * qpk * 128:(j + 1) * qpk * 128].view(qpk, 128).double().numpy()
        k, v = kv[i]
        exp[r * S + j] = head_decode(q, k.double().numpy(), v.double().numpy(), 1 / math.sqrt(128))
    _close(out.cpu().numpy(), exp)
    # the new token was persisted into its page
    items = np.arange(work.n_items)
    last = np.array([lens[work.item_req[i]] - 1 for i in items])
    k2, v2 = cache.read_tokens(items, last)
    for i in items:
        assert torch.equal(k2[i].cpu(), kv[i][0][-1]) and torch.equal(v2[i].cpu(), kv[i][1][-1])
    # semaphores are left zero for the next launch
    assert int(cache.item_sem.abs().sum()) == 0


def _tiny_model(L=2, H=8, qpk=4, hidden=256):
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H * qpk, head_dim=128,
                     hidden_dim=hidden, ffn_intermediate_dim=1024)


def _engine_reference(model, x, kv_hist, lens, seed, mlp=False):
    """torch fp32 reference of the hybrid decode step with bf16 rounding at
    the same points as the engine (qkv, attention output, residual, MLP)."""
    from paper_2511_14116_b200.hybrid import ffn_weights, head_weights
    x = x.float().cuda()
    qpk, hd = model.q_heads_per_kv_head, 128
    all_cols = np.arange(model.ffn_intermediate_dim, dtype=np.int32)
    for layer in range(model.num_layers):
        xb = x.to(torch.bfloat16)
        acc = torch.zeros_like(x)
        for h in range(model.num_kv_heads):
            wq, wk, wv, wo = head_weights(model, layer, h, seed, "cuda")
            q = (xb @ wq).float().view(-1, qpk, hd)
            kn, vn = (xb @ wk), (xb @ wv)
            outs = []
            for r in range(x.shape[0]):
                kp, vp = kv_hist[(layer, h, r)]
                k = torch.cat([kp.cuda(), kn[r:r + 1]]).float()
                v = torch.cat([vp.cuda(), vn[r:r + 1]]).float()
                w = torch.softmax(q[r] @ k.T / math.sqrt(hd), dim=-1)
                outs.append((w @ v).to(torch.bfloat16))
            o = torch.stack(outs).view(x.shape[0], qpk * hd)
            acc += (o @ wo).float()
        x = (xb.float() + acc).to(torch.bfloat16).float()
        if mlp:
            xb = x.to(torch.bfloat16)
            wgu, wd = ffn_weights(model, layer, all_cols, seed, "cuda")
            C = len(all_cols)
            hgu = (xb @ wgu).float()
            act = (torch.nn.functional.silu(hgu[:, :C]) * hgu[:, C:]).to(torch.bfloat16)
            x = (xb.float() + (act @ wd).float()).to(torch.bfloat16).float()
    return x


def _engines(model, mode, world, lens, routing, seed, kv_hist, mlp=False, plan=None):
    from paper_2511_14116_b200.hybrid import HybridDecodeRank
    from paper_2511_14116_b200.placement import make_placement, owner_array
    if plan is None:
        plan = make_placement(mode, model, range(world))
    owner = owner_array(plan, model.num_kv_heads)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    ranks = []
    for g in plan.alive:
        e = HybridDecodeRank(model, owner, g, routing, len(lens), max(lens), seed=seed,
                             page_order="shuffled", mlp=mlp, shard_owner=shards)
        e.set_lengths(lens)
        w = e.work
        seqs, poss, ks, vs = [], [], [], []
        for i in range(w.n_items):
            layer = int(np.searchsorted(w.seg_items, i, side="right") - 1)
            kp, vp = kv_hist[(layer, int(w.item_head[i]), int(w.item_req[i]))]
            if len(kp):
                seqs.append(np.full(len(kp), i))
                poss.append(np.arange(len(kp)))
                ks.append(kp)
                vs.append(vp)
        if seqs:
            e.cache.write_tokens(np.concatenate(seqs), np.concatenate(poss),
                                 torch.cat(ks).cuda(), torch.cat(vs).cuda())
        ranks.append(e)
    return ranks


def _history(model, lens, seed):
    gen = torch.Generator().manual_seed(seed)
    kv_hist = {}
    for layer in range(model.num_layers):
        for h in range(model.num_kv_heads):
            for r in range(len(lens)):
                kv_hist[(layer, h, r)] = (_bf16(torch.randn((lens[r] - 1, 128), generator=gen)),
                                          _bf16(torch.randn((lens[r] - 1, 128), generator=gen)))
    x0 = _bf16(torch.randn((len(lens), model.hidden_dim), generator=gen))
    return kv_hist, x0


@pytest.mark.parametrize("mlp", [False, True])
def test_engine_world_emulation_matches_single_gpu_and_reference(mlp):
    """Decode form of parallel_forward: world 1 == emulated hybrid worlds
    2/7/5 and cyclic 4 (ordered partial sums) == torch fp32 reference."""
    from paper_2511_14116_b200.hybrid import emulated_parallel_step
    model = _tiny_model()
    lens = [5, 17, 1, 33, 16, 2]
    B = len(lens)
    kv_hist, x0 = _history(model, lens, 2)
    ref = _engine_reference(model, x0, kv_hist, lens, seed=4, mlp=mlp)
    one = _engines(model, "hybrid", 1, lens, {r: 0 for r in range(B)}, 4, kv_hist, mlp=mlp)[0]
    y1 = one.step(x0.cuda()).float().clone()
    err = float((y1 - ref).abs().max())
    assert err <= 3e-2 * max(1.0, float(ref.abs().max())), err
    for mode, world in (("hybrid", 2), ("hybrid", 7), ("cyclic", 4), ("hybrid", 5)):
        routing = {r: (r * 3) % world for r in range(B)}
        ranks = _engines(model, mode, world, lens, routing, 4, kv_hist, mlp=mlp)
        yw = emulated_parallel_step(ranks, x0.cuda()).float()
        err = float((yw - y1).abs().max())
        assert err <= 3e-2 * max(1.0, float(y1.abs().max())), (mode, world, err)


def test_engine_on_demand_targets_8_7_6_5_match_single_gpu():
    """The failure states run the on-demand shrink targets (survivors keep
    their heads/shards, lost heads replicated, lost shards redistributed):
    each world's emulated step equals the single-GPU step."""
    from paper_2511_14116_b200.hybrid import emulated_parallel_step
    from paper_2511_14116_b200.placement import make_placement
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    model = _tiny_model()
    lens = [9, 33, 2, 17]
    B = len(lens)
    kv_hist, x0 = _history(model, lens, 8)
    one = _engines(model, "hybrid", 1, lens, {r: 0 for r in range(B)}, 3, kv_hist, mlp=True)[0]
    y1 = one.step(x0.cuda()).float().clone()
    plan = make_placement("hybrid", model, range(8))
    alive = list(range(8))
    for f in (None, 7, 3, 5):
        if f is not None:
            alive = [g for g in alive if g != f]
            plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid",
                                                                                      model)
        routing = {r: alive[r % len(alive)] for r in range(B)}
        ranks = _engines(model, "hybrid", None, lens, routing, 3, kv_hist, mlp=True, plan=plan)
        yw = emulated_parallel_step(ranks, x0.cuda()).float()
        err = float((yw - y1).abs().max())
        assert err <= 3e-2 * max(1.0, float(y1.abs().max())), (f, err)


def test_engine_graph_capture_replays_identically():
    model = _tiny_model(L=3)
    lens = [40, 7, 64]
    kv_hist, x0 = _history(model, lens, 5)
    e = _engines(model, "hybrid", 1, lens, {0: 0, 1: 0, 2: 0}, 1, kv_hist, mlp=True)[0]
    eager = e.step(x0.cuda()).clone()
    e.capture()
    for _ in range(3):
        graphed = e.step(x0.cuda()).clone()
        assert torch.equal(eager, graphed)
    # host in / host out in one graph launch (HybridDecodeRank.step_io)
    x_host, y_host = x0.pin_memory(), torch.empty_like(x0).pin_memory()
    for _ in range(2):
        e.step_io(x_host, y_host)
        torch.cuda.synchronize()
        assert torch.equal(y_host, eager.cpu())


@pytest.mark.parametrize("qpk", [4, 8])
def test_decode_long_context_per_item_tolerance(qpk):
    """The tolerance holds per long item, not only diluted over a launch:
    bf16 P alone gives ~1.5e-3 mean-rel at 4k context; the kernels use a
    bf16 hi + lo pair of P against the bf16 V pages."""
    from oracle.attention import head_decode
    from oracle.placement import owner_table
    owner = owner_table("hybrid", 1, 8, range(8))
    lens = [4096, 3000, 8192]
    routing = {r: 0 for r in range(3)}
    for config in (0, 7):
        work, cache = _build(owner, 0, routing, lens, qpk, config=config)
        gen = torch.Generator().manual_seed(qpk + config)
        kv = _fill(cache, work, lens, gen)
        n_rows = 3 * work.n_slots
        q = _bf16(torch.randn((n_rows, qpk, 128), generator=gen))
        out = torch.zeros((n_rows, qpk, 128), dtype=torch.float32, device="cuda")
        cache.decode_layer(0, q.cuda(), out)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        qn = q.double().numpy()
        for i in range(work.n_items):
            r, j = work.item_req[i], work.item_slot[i]
            row = r * work.n_slots + j
            k, v = kv[i]
            _close(got[row], head_decode(qn[row], k[:lens[r]], v[:lens[r]], 1 / math.sqrt(128)))


@pytest.mark.parametrize("n_req", [1024, 1100])
def test_decode_many_items_table_stage_boundary(n_req):
    """decode_cta_kernel stages the item tables in shared memory for up to
    1024 items per launch and reads them from global memory beyond that:
    both sides of the boundary (one TP head, ragged short contexts) match
    the oracle."""
    from oracle.attention import head_decode
    owner = np.zeros((1, 1), dtype=np.int32)  # one layer, one KV head, rank 0
    rng = np.random.default_rng(n_req)
    lens = [int(x) for x in rng.integers(1, 70, size=n_req)]
    routing = {r: 0 for r in range(n_req)}
    qpk = 4
    gen = torch.Generator().manual_seed(n_req)
    work, cache = _build(owner, 0, routing, lens, qpk, config=0)
    assert work.n_items == n_req
    kv = _fill(cache, work, lens, gen)
    q = _bf16(torch.randn((n_req, qpk, 128), generator=gen))
    out = torch.zeros((n_req, qpk, 128), dtype=torch.float32, device="cuda")
    cache.decode_layer(0, q.cuda(), out)
    torch.cuda.synchronize()
    qn = q.double().numpy()
    exp = np.stack([head_decode(qn[i], kv[i][0][:lens[i]], kv[i][1][:lens[i]], 1 / math.sqrt(128))
                    for i in range(n_req)])
    _close(out.cpu().numpy(), exp)


@pytest.mark.parametrize("kind", ["huge", "tiny", "mixed"])
@pytest.mark.parametrize("config", [0, 7])
def test_v_range_edge_cases_keep_bf16_semantics(kind, config):
    """V values outside f16's range (|v| = 7e4), far below its normal range
    (1e-6) and mixed signs / magnitudes: the pages hold them exactly (read
    back bit-exact, fused append included) and decode matches the float64
    oracle on the same bf16 values -- mean-rel <= 1e-3 and max-abs <= 2e-2
    relative to the output's scale (max(1, max|ref|))."""
    from oracle.attention import head_decode
    from oracle.placement import owner_table
    owner = owner_table("hybrid", 1, 8, range(8))
    lens = [4096, 700, 17, 1]
    routing = {r: 0 for r in range(len(lens))}
    qpk = 4
    work, cache = _build(owner, 0, routing, lens, qpk, config=config)
    gen = torch.Generator().manual_seed(hash(kind) % 1000)
    kv = {}
    seqs, poss, ks, vs = [], [], [], []
    for i in range(work.n_items):
        n = lens[work.item_req[i]]
        k = _bf16(torch.randn((n, 128), generator=gen))
        base = torch.randn((n, 128), generator=gen)
        if kind == "huge":
            v = _bf16(base.sign() * 7e4 * (1 + 0.1 * base.abs()))
        elif kind == "tiny":
            v = _bf16(base * 1e-6)
        else:
            pick = torch.randint(0, 3, (n, 128), generator=gen)
            v = _bf16(torch.where(pick == 0, base * 7e4, torch.where(pick == 1, base * 1e-6, base)))
        kv[i] = (k, v)
        seqs.append(np.full(n, i))
        poss.append(np.arange(n))
        ks.append(k)
        vs.append(v)
    cache.write_tokens(np.concatenate(seqs), np.concatenate(poss), torch.cat(ks).cuda(),
                       torch.cat(vs).cuda())
    k2, v2 = cache.read_tokens(np.concatenate(seqs), np.concatenate(poss))
    assert torch.equal(v2.cpu(), torch.cat(vs)) and torch.equal(k2.cpu(), torch.cat(ks))
    n_rows = len(lens) * work.n_slots
    q = _bf16(torch.randn((n_rows, qpk, 128), generator=gen))
    out = torch.zeros((n_rows, qpk, 128), dtype=torch.float32, device="cuda")
    cache.decode_layer(0, q.cuda(), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    qn = q.double().numpy()
    for i in range(work.n_items):
        r, j = work.item_req[i], work.item_slot[i]
        row = r * work.n_slots + j
        k, v = kv[i]
        ref = head_decode(qn[row], k.double().numpy(), v.double().numpy(), 1 / math.sqrt(128))
        err = np.abs(got[row] - ref)
        scale = max(1.0, float(np.abs(ref).max()))
        assert float(err.max()) <= MAX_ABS * scale, (kind, i, float(err.max()), scale)
        assert float(err.mean() / np.abs(ref).mean()) <= MEAN_REL, (kind, i)
