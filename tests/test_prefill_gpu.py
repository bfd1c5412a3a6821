"""GPU parity of K8 (paged chunked-prefill GQA attention) against the float64
oracle (oracle.attention.head_prefill, the multi-row _head_attention of
refexec.py:85-103) and the live reference's golden prefill rows.

Tolerance (north star): bf16 K/V, fp32 accumulation -> max-abs <= 2e-2 and
mean-rel <= 1e-3 vs the float64 oracle on the same bf16 inputs; the kernel
writes bf16 outputs, whose rounding (<= 2^-9 relative) is inside that.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MEAN_REL = 1e-3


def _close(gpu, ref, scaled=False):
    """scaled: max-abs relative to the output's scale max(1, max|ref|)
    (V far outside O(1))"""
    err = np.abs(np.asarray(gpu, np.float64) - np.asarray(ref, np.float64))
    max_abs = float(err.max())
    mean_rel = float(err.mean() / max(np.abs(ref).mean(), 1e-30))
    lim = MAX_ABS * (max(1.0, float(np.abs(ref).max())) if scaled else 1.0)
    assert max_abs <= lim, (max_abs, mean_rel)
    assert mean_rel <= MEAN_REL, (max_abs, mean_rel)
    return max_abs, mean_rel


def _cache(n_seq, capacity, qpk, seed=0):
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    work = RankWork.build(np.zeros((1, 1), dtype=np.int32), 0, {r: 0 for r in range(n_seq)}, n_seq)
    return PagedKVCache(work, capacity, qpk, device="cuda", page_order="shuffled", seed=seed)


def _run_case(qpk, starts, lens, seed, target_units=None, q_pad=3, out_dtype=torch.float32,
              variant=0, v_scale=None):
    """Items = sequences; q / out rows strided like a fused projection row."""
    from oracle.attention import head_prefill
    from paper_2511_14116_b200.prefill import PrefillLaunch
    gen = torch.Generator().manual_seed(seed)
    n = len(starts)
    total = [s + l for s, l in zip(starts, lens)]
    cache = _cache(n, max(total), qpk, seed)
    kv = []
    seqs, poss, ks, vs = [], [], [], []
    for i in range(n):
        k = torch.randn((total[i], 128), generator=gen).to(torch.bfloat16)
        v = torch.randn((total[i], 128), generator=gen)
        v = (v * v_scale if v_scale is not None else v).to(torch.bfloat16)
        kv.append((k.double().numpy(), v.double().numpy()))
        seqs.append(np.full(total[i], i))
        poss.append(np.arange(total[i]))
        ks.append(k)
        vs.append(v)
    cache.write_tokens(np.concatenate(seqs), np.concatenate(poss), torch.cat(ks).cuda(),
                       torch.cat(vs).cuda())
    # token rows of all chunks back to back; each row = [q heads | padding]
    stride = (qpk + q_pad) * 128
    T = sum(lens)
    q = torch.randn((T, stride), generator=gen).to(torch.bfloat16)
    row0 = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    out = torch.full((T, stride), 7.0, dtype=out_dtype, device="cuda")
    launch = PrefillLaunch(cache, np.arange(n), starts, lens, row0 * stride, row0 * stride,
                           target_units=target_units, variant=variant)
    launch(q.cuda(), stride, out, stride)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    qn = q.double().numpy()
    gots, refs = [], []
    for i in range(n):
        if lens[i] == 0:
            continue
        rows = slice(row0[i], row0[i] + lens[i])
        qi = qn[rows, :qpk * 128].reshape(lens[i], qpk, 128)
        ref = head_prefill(qi, kv[i][0], kv[i][1], starts[i], 1 / math.sqrt(128))
        gots.append(got[rows, :qpk * 128].reshape(-1))
        refs.append(ref.reshape(-1))
        # padding columns untouched
        assert np.all(got[rows, qpk * 128:] == 7.0)
    # metrics over the whole launch output, as for the decode kernel
    if out_dtype == torch.float32:
        _close(np.concatenate(gots), np.concatenate(refs), scaled=v_scale is not None)
    else:  # bf16 output rounding (<= 2^-9 relative): max-abs only
        assert float(np.abs(np.concatenate(gots) - np.concatenate(refs)).max()) <= MAX_ABS
    launch.got = got
    return launch


# 0: tcgen05 / TMEM, 2 x 128-row halves; 1: mma.sync, 64-row tiles; 2: tcgen05, 128 rows
VARIANTS = [0, 1, 2, 3]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("qpk", [1, 2, 3, 4, 5, 6, 7, 8])
def test_prefill_ragged(qpk, variant):
    """Ragged chunks: fresh prompts, continuation chunks at page and
    non-page boundaries, 1-token chunks, a long prefix, an empty item."""
    starts = [0, 0, 16, 37, 100, 1000, 5, 0]
    lens = [1, 70, 16, 9, 130, 40, 0, 17]
    _run_case(qpk, starts, lens, seed=qpk, variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("qpk", [4, 8])
def test_prefill_splits(qpk, variant):
    """Many KV splits per tile (forced by a large target) merge to the same
    result; split ranges cover every tile's causal range exactly once."""
    starts = [3000, 0, 700]
    lens = [33, 200, 64]
    launch = _run_case(qpk, starts, lens, seed=10 + qpk, target_units=100000, variant=variant)
    assert launch.n_comb > 0 and launch.n_slots > launch.n_comb


@pytest.mark.parametrize("variant", VARIANTS)
def test_prefill_single_long_chunk(variant):
    """A 512-token continuation chunk behind a 4096-token prefix."""
    _run_case(8, [4096], [512], seed=99, variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_prefill_bf16_output(variant):
    """The bf16 output the mixed step feeds to the O projection."""
    _run_case(4, [0, 300, 17], [100, 50, 1], seed=5, out_dtype=torch.bfloat16, variant=variant)
    _run_case(8, [1000], [64], seed=6, target_units=100000, out_dtype=torch.bfloat16,
              variant=variant)


def test_prefill_reference_golden(golden):
    """Chunked-prefill rows of the live reference _head_attention
    (oracle/gen_golden.py gen_prefill): GQA by tied K/V, bf16-exact x."""
    from paper_2511_14116_b200.prefill import PrefillLaunch
    g = golden("prefill")
    for c in g["cases"]:
        qpk = c["qpk"]
        x = np.array(c["x"])
        lens = c["seq_lens"]
        cache = _cache(len(lens), max(lens), qpk)
        seqs, poss, starts, clen, off = [], [], [], [], 0
        for i, L in enumerate(lens):
            seqs.append(np.full(L, i))
            poss.append(np.arange(L))
        xt = torch.tensor(x, dtype=torch.float64).to(torch.bfloat16)
        cache.write_tokens(np.concatenate(seqs), np.concatenate(poss), xt.cuda(), xt.cuda())
        q_rows, k = [], 0
        row0 = []
        for i, (L, (c0, cn)) in enumerate(zip(lens, c["chunks"])):
            seg = x[off:off + L]
            q_rows.append(np.stack([seg[c0:c0 + cn] * np.array(d) for d in c["diag"]], axis=1))
            starts.append(c0)
            clen.append(cn)
            row0.append(k)
            k += cn
            off += L
        q = torch.tensor(np.concatenate(q_rows).reshape(k, qpk * 128)).to(torch.bfloat16)
        assert torch.equal(q.double(), torch.tensor(np.concatenate(q_rows).reshape(k, -1)))
        out = torch.zeros((k, qpk * 128), dtype=torch.float32, device="cuda")
        stride = qpk * 128
        launch = PrefillLaunch(cache, np.arange(len(lens)), starts, clen,
                               np.array(row0) * stride, np.array(row0) * stride)
        launch(q.cuda(), stride, out, stride)
        torch.cuda.synchronize()
        _close(out.float().cpu().numpy().reshape(k, qpk, 128), np.array(c["out"]))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("v_scale", [7e4, 1e-6])
def test_prefill_v_range_split_vs_unsplit(variant, v_scale):
    """bf16 V far outside f16's range (7e4) or far below its normal range
    (1e-6): split (fp32 partials + combine) and unsplit tiles both match the
    oracle on the same bf16 values, and each other."""
    starts, lens = [2000, 0], [64, 120]
    a = _run_case(8, starts, lens, seed=21, target_units=100000, variant=variant, v_scale=v_scale)
    b = _run_case(8, starts, lens, seed=21, target_units=1, variant=variant, v_scale=v_scale)
    assert a.n_comb > 0
    ref = np.abs(b.got).max()
    assert float(np.abs(a.got - b.got).max()) <= 1e-3 * max(ref, 1e-30)
