"""GPU tests of the skinny tcgen05 GEMM (fs_gemm_skinny) against a torch
fp32 reference on the same bf16 inputs (bf16 output: max-abs <= 1% of the
output scale, mean-rel <= 5e-3)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(x, w):
    return x.float() @ w.float()


def _close(got, ref):
    scale = float(ref.abs().max()) or 1.0
    err = (got.float() - ref).abs()
    assert float(err.max()) <= 1e-2 * scale, (float(err.max()), scale)
    assert float(err.mean() / ref.abs().mean()) <= 5e-3


@pytest.mark.parametrize("rows,K,N", [(64, 4096, 6144), (37, 8192, 1280), (5, 64, 128),
                                      (64, 1024, 8192), (100, 512, 384), (64, 3584, 256)])
def test_store(rows, K, N):
    from paper_2511_14116_b200.gemm import STORE, SkinnyGemm
    g = torch.Generator(device="cuda").manual_seed(rows + K + N)
    x = torch.randn((rows, K), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    out = torch.empty((rows, N), device="cuda", dtype=torch.bfloat16)
    gemm = SkinnyGemm(N)
    gemm(x, w, out, STORE)
    torch.cuda.synchronize()
    _close(out, _ref(x, w))
    # deterministic and the semaphores are left zero
    out2 = torch.empty_like(out)
    gemm(x, w, out2, STORE)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    assert int(gemm.sems.abs().sum()) == 0


def test_residual_in_place():
    from paper_2511_14116_b200.gemm import RESIDUAL, SkinnyGemm
    g = torch.Generator(device="cuda").manual_seed(1)
    o = torch.randn((64, 1024), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((1024, 4096), device="cuda", generator=g) / 32).to(torch.bfloat16)
    x = torch.randn((64, 4096), device="cuda", generator=g).to(torch.bfloat16)
    ref = x.float() + _ref(o, w)
    SkinnyGemm(4096)(o, w, x, RESIDUAL)
    torch.cuda.synchronize()
    _close(x, ref)


def test_swiglu_epilogue():
    from paper_2511_14116_b200.gemm import SWIGLU, SkinnyGemm, interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(2)
    K, C = 2048, 448
    x = torch.randn((64, K), device="cuda", generator=g).to(torch.bfloat16)
    wg = (torch.randn((K, C), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    wu = (torch.randn((K, C), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    wgu = interleave_gate_up(wg, wu)
    act = torch.empty((64, C), device="cuda", dtype=torch.bfloat16)
    SkinnyGemm(2 * C)(x, wgu, act, SWIGLU)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
    _close(act, ref)


def test_validation():
    from paper_2511_14116_b200 import ValidationError
    from paper_2511_14116_b200.gemm import SkinnyGemm
    x = torch.zeros((4, 100), device="cuda", dtype=torch.bfloat16)
    w = torch.zeros((100, 128), device="cuda", dtype=torch.bfloat16)
    out = torch.zeros((4, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValidationError):
        SkinnyGemm(128)(x, w, out)


@pytest.mark.parametrize("K,N,epi,group", [(4096, 1280, 0, 1), (1024, 4096, 1, 1), (2048, 896, 2, 1),
                                           (4096, 1280, 0, 2), (1024, 4096, 1, 2), (2048, 1024, 2, 2),
                                           (8192, 38912, 2, None)])
def test_packed_panels_match_row_major(K, N, epi, group):
    from paper_2511_14116_b200.gemm import PackedWeight, SkinnyGemm, interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(K + N)
    x = torch.randn((64, K), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    if epi == 2:
        w = interleave_gate_up(w[:, :N // 2], w[:, N // 2:])
    pw = PackedWeight(w, group)
    assert torch.equal(pw.unpack(), w)
    if group is None:  # more 128-column tiles than SMs: two tiles per CTA
        assert pw.group == 2
    n_out = N // 2 if epi == 2 else N
    base = torch.randn((64, n_out), device="cuda", generator=g).to(torch.bfloat16)
    a, b = base.clone(), base.clone()
    gemm = SkinnyGemm(N)
    gemm(x, w, a, epi)
    gemm(x, pw, b, epi)
    torch.cuda.synchronize()
    if pw.group == 1:  # same launch plan as the row-major W: same bits
        assert torch.equal(a, b)
    assert int(gemm.sems.abs().sum()) == 0
    ref = _ref(x, w)
    if epi == 2:
        g_, u_ = ref.view(64, -1, 2, 64)[:, :, 0].reshape(64, -1), ref.view(64, -1, 2, 64)[:, :, 1].reshape(64, -1)
        ref = torch.nn.functional.silu(g_) * u_
    elif epi == 1:
        ref = ref + base.float()
    _close(b, ref)


@pytest.mark.parametrize("rows", [1, 3, 17, 64])
def test_split_reduction_rows(rows):
    """Small row counts with many k-splits per tile (QKV-like: 10 tiles over
    K = 8192): row slices of the in-grid reduction may be empty."""
    from paper_2511_14116_b200.gemm import RESIDUAL, PackedWeight, SkinnyGemm
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn((rows, 8192), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((8192, 1280), device="cuda", generator=g) / 90.0).to(torch.bfloat16)
    base = torch.randn((rows, 1280), device="cuda", generator=g).to(torch.bfloat16)
    out = base.clone()
    gemm = SkinnyGemm(1280)
    for _ in range(3):  # counters reset between launches
        out.copy_(base)
        gemm(x, PackedWeight(w), out, RESIDUAL)
    torch.cuda.synchronize()
    _close(out, base.float() + _ref(x, w))
    assert int(gemm.sems.abs().sum()) == 0


# the decode-step projections at the BASELINE shapes (per rank): C2 (8B,
# world 1) and C3 (70B, hybrid(8) and the 5-survivor on-demand target),
# packed weights and the production epilogues
_CONFIG_SHAPES = {
    "c2": [(4096, 6144, 0), (4096, 4096, 1), (4096, 2 * 14336, 2), (14336, 4096, 1)],
    "c3_n8": [(8192, 1280, 0), (1024, 8192, 0), (8192, 2 * 3584, 2), (3584, 8192, 0)],
    "c3_n5": [(8192, 5120, 0), (4096, 8192, 0), (8192, 2 * 5760, 2), (5760, 8192, 0)],
}


@pytest.mark.parametrize("config", sorted(_CONFIG_SHAPES))
def test_projections_at_baseline_shapes(config):
    from paper_2511_14116_b200.gemm import PackedWeight, SkinnyGemm, interleave_gate_up
    gemm = SkinnyGemm()
    g = torch.Generator(device="cuda").manual_seed(len(config))
    for K, N, epi in _CONFIG_SHAPES[config]:
        x = torch.randn((64, K), device="cuda", generator=g).to(torch.bfloat16)
        w = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
        if epi == 2:
            w = interleave_gate_up(w[:, :N // 2], w[:, N // 2:])
        n_out = N // 2 if epi == 2 else N
        base = torch.randn((64, n_out), device="cuda", generator=g).to(torch.bfloat16)
        out = base.clone()
        gemm(x, PackedWeight(w), out, epi)
        torch.cuda.synchronize()
        ref = _ref(x, w)
        if epi == 2:
            blk = ref.view(64, -1, 2, 64)
            ref = torch.nn.functional.silu(blk[:, :, 0].reshape(64, -1)) * blk[:, :, 1].reshape(64, -1)
        elif epi == 1:
            ref = ref + base.float()
        _close(out, ref)


@pytest.mark.parametrize("t0,nt,s0,ns", [(0, 1, 0, 16), (3, 5, 0, 16), (2, 4, 5, 7), (0, 160, 3, 2)])
def test_packed_pieces_are_canonical_across_column_groups(t0, nt, s0, ns):
    """Failover pieces of packed weights (HybridDecodeRank._blocks): the
    two-tile layout yields the same piece bytes as the one-tile layout
    (the canonical [tile][step] order), and writing a piece back into a
    two-tile weight restores its blocks."""
    from paper_2511_14116_b200.gemm import PackedWeight
    from paper_2511_14116_b200.hostmirror import SegmentCopy
    from paper_2511_14116_b200.hybrid import HybridDecodeRank as H
    g = torch.Generator(device="cuda").manual_seed(t0 + nt + s0 + ns)
    w = torch.randn((1024, 160 * 128), device="cuda", generator=g).to(torch.bfloat16)
    p1, p2 = PackedWeight(w, 1), PackedWeight(w, 2)
    nbytes = nt * ns * 16384
    pieces = []
    for pw in (p1, p2):
        buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        seg = SegmentCopy()
        H._to_piece(seg, H._blocks(pw, t0, nt, s0, ns, 0), buf.data_ptr())
        seg.run(buf.device)
        pieces.append(buf)
    torch.cuda.synchronize()
    assert torch.equal(pieces[0], pieces[1])
    back = PackedWeight.empty(1024, 160 * 128, "cuda", group=2)
    back.panels.copy_(p2.panels)
    for t in range(t0, t0 + nt):  # clobber the target blocks first
        for s in range(s0, s0 + ns):
            back.panels[t // 2, s, t % 2].zero_()
    seg = SegmentCopy()
    H._from_piece(seg, H._blocks(back, t0, nt, s0, ns, 0), pieces[0].data_ptr())
    seg.run(back.panels.device)
    torch.cuda.synchronize()
    assert torch.equal(back.panels, p2.panels)
