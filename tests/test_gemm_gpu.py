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


@pytest.mark.parametrize("K,N,epi", [(4096, 1280, 0), (1024, 4096, 1), (2048, 896, 2)])
def test_packed_panels_match_row_major(K, N, epi):
    from paper_2511_14116_b200.gemm import PackedWeight, SkinnyGemm, interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(K + N)
    x = torch.randn((64, K), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    if epi == 2:
        w = interleave_gate_up(w[:, :N // 2], w[:, N // 2:])
    pw = PackedWeight(w)
    assert torch.equal(pw.unpack(), w)
    n_out = N // 2 if epi == 2 else N
    base = torch.randn((64, n_out), device="cuda", generator=g).to(torch.bfloat16)
    a, b = base.clone(), base.clone()
    gemm = SkinnyGemm(N)
    gemm(x, w, a, epi)
    gemm(x, pw, b, epi)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
