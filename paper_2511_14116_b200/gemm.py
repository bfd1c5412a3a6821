"""Host side of the skinny tcgen05 GEMM (``fs_gemm_skinny``, csrc/gemm.cu).

The decode step's four projections per layer run through it:

* QKV      ``qkv = x @ Wqkv``                       (STORE)
* O-proj   ``x  += o @ Wo``      world 1            (RESIDUAL, in place)
           ``part = o @ Wo``     world > 1          (STORE, then all-reduce)
* gate/up  ``act = silu(x@Wg) * (x@Wu)``            (SWIGLU, fused epilogue)
* down     ``x  += act @ Wd`` / ``part = act @ Wd`` (RESIDUAL / STORE)

Batches above 64 rows are processed in 64-row chunks.
"""

from __future__ import annotations

import torch

from . import _native as N
from .core import ValidationError

STORE, RESIDUAL, SWIGLU = 0, 1, 2
MAX_ROWS = 64


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[K, C] gate and up -> [K, 2C] with 64-column blocks g0 u0 g1 u1 ...
    (the layout the SWIGLU epilogue expects; C % 64 == 0)."""
    K, C = w_gate.shape
    if C % 64:
        raise ValidationError("gate/up width must be a multiple of 64")
    g = w_gate.reshape(K, C // 64, 1, 64)
    u = w_up.reshape(K, C // 64, 1, 64)
    return torch.cat([g, u], dim=2).reshape(K, 2 * C).contiguous()


def _sm_count(device=None) -> int:
    return torch.cuda.get_device_properties(device if device is not None else
                                            torch.cuda.current_device()).multi_processor_count


class PackedWeight:
    """A [K, N] weight pre-packed (once, at load) into the GEMM's streaming
    order: one 16 KB block per (128-column tile t, 64-row k-step s), blocks
    ordered [group][s][g] with t = group * G + g.  A block is W^T's tile as
    the UMMA K-major SWIZZLE_128B A operand, as is: 128 rows (output
    columns) of 64 k x bf16 = 128 B, 16-byte chunk c of row f stored at
    chunk c ^ (f % 8).  A CTA owns a column group and a k-range of it, which
    is ONE contiguous region of HBM, moved in 32 KB bulk copies.

    G (tiles per CTA) is 1, or 2 when the tiles outnumber the SMs (then a
    group's step is 2 tiles x 16 KB, still one 32 KB copy)."""

    def __init__(self, w: torch.Tensor, group: int = None):
        K, n = w.shape
        if n % 128 or K % 64:
            raise ValidationError("packed weights need N % 128 == 0 and K % 64 == 0")
        tiles = n // 128
        if group is None:
            group = auto_group(w.device, tiles)
        if group not in (1, 2) or tiles % group:
            raise ValidationError(f"bad column group {group} for {tiles} tiles")
        self.K, self.N, self.group = K, n, group
        # w[k, col]: k = (s, ch, e), col = (grp, g, f)
        b = w.reshape(K // 64, 8, 8, tiles // group, group, 128)    # s ch e grp g f
        b = b.permute(3, 0, 4, 5, 1, 2)                             # grp s g f ch e
        f, sw = _swizzle_index(w.device)
        self.panels = b[:, :, :, f, sw].contiguous()

    @classmethod
    def empty(cls, K: int, n: int, device, group: int = 1) -> "PackedWeight":
        """Uninitialised panels of a [K, n] weight (filled by block copies:
        failover adoption, hybrid.HybridDecodeRank.adopt)."""
        if n % (128 * group) or K % 64:
            raise ValidationError("packed weights need N % 128 == 0 and K % 64 == 0")
        self = cls.__new__(cls)
        self.K, self.N, self.group = K, n, group
        self.panels = torch.empty((n // (128 * group), K // 64, group, 128, 8, 8),
                                  dtype=torch.bfloat16, device=device)
        return self

    @classmethod
    def empty_layers(cls, L: int, K: int, n: int, device, group: int = None) -> list:
        """``L`` uninitialised [K, n] weights carved from ONE allocation (an
        adoption re-lays out every layer at once; one cudaMalloc, not L);
        ``group`` None: the layout packing would pick."""
        if group is None:
            group = auto_group(device, n // 128)
        if n % (128 * group) or K % 64:
            raise ValidationError("packed weights need N % 128 == 0 and K % 64 == 0")
        buf = torch.empty((L, n // (128 * group), K // 64, group, 128, 8, 8),
                          dtype=torch.bfloat16, device=device)
        out = []
        for layer in range(L):
            self = cls.__new__(cls)
            self.K, self.N, self.group = K, n, group
            self.panels = buf[layer]
            out.append(self)
        return out

    def unpack(self) -> torch.Tensor:
        f, sw = _swizzle_index(self.panels.device)
        b = self.panels[:, :, :, f, sw]                             # the swizzle is an involution
        return b.permute(1, 4, 5, 0, 2, 3).reshape(self.K, self.N)


def auto_group(device, tiles: int) -> int:
    """Tiles per CTA of a packed weight: two when the 128-column tiles
    outnumber the SMs (and pair up), else one."""
    return 2 if tiles > _sm_count(device) and tiles % 2 == 0 else 1


def _swizzle_index(device):
    f = torch.arange(128, device=device)
    return f[:, None], torch.arange(8, device=device)[None, :] ^ (f[:, None] & 7)


class SkinnyGemm:
    """Launcher of ``fs_gemm_skinny`` on one device (shared by all
    projections of an engine; launches are stream-ordered).  The ABI's
    workspace / semaphore arguments are reserved (split tiles are reduced
    over distributed shared memory); minimal buffers are passed."""

    def __init__(self, max_n: int = 0, device=None):
        self.device = torch.device(device if device is not None else "cuda")
        self.index = self.device.index if self.device.index is not None \
            else torch.cuda.current_device()
        floats = N.lib.fs_gemm_workspace_floats(self.index, max_n, 0)
        if floats < 0:
            raise ValidationError("cannot size the GEMM workspace")
        self.max_n = max_n
        self.ws = torch.empty(floats, dtype=torch.float32, device=self.device)
        self.sems = torch.zeros(2, dtype=torch.int32, device=self.device)

    def __call__(self, x: torch.Tensor, w, out: torch.Tensor,
                 epilogue: int = STORE, res: torch.Tensor = None) -> torch.Tensor:
        """``w``: a [K, N] row-major bf16 matrix or a :class:`PackedWeight`."""
        packed = isinstance(w, PackedWeight)
        wt = w.panels if packed else w
        if x.dtype != torch.bfloat16 or wt.dtype != torch.bfloat16 or out.dtype != torch.bfloat16:
            raise ValidationError("skinny GEMM operands must be bf16")
        rows, K = x.shape
        Kw, n = (w.K, w.N) if packed else w.shape
        if Kw != K or x.stride(1) != 1 or wt.stride(-1) != 1 or out.stride(1) != 1:
            raise ValidationError("skinny GEMM: shape / layout mismatch")
        if epilogue == RESIDUAL and res is None:
            res = out
        stream = N.C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        ws_floats = self.ws.numel()
        for r0 in range(0, rows, MAX_ROWS):
            r = min(MAX_ROWS, rows - r0)
            xs, os = x[r0:r0 + r], out[r0:r0 + r]
            rs = res[r0:r0 + r] if res is not None else None
            N.check(N.lib.fs_gemm_skinny(
                N.ptr(xs), x.stride(0), r, K, N.ptr(wt), 128 if packed else wt.stride(0),
                w.group if packed else 0, n, N.ptr(os), out.stride(0),
                N.ptr(rs), res.stride(0) if res is not None else 0, epilogue, N.ptr(self.ws),
                ws_floats, N.ptr(self.sems), self.index, stream), "fs_gemm_skinny")
        return out
