"""The hybrid-attention decode step of one rank (the decode form of the
reference's ``parallel_forward``, ``refexec.py:249-308``).

For each layer, rank ``g``:

1. ``[q|k|v] = x @ Wqkv_g`` for the rank's local KV-head slots (its TP
   heads + the replicated heads; one cuBLAS GEMM);
2. ONE ``fs_decode_attention`` launch appends the new token's K/V of every
   work item into its page (fused K3) and attends every work item: TP
   slots for all requests, replicated slots only for requests routed to
   ``g`` (refexec.py:284-297), merging split items in-kernel (fused K2);
3. ``part = o @ Wo_g`` -- rows of replicated slots for requests routed
   elsewhere are zero, so their contribution is exactly zero;
4. exchange: ``all_reduce(part)`` over the surviving ranks (NCCL over
   NVLink; the reference's exact sum in ascending rank order,
   refexec.py:283-298), ``x += part``;
5. (``mlp=True``) the TP MLP partial over the FFN shards the rank owns
   (``plan.ffn``, refexec.py:299-307): ``act = swiglu(x @ [Wg|Wu]_g)``
   (``fs_swiglu``), ``part = act @ Wd_g``, all-reduce, ``x += part``.

Weights are synthetic and keyed by GLOBAL (row, col) indices
(``fs_fill_normal``): every rank of every world size -- including the
on-demand targets after failures -- materialises bit-identical slices of one
global model, so the sum over ranks reproduces the single-GPU result.
``capture()`` records a whole step (all layers) as one CUDA graph.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import ModelSpec, ValidationError
from .kvcache import PagedKVCache, RankWork

# tensor ids of the synthetic weight salts
_WQ, _WK, _WV, _WO, _WG, _WU, _WD = 1, 2, 3, 4, 5, 6, 7


def _fill(out: torch.Tensor, layer: int, tensor: int, seed: int, scale: float,
          row_off: int = 0, col_off: int = 0, col_map=None) -> None:
    """Fill a 2-D bf16 (view) tensor with its slice of a global matrix."""
    if out.dtype != torch.bfloat16 or out.dim() != 2 or out.stride(1) != 1:
        raise ValidationError("fill target must be a row-major bf16 matrix")
    cm = None
    if col_map is not None:
        cm = torch.as_tensor(np.asarray(col_map, dtype=np.int32)).to(out.device)
    N.check(N.lib.fs_fill_normal(N.ptr(out), out.shape[0], out.shape[1], out.stride(0), None,
                                 row_off, N.ptr(cm), col_off, seed, layer * 16 + tensor,
                                 float(scale), N.C.c_void_p(
                                     torch.cuda.current_stream(out.device).cuda_stream)),
            "fs_fill_normal")


def _scales(model: ModelSpec):
    return (1.0 / math.sqrt(model.hidden_dim),
            0.5 / math.sqrt(model.num_q_heads * model.head_dim),
            0.5 / math.sqrt(model.ffn_intermediate_dim))


def head_weights(model: ModelSpec, layer: int, head: int, seed: int, device):
    """The weights of KV head ``head``'s group in ``layer``:
    wq [hidden, qpk*hd], wk/wv [hidden, hd], wo [qpk*hd, hidden] (bf16)."""
    hd, qpk, hid = model.head_dim, model.q_heads_per_kv_head, model.hidden_dim
    s_in, s_o, _ = _scales(model)
    wq = torch.empty((hid, qpk * hd), dtype=torch.bfloat16, device=device)
    wk = torch.empty((hid, hd), dtype=torch.bfloat16, device=device)
    wv = torch.empty_like(wk)
    wo = torch.empty((qpk * hd, hid), dtype=torch.bfloat16, device=device)
    _fill(wq, layer, _WQ, seed, s_in, col_off=head * qpk * hd)
    _fill(wk, layer, _WK, seed, s_in, col_off=head * hd)
    _fill(wv, layer, _WV, seed, s_in, col_off=head * hd)
    _fill(wo, layer, _WO, seed, s_o, row_off=head * qpk * hd)
    return wq, wk, wv, wo


def ffn_columns(model: ModelSpec, shard_owner, rank: int) -> np.ndarray:
    """Global intermediate columns of the FFN shards ``rank`` owns
    (ShardedView.shard_cols, refexec.py:150-154)."""
    shards = [s for s, g in enumerate(shard_owner) if g == rank]
    width = model.ffn_intermediate_dim // len(shard_owner)
    return np.array([c for s in sorted(shards) for c in range(s * width, (s + 1) * width)],
                    dtype=np.int32)


def ffn_weights(model: ModelSpec, layer: int, cols, seed: int, device):
    """wgu [hidden, 2*C] (gate | up columns), wd [C, hidden] for global
    intermediate columns ``cols``."""
    s_in, _, s_d = _scales(model)
    C = len(cols)
    hid = model.hidden_dim
    wgu = torch.empty((hid, 2 * C), dtype=torch.bfloat16, device=device)
    wd = torch.empty((C, hid), dtype=torch.bfloat16, device=device)
    if C:
        _fill(wgu[:, :C], layer, _WG, seed, s_in, col_map=cols)
        _fill(wgu[:, C:], layer, _WU, seed, s_in, col_map=cols)
        # down projection: generated as its transpose keyed (hidden, intermediate)
        wdt = torch.empty((hid, C), dtype=torch.bfloat16, device=device)
        _fill(wdt, layer, _WD, seed, s_d, col_map=cols)
        wd.copy_(wdt.t())
    return wgu, wd


class HybridDecodeRank:
    """One rank's share of the hybrid decode step.

    ``owner``: int32 [L, H] (``placement.owner_array``); ``routing``:
    request -> GPU; ``shard_owner``: FFN shard -> GPU (``plan.ffn``), needed
    when ``mlp``; ``group``: torch.distributed group of the alive ranks
    (None = no exchange: world 1 or single-GPU emulation).
    """

    def __init__(self, model: ModelSpec, owner, rank: int, routing, batch: int, capacity: int,
                 device=None, seed: int = 0, group=None, page_order: str = "contiguous",
                 config: int = 0, mlp: bool = False, shard_owner=None, gemm: str = "tcgen05",
                 request_capacity=None, exchange: str = "nccl", exchange_elems: int = None,
                 reserve_pages: int = 0):
        if model.head_dim != N.HEAD_DIM:
            raise ValidationError(f"head_dim must be {N.HEAD_DIM} for the CUDA path")
        self.model = model
        self.rank = rank
        self.batch = batch
        self.group = group
        self.mlp = mlp
        self.device = torch.device(device if device is not None else "cuda")
        self.qpk = model.q_heads_per_kv_head
        self.work = RankWork.build(np.asarray(owner, dtype=np.int32), rank, routing, batch)
        self.cache = PagedKVCache(self.work, capacity, self.qpk, self.device,
                                  page_order=page_order, seed=seed, config=config,
                                  request_capacity=request_capacity, reserve_pages=reserve_pages)
        self.backup_ptr = None  # token-granular K5 target (hostmirror.KVMirror), if any
        hd, hid, S = model.head_dim, model.hidden_dim, self.work.n_slots
        self.n_slots = S
        L = model.num_layers
        dev = self.device
        rw = self.cache.set_fused_layout()   # [q slots | k slots | v slots]
        # every decode launch of the step directly follows the QKV GEMM,
        # which writes only qkv: K1 may stage its first pages under PDL
        self.cache.early_prefetch = True
        qw = S * self.qpk * hd
        s_in, s_o, _ = _scales(model)
        self.wqkv = torch.zeros((L, hid, rw), dtype=torch.bfloat16, device=dev)
        self.wo = torch.zeros((L, qw, hid), dtype=torch.bfloat16, device=dev)
        for layer in range(L):
            for j, h in enumerate(self.work.slot_heads[layer]):
                qs = slice(j * self.qpk * hd, (j + 1) * self.qpk * hd)
                _fill(self.wqkv[layer, :, qs], layer, _WQ, seed, s_in, col_off=h * self.qpk * hd)
                _fill(self.wqkv[layer, :, qw + j * hd:qw + (j + 1) * hd], layer, _WK, seed, s_in,
                      col_off=h * hd)
                _fill(self.wqkv[layer, :, qw + (S + j) * hd:qw + (S + j + 1) * hd], layer, _WV,
                      seed, s_in, col_off=h * hd)
                _fill(self.wo[layer, qs, :], layer, _WO, seed, s_o, row_off=h * self.qpk * hd)
        self.qkv = torch.empty((batch, rw), dtype=torch.bfloat16, device=dev)
        self.o = torch.zeros((batch * S, self.qpk, hd), dtype=torch.bfloat16, device=dev)
        self.part = torch.empty((batch, hid), dtype=torch.bfloat16, device=dev)
        self.x = torch.zeros((batch, hid), dtype=torch.bfloat16, device=dev)
        self.ffn_cols = np.zeros(0, dtype=np.int32)
        self.shards = []
        self.num_shards = len(shard_owner) if shard_owner is not None else 0
        if mlp:
            if shard_owner is None:
                raise ValidationError("mlp=True needs the FFN shard owner table")
            self.shards = sorted(s_ for s_, g in enumerate(shard_owner) if g == rank)
            self.ffn_cols = ffn_columns(model, shard_owner, rank)
            C = len(self.ffn_cols)
            self.w_gu = torch.empty((L, hid, 2 * C), dtype=torch.bfloat16, device=dev)
            self.w_d = torch.empty((L, C, hid), dtype=torch.bfloat16, device=dev)
            for layer in range(L):
                gu, d = ffn_weights(model, layer, self.ffn_cols, seed, dev)
                self.w_gu[layer].copy_(gu)
                self.w_d[layer].copy_(d)
            self.h = torch.empty((batch, 2 * C), dtype=torch.bfloat16, device=dev)
            self.act = torch.empty((batch, C), dtype=torch.bfloat16, device=dev)
        if gemm not in ("cublas", "tcgen05"):
            raise ValidationError(f"unknown gemm backend {gemm!r}")
        if exchange not in ("nccl", "fused"):
            raise ValidationError(f"unknown exchange {exchange!r}")
        # exchange "fused": the projection GEMMs write their partials into
        # IPC-shared buffers and fs_ar_residual does the ordered sum + the
        # residual in one kernel over peer memory (collective.py)
        self.exchange = exchange if group is not None else "nccl"
        self.xchg = None
        if self.exchange == "fused":
            from .collective import FusedExchange
            self.xchg = FusedExchange(group, exchange_elems or batch * model.hidden_dim,
                                      self.device)
        self.gemm = gemm
        if gemm == "tcgen05":
            self._use_skinny()
        self._graph = None

    def _use_skinny(self) -> None:
        """Projections through the hand-written tcgen05 GEMM: weights packed
        once into its streaming layout; gate/up interleaved for the fused
        SwiGLU epilogue."""
        from .gemm import PackedWeight, SkinnyGemm, interleave_gate_up
        L = self.model.num_layers
        self.p_qkv = [PackedWeight(self.wqkv[l]) for l in range(L)]
        self.p_o = [PackedWeight(self.wo[l]) for l in range(L)]
        widest = max(self.wqkv.shape[2], self.wo.shape[2])
        if self.mlp and len(self.ffn_cols):
            C = len(self.ffn_cols)
            self.p_gu = [PackedWeight(interleave_gate_up(self.w_gu[l, :, :C], self.w_gu[l, :, C:]))
                         for l in range(L)]
            self.p_d = [PackedWeight(self.w_d[l]) for l in range(L)]
            widest = max(widest, 2 * C, self.w_d.shape[2])
            del self.w_gu, self.w_d
        del self.wqkv, self.wo
        torch.cuda.empty_cache()
        self.skinny = SkinnyGemm(widest, self.device)

    # ------------------------------------------------------------------ api --
    def set_lengths(self, lens) -> None:
        """Per-request attended length of the NEXT step (the new token sits
        at position len-1 and attends itself, refexec.py:97)."""
        self.cache.set_lengths(lens)

    def fill_random_kv(self, seed: int = 0) -> None:
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        self.cache.pool.view(torch.bfloat16).normal_(generator=g)

    def attention_partial(self, layer: int) -> torch.Tensor:
        """This rank's pre-exchange attention contribution of ``layer`` for
        the current ``self.x``: ``o @ Wo_g`` [B, hidden] (into ``self.part``)."""
        B, S, hd = self.batch, self.n_slots, self.model.head_dim
        if self.gemm == "tcgen05":
            from .gemm import STORE
            self.skinny(self.x, self.p_qkv[layer], self.qkv, STORE)
            self.cache.decode_layer_fused(layer, self.qkv, self.o)
            self.skinny(self.o.view(B, S * self.qpk * hd), self.p_o[layer], self.part, STORE)
            return self.part
        torch.matmul(self.x, self.wqkv[layer], out=self.qkv)         # cuBLAS
        self.cache.decode_layer_fused(layer, self.qkv, self.o)       # K1 (+K2, +K3)
        torch.matmul(self.o.view(B, S * self.qpk * hd), self.wo[layer], out=self.part)
        return self.part

    def _swiglu(self) -> None:
        C = self.act.shape[1]
        N.check(N.lib.fs_swiglu(N.ptr(self.h), self.batch, C, 2 * C, N.ptr(self.act), C,
                                N.C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)),
                "fs_swiglu")

    def mlp_partial(self, layer: int) -> torch.Tensor:
        """This rank's pre-exchange MLP contribution (its FFN shards)."""
        if not len(self.ffn_cols):
            return self.part.zero_()
        if self.gemm == "tcgen05":
            from .gemm import STORE, SWIGLU
            self.skinny(self.x, self.p_gu[layer], self.act, SWIGLU)
            self.skinny(self.act, self.p_d[layer], self.part, STORE)
            return self.part
        torch.matmul(self.x, self.w_gu[layer], out=self.h)
        self._swiglu()
        torch.matmul(self.act, self.w_d[layer], out=self.part)
        return self.part

    def _layers_skinny(self) -> None:
        from .gemm import RESIDUAL, STORE, SWIGLU
        B, S, hd = self.batch, self.n_slots, self.model.head_dim
        x, o2, g = self.x, self.o.view(B, S * self.qpk * hd), self.skinny
        for layer in range(self.model.num_layers):
            g(x, self.p_qkv[layer], self.qkv, STORE)
            self.cache.decode_layer_fused(layer, self.qkv, self.o)
            if self.xchg is not None and self.group is not None:
                # partials straight into the symmetric exchange buffers;
                # fs_ar_residual does the ordered sum + residual
                ia, im = (0, 1) if self.mlp else (layer & 1, None)
                g(o2, self.p_o[layer], self.xchg.partial(ia, x.shape), STORE)
                self.xchg.reduce_residual(ia, x)
                if self.mlp:
                    part = self.xchg.partial(im, x.shape)
                    if len(self.ffn_cols):
                        g(x, self.p_gu[layer], self.act, SWIGLU)
                        g(self.act, self.p_d[layer], part, STORE)
                    else:
                        part.zero_()
                    self.xchg.reduce_residual(im, x)
                continue
            if self.group is None:
                g(o2, self.p_o[layer], x, RESIDUAL)
            else:
                g(o2, self.p_o[layer], self.part, STORE)
                torch.distributed.all_reduce(self.part, group=self.group)
                x.add_(self.part)
            if self.mlp and len(self.ffn_cols):
                g(x, self.p_gu[layer], self.act, SWIGLU)
                if self.group is None:
                    g(self.act, self.p_d[layer], x, RESIDUAL)
                else:
                    g(self.act, self.p_d[layer], self.part, STORE)
            if self.mlp and self.group is not None:
                if not len(self.ffn_cols):
                    self.part.zero_()
                torch.distributed.all_reduce(self.part, group=self.group)
                x.add_(self.part)

    def _layers(self) -> None:
        self._layers_inner()
        if self.backup_ptr is not None:
            self.backup_tokens()

    def _layers_inner(self) -> None:
        if self.gemm == "tcgen05":
            return self._layers_skinny()
        B, S, hd = self.batch, self.n_slots, self.model.head_dim
        x, o2 = self.x, self.o.view(B, S * self.qpk * hd)
        for layer in range(self.model.num_layers):
            if self.group is None:
                torch.matmul(x, self.wqkv[layer], out=self.qkv)      # cuBLAS
                self.cache.decode_layer_fused(layer, self.qkv, self.o)
                x.addmm_(o2, self.wo[layer])                         # x += o Wo
                if self.mlp and len(self.ffn_cols):
                    torch.matmul(x, self.w_gu[layer], out=self.h)
                    self._swiglu()
                    x.addmm_(self.act, self.w_d[layer])              # x += act Wd
            elif self.xchg is not None:
                # buffers alternate between consecutive exchanges
                ia, im = (0, 1) if self.mlp else (layer & 1, None)
                torch.matmul(x, self.wqkv[layer], out=self.qkv)
                self.cache.decode_layer_fused(layer, self.qkv, self.o)
                torch.matmul(o2, self.wo[layer], out=self.xchg.partial(ia, x.shape))
                self.xchg.reduce_residual(ia, x)                     # x += sum_r part_r
                if self.mlp:
                    part = self.xchg.partial(im, x.shape)
                    if len(self.ffn_cols):
                        torch.matmul(x, self.w_gu[layer], out=self.h)
                        self._swiglu()
                        torch.matmul(self.act, self.w_d[layer], out=part)
                    else:
                        part.zero_()
                    self.xchg.reduce_residual(im, x)
            else:
                self.attention_partial(layer)
                torch.distributed.all_reduce(self.part, group=self.group)
                x.add_(self.part)
                if self.mlp:
                    self.mlp_partial(layer)
                    torch.distributed.all_reduce(self.part, group=self.group)
                    x.add_(self.part)

    # ------------------------------------------------ failover (in place) --
    def _head_parts(self, layer: int, j: int, wqkv=None, wo=None, S=None):
        """Slot ``j`` of ``layer`` in the fused weights as the 4 parts of a
        canonical head piece (hostmirror.WeightLayout), in piece order:
        [(address, row pitch, row bytes, rows, offset in the piece)]."""
        if self.gemm == "tcgen05":
            return self._head_parts_packed(layer, j, wqkv, wo, S)
        wqkv = self.wqkv if wqkv is None else wqkv
        wo = self.wo if wo is None else wo
        S = self.n_slots if S is None else S
        hd, qpk, hid = self.model.head_dim, self.qpk, self.model.hidden_dim
        qw, rw = S * qpk * hd, wqkv.shape[2]
        base = wqkv.data_ptr() + layer * hid * rw * 2
        qb, kb = hid * qpk * hd * 2, hid * hd * 2
        o_addr = wo.data_ptr() + (layer * wo.shape[1] + j * qpk * hd) * hid * 2
        return [(base + j * qpk * hd * 2, rw * 2, qpk * hd * 2, hid, 0),          # Wq
                (base + (qw + j * hd) * 2, rw * 2, hd * 2, hid, qb),              # Wk
                (base + (qw + (S + j) * hd) * 2, rw * 2, hd * 2, hid, qb + kb),   # Wv
                (o_addr, qpk * hd * hid * 2, qpk * hd * hid * 2, 1, qb + 2 * kb)]  # Wo

    # packed weights (gemm.PackedWeight): 16 KB blocks.  A head piece is [Wq
    # panels (qpk tiles) | Wk panel | Wv panel | Wo: per output tile, the
    # head's 2 qpk k-step blocks]; a shard piece is [gate/up panels (w/64
    # interleaved tiles) | Wd: per output tile, the shard's w/64 k-step
    # blocks] -- the same bytes as the row-major pieces, in the layout the
    # GEMM streams, so adoption is plain block copies.
    _BLK = 16384

    @classmethod
    def _blocks(cls, pw, t0: int, nt: int, s0: int, ns: int, off: int) -> list:
        """Blocks (t, s), t in [t0, t0+nt), s in [s0, s0+ns), of a packed
        weight as parts of a piece in the canonical [t][s] order (the
        one-tile layout's) from piece offset ``off``.  One-tile groups: one
        (2-D) run; two-tile groups interleave the pair's blocks per step,
        so each tile is a strided run of its own."""
        B, nk, base = cls._BLK, pw.K // 64, pw.panels.data_ptr()
        if pw.group == 1:
            if ns == nk:
                return [(base + t0 * nk * B, nt * nk * B, nt * nk * B, 1, off)]
            return [(base + (t0 * nk + s0) * B, nk * B, ns * B, nt, off)]
        return [(base + (((t // 2) * nk + s0) * 2 + t % 2) * B, 2 * B, B, ns, off + i * ns * B)
                for i, t in enumerate(range(t0, t0 + nt))]

    def _head_parts_packed(self, layer: int, j: int, p_qkv=None, p_o=None, S=None):
        p_qkv = self.p_qkv if p_qkv is None else p_qkv
        p_o = self.p_o if p_o is None else p_o
        S = self.n_slots if S is None else S
        qpk, hid, B = self.qpk, self.model.hidden_dim, self._BLK
        q, o = p_qkv[layer], p_o[layer]
        nk = hid // 64
        panel = nk * B
        qb = qpk * panel
        return (self._blocks(q, j * qpk, qpk, 0, nk, 0) +                         # Wq
                self._blocks(q, S * qpk + j, 1, 0, nk, qb) +                      # Wk
                self._blocks(q, S * qpk + S + j, 1, 0, nk, qb + panel) +          # Wv
                self._blocks(o, 0, hid // 128, j * 2 * qpk, 2 * qpk, qb + 2 * panel))  # Wo

    def _shard_parts_packed(self, layer: int, k: int, p_gu=None, p_d=None):
        p_gu = self.p_gu if p_gu is None else p_gu
        p_d = self.p_d if p_d is None else p_d
        hid, B = self.model.hidden_dim, self._BLK
        gu, d = p_gu[layer], p_d[layer]
        tw = (self.model.ffn_intermediate_dim // self.num_shards) // 64
        nk = hid // 64
        return (self._blocks(gu, k * tw, tw, 0, nk, 0) +                          # Wg|Wu
                self._blocks(d, 0, hid // 128, k * tw, tw, tw * nk * B))            # Wd

    def _shard_parts(self, layer: int, k: int, w_gu=None, w_d=None):
        """Local FFN shard ``k`` of ``layer`` as the parts of a canonical
        shard piece ``[Wg | Wu | Wd]`` (same tuple format)."""
        if self.gemm == "tcgen05":
            return self._shard_parts_packed(layer, k, w_gu, w_d)
        w_gu = self.w_gu if w_gu is None else w_gu
        w_d = self.w_d if w_d is None else w_d
        hid = self.model.hidden_dim
        w = self.model.ffn_intermediate_dim // self.num_shards
        C2 = w_gu.shape[2]
        base = w_gu.data_ptr() + layer * hid * C2 * 2
        d_addr = w_d.data_ptr() + (layer * w_d.shape[1] + k * w) * hid * 2
        return [(base + k * w * 2, C2 * 2, w * 2, hid, 0),                        # Wg
                (base + (C2 // 2 + k * w) * 2, C2 * 2, w * 2, hid, hid * w * 2),   # Wu
                (d_addr, w * hid * 2, w * hid * 2, 1, 2 * hid * w * 2)]            # Wd

    @staticmethod
    def _to_piece(seg, parts, piece: int) -> None:
        for addr, pitch, width, rows, off in parts:
            seg.add(piece + off, width, addr, pitch, width, rows)

    @staticmethod
    def _from_piece(seg, parts, piece: int) -> None:
        for addr, pitch, width, rows, off in parts:
            seg.add(addr, pitch, piece + off, width, width, rows)

    @staticmethod
    def _between(seg, src_parts, dst_parts) -> None:
        for (sa, sp, width, rows, _), (da, dp, _, _, _) in zip(src_parts, dst_parts):
            seg.add(da, dp, sa, sp, width, rows)

    def publish_weights(self, store, heads=None) -> int:
        """Write this rank's weight pieces into the node's host weight
        store (hostmirror.WeightStore): its TP heads (or ``heads``: per
        layer the head ids to publish) and its FFN shards.  One launch
        (D2H over PCIe into the mapped store); returns bytes written."""
        from .hostmirror import SegmentCopy
        lay = store.layout
        seg = SegmentCopy()
        for layer in range(self.model.num_layers):
            sel = heads[layer] if heads is not None else \
                self.work.slot_heads[layer][:self.work.n_tp[layer]]
            for j, h in enumerate(self.work.slot_heads[layer]):
                if h in sel:
                    self._to_piece(seg, self._head_parts(layer, j),
                                   store.dev_ptr + lay.head_off(layer, h))
            if self.mlp:
                for k, sh in enumerate(self.shards):
                    self._to_piece(seg, self._shard_parts(layer, k),
                                   store.dev_ptr + lay.shard_off(layer, sh))
        seg.run(self.device)
        return seg.bytes

    def load_pieces(self, pieces) -> int:
        """Overwrite every slot's and shard's weights from canonical pieces
        (``adopt``'s ``pieces`` map): a GPU reloading its whole assignment
        (expansion, recovery.py:366-394).  One launch; returns bytes."""
        from .hostmirror import SegmentCopy
        seg = SegmentCopy()
        for layer in range(self.model.num_layers):
            for j, h in enumerate(self.work.slot_heads[layer]):
                self._from_piece(seg, self._head_parts(layer, j), pieces[("head", layer, h)])
            if self.mlp:
                for k, sh in enumerate(self.shards):
                    self._from_piece(seg, self._shard_parts(layer, k), pieces[("shard", layer, sh)])
        seg.run(self.device)
        torch.cuda.current_stream(self.device).synchronize()
        return seg.bytes

    def adopt(self, owner, routing, shard_owner, pieces) -> np.ndarray:
        """Adopt a new placement IN PLACE (the on-demand shrink target,
        recovery.py:396-427, after re-routing): KV pages of every (layer,
        head, request) the rank keeps stay where they are (new items get
        reserve pages, PagedKVCache.adopt); the fused weights are re-laid
        out for the new slots in ONE copy launch -- kept slots / shards from
        the current tensors, new ones from ``pieces``: {("head", layer,
        head) | ("shard", layer, shard): device address of the canonical
        piece} (the K7 staging buffer).  Returns the new items (their KV is
        restored by the caller).  The step graph must be captured again."""
        from .hostmirror import SegmentCopy
        old_work = self.work
        work = RankWork.build(np.asarray(owner, dtype=np.int32), self.rank, routing, self.batch)
        new_shards = sorted(s_ for s_, g in enumerate(shard_owner) if g == self.rank) \
            if self.mlp else self.shards
        if work.slot_heads == old_work.slot_heads and new_shards == self.shards:
            # same slots and shards (a routing change): only the KV tables move
            fresh = self.cache.adopt(work)
            self.work = work
            self._graph = None
            return fresh
        L, hd, hid, qpk = self.model.num_layers, self.model.head_dim, self.model.hidden_dim, self.qpk
        S = work.n_slots
        rw = S * (qpk + 2) * hd
        dev = self.device
        packed = self.gemm == "tcgen05"
        if packed:
            from .gemm import PackedWeight
            wqkv = PackedWeight.empty_layers(L, hid, rw, dev)
            wo = PackedWeight.empty_layers(L, S * qpk * hd, hid, dev)
        else:
            wqkv = torch.zeros((L, hid, rw), dtype=torch.bfloat16, device=dev)
            wo = torch.zeros((L, S * qpk * hd, hid), dtype=torch.bfloat16, device=dev)
        seg = SegmentCopy()
        for layer in range(L):
            old_heads = old_work.slot_heads[layer]
            for j, h in enumerate(work.slot_heads[layer]):
                new_parts = self._head_parts(layer, j, wqkv=wqkv, wo=wo, S=S)
                if h in old_heads:  # kept slot: straight from the current tensors
                    self._between(seg, self._head_parts(layer, old_heads.index(h)), new_parts)
                else:
                    key = ("head", layer, h)
                    if key not in pieces:
                        raise SimulationError(f"no recovered weights for layer {layer} head {h}")
                    self._from_piece(seg, new_parts, pieces[key])
        shards = self.shards
        if self.mlp:
            shards = sorted(s_ for s_, g in enumerate(shard_owner) if g == self.rank)
            C = len(shards) * (self.model.ffn_intermediate_dim // self.num_shards)
            if packed:
                w_gu = PackedWeight.empty_layers(L, hid, 2 * C, dev)
                w_d = PackedWeight.empty_layers(L, C, hid, dev)
            else:
                w_gu = torch.zeros((L, hid, 2 * C), dtype=torch.bfloat16, device=dev)
                w_d = torch.zeros((L, C, hid), dtype=torch.bfloat16, device=dev)
            for layer in range(L):
                for k, sh in enumerate(shards):
                    new_parts = self._shard_parts(layer, k, w_gu=w_gu, w_d=w_d)
                    if sh in self.shards:
                        self._between(seg, self._shard_parts(layer, self.shards.index(sh)),
                                      new_parts)
                    else:
                        key = ("shard", layer, sh)
                        if key not in pieces:
                            raise SimulationError(f"no recovered weights for layer {layer} "
                                                  f"shard {sh}")
                        self._from_piece(seg, new_parts, pieces[key])
        seg.run(dev)
        torch.cuda.current_stream(dev).synchronize()
        fresh = self.cache.adopt(work)
        self.work, self.n_slots = work, S
        if packed:
            self.p_qkv, self.p_o = wqkv, wo
        else:
            self.wqkv, self.wo = wqkv, wo
        if self.mlp:
            if packed:
                self.p_gu, self.p_d = w_gu, w_d
            else:
                self.w_gu, self.w_d = w_gu, w_d
            self.shards = shards
            self.ffn_cols = ffn_columns(self.model, shard_owner, self.rank)
            C = len(self.ffn_cols)
            self.h = torch.empty((self.batch, 2 * C), dtype=torch.bfloat16, device=dev)
            self.act = torch.empty((self.batch, C), dtype=torch.bfloat16, device=dev)
        self.qkv = torch.empty((self.batch, rw), dtype=torch.bfloat16, device=dev)
        self.o = torch.zeros((self.batch * S, qpk, hd), dtype=torch.bfloat16, device=dev)
        self._graph = None
        return fresh

    def backup_tokens(self) -> None:
        """K5 (token-granular): the token each item appended this step ->
        the rank's host mirror (``self.backup_ptr``), one launch."""
        c = self.cache
        N.check(N.lib.fs_kv_backup_tokens(N.ptr(c.pool), N.ptr(c.block_table), c.pages_per_seq,
                                          N.ptr(c.item_seq), N.ptr(c.item_len), c.work.n_items,
                                          N.C.c_void_p(self.backup_ptr), N.C.c_void_p(
                                              torch.cuda.current_stream(self.device).cuda_stream)),
                "fs_kv_backup_tokens")

    def launches_per_step(self) -> int:
        """Our kernel launches per step: the fused decode launch per layer
        plus its 4 tcgen05 GEMM launches (2 without the MLP; gemm="tcgen05"),
        or the decode + swiglu launches per layer (cuBLAS GEMMs)."""
        has_mlp = self.mlp and len(self.ffn_cols)
        if self.gemm == "tcgen05":
            n = self.model.num_layers * (1 + (4 if has_mlp else 2))
        else:
            n = self.model.num_layers * (2 if has_mlp else 1)
        if self.xchg is not None:  # one fs_ar_residual per exchange
            n += self.model.num_layers * (2 if self.mlp else 1)
        if self.backup_ptr is not None:  # token backup
            n += 1
        return n

    def weight_bytes(self) -> int:
        if self.gemm == "tcgen05":
            ws = self.p_qkv + self.p_o + (getattr(self, "p_gu", []) + getattr(self, "p_d", []))
            return 2 * sum(w.panels.numel() for w in ws)
        n = self.wqkv.numel() + self.wo.numel()
        if self.mlp:
            n += self.w_gu.numel() + self.w_d.numel()
        return 2 * n

    def capture(self) -> None:
        """Capture one decode step (all layers) into a CUDA graph."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        x_saved = self.x.clone()
        with torch.cuda.stream(s):
            self._layers()  # warm cuBLAS workspaces outside capture
            # the warm-up must not advance the state: x back; the token it
            # appended at len-1 is rewritten by the next step
            self.x.copy_(x_saved)
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._layers()
        self._graph = g

    def step_io(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """One decode step from pinned host ``x_host`` into pinned host
        ``y_host``: the input copy, every layer and the result copy are ONE
        CUDA-graph launch (captured on first use for this pair of buffers);
        the caller synchronizes before reading ``y_host``."""
        io = getattr(self, "_io", None)
        if io is None or io[1] is not x_host or io[2] is not y_host or self._graph is None:
            if self._graph is None:
                self.capture()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.x.copy_(x_host, non_blocking=True)
                self._layers()
                y_host.copy_(self.x, non_blocking=True)
            self._io = io = (g, x_host, y_host)
        io[0].replay()
        return y_host

    def step(self, x: torch.Tensor = None) -> torch.Tensor:
        """One decode step: x [B, hidden] bf16 (device or pinned host) ->
        updated x (device tensor owned by the engine)."""
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        if self._graph is not None:
            self._graph.replay()
        else:
            self._layers()
        return self.x


def emulated_parallel_step(ranks, x: torch.Tensor) -> torch.Tensor:
    """Single-process emulation of one hybrid decode step over several
    ranks (all on one GPU): per layer every rank computes its partial, the
    partials are summed in ascending rank order in fp32 (the reference's
    ordered all-reduce, refexec.py:283-298) and the residual is applied;
    likewise for the MLP partials when the ranks carry the MLP."""
    ranks = sorted(ranks, key=lambda r: r.rank)
    x = x.to(torch.bfloat16)
    for layer in range(ranks[0].model.num_layers):
        for part_fn in ("attention_partial", "mlp_partial"):
            if part_fn == "mlp_partial" and not ranks[0].mlp:
                continue
            total = None
            for r in ranks:
                r.x.copy_(x)
                part = getattr(r, part_fn)(layer).float()
                total = part if total is None else total + part
            x = x + total.to(torch.bfloat16)
    return x
