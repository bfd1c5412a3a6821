"""The hybrid-attention decode step of one rank (the decode form of the
reference's ``parallel_forward``, ``refexec.py:249-308``).

For each layer, rank ``g``:

1. ``[q|k|v] = x @ Wqkv_g`` for the rank's local KV-head slots (its TP
   heads + the replicated heads; one cuBLAS GEMM);
2. ONE ``fs_decode_attention`` launch appends the new token's K/V of every
   work item into its page (fused K3) and attends every work item: TP
   slots for all requests, replicated slots only for requests routed to
   ``g`` (refexec.py:284-297), merging split items in-kernel (fused K2);
4. ``part = o @ Wo_g`` -- rows of replicated slots for requests routed
   elsewhere are zero, so their contribution is exactly zero
   (refexec.py:290-297);
5. the exchange: ``all_reduce(part)`` over the surviving ranks (NCCL over
   NVLink; the reference's "exact sum in ascending rank order",
   refexec.py:283-298), then ``x += part``.

Weights are derived per (layer, KV head) from a seed, so every rank of every
world size builds bit-identical slices of one global model; the sum over
ranks therefore reproduces the single-GPU result.  ``step`` can be captured
into one CUDA graph (``capture=True``): a whole decode step is then a single
graph launch.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import ModelSpec, ValidationError
from .kvcache import PagedKVCache, RankWork


def head_weights(model: ModelSpec, layer: int, head: int, seed: int, device):
    """Deterministic weights of one KV head's group in one layer:
    wq [hidden, qpk*hd], wk/wv [hidden, hd], wo [qpk*hd, hidden] (bf16)."""
    hd, qpk, hid = model.head_dim, model.q_heads_per_kv_head, model.hidden_dim
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + layer * 4099 + head * 31) & 0x7FFFFFFF)
    s_in = 1.0 / math.sqrt(hid)
    s_out = 0.5 / math.sqrt(model.num_q_heads * hd)
    wq = torch.randn((hid, qpk * hd), generator=g, device=device) * s_in
    wk = torch.randn((hid, hd), generator=g, device=device) * s_in
    wv = torch.randn((hid, hd), generator=g, device=device) * s_in
    wo = torch.randn((qpk * hd, hid), generator=g, device=device) * s_out
    return [w.to(torch.bfloat16) for w in (wq, wk, wv, wo)]


class HybridDecodeRank:
    """One rank's share of the hybrid-attention decode step.

    ``owner``: int32 [L, H] table (``placement.owner_array``), ``routing``:
    request -> GPU, ``group``: torch.distributed process group of the alive
    ranks (None = no exchange, e.g. world 1 or single-GPU emulation).
    """

    def __init__(self, model: ModelSpec, owner, rank: int, routing, batch: int, capacity: int,
                 device=None, seed: int = 0, group=None, page_order: str = "contiguous",
                 config: int = 0):
        if model.head_dim != N.HEAD_DIM:
            raise ValidationError(f"head_dim must be {N.HEAD_DIM} for the CUDA path")
        self.model = model
        self.rank = rank
        self.batch = batch
        self.group = group
        self.device = torch.device(device if device is not None else "cuda")
        self.qpk = model.q_heads_per_kv_head
        self.work = RankWork.build(np.asarray(owner, dtype=np.int32), rank, routing, batch)
        self.cache = PagedKVCache(self.work, capacity, self.qpk, self.device,
                                  page_order=page_order, seed=seed, config=config)
        hd, hid, S = model.head_dim, model.hidden_dim, self.work.n_slots
        self.n_slots = S
        L = model.num_layers
        dev = self.device
        rw = self.cache.set_fused_layout()   # [q slots | k slots | v slots]
        qw = S * self.qpk * hd
        self.wqkv = torch.zeros((L, hid, rw), dtype=torch.bfloat16, device=dev)
        self.wo = torch.zeros((L, qw, hid), dtype=torch.bfloat16, device=dev)
        for layer in range(L):
            for j, h in enumerate(self.work.slot_heads[layer]):
                wq, wk, wv, wo = head_weights(model, layer, h, seed, dev)
                qs = slice(j * self.qpk * hd, (j + 1) * self.qpk * hd)
                self.wqkv[layer, :, qs] = wq
                self.wqkv[layer, :, qw + j * hd:qw + (j + 1) * hd] = wk
                self.wqkv[layer, :, qw + (S + j) * hd:qw + (S + j + 1) * hd] = wv
                self.wo[layer, qs, :] = wo
        self.qkv = torch.empty((batch, rw), dtype=torch.bfloat16, device=dev)
        self.o = torch.zeros((batch * S, self.qpk, hd), dtype=torch.bfloat16, device=dev)
        self.part = torch.empty((batch, hid), dtype=torch.bfloat16, device=dev)
        self.x = torch.zeros((batch, hid), dtype=torch.bfloat16, device=dev)
        self._graph = None

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
        """This rank's pre-exchange contribution of ``layer`` for the
        current ``self.x``: ``o @ Wo_g`` [B, hidden] (into ``self.part``)."""
        B, S, hd = self.batch, self.n_slots, self.model.head_dim
        torch.matmul(self.x, self.wqkv[layer], out=self.qkv)         # cuBLAS
        self.cache.decode_layer_fused(layer, self.qkv, self.o)       # K1 (+K2, +K3)
        torch.matmul(self.o.view(B, S * self.qpk * hd), self.wo[layer], out=self.part)
        return self.part

    def _layers(self) -> None:
        B, S, hd = self.batch, self.n_slots, self.model.head_dim
        x, o2 = self.x, self.o.view(B, S * self.qpk * hd)
        for layer in range(self.model.num_layers):
            if self.group is None:
                torch.matmul(x, self.wqkv[layer], out=self.qkv)      # cuBLAS
                self.cache.decode_layer_fused(layer, self.qkv, self.o)
                x.addmm_(o2, self.wo[layer])                         # x += o Wo
            else:
                self.attention_partial(layer)
                torch.distributed.all_reduce(self.part, group=self.group)
                x.add_(self.part)

    def launches_per_step(self) -> int:
        """Our kernel launches per step: one fused decode launch per layer."""
        return self.model.num_layers

    def capture(self) -> None:
        """Capture one decode step (all layers) into a CUDA graph."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self._layers()  # warm cuBLAS workspaces outside capture
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._layers()
        self._graph = g

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
    ordered all-reduce, refexec.py:283-298) and the residual is applied.
    Returns x after all layers."""
    ranks = sorted(ranks, key=lambda r: r.rank)
    x = x.to(torch.bfloat16)
    for layer in range(ranks[0].model.num_layers):
        total = None
        for r in ranks:
            r.x.copy_(x)
            part = r.attention_partial(layer).float()
            total = part if total is None else total + part
        x = x + total.to(torch.bfloat16)
    return x
