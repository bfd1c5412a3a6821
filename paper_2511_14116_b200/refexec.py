"""GPU drop-in for the reference's toy executor API (``failsafe.refexec``).

``parallel_forward(view, plan, routing, activations, seq_lens)`` and
``reference_forward(weights, activations, seq_lens)`` keep the reference
signatures and semantics (refexec.py:111-125, 249-308) -- every rank of the
plan is emulated on one GPU in ascending rank order, TP heads attend for
every token, replicated heads only for the rows of requests routed to the
rank, the per-rank partials are summed in rank order, residual, then the FFN
partial of each rank's shards -- but the attention itself runs through the
CUDA hot path: every (head, request) becomes a paged KV sequence written by
K3 (``fs_kv_write``) and every (head, token row) a work item of the
stream-K decode kernel (``fs_decode_attention``) with its own causal length
(the row attends its request's prefix including itself, refexec.py:97).
Head dims below 128 are zero-padded (exact: padding adds 0 to every dot
product); the softmax scale stays 1/sqrt(true head_dim).

Numerics: q/K/V are rounded to bf16 for the kernel and accumulated in fp32;
results match the reference's float64 within the bf16 tolerance, not to
1e-10.  Inputs may be the reference's own ``ToyModelWeights`` /
``ShardedView`` objects (duck-typed) or this module's mirrors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Mapping, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .core import SimulationError, ValidationError
from .placement import PlacementPlan


@dataclass
class ToyLayerWeights:
    """One layer (refexec.py:29-38): per-head QKVO plus a two-matrix FFN."""

    wq: np.ndarray  # (heads, head_dim, hidden)
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray  # (heads, hidden, head_dim)
    w_up: np.ndarray  # (intermediate, hidden)
    w_down: np.ndarray  # (hidden, intermediate)


@dataclass
class ToyModelWeights:
    hidden: int
    num_heads: int
    head_dim: int
    intermediate: int
    layers: list

    @classmethod
    def random(cls, seed: int, num_layers: int = 2, num_heads: int = 4, head_dim: int = 4,
               hidden: int = 16, intermediate: int = 24) -> "ToyModelWeights":
        """Same draw order as the reference (refexec.py:49-66)."""
        rng = np.random.default_rng(seed)
        s = 1.0 / np.sqrt(hidden)
        layers = []
        for _ in range(num_layers):
            draws = [rng.standard_normal(shape) * s for shape in
                     ((num_heads, head_dim, hidden), (num_heads, head_dim, hidden),
                      (num_heads, head_dim, hidden), (num_heads, hidden, head_dim),
                      (intermediate, hidden), (hidden, intermediate))]
            layers.append(ToyLayerWeights(*draws))
        return cls(hidden=hidden, num_heads=num_heads, head_dim=head_dim,
                   intermediate=intermediate, layers=layers)


def _segments(n_tokens: int, seq_lens: Optional[Sequence[int]]):
    if seq_lens is None:
        return [(0, n_tokens)]
    if sum(seq_lens) != n_tokens:
        raise ValidationError("seq_lens must sum to the token count")
    out, s = [], 0
    for length in seq_lens:
        out.append((s, s + length))
        s += length
    return out


def _stream():
    return N.C.c_void_p(torch.cuda.current_stream().cuda_stream)


def paged_attend(q_items: torch.Tensor, k_tok: torch.Tensor, v_tok: torch.Tensor,
                 tok_seq, tok_pos, item_seq, item_len, scale: float) -> torch.Tensor:
    """Attention of ``n`` single-query items over paged sequences.

    k_tok/v_tok: [T, 128] bf16 tokens, token t belongs to sequence
    tok_seq[t] at position tok_pos[t] (written into pages by K3); item i
    attends the first item_len[i] tokens of sequence item_seq[i] with query
    q_items[i] ([n, 128] bf16).  Returns [n, 128] fp32 (K1 + in-kernel merge)."""
    dev = q_items.device
    n = q_items.shape[0]
    tok_seq = np.asarray(tok_seq, dtype=np.int32)
    tok_pos = np.asarray(tok_pos, dtype=np.int32)
    n_seq = int(tok_seq.max()) + 1 if len(tok_seq) else 1
    seq_len = np.zeros(n_seq, dtype=np.int64)
    np.maximum.at(seq_len, tok_seq, tok_pos + 1)
    ppseq = max(1, int(math.ceil(seq_len.max() / N.PAGE_TOKENS)))
    pool = torch.zeros((n_seq * ppseq, N.PAGE_BYTES), dtype=torch.uint8, device=dev)
    bt = torch.arange(n_seq * ppseq, dtype=torch.int32, device=dev).view(n_seq, ppseq)
    ts = torch.from_numpy(tok_seq).to(dev)
    tp = torch.from_numpy(tok_pos).to(dev)
    src = torch.arange(len(tok_seq), dtype=torch.int32, device=dev)
    N.check(N.lib.fs_kv_write(N.ptr(pool), N.ptr(bt), ppseq, N.ptr(ts), N.ptr(tp), N.ptr(src),
                              len(tok_seq), N.ptr(k_tok.contiguous()), N.ptr(v_tok.contiguous()),
                              N.HEAD_DIM, _stream()), "fs_kv_write")
    iseq = torch.as_tensor(np.asarray(item_seq, dtype=np.int32)).to(dev)
    ilen = torch.as_tensor(np.asarray(item_len, dtype=np.int32)).to(dev)
    off = (torch.arange(n, dtype=torch.int32, device=dev) * N.HEAD_DIM)
    seg = torch.tensor([0, n], dtype=torch.int32, device=dev)
    page_off = torch.zeros(n + 1, dtype=torch.int32, device=dev)
    N.check(N.lib.fs_plan_pages(N.ptr(ilen), N.ptr(seg), 1, N.ptr(page_off), _stream()),
            "fs_plan_pages")
    index = dev.index if dev.index is not None else torch.cuda.current_device()
    slots = N.lib.fs_decode_partial_slots(index, n, 0)
    part_o = torch.empty((slots, 1, N.HEAD_DIM), dtype=torch.float32, device=dev)
    part_lse = torch.empty((slots, 1), dtype=torch.float32, device=dev)
    sem = torch.zeros(n, dtype=torch.int32, device=dev)
    out = torch.zeros((n, N.HEAD_DIM), dtype=torch.float32, device=dev)
    q = q_items.contiguous()
    d = N.DecodeDesc()
    d.q, d.kv_pool, d.block_table, d.bt_stride = q.data_ptr(), pool.data_ptr(), bt.data_ptr(), ppseq
    d.item_seq, d.item_len = iseq.data_ptr(), ilen.data_ptr()
    d.item_qoff = d.item_ooff = off.data_ptr()
    d.page_off, d.item_sem, d.n_items, d.q_per_kv = page_off.data_ptr(), sem.data_ptr(), n, 1
    d.scale, d.out_fp32, d.out = float(scale), 1, out.data_ptr()
    d.part_o, d.part_lse, d.partial_slots = part_o.data_ptr(), part_lse.data_ptr(), slots
    d.device, d.config = index, 0
    N.check(N.lib.fs_decode_attention(N.C.byref(d), _stream()), "fs_decode_attention")
    return out


def _rank_attention(lw, heads_rows, x: torch.Tensor, segs, hd: int) -> torch.Tensor:
    """Sum over (head, rows) of causal head attention projected by wo, as
    one batch of kernel work items; rows=None means every row."""
    dev = x.device
    pad = N.HEAD_DIM
    toks_k, toks_v, tok_seq, tok_pos = [], [], [], []
    q_items, item_seq, item_len, item_row, item_head = [], [], [], [], []
    seq_id = 0
    for head, rows in heads_rows:
        wq = torch.from_numpy(np.asarray(lw.wq[head], dtype=np.float32)).to(dev)
        wk = torch.from_numpy(np.asarray(lw.wk[head], dtype=np.float32)).to(dev)
        wv = torch.from_numpy(np.asarray(lw.wv[head], dtype=np.float32)).to(dev)
        q, k, v = x @ wq.T, x @ wk.T, x @ wv.T          # (tokens, hd) fp32
        qp = torch.zeros((x.shape[0], pad), device=dev)
        kp = torch.zeros_like(qp)
        vp = torch.zeros_like(qp)
        qp[:, :hd], kp[:, :hd], vp[:, :hd] = q, k, v
        for s, e in segs:
            want = [t for t in range(s, e) if rows is None or rows[t]]
            if not want:
                continue
            toks_k.append(kp[s:e])
            toks_v.append(vp[s:e])
            tok_seq.extend([seq_id] * (e - s))
            tok_pos.extend(range(e - s))
            for t in want:
                q_items.append(qp[t])
                item_seq.append(seq_id)
                item_len.append(t - s + 1)
                item_row.append(t)
                item_head.append(head)
            seq_id += 1
    out = torch.zeros_like(x)
    if not q_items:
        return out
    o = paged_attend(torch.stack(q_items).to(torch.bfloat16),
                     torch.cat(toks_k).to(torch.bfloat16), torch.cat(toks_v).to(torch.bfloat16),
                     tok_seq, tok_pos, item_seq, item_len, 1.0 / math.sqrt(hd))[:, :hd]
    rows_t = torch.tensor(item_row, device=dev)
    for head in sorted(set(item_head)):
        sel = torch.tensor([i for i, h in enumerate(item_head) if h == head], device=dev)
        wo = torch.from_numpy(np.asarray(lw.wo[head], dtype=np.float32)).to(dev)
        out.index_add_(0, rows_t[sel], o[sel] @ wo.T)
    return out


def _ffn_partial(lw, x: torch.Tensor, cols) -> torch.Tensor:
    dev = x.device
    up = torch.from_numpy(np.asarray(lw.w_up[cols], dtype=np.float32)).to(dev)
    down = torch.from_numpy(np.asarray(lw.w_down[:, cols], dtype=np.float32)).to(dev)
    return torch.nn.functional.silu(x @ up.T) @ down.T


def _residency(view, plan):
    """rank -> layer -> resident heads, and rank -> shards (ShardedView
    semantics, refexec.py:136-148); taken from ``view`` when it carries them."""
    if hasattr(view, "rank_heads") and hasattr(view, "rank_shards"):
        return view.rank_heads, view.rank_shards
    heads = {g: {l: set(a.tp_heads.get(g, ())) | set(a.dp_heads)
                 for l, a in enumerate(plan.per_layer)} for g in plan.alive}
    shards = {g: set(plan.ffn.shards_of(g)) for g in plan.alive}
    return heads, shards


def parallel_forward(view, plan: PlacementPlan, routing: Optional[Mapping[int, int]],
                     activations, seq_lens: Optional[Sequence[int]] = None,
                     device=None) -> np.ndarray:
    """Hybrid-parallel forward on the GPU (refexec.py:249-308 semantics)."""
    weights = getattr(view, "weights", view)
    dev = torch.device(device if device is not None else "cuda")
    x64 = np.asarray(activations, dtype=np.float64)
    if x64.ndim != 2 or x64.shape[1] != weights.hidden:
        raise ValidationError(f"activations must be (tokens, {weights.hidden})")
    if weights.head_dim > N.HEAD_DIM:
        raise ValidationError(f"head_dim {weights.head_dim} > {N.HEAD_DIM}")
    segs = _segments(x64.shape[0], seq_lens)
    has_dp = any(a.dp_heads for a in plan.per_layer)
    if has_dp and routing is None:
        raise ValidationError("routing is required for plans with replicated heads")
    if has_dp:
        for idx in range(len(segs)):
            if routing.get(idx) is None:
                raise ValidationError(f"missing routing entry for request {idx}")
            if routing[idx] not in plan.alive:
                raise ValidationError(f"request {idx} routed to a dead rank")
    rows_by_rank = {}
    for g in plan.alive:
        rows = np.zeros(x64.shape[0], dtype=bool)
        if routing is not None:
            for idx, (s, e) in enumerate(segs):
                if routing.get(idx) == g:
                    rows[s:e] = True
        rows_by_rank[g] = rows
    rank_heads, rank_shards = _residency(view, plan)
    width = weights.intermediate // plan.ffn.num_shards
    x = torch.from_numpy(x64.astype(np.float32)).to(dev)
    for layer, lw in enumerate(weights.layers):
        assign = plan.per_layer[layer]
        attn = torch.zeros_like(x)
        for g in sorted(plan.alive):
            resident = rank_heads[g][layer]
            hr = []
            for head in sorted(assign.tp_heads.get(g, ())):
                if head not in resident:
                    raise SimulationError(f"rank {g} does not hold head {head} (layer {layer})")
                hr.append((head, None))
            if assign.dp_heads and rows_by_rank[g].any():
                for head in sorted(assign.dp_heads):
                    if head not in resident:
                        raise SimulationError(
                            f"rank {g} does not hold replicated head {head} (layer {layer})")
                    hr.append((head, rows_by_rank[g]))
            attn += _rank_attention(lw, hr, x, segs, weights.head_dim)
        x = x + attn
        ffn = torch.zeros_like(x)
        for g in sorted(plan.alive):
            needed = set(plan.ffn.shards_of(g)) - set(rank_shards[g])
            if needed:
                raise SimulationError(f"rank {g} does not hold FFN shards {sorted(needed)}")
            cols = [c for s in sorted(plan.ffn.shards_of(g))
                    for c in range(s * width, (s + 1) * width)]
            if cols:
                ffn += _ffn_partial(lw, x, np.array(cols))
        x = x + ffn
    torch.cuda.synchronize(dev)
    return x.double().cpu().numpy()


def reference_forward(weights, activations, seq_lens: Optional[Sequence[int]] = None,
                      device=None) -> np.ndarray:
    """Single-device forward (refexec.py:111-125) on the GPU path: one rank
    owning every head and every shard."""
    from .placement import HeadAssignment, ShardAssignment
    L, H = len(weights.layers), weights.num_heads
    per_layer = tuple(HeadAssignment(layer=l, tp_heads={0: frozenset(range(H))},
                                     dp_heads=frozenset()) for l in range(L))
    plan = PlacementPlan(mode="single", world_size=1, alive=(0,), per_layer=per_layer,
                         ffn=ShardAssignment(num_shards=1, owner={0: 0}))
    return parallel_forward(weights, plan, None, activations, seq_lens, device)
