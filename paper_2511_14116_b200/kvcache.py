"""Device-resident paged KV cache and per-rank work tables.

This is where the reference's placement + routing become device tables
(north star item 1).  For one rank ``g`` of a plan:

* local KV-head slots of layer ``l`` = ``g``'s TP heads (ascending) followed
  by the replicated (DP) heads (ascending) -- the residency of
  ``ShardedView.rank_heads`` (refexec.py:143-147);
* one *work item* per (layer, slot, request) the rank serves: every request
  for a TP slot, only requests routed to ``g`` for a DP slot -- exactly the
  (head, rows) pairs ``parallel_forward`` evaluates on rank ``g``
  (refexec.py:284-297);
* one KV *sequence* (a block-table row of 16-token pages) per work item,
  so the bytes resident on ``g`` equal ``memory_footprint``
  (placement.py:206-236) rounded up to whole pages.

Query / output rows are ``request * n_slots + slot`` (each row holds the
``q_per_kv`` query heads of the slot's KV head); the appended K/V rows of a
step are ``request * 2 * n_slots + slot`` (K) in a fused [B, 2*n_slots*128]
projection output, V following K.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .core import SimulationError, ValidationError


@dataclass
class RankWork:
    """Host-side work tables of one rank (numpy, built once per plan)."""

    rank: int
    num_layers: int
    n_slots: int                 # max local heads over layers
    slot_heads: list             # per layer: KV head id of each local slot
    n_tp: list                   # per layer: number of TP slots
    seg_items: np.ndarray        # [L+1] item offsets per layer
    item_req: np.ndarray         # [n_items] request index
    item_slot: np.ndarray        # [n_items] local slot
    item_head: np.ndarray        # [n_items] KV head id

    @property
    def n_items(self) -> int:
        return int(self.seg_items[-1])

    @classmethod
    def build(cls, owner: np.ndarray, rank: int, routing, num_requests: int) -> "RankWork":
        """owner: int32 [L, H] (-1 = replicated); routing: request -> GPU
        (array-like or mapping; only consulted for replicated heads)."""
        owner = np.asarray(owner)
        L, H = owner.shape
        route = np.array([routing[r] for r in range(num_requests)], dtype=np.int64) \
            if num_requests else np.zeros(0, dtype=np.int64)
        mine = np.flatnonzero(route == rank)
        slot_heads, n_tp, reqs, slots, heads, seg = [], [], [], [], [], [0]
        for layer in range(L):
            tp = [int(h) for h in np.flatnonzero(owner[layer] == rank)]
            dp = [int(h) for h in np.flatnonzero(owner[layer] == N.REPLICATED)]
            slot_heads.append(tp + dp)
            n_tp.append(len(tp))
            for j, h in enumerate(tp + dp):
                served = np.arange(num_requests) if j < len(tp) else mine
                reqs.append(served)
                slots.append(np.full(len(served), j))
                heads.append(np.full(len(served), h))
            seg.append(seg[-1] + sum(len(x) for x in reqs[len(reqs) - len(tp + dp):]))
        cat = (lambda xs: np.concatenate(xs).astype(np.int32) if xs else np.zeros(0, np.int32))
        return cls(rank=rank, num_layers=L,
                   n_slots=max([len(s) for s in slot_heads] + [1]),
                   slot_heads=slot_heads, n_tp=n_tp, seg_items=np.array(seg, dtype=np.int32),
                   item_req=cat(reqs), item_slot=cat(slots), item_head=cat(heads))

    def keys(self) -> np.ndarray:
        return item_keys(self)

    def kv_tokens(self, lens) -> int:
        """KV tokens resident on this rank for per-request lengths ``lens``."""
        lens = np.asarray(lens, dtype=np.int64)
        return int(lens[self.item_req].sum()) if self.n_items else 0


def item_keys(work: RankWork) -> np.ndarray:
    """Per item the packed key (layer << 40) | (head << 20) | request."""
    if not work.n_items:
        return np.zeros(0, np.int64)
    layer = np.repeat(np.arange(work.num_layers, dtype=np.int64), np.diff(work.seg_items))
    return (layer << 40) | (work.item_head.astype(np.int64) << 20) | work.item_req.astype(np.int64)


def unpack_keys(keys: np.ndarray) -> np.ndarray:
    """[n, 3] int32 (layer, head, request) of packed item keys."""
    keys = np.asarray(keys, dtype=np.int64)
    return np.stack([keys >> 40, (keys >> 20) & 0xFFFFF, keys & 0xFFFFF], axis=1).astype(np.int32)


def pack_keys(lhr: np.ndarray) -> np.ndarray:
    lhr = np.asarray(lhr, dtype=np.int64).reshape(-1, 3)
    return (lhr[:, 0] << 40) | (lhr[:, 1] << 20) | lhr[:, 2]


def _stream():
    return N.C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _at(t: torch.Tensor, index: int) -> N.C.c_void_p:
    """Pointer to element ``index`` of a 1-D tensor."""
    return N.C.c_void_p(t.data_ptr() + index * t.element_size())


class PagedKVCache:
    """Page pool + block table + work/page tables of one rank on one GPU.

    ``capacity`` tokens of pages are reserved per sequence.  ``page_order``
    "shuffled" scatters the page ids (exercises the indirection);
    "contiguous" lays each sequence out linearly.
    """

    def __init__(self, work: RankWork, capacity: int, q_per_kv: int, device=None,
                 page_order: str = "contiguous", seed: int = 0, config: int = 0,
                 request_capacity=None, reserve_pages: int = 0):
        if not (1 <= q_per_kv <= N.MAX_Q_PER_KV):
            raise ValidationError(f"q_per_kv must be in [1, {N.MAX_Q_PER_KV}]")
        if capacity < 1:
            raise ValidationError("capacity must be >= 1 token")
        if reserve_pages < 0:
            raise ValidationError("reserve_pages must be nonnegative")
        self.qpk = q_per_kv
        self.capacity = capacity
        self.config = config
        self.device = torch.device(device if device is not None else "cuda")
        self.dev_index = self.device.index if self.device.index is not None \
            else torch.cuda.current_device()
        self.pages_per_seq = math.ceil(capacity / N.PAGE_TOKENS)
        self.request_capacity = None if request_capacity is None else \
            np.asarray(request_capacity, dtype=np.int64)
        cap = self.request_capacity
        if cap is not None and cap.size and (cap.max() > capacity or cap.min() < 0):
            raise ValidationError("request capacities must lie in [0, capacity]")
        seq_pages = self._seq_pages(work.item_req)
        used = int(seq_pages.sum())
        # reserve: free pages for the items an on-demand adoption adds
        # (replicated heads of a failed GPU, re-routed requests)
        self.n_pages = max(1, used + reserve_pages)
        ids = np.arange(self.n_pages, dtype=np.int64)
        if page_order == "shuffled":
            ids = np.random.default_rng(seed).permutation(self.n_pages)
        elif page_order != "contiguous":
            raise ValidationError(f"unknown page_order {page_order!r}")
        self.page_order = page_order
        bt = np.zeros((work.n_items, self.pages_per_seq), dtype=np.int64)
        cols = np.arange(self.pages_per_seq)
        mask = cols[None, :] < seq_pages[:, None]
        bt[mask] = ids[:used]
        self.free_pages = list(ids[used:])
        # zero-filled: unwritten rows hold finite values (0), never NaN bit patterns
        self.pool = torch.zeros((self.n_pages, N.PAGE_BYTES), dtype=torch.uint8,
                                device=self.device)
        # FS_DECODE_EARLY_PREFETCH: set by callers whose decode launches always
        # follow a kernel that writes none of the tables / pages (the QKV GEMM
        # in HybridDecodeRank); otherwise (K3 / K4 / restores just before) the
        # launch reads nothing before its PDL wait
        self.early_prefetch = False
        self.fused = None  # (qoff, koff, voff) of the fused-qkv layout
        self._install(work, bt.astype(np.int32))

    def _seq_pages(self, item_req) -> np.ndarray:
        """Pages backed per item: the full row, or the request's capacity."""
        if self.request_capacity is None:
            return np.full(len(item_req), self.pages_per_seq, dtype=np.int64)
        if not len(item_req):
            return np.zeros(0, np.int64)
        return (self.request_capacity[item_req] + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS

    def _install(self, work: RankWork, bt: np.ndarray) -> None:
        """(Re)build every device table of ``work`` over block table ``bt``."""
        dev = self.device
        n_seq = work.n_items
        self.work = work
        self.seq_tokens = self._seq_pages(work.item_req) * N.PAGE_TOKENS
        self.block_table = torch.from_numpy(np.ascontiguousarray(bt, dtype=np.int32)).to(dev)
        self.item_seq = torch.arange(n_seq, dtype=torch.int32, device=dev)
        self.item_len = torch.zeros(n_seq, dtype=torch.int32, device=dev)
        self.item_pos = torch.zeros(n_seq, dtype=torch.int32, device=dev)
        self.item_sem = torch.zeros(n_seq, dtype=torch.int32, device=dev)
        self._req = torch.from_numpy(work.item_req.astype(np.int64)).to(dev)
        self._slot = torch.from_numpy(work.item_slot.astype(np.int64)).to(dev)
        # default ("blocks") layout: the query / output block of item i is
        # row request*n_slots + slot of a [B*n_slots, qpk, 128] tensor
        row = self._req * work.n_slots + self._slot
        self.item_qoff = (row * self.qpk * N.HEAD_DIM).to(torch.int32)
        self.item_ooff = self.item_qoff
        self.seg_items = torch.from_numpy(work.seg_items).to(dev)
        self.page_off = torch.zeros(n_seq + work.num_layers, dtype=torch.int32, device=dev)
        seg = work.seg_items
        self.max_items = int(max(seg[1:] - seg[:-1])) if work.num_layers else 0
        slots = N.lib.fs_decode_partial_slots(self.dev_index, self.max_items, -1)
        if slots < 0:
            raise SimulationError(f"cannot size decode partials: {N.lib.fs_last_error()}")
        if getattr(self, "part_o", None) is None or self.part_o.shape[0] < slots:
            self.part_o = torch.empty((slots, self.qpk, N.HEAD_DIM), dtype=torch.float32,
                                      device=dev)
            self.part_lse = torch.empty((slots, self.qpk), dtype=torch.float32, device=dev)
        self._descs = {}
        if self.fused is not None:
            self.set_fused_layout()

    def adopt(self, work: RankWork):
        """In-place adoption of a new work table (the on-demand shrink
        target, recovery.py:396-427, with re-routed requests): items whose
        (layer, head, request) this rank already serves keep their pages --
        no KV moves; new items get pages from the free reserve; dropped
        items return theirs.  Lengths must be set again afterwards.
        Returns the indices (into the new work) of the new items, whose
        pages the caller restores (K6) or recomputes."""
        old_keys = item_keys(self.work)
        new_keys = item_keys(work)
        old_bt = self.block_table.cpu().numpy()
        old_pages = self._seq_pages(self.work.item_req)
        index = {k: i for i, k in enumerate(old_keys.tolist())}
        kept = np.array([index.get(k, -1) for k in new_keys.tolist()], dtype=np.int64) \
            if len(new_keys) else np.zeros(0, np.int64)
        new_set = set(new_keys.tolist())
        for i, k in enumerate(old_keys.tolist()):
            if k not in new_set:  # dropped: its pages return to the reserve
                self.free_pages.extend(int(x) for x in old_bt[i, :old_pages[i]])
        need = self._seq_pages(work.item_req)
        bt = np.zeros((work.n_items, self.pages_per_seq), dtype=np.int32)
        fresh = np.flatnonzero(kept < 0)
        if int(need[fresh].sum()) > len(self.free_pages):
            raise SimulationError(
                f"KV reserve exhausted: {int(need[fresh].sum())} pages needed, "
                f"{len(self.free_pages)} free (raise reserve_pages)")
        for i in range(work.n_items):
            if kept[i] >= 0:
                bt[i] = old_bt[kept[i]]
            else:
                n = int(need[i])
                bt[i, :n] = self.free_pages[:n]
                del self.free_pages[:n]
        self._install(work, bt)
        return fresh

    def set_fused_layout(self) -> int:
        """Use the fused projection layout: per request one row
        ``[q slots (S*qpk*128) | k slots (S*128) | v slots (S*128)]``.
        Returns the row width in elements."""
        S, hd, qpk = self.work.n_slots, N.HEAD_DIM, self.qpk
        rw = S * (qpk + 2) * hd
        base = self._req * rw
        self.fused = ((base + self._slot * qpk * hd).to(torch.int32),
                      (base + S * qpk * hd + self._slot * hd).to(torch.int32),
                      (base + S * (qpk + 1) * hd + self._slot * hd).to(torch.int32))
        self._descs.clear()
        return rw

    # ------------------------------------------------------------ lengths --
    def set_lengths(self, lens_per_request) -> None:
        """Set every sequence's attended length from per-request lengths
        (host call; re-plans the page tables)."""
        lens = np.asarray(lens_per_request, dtype=np.int32)
        if lens.size and (lens.max() > self.capacity or lens.min() < 0):
            raise ValidationError("lengths must lie in [0, capacity]")
        per_item = lens[self.work.item_req] if self.work.n_items else lens[:0]
        self.item_len.copy_(torch.from_numpy(np.ascontiguousarray(per_item)))
        torch.sub(self.item_len, 1, out=self.item_pos)
        self.plan()

    def advance(self, n: int = 1) -> None:
        """Grow every sequence by ``n`` tokens on the device (no host sync)."""
        self.item_len.add_(n)
        torch.sub(self.item_len, 1, out=self.item_pos)
        self.plan()

    def plan(self) -> None:
        """K4: device page prefix per layer."""
        N.check(N.lib.fs_plan_pages(N.ptr(self.item_len), N.ptr(self.seg_items),
                                    self.work.num_layers, N.ptr(self.page_off), _stream()),
                "fs_plan_pages")

    # -------------------------------------------------------------- writes --
    def write_tokens(self, seq, pos, k, v) -> None:
        """K3 over explicit tokens: k/v [n, 128] bf16 (device), seq/pos int."""
        seq = torch.as_tensor(seq, dtype=torch.int32, device=self.device)
        pos = torch.as_tensor(pos, dtype=torch.int32, device=self.device)
        n = seq.numel()
        src = torch.arange(n, dtype=torch.int32, device=self.device)
        k = k.contiguous()
        v = v.contiguous()
        if k.dtype != torch.bfloat16 or k.shape[-1] != N.HEAD_DIM:
            raise ValidationError("k/v must be bf16 [n, 128]")
        N.check(N.lib.fs_kv_write(N.ptr(self.pool), N.ptr(self.block_table), self.pages_per_seq,
                                  N.ptr(seq), N.ptr(pos), N.ptr(src), n, N.ptr(k), N.ptr(v),
                                  N.HEAD_DIM, _stream()), "fs_kv_write")

    def read_tokens(self, seq, pos):
        seq = torch.as_tensor(seq, dtype=torch.int32, device=self.device)
        pos = torch.as_tensor(pos, dtype=torch.int32, device=self.device)
        n = seq.numel()
        dst = torch.arange(n, dtype=torch.int32, device=self.device)
        k = torch.empty((n, N.HEAD_DIM), dtype=torch.bfloat16, device=self.device)
        v = torch.empty_like(k)
        N.check(N.lib.fs_kv_read(N.ptr(self.pool), N.ptr(self.block_table), self.pages_per_seq,
                                 N.ptr(seq), N.ptr(pos), N.ptr(dst), n, N.ptr(k), N.ptr(v),
                                 N.HEAD_DIM, _stream()), "fs_kv_read")
        return k, v

    # -------------------------------------------------------------- decode --
    def _desc(self, layer, q, out, qkv, scale):
        key = (layer, q.data_ptr(), out.data_ptr(), out.dtype, qkv, scale, self.config,
               self.early_prefetch)
        d = self._descs.get(key)
        if d is not None:
            return d
        a = int(self.work.seg_items[layer])
        n = int(self.work.seg_items[layer + 1]) - a
        d = N.DecodeDesc()
        d.q = q.data_ptr()
        d.kv_pool = self.pool.data_ptr()
        d.block_table = self.block_table.data_ptr()
        d.bt_stride = self.pages_per_seq
        d.item_seq = _at(self.item_seq, a).value
        d.item_len = _at(self.item_len, a).value
        if qkv:
            qoff, koff, voff = self.fused
            d.item_qoff = _at(qoff, a).value
            d.kv_new = q.data_ptr()
            d.item_koff = _at(koff, a).value
            d.item_voff = _at(voff, a).value
        else:
            d.item_qoff = _at(self.item_qoff, a).value
        d.item_ooff = _at(self.item_ooff, a).value
        d.page_off = _at(self.page_off, a + layer).value
        d.item_sem = _at(self.item_sem, a).value
        d.n_items = n
        d.q_per_kv = self.qpk
        d.scale = (1.0 / math.sqrt(N.HEAD_DIM)) if scale is None else float(scale)
        d.out_fp32 = 1 if out.dtype == torch.float32 else 0
        d.out = out.data_ptr()
        d.part_o = self.part_o.data_ptr()
        d.part_lse = self.part_lse.data_ptr()
        d.partial_slots = self.part_o.shape[0]
        d.device = self.dev_index
        d.config = self.config
        d.flags = N.DECODE_EARLY_PREFETCH if self.early_prefetch else 0
        self._descs[key] = d
        return d

    def decode_layer(self, layer: int, q: torch.Tensor, out: torch.Tensor,
                     scale: float = None) -> None:
        """K1 (+ fused combine) for every item of ``layer``.  q / out are
        [B*n_slots, qpk, 128] blocks (out bf16 or fp32); the KV must already
        hold every token (see :meth:`write_tokens`)."""
        if int(self.work.seg_items[layer + 1]) == int(self.work.seg_items[layer]):
            return
        d = self._desc(layer, q, out, False, scale)
        N.check(N.lib.fs_decode_attention(N.C.byref(d), _stream()), "fs_decode_attention")

    def decode_layer_fused(self, layer: int, qkv: torch.Tensor, out: torch.Tensor,
                           scale: float = None) -> None:
        """One decode step of ``layer`` from the fused projection output
        ``qkv`` [B, row] (:meth:`set_fused_layout`): the new token's K/V are
        appended into their pages inside the same launch (fused K3), then
        attention over ``len`` tokens.  ``out`` is [B*n_slots, qpk, 128]."""
        if self.fused is None:
            raise ValidationError("call set_fused_layout() first")
        if int(self.work.seg_items[layer + 1]) == int(self.work.seg_items[layer]):
            return
        d = self._desc(layer, qkv, out, True, scale)
        N.check(N.lib.fs_decode_attention(N.C.byref(d), _stream()), "fs_decode_attention")

    def layer_kv_bytes(self, layer: int) -> int:
        """Algorithmic KV bytes one decode of ``layer`` reads (512 B per
        (head, token); SURVEY 8d / memory_footprint)."""
        a, b = int(self.work.seg_items[layer]), int(self.work.seg_items[layer + 1])
        return int(self.item_len[a:b].sum().item()) * 2 * N.HEAD_DIM * 2
