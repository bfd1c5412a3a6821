"""Chunked-prefill attention over the paged KV cache (K8).

The device form of the multi-row ``_head_attention`` (refexec.py:85-103)
for the batches the adaptive chunked-prefill scheduler forms
(``scheduler.build_prefill_batch``, scheduler.py:189-245): one *item* per
(KV-head slot, request chunk) a rank serves -- the chunk's tokens sit at
prompt positions ``start .. start+len-1`` and attend causally, including
themselves, to the request's prefix.  The tile / split plan is made on the
host by the native planner (``fs_plan_prefill_tiles``); the kernel streams
KV pages with TMA and runs the 64-row GQA tile on tensor cores
(csrc/prefill.cu).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import ValidationError

# kernel variants: 0 = tcgen05 (TMEM accumulators, two 128-row halves per
# tile, 64-key blocks), 1 = mma.sync (64-row tiles), 2 = tcgen05 with one
# 128-row half, 3 = tcgen05, two halves, 128-key blocks
VARIANT_ROWS = {0: 256, 1: 64, 2: 128, 3: 256}
DEFAULT_VARIANT = 3


def default_target_units(device_index: int, variant: int = DEFAULT_VARIANT) -> int:
    """CTAs that run at once, the planner's parallel slots: one ~225-KB
    tcgen05 CTA per SM, 4 per SM for the mma.sync variant."""
    return (4 if variant == 1 else 1) * N.lib.fs_device_sms(device_index)


def _stream():
    return N.C.c_void_p(torch.cuda.current_stream().cuda_stream)


class PrefillTilePlan:
    """Host tile / split plan of one launch: depends only on the items'
    (start, length) lists, so layers with the same item structure share it."""

    def __init__(self, starts, lens, q_per_kv: int, target_units: int,
                 variant: int = DEFAULT_VARIANT):
        starts = np.ascontiguousarray(np.asarray(starts, dtype=np.int32))
        lens = np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
        n = starts.size
        tpt = N.lib.fs_prefill_tokens_per_tile(q_per_kv, variant)
        if tpt < 0:
            raise ValidationError(f"q_per_kv must be in [1, {N.MAX_Q_PER_KV}] and variant in "
                                  f"{sorted(VARIANT_ROWS)}")
        self.variant, self.rows = variant, VARIANT_ROWS[variant]
        # capacity bounds: one tile per token tile plus one per 32 pages of
        # its causal range (splits are >= 32 pages)
        n_tok = (lens.astype(np.int64) + tpt - 1) // tpt
        max_comb = int(n_tok.sum()) + 1
        max_tiles = max_comb + int(np.sum(n_tok * ((starts.astype(np.int64) + lens) //
                                                   (32 * N.PAGE_TOKENS) + 1)))
        I32 = N.C.c_int32
        out = {k: (I32 * max_tiles)() for k in ("item", "tok0", "p0", "p1", "slot")}
        comb = {k: (I32 * max_comb)() for k in ("item", "tok0", "slot0", "ns")}
        nt, nc, ns = I32(), I32(), I32()
        P = N.C.POINTER(I32)
        cast = (lambda a: a.ctypes.data_as(P))
        N.check(N.lib.fs_plan_prefill_tiles(
            n, cast(starts), cast(lens), q_per_kv, variant, int(target_units), max_tiles,
            out["item"], out["tok0"], out["p0"], out["p1"], out["slot"], N.C.byref(nt),
            max_comb, comb["item"], comb["tok0"], comb["slot0"], comb["ns"], N.C.byref(nc),
            N.C.byref(ns)), "fs_plan_prefill_tiles")
        self.n_tiles, self.n_comb, self.n_slots = nt.value, nc.value, ns.value
        self.tiles = np.stack([np.frombuffer(out[k], dtype=np.int32)[:self.n_tiles]
                               for k in ("item", "tok0", "p0", "p1", "slot")])
        self.combs = np.stack([np.frombuffer(comb[k], dtype=np.int32)[:self.n_comb]
                               for k in ("item", "tok0", "slot0", "ns")])
        # algorithmic work: KV pages the tiles stream (each token tile reads
        # its causal range once) and 4*hd FLOP per (query head, visible key)
        self.kv_page_reads = int(np.sum(self.tiles[3] - self.tiles[2]))
        vis = starts.astype(np.int64) * lens + lens.astype(np.int64) * (lens + 1) // 2
        self.flops = int(4 * N.HEAD_DIM * q_per_kv * vis.sum())


class PrefillLaunch:
    """Tables of one ``fs_prefill_attention`` launch.

    ``cache``: the :class:`~.kvcache.PagedKVCache` holding the pages (the
    chunk tokens' K/V must be written before the launch); per item: block-
    table row ``item_seq``, first position ``item_start``, chunk length
    ``item_len``, element offsets ``item_qoff`` / ``item_ooff`` of the
    chunk's first token in q / out (token ``j`` at ``+ j*stride``).

    By default the tables are uploaded at once; with ``upload=False`` the
    caller concatenates :attr:`host_table` of several launches, uploads them
    in one copy and calls :meth:`bind` (what the serving iteration does).
    """

    def __init__(self, cache, item_seq, item_start, item_len, item_qoff, item_ooff,
                 target_units: int = None, tile_plan: PrefillTilePlan = None,
                 upload: bool = True, variant: int = DEFAULT_VARIANT):
        arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.int32))
                for a in (item_seq, item_start, item_len, item_qoff, item_ooff)]
        n = arrs[0].size
        if any(a.shape != (n,) for a in arrs):
            raise ValidationError("item arrays must be 1-D of equal length")
        if n and (arrs[1].min() < 0 or arrs[2].min() < 0):
            raise ValidationError("item_start / item_len must be nonnegative")
        if n and int((arrs[1].astype(np.int64) + arrs[2]).max()) > cache.capacity:
            raise ValidationError("chunk exceeds the cache capacity")
        self.cache = cache
        self.qpk = cache.qpk
        if tile_plan is None:
            if target_units is None:
                target_units = default_target_units(cache.dev_index, variant)
            tile_plan = PrefillTilePlan(arrs[1], arrs[2], self.qpk, target_units, variant)
        tp = tile_plan
        self.plan = tp
        self.n_items, self.n_tiles, self.n_comb, self.n_slots = n, tp.n_tiles, tp.n_comb, \
            tp.n_slots
        self.kv_page_reads, self.flops = tp.kv_page_reads, tp.flops
        self.tiles_host = tp.tiles
        self.host_table = np.concatenate([np.stack(arrs).ravel(), tp.tiles.ravel(),
                                          tp.combs.ravel()])
        self._off = {}
        o = 0
        for name, size in (("seq", n), ("start", n), ("len", n), ("qoff", n), ("ooff", n),
                           ("t_item", tp.n_tiles), ("t_tok0", tp.n_tiles), ("t_p0", tp.n_tiles),
                           ("t_p1", tp.n_tiles), ("t_slot", tp.n_tiles), ("c_item", tp.n_comb),
                           ("c_tok0", tp.n_comb), ("c_slot0", tp.n_comb), ("c_ns", tp.n_comb)):
            self._off[name] = o
            o += size
        self._tab = None
        self._base = 0
        self.part_o = self.part_lse = None
        if upload:
            tab = torch.from_numpy(self.host_table).to(cache.device)
            po = pl = None
            if self.n_slots:
                po = torch.empty((self.n_slots, tp.rows, N.HEAD_DIM), dtype=torch.float32,
                                 device=cache.device)
                pl = torch.empty((self.n_slots, tp.rows), dtype=torch.float32,
                                 device=cache.device)
            self.bind(tab, 0, po, pl)

    def bind(self, table: torch.Tensor, base: int, part_o=None, part_lse=None) -> None:
        """Use ``table[base : base + len(host_table)]`` (int32, on the device)
        and the given partial buffers (>= n_slots slots of the variant's rows)."""
        if self.n_slots and (part_o is None or
                             part_o.numel() < self.n_slots * self.plan.rows * N.HEAD_DIM):
            raise ValidationError("split tiles need partial buffers of n_slots slots")
        self._tab, self._base = table, base
        self.part_o, self.part_lse = part_o, part_lse

    def _p(self, name):
        return self._tab.data_ptr() + 4 * (self._base + self._off[name])

    def __call__(self, q: torch.Tensor, q_stride: int, out: torch.Tensor, o_stride: int,
                 scale: float = None) -> None:
        if self.n_tiles == 0:
            return
        if q.dtype != torch.bfloat16 or out.dtype not in (torch.bfloat16, torch.float32):
            raise ValidationError("q must be bf16 and out bf16 or fp32")
        if self._tab is None:
            raise ValidationError("tables not bound (upload=False needs bind())")
        c = self.cache
        d = N.PrefillDesc()
        d.q, d.out = q.data_ptr(), out.data_ptr()
        d.q_stride, d.o_stride = int(q_stride), int(o_stride)
        d.out_fp32 = 1 if out.dtype == torch.float32 else 0
        d.kv_pool = c.pool.data_ptr()
        d.block_table = c.block_table.data_ptr()
        d.bt_stride = c.pages_per_seq
        d.item_seq, d.item_start, d.item_len = self._p("seq"), self._p("start"), self._p("len")
        d.item_qoff, d.item_ooff = self._p("qoff"), self._p("ooff")
        d.tile_item, d.tile_tok0 = self._p("t_item"), self._p("t_tok0")
        d.tile_page0, d.tile_page1 = self._p("t_p0"), self._p("t_p1")
        d.tile_slot = self._p("t_slot")
        d.n_tiles = self.n_tiles
        if self.n_comb:
            d.comb_item, d.comb_tok0 = self._p("c_item"), self._p("c_tok0")
            d.comb_slot0, d.comb_nsplit = self._p("c_slot0"), self._p("c_ns")
            d.part_o, d.part_lse = self.part_o.data_ptr(), self.part_lse.data_ptr()
            d.partial_slots = self.part_o.numel() // (self.plan.rows * N.HEAD_DIM)
        d.n_comb = self.n_comb
        d.q_per_kv = self.qpk
        d.variant = self.plan.variant
        d.scale = (1.0 / math.sqrt(N.HEAD_DIM)) if scale is None else float(scale)
        N.check(N.lib.fs_prefill_attention(N.C.byref(d), _stream()), "fs_prefill_attention")
