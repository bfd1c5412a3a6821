"""Chunked-prefill attention over the paged KV cache (K8).

The device form of the multi-row ``_head_attention`` (refexec.py:85-103)
for the batches the adaptive chunked-prefill scheduler forms
(``scheduler.build_prefill_batch``, scheduler.py:189-245): one *item* per
(KV-head slot, request chunk) a rank serves -- the chunk's tokens sit at
prompt positions ``start .. start+len-1`` and attend causally, including
themselves, to the request's prefix.  The tile / split plan is made on the
host by the native planner (``fs_plan_prefill_tiles``) and uploaded once per
launch; the kernel streams KV pages with TMA and runs the 64-row GQA tile on
tensor cores (csrc/prefill.cu).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import ValidationError

_TILE_ROWS = 64


def _stream():
    return N.C.c_void_p(torch.cuda.current_stream().cuda_stream)


class PrefillLaunch:
    """Device tables of one ``fs_prefill_attention`` launch.

    ``cache``: the :class:`~.kvcache.PagedKVCache` holding the pages (the
    chunk tokens' K/V must be written before the launch); per item: block-
    table row ``item_seq``, first position ``item_start``, chunk length
    ``item_len``, element offsets ``item_qoff`` / ``item_ooff`` of the
    chunk's first token in q / out (token ``j`` at ``+ j*stride``).
    """

    def __init__(self, cache, item_seq, item_start, item_len, item_qoff, item_ooff,
                 target_units: int = None):
        arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.int32))
                for a in (item_seq, item_start, item_len, item_qoff, item_ooff)]
        n = arrs[0].size
        if any(a.shape != (n,) for a in arrs):
            raise ValidationError("item arrays must be 1-D of equal length")
        if n and (arrs[1].min() < 0 or arrs[2].min() < 0):
            raise ValidationError("item_start / item_len must be nonnegative")
        if n and int((arrs[1] + arrs[2]).max()) > cache.capacity:
            raise ValidationError("chunk exceeds the cache capacity")
        self.cache = cache
        self.qpk = cache.qpk
        tpt = N.lib.fs_prefill_tokens_per_tile(self.qpk)
        if target_units is None:
            target_units = 4 * N.lib.fs_device_sms(cache.dev_index)
        starts, lens = arrs[1], arrs[2]
        max_tiles = max_comb = 1
        for st, ln in zip(starts.tolist(), lens.tolist()):
            last = np.minimum(np.arange(0, ln, tpt) + tpt, ln)
            pages = (st + last + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS
            max_tiles += int(np.sum(pages // 32 + 1))  # splits are >= 32 pages
            max_comb += last.size
        I32 = N.C.c_int32
        out = {k: (I32 * max_tiles)() for k in ("item", "tok0", "p0", "p1", "slot")}
        comb = {k: (I32 * max_comb)() for k in ("item", "tok0", "slot0", "ns")}
        nt, nc, ns = I32(), I32(), I32()
        P = N.C.POINTER(I32)
        cast = (lambda a: a.ctypes.data_as(P))
        N.check(N.lib.fs_plan_prefill_tiles(
            n, cast(starts), cast(lens), self.qpk, int(target_units), max_tiles,
            out["item"], out["tok0"], out["p0"], out["p1"], out["slot"], N.C.byref(nt),
            max_comb, comb["item"], comb["tok0"], comb["slot0"], comb["ns"], N.C.byref(nc),
            N.C.byref(ns)), "fs_plan_prefill_tiles")
        self.n_items, self.n_tiles, self.n_comb, self.n_slots = n, nt.value, nc.value, ns.value
        tiles = np.stack([np.frombuffer(out[k], dtype=np.int32)[:self.n_tiles]
                          for k in ("item", "tok0", "p0", "p1", "slot")]) \
            if self.n_tiles else np.zeros((5, 0), np.int32)
        combs = np.stack([np.frombuffer(comb[k], dtype=np.int32)[:self.n_comb]
                          for k in ("item", "tok0", "slot0", "ns")]) \
            if self.n_comb else np.zeros((4, 0), np.int32)
        self.tiles_host = tiles
        # one H2D copy of every table
        flat = np.concatenate([np.stack(arrs).ravel(), tiles.ravel(), combs.ravel()])
        self._tab = torch.from_numpy(flat).to(cache.device, non_blocking=False)
        self._off = {}
        o = 0
        for name in ("seq", "start", "len", "qoff", "ooff"):
            self._off[name] = o
            o += n
        for name in ("t_item", "t_tok0", "t_p0", "t_p1", "t_slot"):
            self._off[name] = o
            o += self.n_tiles
        for name in ("c_item", "c_tok0", "c_slot0", "c_ns"):
            self._off[name] = o
            o += self.n_comb
        dev = cache.device
        slots = max(1, self.n_slots)
        self.part_o = torch.empty((slots, _TILE_ROWS, N.HEAD_DIM), dtype=torch.float32,
                                  device=dev) if self.n_slots else None
        self.part_lse = torch.empty((slots, _TILE_ROWS), dtype=torch.float32,
                                    device=dev) if self.n_slots else None
        # algorithmic KV bytes: each (query-row tile, key) pair's page read
        # once per token tile (the tile's causal range)
        self.kv_page_reads = int(np.sum(tiles[3] - tiles[2])) if self.n_tiles else 0
        self.flops = 0
        if n:
            # 4*hd FLOP per (query head, visible key): QK^T and PV
            vis = (starts.astype(np.int64) * lens + lens * (lens.astype(np.int64) + 1) // 2)
            self.flops = int(4 * N.HEAD_DIM * self.qpk * vis.sum())

    def _p(self, name):
        return N.C.c_void_p(self._tab.data_ptr() + 4 * self._off[name])

    def __call__(self, q: torch.Tensor, q_stride: int, out: torch.Tensor, o_stride: int,
                 scale: float = None) -> None:
        if self.n_tiles == 0:
            return
        if q.dtype != torch.bfloat16 or out.dtype not in (torch.bfloat16, torch.float32):
            raise ValidationError("q must be bf16 and out bf16 or fp32")
        c = self.cache
        d = N.PrefillDesc()
        d.q, d.out = q.data_ptr(), out.data_ptr()
        d.q_stride, d.o_stride = int(q_stride), int(o_stride)
        d.out_fp32 = 1 if out.dtype == torch.float32 else 0
        d.kv_pool = c.pool.data_ptr()
        d.block_table = c.block_table.data_ptr()
        d.bt_stride = c.pages_per_seq
        d.item_seq, d.item_start, d.item_len = (self._p("seq").value, self._p("start").value,
                                                self._p("len").value)
        d.item_qoff, d.item_ooff = self._p("qoff").value, self._p("ooff").value
        d.tile_item, d.tile_tok0 = self._p("t_item").value, self._p("t_tok0").value
        d.tile_page0, d.tile_page1 = self._p("t_p0").value, self._p("t_p1").value
        d.tile_slot = self._p("t_slot").value
        d.n_tiles = self.n_tiles
        if self.n_comb:
            d.comb_item, d.comb_tok0 = self._p("c_item").value, self._p("c_tok0").value
            d.comb_slot0, d.comb_nsplit = self._p("c_slot0").value, self._p("c_ns").value
            d.part_o, d.part_lse = self.part_o.data_ptr(), self.part_lse.data_ptr()
            d.partial_slots = self.n_slots
        d.n_comb = self.n_comb
        d.q_per_kv = self.qpk
        d.scale = (1.0 / math.sqrt(N.HEAD_DIM)) if scale is None else float(scale)
        N.check(N.lib.fs_prefill_attention(N.C.byref(d), _stream()), "fs_prefill_attention")
