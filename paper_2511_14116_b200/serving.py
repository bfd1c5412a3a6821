"""The mixed prefill/decode serving iteration of one rank (BASELINE config 5).

One iteration of the reference's serving loop (``Simulation._start_iteration``,
simulation.py:404-443) combines an Alg. 1 prefill batch
(``scheduler.build_prefill_batch``, scheduler.py:189-245: ``(request, chunk
start, chunk length)`` entries under the token budget) with one decode token
per resident request whose prefill finished.  This module executes that
iteration for real on a rank of the hybrid-attention layout -- the same
per-rank decomposition as ``parallel_forward`` (refexec.py:249-308): TP heads
for every token, replicated (DP) heads only for tokens of requests routed to
the rank, FFN shards the rank owns, partials summed over the ranks.

Per layer, for the T tokens of the iteration (prefill chunk tokens first,
then the decode tokens):

1. ``[q|k|v] = x @ Wqkv_g`` for the rank's local KV-head slots (cuBLAS);
2. K3 writes every served token's K/V into its pages (one launch);
3. K8 ``fs_prefill_attention`` over the prefill items (one launch) and K1
   ``fs_decode_attention`` over the decode items (one launch);
4. ``o @ Wo_g`` (+ NCCL all-reduce over the alive ranks), residual;
5. the TP MLP partial over the rank's FFN shards (+ all-reduce), residual.

The host builds a :class:`StepPlan` per iteration (work tables of every
layer, uploaded in one copy; K8 tile plans from the native planner); the
device work is then launch-only.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .core import ValidationError
from .hybrid import HybridDecodeRank
from .prefill import PrefillLaunch, PrefillTilePlan, default_target_units


@dataclass
class StepBatch:
    """One serving iteration: Alg. 1 prefill entries ``(request, start,
    length)`` and decode tokens ``(request, position)`` -- the new token at
    ``position`` attends positions ``0..position`` (refexec.py:97)."""

    prefill: list = field(default_factory=list)
    decode: list = field(default_factory=list)

    @property
    def num_tokens(self) -> int:
        return sum(n for _, _, n in self.prefill) + len(self.decode)


class StepPlan:
    """Device work tables of one iteration on one rank (all layers), built
    with vectorised numpy and uploaded in ONE host->device copy; the K8 tile
    plans are shared by the layers with the same item structure."""

    def __init__(self, eng: "HybridServingRank", batch: StepBatch):
        self.batch = batch
        T = batch.num_tokens
        if T > eng.max_tokens:
            raise ValidationError(f"iteration has {T} tokens > max_tokens {eng.max_tokens}")
        cap = eng.request_capacity
        E = np.array(batch.prefill, dtype=np.int64).reshape(-1, 3)
        D = np.array(batch.decode, dtype=np.int64).reshape(-1, 2)
        e_req, e_st, e_len = E[:, 0], E[:, 1], E[:, 2]
        d_req, d_pos = D[:, 0], D[:, 1]
        if E.size and (e_len.min() < 1 or e_st.min() < 0 or np.any(e_st + e_len > cap[e_req])):
            raise ValidationError("a prefill chunk lies outside its request's capacity")
        if D.size and (d_pos.min() < 0 or np.any(d_pos + 1 > cap[d_req])):
            raise ValidationError("a decode token lies outside its request's capacity")
        self.T = T
        L, qpk, hd = eng.model.num_layers, eng.qpk, eng.model.head_dim
        rw, ow = eng.row_width, eng.n_slots * qpk * hd
        rpt = rw // hd  # 128-element rows per token row of qkv
        Tp = int(e_len.sum())
        e_row = np.concatenate([[0], np.cumsum(e_len)[:-1]]).astype(np.int64) if E.size \
            else np.zeros(0, np.int64)
        d_row = Tp + np.arange(D.shape[0], dtype=np.int64)
        # every (layer, slot, entry) at once: item index -1 = replicated
        # head whose request is routed elsewhere; np.nonzero keeps the
        # layer-major, slot, entry order of the per-layer tables
        IDX = eng.item_index_all                             # [L, S, requests]
        z = np.zeros(0, np.int64)
        if E.size:
            itE = IDX[:, :, e_req]
            l_p, j_p, e_p = np.nonzero(itE >= 0)
            p_seq, p_st, p_ln, p_row = itE[l_p, j_p, e_p], e_st[e_p], e_len[e_p], e_row[e_p]
            p_qoff, p_ooff = p_row * rw + j_p * qpk * hd, p_row * ow + j_p * qpk * hd
            p_src = p_row * rpt + j_p                        # K/V row of the run's first token
        else:
            l_p = p_seq = p_st = p_ln = p_qoff = p_ooff = p_src = z
        if D.size:
            itD = IDX[:, :, d_req]
            l_d, j_d, k_d = np.nonzero(itD >= 0)
            dd_seq, dd_len = itD[l_d, j_d, k_d], d_pos[k_d] + 1
            dd_qoff, dd_ooff = d_row[k_d] * rw + j_d * qpk * hd, d_row[k_d] * ow + j_d * qpk * hd
            td_pos, td_src = d_pos[k_d], d_row[k_d] * rpt + j_d
        else:
            l_d = dd_seq = dd_len = dd_qoff = dd_ooff = td_pos = td_src = z
        # K3 runs (consecutive tokens of one entry and head slot) per layer:
        # its prefill runs, then its decode tokens (runs of 1); the device
        # expands them (fs_kv_write_runs), the host never lists tokens
        lay = np.arange(L + 1)
        p_cut = np.searchsorted(l_p, lay)                    # prefill runs per layer
        d_cut = np.searchsorted(l_d, lay)
        n_pr, n_dr = np.diff(p_cut), np.diff(d_cut)
        run_cut = np.concatenate([[0], np.cumsum(n_pr + n_dr)])
        n_run, n_dec = int(run_cut[-1]), int(d_cut[-1])
        runs = np.empty((4, n_run), dtype=np.int64)          # seq, pos, src, len
        pos_p = run_cut[l_p] + (np.arange(l_p.size) - p_cut[l_p])
        pos_d = run_cut[l_d] + n_pr[l_d] + (np.arange(l_d.size) - d_cut[l_d])
        runs[:, pos_p] = np.stack([p_seq, p_st, p_src, p_ln])
        runs[:, pos_d] = np.stack([dd_seq, td_pos, td_src, np.ones_like(dd_seq)])
        run_off = np.concatenate([[0], np.cumsum(runs[3])])
        kv_seg = [int(x) for x in run_cut]
        self.kv_tokens = [int(run_off[run_cut[l + 1]] - run_off[run_cut[l]]) for l in range(L)]
        self.src_step = rpt
        dec_seg = [int(x) for x in d_cut]
        self.prefill = []
        tile_plans = {}
        target = default_target_units(eng.cache.dev_index)
        for layer in range(L):
            a_, b_ = int(p_cut[layer]), int(p_cut[layer + 1])
            launch = None
            if b_ > a_ and int(p_ln[a_:b_].sum()):
                st_, ln_ = p_st[a_:b_], p_ln[a_:b_]
                key = (st_.tobytes(), ln_.tobytes())
                tp = tile_plans.get(key)
                if tp is None:
                    tp = tile_plans[key] = PrefillTilePlan(st_, ln_, qpk, target)
                launch = PrefillLaunch(eng.cache, p_seq[a_:b_], st_, ln_, p_qoff[a_:b_],
                                       p_ooff[a_:b_], tile_plan=tp, upload=False)
            self.prefill.append(launch)
        dec = {"seq": [dd_seq], "len": [dd_len], "qoff": [dd_qoff], "ooff": [dd_ooff]}
        cat = (lambda xs: np.concatenate(xs).astype(np.int32) if xs else np.zeros(0, np.int32))
        self.kv_seg = kv_seg
        self.dec_seg = np.array(dec_seg, dtype=np.int32)
        d_len = cat(dec["len"])
        parts = [runs[0].astype(np.int32), runs[1].astype(np.int32), runs[2].astype(np.int32),
                 run_off.astype(np.int32), cat(dec["seq"]), d_len,
                 cat(dec["qoff"]), cat(dec["ooff"]), self.dec_seg]
        pf_base = sum(x.size for x in parts)
        for lp in self.prefill:
            if lp is not None:
                parts.append(lp.host_table)
        dev = eng.device
        self._tab = torch.from_numpy(np.concatenate(parts)).to(dev)
        o = 0
        self._off = {}
        for name, size in (("run_seq", n_run), ("run_pos", n_run), ("run_src", n_run),
                           ("run_off", n_run + 1), ("d_seq", n_dec), ("d_len", n_dec), ("d_qoff", n_dec),
                           ("d_ooff", n_dec), ("d_seg", L + 1)):
            self._off[name] = o
            o += size
        slots = max([lp.n_slots for lp in self.prefill if lp is not None] + [0])
        rows = max([lp.plan.rows for lp in self.prefill if lp is not None] + [64])
        self.pf_part_o = torch.empty((max(1, slots), rows, hd), dtype=torch.float32, device=dev)
        self.pf_part_lse = torch.empty((max(1, slots), rows), dtype=torch.float32, device=dev)
        o = pf_base
        for lp in self.prefill:
            if lp is not None:
                lp.bind(self._tab, o, self.pf_part_o, self.pf_part_lse)
                o += lp.host_table.size
        self.n_dec = n_dec
        self.dec_sem = torch.zeros(max(1, n_dec), dtype=torch.int32, device=dev)
        self.page_off = torch.zeros(n_dec + L, dtype=torch.int32, device=dev)
        if n_dec:
            N.check(N.lib.fs_plan_pages(self.ptr("d_len"), self.ptr("d_seg"), L,
                                        N.ptr(self.page_off), _stream()), "fs_plan_pages")
        self._descs = [self._decode_desc(eng, layer) for layer in range(L)]
        # algorithmic KV bytes of the iteration on this rank (512 B per
        # (head, token) read: decode items read len, prefill tiles their
        # causal page range)
        self.kv_read_bytes = 512 * int(d_len.astype(np.int64).sum()) + sum(
            (p.kv_page_reads * N.PAGE_BYTES) for p in self.prefill if p is not None)
        self.attn_flops = sum(p.flops for p in self.prefill if p is not None)

    def ptr(self, name, index=0):
        return N.C.c_void_p(self._tab.data_ptr() + 4 * (self._off[name] + index))

    def _decode_desc(self, eng, layer):
        a, b = int(self.dec_seg[layer]), int(self.dec_seg[layer + 1])
        if a == b:
            return None
        d = N.DecodeDesc()
        c = eng.cache
        d.q = eng.qkv_s.data_ptr()
        d.kv_pool = c.pool.data_ptr()
        d.block_table = c.block_table.data_ptr()
        d.bt_stride = c.pages_per_seq
        d.item_seq = self.ptr("d_seq", a).value
        d.item_len = self.ptr("d_len", a).value
        d.item_qoff = self.ptr("d_qoff", a).value
        d.item_ooff = self.ptr("d_ooff", a).value
        d.page_off = self.page_off.data_ptr() + 4 * (a + layer)
        d.kv_new = None
        d.item_sem = self.dec_sem.data_ptr() + 4 * a
        d.n_items = b - a
        d.q_per_kv = eng.qpk
        d.scale = 1.0 / math.sqrt(eng.model.head_dim)
        d.out_fp32 = 0
        d.out = eng.o_s.data_ptr()
        d.part_o = eng.part_o.data_ptr()
        d.part_lse = eng.part_lse.data_ptr()
        d.partial_slots = eng.part_o.shape[0]
        d.device = c.dev_index
        d.config = c.config
        return d


def _stream():
    return N.C.c_void_p(torch.cuda.current_stream().cuda_stream)


class HybridServingRank(HybridDecodeRank):
    """One rank of the mixed prefill/decode iteration.

    ``routing``: request -> GPU for every request of the serving window
    (drives which requests' replicated heads live here); ``request_capacity``:
    per-request KV token capacity (final context, ``Request.final_context_
    tokens``, core.py:155-156) -- only those pages are backed; ``max_tokens``:
    largest iteration (the token budget plus the decode batch).
    """

    def __init__(self, model, owner, rank: int, routing, request_capacity, max_tokens: int,
                 device=None, seed: int = 0, group=None, mlp: bool = True, shard_owner=None,
                 config: int = 0, page_order: str = "contiguous", exchange: str = "nccl",
                 reserve_pages: int = 0):
        cap = np.asarray(request_capacity, dtype=np.int64)
        if cap.ndim != 1 or cap.size == 0 or cap.min() < 1:
            raise ValidationError("request_capacity must list >= 1 token per request")
        super().__init__(model, owner, rank, routing, int(cap.size), int(cap.max()),
                         device=device, seed=seed, group=group, page_order=page_order,
                         config=config, mlp=mlp, shard_owner=shard_owner,
                         request_capacity=cap, exchange=exchange,
                         exchange_elems=int(max_tokens) * model.hidden_dim,
                         reserve_pages=reserve_pages,
                         gemm="cublas")  # iterations of ~2k tokens: compute-bound library GEMMs
        self.request_capacity = cap
        self.max_tokens = int(max_tokens)
        self._derive()

    def _derive(self) -> None:
        """Buffers and tables that follow the work / slot layout (rebuilt
        after an in-place adoption)."""
        model = self.model
        cap = self.request_capacity
        S, hd, qpk, hid = self.n_slots, model.head_dim, self.qpk, model.hidden_dim
        self.row_width = S * (qpk + 2) * hd
        dev = self.device
        T = self.max_tokens
        self.x_s = torch.zeros((T, hid), dtype=torch.bfloat16, device=dev)
        self.qkv_s = torch.empty((T, self.row_width), dtype=torch.bfloat16, device=dev)
        self.o_s = torch.zeros((T, S * qpk * hd), dtype=torch.bfloat16, device=dev)
        self.part_s = torch.empty((T, hid), dtype=torch.bfloat16, device=dev)
        if self.mlp and len(self.ffn_cols):
            C = len(self.ffn_cols)
            self.h_s = torch.empty((T, 2 * C), dtype=torch.bfloat16, device=dev)
            self.act_s = torch.empty((T, C), dtype=torch.bfloat16, device=dev)
        # decode partials: enough slots for every decode item of one layer
        w = self.work
        per_layer = max(int(w.seg_items[l + 1] - w.seg_items[l]) for l in range(model.num_layers))
        slots = N.lib.fs_decode_partial_slots(self.cache.dev_index, per_layer, -1)
        self.part_o = torch.empty((slots, qpk, hd), dtype=torch.float32, device=dev)
        self.part_lse = torch.empty((slots, qpk), dtype=torch.float32, device=dev)
        # (layer, slot, request) -> work item (= block-table row), -1 if the
        # replicated head's request is routed elsewhere
        self.item_index = []
        for layer in range(model.num_layers):
            idx = np.full((S, int(cap.size)), -1, dtype=np.int64)
            a, b = int(w.seg_items[layer]), int(w.seg_items[layer + 1])
            idx[w.item_slot[a:b], w.item_req[a:b]] = np.arange(a, b)
            self.item_index.append(idx)
        self.item_index_all = np.stack(self.item_index)  # [L, S, requests]
        # head slots a layer's kernels do not fill for every request (the
        # replicated heads: only routed requests): their o columns are zeroed
        # per iteration, the fully served (TP) slots are not
        self.partial_slots = [np.nonzero((self.item_index_all[l] < 0).any(axis=1))[0].tolist()
                              for l in range(model.num_layers)]

    def adopt(self, owner, routing, shard_owner, pieces) -> np.ndarray:
        """In-place adoption (HybridDecodeRank.adopt) + the serving tables."""
        fresh = super().adopt(owner, routing, shard_owner, pieces)
        self._derive()
        return fresh

    def plan(self, batch: StepBatch) -> StepPlan:
        return StepPlan(self, batch)

    # ------------------------------------------------------------ pieces --
    def _attention(self, layer: int, plan: StepPlan) -> None:
        T = plan.T
        x, qkv, o = self.x_s[:T], self.qkv_s[:T], self.o_s[:T]
        torch.matmul(x, self.wqkv[layer], out=qkv)                       # cuBLAS
        a, b = plan.kv_seg[layer], plan.kv_seg[layer + 1]
        if b > a:                                                        # K3
            hd = self.model.head_dim
            qw = self.n_slots * self.qpk * hd
            N.check(N.lib.fs_kv_write_runs(
                N.ptr(self.cache.pool), N.ptr(self.cache.block_table), self.cache.pages_per_seq,
                plan.ptr("run_seq", a), plan.ptr("run_pos", a), plan.ptr("run_src", a),
                plan.ptr("run_off", a), b - a, plan.kv_tokens[layer], plan.src_step,
                N.C.c_void_p(qkv.data_ptr() + 2 * qw),
                N.C.c_void_p(qkv.data_ptr() + 2 * (qw + self.n_slots * hd)), hd, _stream()),
                "fs_kv_write_runs")
        w = self.qpk * self.model.head_dim
        for j in self.partial_slots[layer]:  # replicated slots: rows routed elsewhere stay 0
            o[:, j * w:(j + 1) * w].zero_()
        pf = plan.prefill[layer]
        if pf is not None:                                               # K8
            pf(qkv, self.row_width, o, o.shape[1])
        d = plan._descs[layer]
        if d is not None:                                                # K1
            N.check(N.lib.fs_decode_attention(N.C.byref(d), _stream()), "fs_decode_attention")

    def serve_attention_partial(self, layer: int, plan: StepPlan) -> torch.Tensor:
        """This rank's pre-exchange attention contribution ``o @ Wo_g``."""
        self._attention(layer, plan)
        T = plan.T
        torch.matmul(self.o_s[:T], self.wo[layer], out=self.part_s[:T])
        return self.part_s[:T]

    def serve_mlp_partial(self, layer: int, plan: StepPlan) -> torch.Tensor:
        T = plan.T
        if not len(self.ffn_cols):
            return self.part_s[:T].zero_()
        C = len(self.ffn_cols)
        torch.matmul(self.x_s[:T], self.w_gu[layer], out=self.h_s[:T])
        N.check(N.lib.fs_swiglu(N.ptr(self.h_s), T, C, 2 * C, N.ptr(self.act_s), C, _stream()),
                "fs_swiglu")
        torch.matmul(self.act_s[:T], self.w_d[layer], out=self.part_s[:T])
        return self.part_s[:T]

    def serve(self, plan: StepPlan, x: torch.Tensor = None) -> torch.Tensor:
        """Run one iteration: ``x`` [T, hidden] (device or pinned host; None
        = the resident ``x_s``) -> the updated residual stream [T, hidden]."""
        T = plan.T
        xs = self.x_s[:T]
        if x is not None:
            xs.copy_(x, non_blocking=True)
        if self.xchg is not None:
            return self._serve_fused(plan, xs)
        if self.group is None:
            # no exchange: the residual add rides on the projection GEMMs
            # (cuBLAS beta = 1) instead of a separate elementwise pass
            has_ffn = self.mlp and len(self.ffn_cols)
            C = len(self.ffn_cols)
            for layer in range(self.model.num_layers):
                self._attention(layer, plan)
                xs.addmm_(self.o_s[:T], self.wo[layer])
                if has_ffn:
                    torch.matmul(xs, self.w_gu[layer], out=self.h_s[:T])
                    N.check(N.lib.fs_swiglu(N.ptr(self.h_s), T, C, 2 * C, N.ptr(self.act_s), C,
                                            _stream()), "fs_swiglu")
                    xs.addmm_(self.act_s[:T], self.w_d[layer])
            return xs
        for layer in range(self.model.num_layers):
            part = self.serve_attention_partial(layer, plan)
            if self.group is not None:
                torch.distributed.all_reduce(part, group=self.group)
            xs.add_(part)
            if self.mlp:
                part = self.serve_mlp_partial(layer, plan)
                if self.group is not None:
                    torch.distributed.all_reduce(part, group=self.group)
                xs.add_(part)
        return xs

    def _serve_fused(self, plan: StepPlan, xs: torch.Tensor) -> torch.Tensor:
        """serve() with the fused exchange: the O / down projections write
        into the IPC-shared buffers, fs_ar_residual adds the ordered sum."""
        T = plan.T
        for layer in range(self.model.num_layers):
            ia, im = (0, 1) if self.mlp else (layer & 1, None)
            self._attention(layer, plan)
            torch.matmul(self.o_s[:T], self.wo[layer], out=self.xchg.partial(ia, xs.shape))
            self.xchg.reduce_residual(ia, xs)
            if self.mlp:
                part = self.xchg.partial(im, xs.shape)
                if len(self.ffn_cols):
                    C = len(self.ffn_cols)
                    torch.matmul(xs, self.w_gu[layer], out=self.h_s[:T])
                    N.check(N.lib.fs_swiglu(N.ptr(self.h_s), T, C, 2 * C, N.ptr(self.act_s), C,
                                            _stream()), "fs_swiglu")
                    torch.matmul(self.act_s[:T], self.w_d[layer], out=part)
                else:
                    part.zero_()
                self.xchg.reduce_residual(im, xs)
        return xs

    def serve_launches(self, plan: StepPlan) -> int:
        """Our kernel launches per iteration (K3 + K8 (+combine) + K1 per
        layer, swiglu per layer with the MLP)."""
        n = 0
        for layer in range(self.model.num_layers):
            n += plan.kv_seg[layer + 1] > plan.kv_seg[layer]
            pf = plan.prefill[layer]
            n += 0 if pf is None else 1 + (pf.n_comb > 0)
            n += plan._descs[layer] is not None
            n += bool(self.mlp and len(self.ffn_cols))
        return int(n)


def emulated_serving_step(ranks, plans, x: torch.Tensor) -> torch.Tensor:
    """Single-process emulation of one iteration over several ranks on one
    GPU: per layer each rank's partial, summed in ascending rank order in
    fp32 (refexec.py:283-307), then the residual."""
    order = sorted(range(len(ranks)), key=lambda i: ranks[i].rank)
    x = x.to(torch.bfloat16)
    T = x.shape[0]
    model = ranks[0].model
    for layer in range(model.num_layers):
        for fn in ("serve_attention_partial", "serve_mlp_partial"):
            if fn == "serve_mlp_partial" and not ranks[0].mlp:
                continue
            total = None
            for i in order:
                ranks[i].x_s[:T].copy_(x)
                part = getattr(ranks[i], fn)(layer, plans[i]).float()
                total = part if total is None else total + part
            x = x + total.to(torch.bfloat16)
    return x
