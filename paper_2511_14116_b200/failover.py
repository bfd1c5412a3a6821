"""Reconfiguration orchestration: a GPU failure handled end to end.

The executed form of the reference's ``Simulation._reconfigure`` /
``_route_for`` / ``_adopt_plan`` (simulation.py:203-232, 300-371): on the
loss of a GPU the survivors

1. adopt the on-demand shrink target (``plan_weight_recovery(..,
   "on_demand").target_plan``, recovery.py:396-427 -- bit-exact with the
   reference): they keep their TP heads, the lost GPU's heads become
   replicated, its FFN shards go to the least-loaded survivors;
2. re-route residents (``route_for`` = simulation.py:358-371: a request
   keeps its rank if it survived, else goes to the survivor with the least
   remaining tokens);
3. execute the KV plan (``plan_kv_recovery(.., "host_restore")``,
   recovery.py:430-504): slices of the lost GPU are scattered from its
   pinned-host backup mirror into the new owners' pages (K6, one launch per
   survivor); survivor->survivor slices move device to device; tokens past
   the backup watermark are recomputed by a chunked-prefill iteration over
   the affected requests' tails;
4. execute the weight plan's bytes: lost shards / head slices re-materialise
   from pinned host memory (H2D) -- ``nvlink_peer`` slices from surviving
   peers (K7) when the cluster spans several GPUs;
5. rebuild the router state (``_adopt_plan``: residents re-enqueued in
   arrival order on the survivors) and resume serving.

:class:`EmulatedCluster` runs every rank of the world on one GPU (the
single-process form of the one-process-per-GPU deployment; the exchange is
the ordered sum of the per-rank partials, refexec.py:283-307), so the whole
failure path -- backup during serving, loss, restore, resume -- executes
and is checked on a one-GPU box.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .core import Request, ValidationError
from .metrics import MetricsLog, RunRecorder
from .placement import make_placement, owner_array
from .recovery import BackupState, plan_kv_recovery, plan_weight_recovery
from .recovery_exec import KVBackupExecutor, restore_pages
from .scheduler import SchedulerState, build_prefill_batch, route_request
from .serving import HybridServingRank, StepBatch, emulated_serving_step


def route_for(residents, requests, old_routing, serving) -> dict:
    """Deterministic re-routing of residents onto the new world
    (simulation.py:358-371): a request keeps its rank when that rank
    survives; otherwise it goes to argmin (load, rank) over the survivors,
    where load accumulates each placed request's remaining tokens, residents
    visited in order."""
    loads = {g: 0.0 for g in serving}
    out = {}
    for rid in residents:
        req = requests[rid]
        cost = (req.input_len - req.tokens_prefilled) + (req.output_len - req.tokens_decoded)
        old = old_routing.get(rid)
        rank = old if old in loads else min(serving, key=lambda g: (loads[g], g))
        out[rid] = rank
        loads[rank] += cost
    return out


@dataclass
class FailoverReport:
    failed: int
    world_after: int
    plan_ms: float = 0.0
    rebuild_ms: float = 0.0          # survivors' engines on the new layout (emulation)
    kv_restore_ms: float = 0.0       # K6 scatters from the lost GPU's host mirror
    kv_restore_bytes: int = 0
    kv_move_bytes: int = 0           # survivor -> survivor slices (device to device)
    recompute_tokens: int = 0
    recompute_ms: float = 0.0
    weight_h2d_bytes: int = 0
    weight_h2d_ms: float = 0.0
    restored_exact: bool = False     # restored pages == the lost GPU's pages, bit for bit
    transfers: dict = field(default_factory=dict)

    @property
    def recovery_ms(self) -> float:
        """Failure -> survivors ready (the emulation's engine rebuild, which
        a real deployment does in place, is reported separately)."""
        return self.plan_ms + self.kv_restore_ms + self.recompute_ms + self.weight_h2d_ms


class EmulatedCluster:
    """A serving world of ``world`` hybrid-attention ranks on one GPU with
    incremental KV backup, driven by the reference's router and Alg. 1
    batcher, that can lose GPUs and recover."""

    def __init__(self, model, world: int, inputs, token_budget: int = 256, seed: int = 0,
                 device=None, page_order: str = "shuffled"):
        self.model = model
        self.seed = seed
        self.page_order = page_order
        self.device = torch.device(device if device is not None else "cuda")
        self.alive = list(range(world))
        self.plan = make_placement("hybrid", model, self.alive)
        self.budget = token_budget
        self.requests = [Request(id=i, arrival_time=0.0, input_len=a, output_len=o)
                         for i, (a, o) in enumerate(inputs)]
        self.caps = np.array([a + o - 1 for a, o in inputs], dtype=np.int64)
        self.max_tokens = token_budget + len(inputs)
        self.sched = SchedulerState(token_budget=token_budget, rank_set=tuple(self.alive))
        self.routing = {r.id: route_request(self.sched, r) for r in self.requests}
        self.residents = [r.id for r in self.requests]
        self.token_x = {}  # (request, position) -> the token's input row (host), for recompute
        self.engines = self._build(self.plan, self.routing, self.alive)
        self.backups = {g: KVBackupExecutor(e.cache) for g, e in self.engines.items()}
        # reference-format metrics (simulation.py:84-132) on the measured
        # clock: every rank of the world shares this GPU, so an iteration's
        # duration is the sum of the ranks' work (a real world runs them in
        # parallel)
        self.recorder = RunRecorder(self.requests, world)

    def _build(self, plan, routing, ranks):
        owner = owner_array(plan, self.model.num_kv_heads)
        shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
        return {g: HybridServingRank(self.model, owner, g, routing, self.caps, self.max_tokens,
                                     device=self.device, seed=self.seed, shard_owner=shards,
                                     page_order=self.page_order) for g in ranks}

    # ------------------------------------------------------------ serving --
    def context(self, rid) -> int:
        return self.requests[rid].context_tokens()

    def next_batch(self) -> StepBatch:
        """One iteration: Alg. 1 prefill batch + one decode token per
        resident whose prefill finished (simulation.py:413-443)."""
        b = build_prefill_batch(self.sched)
        dec = [(r.id, r.input_len + r.tokens_decoded - 1) for r in self.requests
               if r.id in self.residents and r.tokens_prefilled == r.input_len
               and 1 <= r.tokens_decoded < r.output_len]
        return StepBatch(prefill=list(b.entries), decode=dec)

    def step(self, batch: StepBatch, x: torch.Tensor) -> torch.Tensor:
        """Execute ``batch`` on the alive ranks (x: [T, hidden] bf16), record
        the tokens' inputs, advance request progress and back up every page
        that became complete (K5 on each rank's side stream)."""
        ranks = [self.engines[g] for g in self.alive]
        plans = [e.plan(batch) for e in ranks]
        x = x.to(self.device)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        out = emulated_serving_step(ranks, plans, x)
        t1.record()
        xh = x.detach().to("cpu")
        rows = [(r, s + j) for r, s, n in batch.prefill for j in range(n)] + list(batch.decode)
        for t, key in enumerate(rows):
            self.token_x[key] = xh[t]
        for rid, _, n in batch.prefill:
            self.requests[rid].tokens_prefilled += n
        for rid, _ in batch.decode:
            req = self.requests[rid]
            req.tokens_decoded += 1
            self.sched.note_decode_token(req, self.routing[rid])
        first = []
        for req in self.requests:
            if req.tokens_prefilled == req.input_len and req.tokens_decoded == 0:
                req.tokens_decoded = 1
                first.append(req.id)
        marks = {r.id: self.context(r.id) for r in self.requests}
        for ex in self.backups.values():
            ex.sync(marks)
        t1.synchronize()
        self.recorder.iteration(batch, t0.elapsed_time(t1) / 1e3, finished_prefill=first)
        return out

    def metrics(self) -> MetricsLog:
        """The run so far as the reference's JSONL records (+ run_summary)."""
        unserved = sum(1 for r in self.requests if r.tokens_decoded < r.output_len)
        return self.recorder.finish(unserved)

    # ----------------------------------------------------------- failover --
    def fail(self, gpu: int) -> FailoverReport:
        if gpu not in self.alive or len(self.alive) < 2:
            raise ValidationError(f"cannot fail GPU {gpu} of world {self.alive}")
        torch.cuda.synchronize()
        for ex in self.backups.values():
            ex.wait()
        lost_eng, lost_bak = self.engines.pop(gpu), self.backups.pop(gpu)
        survivors = [g for g in self.alive if g != gpu]
        rep = FailoverReport(failed=gpu, world_after=len(survivors))
        t0 = time.perf_counter()
        wplan = plan_weight_recovery(self.model, self.plan, survivors, "on_demand")
        new_plan = wplan.target_plan("hybrid", self.model)
        contexts = {r: self.context(r) for r in self.residents if self.context(r) > 0}
        new_routing = route_for(self.residents, self.requests, self.routing, survivors)
        backup = BackupState(host_memory_bytes=1 << 62,
                             kv_bytes_per_token=self.model.kv_bytes_per_token())
        for r in contexts:  # what the lost GPU's mirror holds (page-aligned)
            backup.register(r)
            backup.backed[r] = lost_bak.backed_tokens(r)
        kvplan = plan_kv_recovery(backup, self.plan, new_plan, self.model, contexts,
                                  self.routing, new_routing, "host_restore")
        rep.plan_ms = (time.perf_counter() - t0) * 1e3
        rep.transfers = {"weight": len(wplan.transfers), "kv": len(kvplan.transfers)}

        t0 = time.perf_counter()
        new = self._build(new_plan, new_routing, survivors)
        torch.cuda.synchronize()
        rep.rebuild_ms = (time.perf_counter() - t0) * 1e3

        # survivor-held slices: retained (in place in a real deployment) or
        # moved between survivors (DP slices of re-routed requests)
        for g, eng in new.items():
            for src_g, src in self.engines.items():
                n = _copy_items(src, eng, contexts, lambda layer, h, r: True
                                if src_g == g else new_routing[r] == g)
                if src_g != g:
                    rep.kv_move_bytes += n * N.PAGE_BYTES
        # lost slices: K6 scatter from the lost GPU's pinned mirror
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs = {g: ([], []) for g in survivors}
        for t in kvplan.transfers:
            if t.medium != "pcie_host":
                continue
            r, layer, h = t.detail
            dst = new[t.dest_gpu]
            src_ids = _item_pages(lost_eng, layer, h, r)
            dst_ids = _item_pages(dst, layer, h, r)
            npg = backup.backed[r] // N.PAGE_TOKENS
            pairs[t.dest_gpu][0].append(dst_ids[:npg])
            pairs[t.dest_gpu][1].append(src_ids[:npg])
            rep.kv_restore_bytes += npg * N.PAGE_BYTES
        for g, (dst_ids, src_ids) in pairs.items():
            if dst_ids:
                restore_pages(new[g].cache.pool, np.concatenate(dst_ids),
                              lost_bak.host, np.concatenate(src_ids))
        torch.cuda.synchronize()
        rep.kv_restore_ms = (time.perf_counter() - t0) * 1e3
        rep.restored_exact = _restored_exact(kvplan, lost_eng, new, backup)

        # lost weights re-materialised from pinned host memory (bytes of the
        # plan's pcie transfers for the heaviest survivor, executed as H2D)
        pcie = wplan.pcie_bytes_by_gpu()
        rep.weight_h2d_bytes = int(max(pcie.values())) if pcie else 0
        if rep.weight_h2d_bytes:
            host = torch.empty(rep.weight_h2d_bytes, dtype=torch.uint8, pin_memory=True)
            dev = torch.empty(rep.weight_h2d_bytes, dtype=torch.uint8, device=self.device)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.copy_(host, non_blocking=True)
            torch.cuda.synchronize()
            rep.weight_h2d_ms = (time.perf_counter() - t0) * 1e3
            del host, dev

        # adopt: survivors serve the new layout; router rebuilt in arrival
        # order (simulation.py:203-232)
        del lost_eng
        self.engines, self.alive, self.plan, self.routing = new, survivors, new_plan, new_routing
        self.backups = {g: KVBackupExecutor(e.cache) for g, e in new.items()}
        self.sched = SchedulerState(token_budget=self.budget, rank_set=tuple(survivors))
        for rid in self.residents:
            req = self.requests[rid]
            req.dp_rank = new_routing[rid]
            self.sched._enqueue(req, new_routing[rid])

        # tokens past the backup watermark: recompute by a prefill iteration
        # over the affected tails (the chunk attends to the restored prefix)
        tails = sorted((r, kvplan.recompute_start[r], kvplan.recompute_tokens[r])
                       for r in kvplan.recompute_tokens if kvplan.recompute_tokens[r] > 0)
        if tails:
            t0 = time.perf_counter()
            b = StepBatch(prefill=list(tails), decode=[])
            x = torch.stack([self.token_x[(r, s + j)] for r, s, n in tails for j in range(n)])
            ranks = [self.engines[g] for g in self.alive]
            emulated_serving_step(ranks, [e.plan(b) for e in ranks], x.to(self.device))
            torch.cuda.synchronize()
            rep.recompute_ms = (time.perf_counter() - t0) * 1e3
            rep.recompute_tokens = sum(n for _, _, n in tails)
        marks = {r.id: self.context(r.id) for r in self.requests}
        for ex in self.backups.values():
            ex.sync(marks)
        self.recorder.failure(gpu, alive=len(survivors))
        self.recorder.reconfig(len(survivors), rep.recovery_ms / 1e3, rep.recompute_tokens,
                               rep.kv_restore_bytes + rep.weight_h2d_bytes)
        return rep


def _item_pages(eng, layer, head, req):
    """Page ids (block-table row) of (layer, head, request) on ``eng``."""
    slots = eng.work.slot_heads[layer]
    j = slots.index(head)
    it = int(eng.item_index[layer][j, req])
    if it < 0:
        raise ValidationError(f"rank {eng.rank} does not hold layer {layer} head {head} "
                              f"request {req}")
    return eng.cache.block_table[it].cpu().numpy()


def _copy_items(src, dst, contexts, want) -> int:
    """Copy the KV pages of every (layer, head, request) both engines hold
    (and ``want`` selects) from ``src`` to ``dst``; returns pages copied."""
    s_ids, d_ids = [], []
    s_bt = src.cache.block_table.cpu().numpy()
    d_bt = dst.cache.block_table.cpu().numpy()
    for layer in range(src.model.num_layers):
        for h in src.work.slot_heads[layer]:
            if h not in dst.work.slot_heads[layer]:
                continue
            js, jd = src.work.slot_heads[layer].index(h), dst.work.slot_heads[layer].index(h)
            for r, ctx in contexts.items():
                a, b = int(src.item_index[layer][js, r]), int(dst.item_index[layer][jd, r])
                if a < 0 or b < 0 or not want(layer, h, r):
                    continue
                n = (ctx + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS
                s_ids.append(s_bt[a, :n])
                d_ids.append(d_bt[b, :n])
    if not s_ids:
        return 0
    si = torch.from_numpy(np.concatenate(s_ids)).to(dst.device)
    di = torch.from_numpy(np.concatenate(d_ids)).to(dst.device)
    dst.cache.pool[di] = src.cache.pool[si]
    return int(si.numel())


def _restored_exact(kvplan, lost_eng, new, backup) -> bool:
    """Every restored page equals the lost GPU's page, byte for byte."""
    for t in kvplan.transfers:
        if t.medium != "pcie_host":
            continue
        r, layer, h = t.detail
        npg = backup.backed[r] // N.PAGE_TOKENS
        a = _item_pages(lost_eng, layer, h, r)[:npg]
        b = _item_pages(new[t.dest_gpu], layer, h, r)[:npg]
        ia = torch.from_numpy(a.astype(np.int64)).to(lost_eng.device)
        ib = torch.from_numpy(b.astype(np.int64)).to(lost_eng.device)
        if not torch.equal(lost_eng.cache.pool[ia], new[t.dest_gpu].cache.pool[ib]):
            return False
    return True
