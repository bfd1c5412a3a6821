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
from .core import ClusterSpec, Request, ValidationError
from .metrics import MetricsLog, RunRecorder
from .placement import owner_array
from .recovery_exec import KVBackupExecutor, restore_pages
from .scheduler import build_prefill_batch
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
    weights_ms: float = 0.0          # K7: pcie_host slices + nvlink_peer remainders
    adopt_ms: float = 0.0            # in-place adoption (tables + weight re-layout)
    kv_restore_ms: float = 0.0       # K6 scatters from the lost GPU's host mirror
    kv_restore_bytes: int = 0
    kv_move_bytes: int = 0           # survivor -> survivor KV (re-routed / re-placed)
    recompute_tokens: int = 0
    recompute_ms: float = 0.0
    weight_pcie_bytes: int = 0
    weight_nvlink_bytes: int = 0
    preempted: list = field(default_factory=list)
    restored_exact: bool = False     # restored pages == the lost GPU's pages, bit for bit
    transfers: dict = field(default_factory=dict)

    @property
    def recovery_ms(self) -> float:
        """Failure -> survivors ready (each phase timed on the device)."""
        return (self.plan_ms + self.weights_ms + self.adopt_ms + self.kv_restore_ms +
                self.recompute_ms)


_BIG = 1 << 50


def default_cluster(world: int) -> ClusterSpec:
    """A cluster whose HBM / host memory never bind (no preemption)."""
    return ClusterSpec(num_gpus=world, hbm_bytes_per_gpu=_BIG, pcie_bw_per_gpu=5.0e10,
                       nvlink_bw_per_gpu=9.0e11, allreduce_alpha=1e-5, allreduce_beta=1e-12,
                       host_memory_bytes=_BIG, switch_latency=0.0)


class EmulatedCluster:
    """A serving world of hybrid-attention ranks on one GPU with incremental
    KV backup, driven by the reference's router, Alg. 1 batcher and world
    management (controller.WorldController), that loses GPUs, gets them
    back, and preempts over KV capacity -- executing every decision.

    ``cluster`` (ClusterSpec): HBM per GPU for the capacity / preemption
    decisions (default: never binding)."""

    def __init__(self, model, world: int, inputs, token_budget: int = 256, seed: int = 0,
                 device=None, page_order: str = "shuffled", cluster: ClusterSpec = None):
        from .controller import WorldController
        from .hostmirror import HostWeightStore, WeightLayout
        self.model = model
        self.seed = seed
        self.page_order = page_order
        self.device = torch.device(device if device is not None else "cuda")
        self.budget = token_budget
        self.requests = [Request(id=i, arrival_time=0.0, input_len=a, output_len=o)
                         for i, (a, o) in enumerate(inputs)]
        self.caps = np.array([a + o - 1 for a, o in inputs], dtype=np.int64)
        self.max_tokens = token_budget + len(inputs)
        self.ctrl = WorldController(model, cluster or default_cluster(world),
                                    token_budget=token_budget)
        self.ctrl.alive = set(range(world))
        for r in self.requests:
            self.ctrl.add_request(r)
        self.ctrl.start()
        self.ctrl.admit()
        self.token_x = {}  # (request, position) -> the token's input row (host), for recompute
        self.engines = self._build(self.plan, self.ctrl.serving)
        self.layout = WeightLayout(model, self.plan.ffn.num_shards)
        self.store = HostWeightStore(self.layout)
        first = self.alive[0]
        for g, e in self.engines.items():  # each piece published once (DP heads by the first)
            heads = [e.work.slot_heads[l] if g == first else e.work.slot_heads[l][:e.work.n_tp[l]]
                     for l in range(model.num_layers)]
            e.publish_weights(self.store, heads)
        torch.cuda.synchronize(self.device)
        self.backups = {g: KVBackupExecutor(e.cache) for g, e in self.engines.items()}
        # reference-format metrics (simulation.py:84-132) on the measured
        # clock: every rank of the world shares this GPU, so an iteration's
        # duration is the sum of the ranks' work (a real world runs them in
        # parallel)
        self.recorder = RunRecorder(self.requests, world)

    # -------------------------------------------------------------- state --
    @property
    def alive(self) -> list:
        return list(self.ctrl.serving)

    @property
    def plan(self):
        return self.ctrl.plan

    @property
    def sched(self):
        return self.ctrl.sched

    @property
    def residents(self) -> list:
        return list(self.ctrl.residents)

    def engine_routing(self) -> dict:
        """Routing of every request for the engines' work tables: residents
        by the controller; waiting requests (no KV yet) on the first GPU."""
        first = self.alive[0]
        return {r.id: self.ctrl.routing.get(r.id, first) for r in self.requests}

    def _reserve(self) -> int:
        """KV pages each engine keeps free for in-place adoptions: enough
        for every (layer, head) of every request (the emulation's models
        are small; a deployment sizes it from the planned chain, see
        bench.chain_reserve_pages)."""
        pages = int(((self.caps + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS).sum())
        return self.model.num_layers * self.model.num_kv_heads * pages

    def _engine(self, plan, g, routing):
        owner = owner_array(plan, self.model.num_kv_heads)
        shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
        e = HybridServingRank(self.model, owner, g, routing, self.caps, self.max_tokens,
                              device=self.device, seed=self.seed, shard_owner=shards,
                              page_order=self.page_order, reserve_pages=self._reserve())
        return e

    def _build(self, plan, ranks):
        routing = self.engine_routing()
        return {g: self._engine(plan, g, routing) for g in ranks}

    def _tables(self, plan):
        return (owner_array(plan, self.model.num_kv_heads),
                [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)])

    # ------------------------------------------------------------ serving --
    def context(self, rid) -> int:
        return self.requests[rid].context_tokens()

    def _admit(self) -> None:
        """Admission (simulation.py:401-446); a request admitted onto
        another rank than its engine placeholder moves its (empty) DP items
        there by an in-place adoption."""
        before = self.engine_routing()
        admitted = self.ctrl.admit()
        after = self.engine_routing()
        if any(before[r] != after[r] for r in admitted):
            owner, shards = self._tables(self.plan)
            for e in self.engines.values():
                e.adopt(owner, after, shards, {})
            self.backups = {g: KVBackupExecutor(e.cache) for g, e in self.engines.items()}
            self._sync_backups()

    def next_batch(self) -> StepBatch:
        """One iteration: admission, Alg. 1 prefill batch + one decode token
        per resident whose prefill finished (simulation.py:413-443)."""
        self._admit()
        b = build_prefill_batch(self.sched)
        res = set(self.ctrl.residents)
        dec = [(r.id, r.input_len + r.tokens_decoded - 1) for r in self.requests
               if r.id in res and r.tokens_prefilled == r.input_len
               and 1 <= r.tokens_decoded < r.output_len]
        return StepBatch(prefill=list(b.entries), decode=dec)

    def _sync_backups(self) -> None:
        marks = {r.id: self.context(r.id) for r in self.requests}
        for ex in self.backups.values():
            ex.sync(marks)

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
            self.sched.note_decode_token(req, self.ctrl.routing[rid])
        first = []
        res = set(self.ctrl.residents)
        for req in self.requests:
            if req.id in res and req.tokens_prefilled == req.input_len and \
                    req.tokens_decoded == 0:
                req.tokens_decoded = 1
                first.append(req.id)
        for req in self.requests:  # finished: leave the world, free the reservation
            if req.id in res and req.tokens_decoded >= req.output_len:
                self.ctrl.finish(req.id)
        self._sync_backups()
        t1.synchronize()
        self.recorder.iteration(batch, t0.elapsed_time(t1) / 1e3, finished_prefill=first)
        return out

    def metrics(self) -> MetricsLog:
        """The run so far as the reference's JSONL records (+ run_summary)."""
        unserved = sum(1 for r in self.requests if r.tokens_decoded < r.output_len)
        return self.recorder.finish(unserved)

    # ----------------------------------------------------------- failover --
    def _stage_weights(self, wplan, survivors, rep):
        """K7 on every survivor: the plan's pcie_host transfers from the host
        weight store, then the nvlink_peer remainders from the other
        survivors' staging (device to device here; NVLink on a node)."""
        from .cluster import WeightStaging
        stg, bufs, pieces = {}, {}, {}
        for g in survivors:
            stg[g] = WeightStaging(wplan, g, survivors, self.layout, self.model.num_layers)
            bufs[g] = torch.empty(max(stg[g].nbytes, 16), dtype=torch.uint8, device=self.device)
            pieces[g] = stg[g].bind(bufs[g].data_ptr())
            seg = stg[g].pcie(self.store.dev_ptr)
            seg.run(self.device)
            rep.weight_pcie_bytes += seg.bytes
        bases = {j: bufs[g].data_ptr() for j, g in enumerate(survivors)}
        for g in survivors:
            seg = stg[g].nvlink(bases)
            seg.run(self.device)
            rep.weight_nvlink_bytes += seg.bytes
        torch.cuda.synchronize(self.device)
        return pieces, bufs

    def _preempted(self, pre, rep) -> None:
        for rid in pre:
            self.recorder.preemption(rid)
        rep.preempted = list(pre)

    def fail(self, gpu: int) -> FailoverReport:
        if gpu not in self.alive or len(self.alive) < 2:
            raise ValidationError(f"cannot fail GPU {gpu} of world {self.alive}")
        torch.cuda.synchronize()
        for ex in self.backups.values():
            ex.wait()
        lost_eng, lost_bak = self.engines.pop(gpu), self.backups.pop(gpu)
        old_plan, old_routing = self.plan, dict(self.ctrl.routing)
        t0 = time.perf_counter()
        # what the lost GPU's mirror holds (page-aligned) -> the watermarks
        for r in self.ctrl.residents:
            self.ctrl.backup.register(r)
            self.ctrl.backup.backed[r] = lost_bak.backed_tokens(r)
        d = self.ctrl.fail(gpu)
        survivors = d.desired
        rep = FailoverReport(failed=gpu, world_after=len(survivors))
        kvplan = d.kv_plan
        rep.plan_ms = (time.perf_counter() - t0) * 1e3
        rep.transfers = {"weight": len(d.weight_plan.transfers),
                         "kv": len(kvplan.transfers) if kvplan else 0}

        t0 = time.perf_counter()
        pieces, bufs = self._stage_weights(d.weight_plan, survivors, rep)
        rep.weights_ms = (time.perf_counter() - t0) * 1e3

        # in-place adoption of the on-demand target by every survivor (kept
        # KV pages stay; new items get reserve pages)
        t0 = time.perf_counter()
        owner, shards = self._tables(d.new_plan)
        routing = {r.id: d.new_routing.get(r.id, old_routing.get(r.id, survivors[0]))
                   for r in self.requests}
        routing = {r: (g if g in survivors else survivors[0]) for r, g in routing.items()}
        for g in survivors:
            self.engines[g].adopt(owner, routing, shards, pieces[g])
        del bufs
        torch.cuda.synchronize()
        rep.adopt_ms = (time.perf_counter() - t0) * 1e3

        # lost slices: K6 scatter from the lost GPU's pinned mirror
        t0 = time.perf_counter()
        backup = self.ctrl.backup
        pairs = {g: ([], []) for g in survivors}
        if kvplan is not None:
            for t in kvplan.transfers:
                if t.medium != "pcie_host":
                    continue
                r, layer, h = t.detail
                dst = self.engines[t.dest_gpu]
                src_ids = _item_pages(lost_eng, layer, h, r)
                dst_ids = _item_pages(dst, layer, h, r)
                npg = backup.backed[r] // N.PAGE_TOKENS
                pairs[t.dest_gpu][0].append(dst_ids[:npg])
                pairs[t.dest_gpu][1].append(src_ids[:npg])
                rep.kv_restore_bytes += npg * N.PAGE_BYTES
        for g, (dst_ids, src_ids) in pairs.items():
            if dst_ids:
                restore_pages(self.engines[g].cache.pool, np.concatenate(dst_ids),
                              lost_bak.host, np.concatenate(src_ids))
        torch.cuda.synchronize()
        rep.kv_restore_ms = (time.perf_counter() - t0) * 1e3
        rep.restored_exact = _restored_exact(kvplan, lost_eng, self.engines, backup)
        del lost_eng

        # adopt (simulation.py:225-258): router rebuilt in arrival order,
        # over-capacity preemption
        self._preempted(self.ctrl.apply(d), rep)
        self.backups = {g: KVBackupExecutor(e.cache) for g, e in self.engines.items()}

        # tokens past the backup watermark: recompute by a prefill iteration
        # over the affected tails (the chunk attends to the restored prefix)
        tails = sorted((r, kvplan.recompute_start[r], kvplan.recompute_tokens[r])
                       for r in (kvplan.recompute_tokens if kvplan else {})
                       if kvplan.recompute_tokens[r] > 0 and r in self.ctrl.routing)
        if tails:
            t0 = time.perf_counter()
            b = StepBatch(prefill=list(tails), decode=[])
            x = torch.stack([self.token_x[(r, s + j)] for r, s, n in tails for j in range(n)])
            ranks = [self.engines[g] for g in self.alive]
            emulated_serving_step(ranks, [e.plan(b) for e in ranks], x.to(self.device))
            torch.cuda.synchronize()
            rep.recompute_ms = (time.perf_counter() - t0) * 1e3
            rep.recompute_tokens = sum(n for _, _, n in tails)
        self._sync_backups()
        self.recorder.failure(gpu, alive=len(survivors))
        self.recorder.reconfig(len(survivors), rep.recovery_ms / 1e3, rep.recompute_tokens,
                               rep.kv_restore_bytes + rep.weight_pcie_bytes)
        return rep

    def rejoin(self, gpu: int) -> FailoverReport:
        """A GPU comes back (simulation.py:626-633): the expanded world gets
        a FRESH placement that every GPU reloads from host (recovery.py:
        366-394); KV of every (layer, head, request) whose owner changed moves
        from the GPU that held it (nvlink_peer, plan_kv_recovery); the
        survivors adopt in place, the rejoined GPU starts empty."""
        if gpu in self.ctrl.alive:
            raise ValidationError(f"GPU {gpu} is alive")
        torch.cuda.synchronize()
        for ex in self.backups.values():
            ex.wait()
        t0 = time.perf_counter()
        d = self.ctrl.rejoin(gpu)
        rep = FailoverReport(failed=-gpu - 1, world_after=len(d.desired))
        rep.plan_ms = (time.perf_counter() - t0) * 1e3
        rep.transfers = {"weight": len(d.weight_plan.transfers),
                         "kv": len(d.kv_plan.transfers) if d.kv_plan else 0}
        t0 = time.perf_counter()
        pieces, bufs = self._stage_weights(d.weight_plan, d.desired, rep)
        rep.weights_ms = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        owner, shards = self._tables(d.new_plan)
        old_tabs = {g: (e.work, e.cache.block_table.cpu().numpy()) for g, e in
                    self.engines.items()}
        routing = {r.id: d.new_routing.get(r.id, d.desired[0]) for r in self.requests}
        for g in d.desired:
            if g in self.engines:
                self.engines[g].adopt(owner, routing, shards, pieces[g])
            else:  # the rejoined GPU: a fresh engine, every piece reloaded
                e = self._engine(d.new_plan, g, routing)
                e.load_pieces(pieces[g])  # the fresh reload from host
                self.engines[g] = e
        del bufs
        # KV moves: every new item's pages from the engine that held the key
        src, dst = [], []
        from .kvcache import item_keys
        where = {}
        for g, (w, bt) in old_tabs.items():
            for i, k in enumerate(item_keys(w).tolist()):
                where.setdefault(k, (g, bt[i]))
        for g, e in self.engines.items():
            bt = e.cache.block_table.cpu().numpy()
            for i, k in enumerate(item_keys(e.work).tolist()):
                og = where.get(k)
                req = (k & 0xFFFFF)
                n = (self.context(req) + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS
                if og is None or n == 0:
                    continue
                g0, row = og
                if g0 == g and np.array_equal(row[:n], bt[i, :n]):
                    continue  # kept in place
                src.append((g0, row[:n]))
                dst.append((g, bt[i, :n]))
        if src:  # stage every source page first: freed pages may be reused
            stage = torch.cat([self.engines[g].cache.pool[torch.from_numpy(r.astype(np.int64))
                                                          .to(self.device)] for g, r in src])
            o = 0
            for (g, ids) in dst:
                n = len(ids)
                self.engines[g].cache.pool[torch.from_numpy(ids.astype(np.int64))
                                           .to(self.device)] = stage[o:o + n]
                o += n
            rep.kv_move_bytes = int(stage.numel())
            del stage
        torch.cuda.synchronize()
        rep.adopt_ms = (time.perf_counter() - t0) * 1e3
        self._preempted(self.ctrl.apply(d), rep)
        self.backups = {g: KVBackupExecutor(e.cache) for g, e in self.engines.items()}
        self._sync_backups()
        self.recorder.recovery(gpu, alive=len(self.ctrl.alive))
        self.recorder.reconfig(len(d.desired), rep.recovery_ms / 1e3, 0, rep.weight_pcie_bytes)
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


def _restored_exact(kvplan, lost_eng, engines, backup) -> bool:
    """Every restored page equals the lost GPU's page, byte for byte."""
    if kvplan is None:
        return True
    for t in kvplan.transfers:
        if t.medium != "pcie_host":
            continue
        r, layer, h = t.detail
        npg = backup.backed[r] // N.PAGE_TOKENS
        a = _item_pages(lost_eng, layer, h, r)[:npg]
        b = _item_pages(engines[t.dest_gpu], layer, h, r)[:npg]
        ia = torch.from_numpy(a.astype(np.int64)).to(lost_eng.device)
        ib = torch.from_numpy(b.astype(np.int64)).to(lost_eng.device)
        if not torch.equal(lost_eng.cache.pool[ia], engines[t.dest_gpu].cache.pool[ib]):
            return False
    return True
