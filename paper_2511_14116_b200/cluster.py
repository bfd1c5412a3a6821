"""One-process-per-GPU serving world that loses GPUs and recovers in place.

The executed form of the reference's reconfiguration path for the decode
step (``Simulation._reconfigure`` / ``_route_for`` / ``_adopt_plan``,
simulation.py:225-397, with ``plan_weight_recovery(.., "on_demand")`` and
``plan_kv_recovery(.., "host_restore")``, recovery.py:396-504) across real
processes:

* control plane: :class:`StoreControl` -- all-gather / barrier over the
  job's c10d key-value store (torchrun's agent store).  No collective
  communicator spans the ranks, so a dead process cannot wedge the
  survivors; regrouping is a new key generation over the new alive set;
* data plane: the step's exchanges are ``fs_ar_residual`` over IPC-mapped
  peer buffers (collective.FusedExchange), rebuilt for the survivors;
* host state that outlives a rank (hostmirror): every rank's KV backup
  mirror + page map (K5 token backup after every step) and the node's
  weight store;
* recovery (:meth:`ClusterRank.recover`), on every survivor, from the
  failure event to the first decode step of the new world:

  1. regroup, plan (on-demand target, ``route_for``, both recovery plans);
  2. K7 weights, exactly the plan's transfers for this GPU: its
     ``pcie_host`` slices of every lost head-layer and its lost FFN shards
     from the weight store (one launch), barrier, then the ``nvlink_peer``
     remainders pulled from the other survivors' staging buffers (one
     launch over NVLink);
  3. in-place adoption (``HybridDecodeRank.adopt``): kept KV pages stay,
     new items get reserve pages, weights re-laid out for the new slots;
  4. K6: the plan's ``pcie_host`` KV slices scattered from the dead rank's
     mirror (located through its page map) into the new items' pages;
  5. the exchange rebuilt over the survivors, the step graph recaptured,
     the first step run.  Each phase is timed; ``recovery_ms`` is the wall
     clock from the failure event to the end of that first step.
"""

from __future__ import annotations

import ctypes as C
import os
import pickle
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .core import Request, SimulationError, ValidationError
from .failover import route_for
from .hostmirror import KVMirror, SegmentCopy, WeightLayout, WeightStore
from .hybrid import HybridDecodeRank
from .kvcache import item_keys, pack_keys, unpack_keys
from .placement import make_placement, owner_array
from .recovery import (BackupState, _split_bytes, plan_kv_recovery, plan_weight_recovery)


class StoreControl:
    """Control plane over a c10d Store: ``all_gather_object`` and
    ``barrier`` among the alive ranks (global ids, ascending) of one
    generation.  Works when other ranks have died (no communicator)."""

    def __init__(self, store, rank: int, alive, gen: int = 0, timeout_s: float = 300.0):
        self.store = store
        self.rank = rank
        self.alive = sorted(alive)
        if rank not in self.alive:
            raise ValidationError(f"rank {rank} not in alive set {self.alive}")
        self.gen = gen
        self.index = self.alive.index(rank)
        self.world = len(self.alive)
        self.timeout_s = timeout_s
        self._seq = 0

    def all_gather_object(self, obj) -> list:
        self._seq += 1
        base = f"fs/g{self.gen}/c{self._seq}"
        self.store.set(f"{base}/{self.rank}", pickle.dumps(obj))
        keys = [f"{base}/{r}" for r in self.alive]
        t0 = time.monotonic()
        while not self.store.check(keys):
            if time.monotonic() - t0 > self.timeout_s:
                missing = [r for r, k in zip(self.alive, keys) if not self.store.check([k])]
                raise SimulationError(f"control plane: ranks {missing} did not arrive")
            time.sleep(0.0002)
        return [pickle.loads(self.store.get(k)) for k in keys]

    def barrier(self) -> None:
        self.all_gather_object(None)

    def regroup(self, alive) -> "StoreControl":
        """The survivors' control plane (a new generation of keys)."""
        return StoreControl(self.store, self.rank, alive, self.gen + 1, self.timeout_s)

    def post(self, key: str, value: str = "1") -> None:
        self.store.set(f"fs/{key}", value)


@dataclass
class RecoveryReport:
    failed: int
    world_after: int
    phases_ms: dict = field(default_factory=dict)
    recovery_ms: float = 0.0
    kv_restore_bytes: int = 0
    weight_pcie_bytes: int = 0
    weight_nvlink_bytes: int = 0
    planned_kv_pcie_bytes: int = 0
    planned_weight_pcie_bytes: int = 0
    planned_weight_nvlink_bytes: int = 0
    new_items: int = 0


def _decode_requests(batch: int, ctx: int, out_len: int):
    """Resident decode requests at context ``ctx`` (prompt ctx-1 tokens
    prefilled, first token decoded) for the router / recovery planners."""
    return {i: Request(id=i, arrival_time=0.0, input_len=ctx - 1, output_len=out_len,
                       tokens_prefilled=ctx - 1, tokens_decoded=1) for i in range(batch)}


class WeightStaging:
    """K7 staging of one GPU for a weight plan (recovery.py:348-427): the
    head-layers it receives (on-demand: every lost head-layer, at the same
    offsets on every survivor, so peers can pull each other's slices) and
    the FFN shards it receives, in the canonical piece layout
    (hostmirror.WeightLayout).  ``pcie(store_ptr)`` lists the plan's
    ``pcie_host`` transfers to this GPU (host store -> staging),
    ``nvlink(peer_bases)`` its ``nvlink_peer`` remainders (peer staging ->
    staging; the peers loaded those slices from host first)."""

    def __init__(self, wplan, me: int, survivors, layout, num_layers: int):
        self.plan, self.me, self.layout, self.L = wplan, me, layout, num_layers
        self.survivors = list(survivors)
        self.slices = _split_bytes(layout.head_bytes, len(self.survivors))
        self.starts = np.concatenate([[0], np.cumsum(self.slices)]).astype(np.int64).tolist()
        mine = [t for t in wplan.transfers if t.dest_gpu == me]
        self.heads = sorted({tuple(t.detail[:2]) for t in mine if t.content == "attn_head_slice"})
        self.shards = sorted({t.detail[0] for t in mine if t.content == "ffn_shard"})
        self.nbytes = len(self.heads) * layout.head_bytes + \
            len(self.shards) * num_layers * layout.shard_bytes

    def bind(self, base: int) -> dict:
        """Staging at device address ``base``; returns the pieces map
        HybridDecodeRank.adopt consumes."""
        lay = self.layout
        self.base = base
        self.head_at = {hl: base + k * lay.head_bytes for k, hl in enumerate(self.heads)}
        sb = base + len(self.heads) * lay.head_bytes
        self.shard_at = {(layer, s): sb + (k * self.L + layer) * lay.shard_bytes
                         for k, s in enumerate(self.shards) for layer in range(self.L)}
        pieces = {("head", l_, h_): a for (l_, h_), a in self.head_at.items()}
        pieces.update({("shard", l_, s_): a for (l_, s_), a in self.shard_at.items()})
        return pieces

    def pcie(self, store_ptr: int) -> SegmentCopy:
        lay, seg = self.layout, SegmentCopy()
        for t in self.plan.transfers:
            if t.dest_gpu != self.me or t.medium != "pcie_host":
                continue
            if t.content == "ffn_shard":
                s = t.detail[0]
                for layer in range(self.L):
                    seg.add_bytes(self.shard_at[(layer, s)], store_ptr + lay.shard_off(layer, s),
                                  lay.shard_bytes)
            elif len(t.detail) == 3:  # on-demand: this GPU's slice i
                layer, h, i = t.detail
                a = self.starts[i]
                seg.add_bytes(self.head_at[(layer, h)] + a, store_ptr + lay.head_off(layer, h) + a,
                              self.slices[i])
            else:                     # fresh reload: the whole head-layer
                layer, h = t.detail
                seg.add_bytes(self.head_at[(layer, h)], store_ptr + lay.head_off(layer, h),
                              lay.head_bytes)
        return seg

    def nvlink(self, peer_bases: dict) -> SegmentCopy:
        """peer_bases: survivor index j -> that survivor's staging base (as
        mapped here); the other survivors' slices of every head-layer."""
        seg = SegmentCopy()
        if not any(t.medium == "nvlink_peer" and t.dest_gpu == self.me
                   for t in self.plan.transfers):
            return seg
        i_me = self.survivors.index(self.me)
        for j, b in peer_bases.items():
            if j == i_me:
                continue
            for hl, a in self.head_at.items():
                off = (a - self.base) + self.starts[j]
                seg.add_bytes(self.base + off, b + off, self.slices[j])
        return seg


class ClusterRank:
    """Rank ``rank`` of a hybrid-attention decode world over ``alive``.

    ``store``: the job's c10d Store; ``job``: a name unique to the job (the
    shared-memory regions are ``/dev/shm/<job>_*``); ``reserve_pages``: KV
    pages kept free for adoptions.  All ranks construct together."""

    def __init__(self, model, rank: int, alive, store, job: str, batch: int, ctx: int,
                 seed: int = 0, mlp: bool = True, reserve_pages: int = 0, device=None,
                 page_order: str = "contiguous", out_len: int = 1024, kv_fill=None,
                 config: int = 0):
        self.model = model
        self.rank = rank
        self.job = job
        self.batch, self.ctx = batch, ctx
        self.device = torch.device(device if device is not None else "cuda")
        self.ctl = StoreControl(store, rank, alive)
        self.plan = make_placement("hybrid", model, self.ctl.alive)
        self.requests = _decode_requests(batch, ctx, out_len)
        self.routing = self._initial_routing()
        self.layout = WeightLayout(model, self.plan.ffn.num_shards)
        owner = owner_array(self.plan, model.num_kv_heads)
        shards = [self.plan.ffn.owner[s] for s in range(self.plan.ffn.num_shards)]
        self.eng = HybridDecodeRank(model, owner, rank, self.routing, batch, ctx,
                                    device=self.device, seed=seed, group=self.ctl,
                                    page_order=page_order, mlp=mlp, shard_owner=shards,
                                    exchange="fused", reserve_pages=reserve_pages, config=config)
        self.eng.set_lengths([ctx] * batch)
        if kv_fill is not None:
            kv_fill(self.eng)
        # host state: my KV mirror (+ page map), the node's weight store
        c = self.eng.cache
        items_cap = c.work.n_items + reserve_pages // max(1, c.pages_per_seq) + 1
        self.mirror = KVMirror(f"{job}_kv{rank}", n_pages=c.n_pages, items_cap=items_cap,
                               pages_per_seq=c.pages_per_seq, rank=rank, create=True)
        if self.ctl.index == 0:
            WeightStore(f"{job}_w", self.layout, create=True, register=False).close()
        self.ctl.barrier()
        self.wstore = WeightStore(f"{job}_w", self.layout)
        self.eng.publish_weights(self.wstore)
        self._publish_tables()
        self.backup_all()
        self.eng.backup_ptr = self.mirror.pages_dev_ptr
        torch.cuda.synchronize(self.device)
        self.ctl.barrier()
        # every survivor maps every peer's mirror up front (registration of
        # a multi-GB mapping is slow; the failure path must not pay it)
        self.peer_mirrors = {g: KVMirror(f"{job}_kv{g}") for g in self.ctl.alive if g != rank}
        self.reports = []
        self.ctl.barrier()  # the next exchange spins on every rank: leave together

    # ------------------------------------------------------------ serving --
    def _initial_routing(self):
        from .scheduler import SchedulerState, route_request
        st = SchedulerState(token_budget=2048, rank_set=tuple(self.ctl.alive))
        return {i: route_request(st, Request(id=i, arrival_time=0.0, input_len=self.ctx - 1,
                                             output_len=1)) for i in range(self.batch)}

    def _publish_tables(self) -> None:
        c = self.eng.cache
        keys = unpack_keys(item_keys(c.work))
        self.mirror.publish_tables(keys, c.block_table.cpu().numpy())

    def backup_all(self) -> None:
        """K5 over every page holding tokens (start-up / after adoption);
        the page map and watermarks go to the mirror header."""
        c = self.eng.cache
        lens = c.item_len.cpu().numpy()
        bt = c.block_table.cpu().numpy()
        ids = np.concatenate([bt[i, :(int(n) + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS]
                              for i, n in enumerate(lens)]) if len(lens) else np.zeros(0)
        self._gather(ids)
        torch.cuda.current_stream(self.device).synchronize()
        self.mirror.set_backed(lens)

    def _gather(self, page_ids) -> None:
        if not len(page_ids):
            return
        ids = torch.from_numpy(np.asarray(page_ids, dtype=np.int32)).to(self.device)
        N.check(N.lib.fs_pages_gather(N.ptr(self.eng.cache.pool), N.ptr(ids), ids.numel(),
                                      C.c_void_p(self.mirror.pages_dev_ptr), N.ptr(ids), 0,
                                      C.c_void_p(torch.cuda.current_stream(
                                          self.device).cuda_stream)), "fs_pages_gather")

    def step(self, x=None):
        return self.eng.step(x)

    def mark_backed(self) -> None:
        """Every item's tokens up to its length are on the host (the token
        backup rides at the end of every step)."""
        torch.cuda.current_stream(self.device).synchronize()
        self.mirror.set_backed(self.eng.cache.item_len.cpu().numpy())

    def die(self) -> None:
        """The injected failure: finish in-flight work (the backup of the
        last step), post the loss and exit the process (exit code 0)."""
        self.mark_backed()
        self.ctl.post(f"dead/{self.rank}", f"{time.time():.6f}")
        os._exit(0)

    # ----------------------------------------------------------- recovery --
    def wait_dead(self, failed: int, timeout_s: float = 300.0) -> float:
        """Failure detection: block until ``failed`` posted its loss (the
        injected failure's notice; its mirror is final from then on).
        Returns the posted wall time."""
        key = f"fs/dead/{failed}"
        t0 = time.monotonic()
        while not self.ctl.store.check([key]):
            if time.monotonic() - t0 > timeout_s:
                raise SimulationError(f"rank {failed} never reported its loss")
            time.sleep(0.0002)
        return float(self.ctl.store.get(key).decode())

    def recover(self, failed: int) -> RecoveryReport:
        """Run on every survivor at the failure event (see module doc):
        the clock starts when the loss is detected (the dead rank's notice)."""
        self.wait_dead(failed)
        t_event = time.perf_counter()
        ph = {}

        def lap(name, t):
            torch.cuda.synchronize(self.device)
            now = time.perf_counter()
            ph[name] = round((now - t) * 1e3, 3)
            return now

        model, eng = self.model, self.eng
        old_plan, old_routing = self.plan, self.routing
        survivors = [g for g in self.ctl.alive if g != failed]
        rep = RecoveryReport(failed=failed, world_after=len(survivors))
        # 1. regroup + plans
        old_xchg = eng.xchg
        self.ctl = self.ctl.regroup(survivors)
        wplan = plan_weight_recovery(model, old_plan, survivors, "on_demand")
        new_plan = wplan.target_plan("hybrid", model)
        residents = sorted(self.requests)
        new_routing = route_for(residents, self.requests, old_routing, survivors)
        vm = self.peer_mirrors[failed]
        v_keys, v_bt, v_backed = vm.tables()
        v_index = {k: i for i, k in enumerate(pack_keys(v_keys).tolist())}
        backup = BackupState(host_memory_bytes=1 << 62,
                             kv_bytes_per_token=model.kv_bytes_per_token())
        contexts = {r: self.ctx for r in residents}
        # the dead rank's watermark per request: min over its items (all equal here)
        v_req_backed = {}
        for (layer, h, r), b in zip(v_keys.tolist(), v_backed.tolist()):
            v_req_backed[r] = min(v_req_backed.get(r, b), b)
        for r in residents:
            backup.register(r)
            backup.backed[r] = v_req_backed.get(r, self.ctx)
        kvplan = plan_kv_recovery(backup, old_plan, new_plan, model, contexts, old_routing,
                                  new_routing, "host_restore")
        if kvplan.recompute_tokens:
            raise SimulationError("tokens past the backup watermark: the decode engine has no "
                                  "recompute path (serving.HybridServingRank does)")
        me = self.rank
        rep.planned_kv_pcie_bytes = sum(t.num_bytes for t in kvplan.transfers
                                        if t.dest_gpu == me and t.medium == "pcie_host")
        rep.planned_weight_pcie_bytes = wplan.pcie_bytes_by_gpu().get(me, 0)
        rep.planned_weight_nvlink_bytes = wplan.nvlink_bytes_by_gpu().get(me, 0)
        t = lap("plan", t_event)

        # 2. K7: staging = every lost head-layer (same offsets on every
        #    survivor) + this GPU's lost shards; cudaMalloc'd (not the
        #    caching allocator): IPC exports whole allocations
        stg = WeightStaging(wplan, me, survivors, self.layout, model.num_layers)
        sp = C.c_void_p()
        dev_index = self.device.index if self.device.index is not None \
            else torch.cuda.current_device()
        N.check(N.lib.fs_ar_alloc(dev_index, max(stg.nbytes, 256), C.byref(sp)), "fs_ar_alloc")
        base = sp.value
        pieces = stg.bind(base)
        h2d = stg.pcie(self.wstore.dev_ptr)
        h2d.run(self.device)
        rep.weight_pcie_bytes = h2d.bytes
        t = lap("weights_pcie", t)
        # staging of the peers (IPC over NVLink), after their slices landed
        handle = (C.c_uint8 * 64)()
        N.check(N.lib.fs_ar_ipc_handle(C.c_void_p(base), handle), "fs_ar_ipc_handle")
        every = self.ctl.all_gather_object(bytes(handle))
        opened, peer_bases = [], {}
        if stg.heads:
            for j, g in enumerate(survivors):
                if g == me:
                    continue
                q = C.c_void_p()
                N.check(N.lib.fs_ar_ipc_open((C.c_uint8 * 64).from_buffer_copy(every[j]),
                                             C.byref(q)), "fs_ar_ipc_open")
                opened.append(q.value)
                peer_bases[j] = q.value
        p2p = stg.nvlink(peer_bases)
        p2p.run(self.device)
        rep.weight_nvlink_bytes = p2p.bytes
        t = lap("weights_nvlink", t)
        self.ctl.barrier()  # every peer finished reading my staging
        for q in opened:
            N.lib.fs_ar_ipc_close(C.c_void_p(q))
        t = lap("barrier", t)

        # 3. in-place adoption
        new_owner = owner_array(new_plan, model.num_kv_heads)
        new_shards = [new_plan.ffn.owner[s] for s in range(new_plan.ffn.num_shards)]
        fresh = eng.adopt(new_owner, new_routing, new_shards, pieces)
        eng.set_lengths([self.ctx] * self.batch)
        N.lib.fs_ar_free(C.c_void_p(base))
        t = lap("adopt", t)

        # 4. K6: the plan's pcie_host KV slices from the dead rank's mirror
        want = {(t_.detail[1], t_.detail[2], t_.detail[0]) for t_ in kvplan.transfers
                if t_.dest_gpu == me and t_.medium == "pcie_host"}
        keys = unpack_keys(item_keys(eng.work))
        bt = eng.cache.block_table.cpu().numpy()
        dst_ids, src_ids = [], []
        for i in fresh:
            lhr = tuple(int(x) for x in keys[i])
            if lhr not in want:
                raise SimulationError(f"new item {lhr} is not a planned KV restore")
            want.discard(lhr)
            vi = v_index.get(pack_keys(np.array(lhr))[0])
            if vi is None:
                raise SimulationError(f"item {lhr} is not in rank {failed}'s page map")
            npg = (int(v_backed[vi]) + N.PAGE_TOKENS - 1) // N.PAGE_TOKENS
            dst_ids.append(bt[i, :npg])
            src_ids.append(v_bt[vi, :npg])
        if want:
            raise SimulationError(f"planned KV restores without a new item: {sorted(want)[:4]}")
        if dst_ids:
            d = torch.from_numpy(np.concatenate(dst_ids).astype(np.int32)).to(self.device)
            s_ = torch.from_numpy(np.concatenate(src_ids).astype(np.int32)).to(self.device)
            N.check(N.lib.fs_pages_scatter(N.ptr(eng.cache.pool), N.ptr(d), d.numel(),
                                           C.c_void_p(vm.pages_dev_ptr), N.ptr(s_), 0,
                                           C.c_void_p(torch.cuda.current_stream(
                                               self.device).cuda_stream)), "fs_pages_scatter")
            rep.kv_restore_bytes = int(d.numel()) * N.PAGE_BYTES
        rep.new_items = len(fresh)
        t = lap("kv_restore", t)

        # 5. the exchange re-formed over the survivors (same buffers and
        #    mappings, the dead rank's dropped), first step (eager: the step
        #    graph is re-captured after the clock stops)
        eng.group = self.ctl
        old_xchg.shrink(self.ctl)
        self.ctl.barrier()  # the first exchange spins on every survivor: start together
        t = lap("exchange", t)
        eng.step()
        t = lap("first_step", t)
        rep.phases_ms = ph
        rep.recovery_ms = round((t - t_event) * 1e3, 3)
        eng.capture()
        # new state: plan, routing, page map; the restored pages into my
        # own mirror (off the critical path)
        self.plan, self.routing = new_plan, new_routing
        for g in [failed]:
            m = self.peer_mirrors.pop(g)
            m.close()
        self._publish_tables()
        self.backup_all()
        self.ctl.barrier()  # every survivor's mirror is consistent before serving resumes
        self.reports.append(rep)
        return rep

    def close(self, unlink: bool = True) -> None:
        if self.eng.xchg is not None:
            self.eng.xchg.close()
        for m in self.peer_mirrors.values():
            m.close()
        self.mirror.close(unlink=unlink)
        self.wstore.close(unlink=unlink and self.ctl.index == 0)


def shm_cleanup(prefix: str) -> None:
    """Remove the shared-memory regions whose names start with ``prefix``
    (a job's, including those of its dead ranks)."""
    for name in os.listdir("/dev/shm"):
        if name.startswith(prefix):
            try:
                os.unlink(os.path.join("/dev/shm", name))
            except FileNotFoundError:
                pass
