#!/usr/bin/env python
"""bench.py -- FailSafe (arXiv 2511.14116) hybrid-attention decode on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 (default) runs BASELINE config 2 -- the Llama-3-8B-shaped hybrid-
attention decode step, batch 64, context 4096, hybrid placement -- on one
GPU; N>1 (torchrun, one process per GPU, NCCL) runs the same job split over
N ranks (hybrid placement, least-loaded routing, NCCL all-reduce of the
attention output).  One JSON line on rank 0.

A *step* = one decode token for all 64 requests through every layer:
fused QKV GEMM (fs_gemm_skinny, tcgen05; ``--gemm cublas`` for cuBLAS) -> ONE
fs_decode_attention launch (KV append + paged GQA decode + split merge) ->
output projection (+ residual at N=1) -> exchange + residual (N>1: one
fs_ar_residual kernel over IPC-mapped peer buffers, ``--exchange nccl`` for an
NCCL all-reduce) -> TP MLP partial over the rank's FFN shards (gate/up GEMM
with the SwiGLU epilogue, down GEMM) -> exchange -> residual (``--no-mlp``:
attention sublayer only).  The whole step is one CUDA-graph replay.  The KV working set
(34 GB at N=1) is far larger than L2, so no flush is needed between steps.

At N=1 the line also carries (rank 0 only):
* ``failure_states`` -- BASELINE config 3 (Llama-3-70B-shaped, B=64,
  ctx 4096) at the 8 -> 7 -> 6 -> 5 on-demand shrink chain, every rank of
  every world emulated on this GPU (exchange excluded: one GPU);
* ``mixed_trace`` -- config 5: mixed prefill/decode iterations (Alg. 1
  chunked prefill + decode, 32k prompts) on the 7 survivors, every rank
  emulated on this GPU;
* ``cost_calibration`` -- the reference's iteration-time model fitted to
  the per-rank times above;
* ``recovery`` -- config 4 microbenchmark (KV restore from the pinned host
  backup, weight shards) after 1-3 losses;
* ``cpu_baseline`` -- the CPU oracle port on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("decode tokens/s at 8→7→6→5 B200 (fraction of HBM roofline); "
          "failure recovery ms")
UNIT = "tokens/s"
KV_UNIT = 512  # bytes per (kv head, token): K+V, head_dim 128, bf16 (core.py:101-103)
GEMM_BACKEND = "tcgen05"  # --gemm: projections via the tcgen05 skinny GEMM (default) or cuBLAS
EXCHANGE = "fused"
# fs_decode_attention configs -> the kernel instance that runs (csrc/decode.cu)
KERNEL_NAMES = {0: "decode_cta_kernel<8,2>", 3: "decode_cta_kernel<16,1>",
                7: "decode_kernel<4,4,1>", 9: "decode_kernel<8,2,1>"}  # --exchange (N>1): fs_ar_residual over peer memory, or NCCL all-reduce


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every 10 ms."""

    HW = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
          "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [k for k, bit in self.HW.items() if self.reasons & bit],
                "samples": len(self.samples)}


# -------------------------------------------------------------- workloads --
def llama8b():
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=32, num_kv_heads=8, num_q_heads=32, head_dim=128,
                     hidden_dim=4096, ffn_intermediate_dim=14336)


def llama70b():
    from paper_2511_14116_b200.core import load_config
    return load_config(os.path.join(ROOT, "paper_2511_14116_b200", "data", "llama70b.toml"))[0]


def route(n_requests, ranks, ctx):
    """Least-loaded routing of equal requests (scheduler.py:160-164)."""
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.scheduler import SchedulerState, route_request
    st = SchedulerState(token_budget=2048, rank_set=tuple(ranks))
    return {i: route_request(st, Request(id=i, arrival_time=0.0, input_len=ctx - 1,
                                         output_len=1)) for i in range(n_requests)}


def build_rank(model, plan, rank, routing, batch, ctx, group, config, seed=0, mlp=True):
    import torch
    from paper_2511_14116_b200.hybrid import HybridDecodeRank
    from paper_2511_14116_b200.placement import owner_array
    owner = owner_array(plan, model.num_kv_heads)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    eng = HybridDecodeRank(model, owner, rank, routing, batch, ctx, group=group, seed=seed,
                           config=config, mlp=mlp, shard_owner=shards, gemm=GEMM_BACKEND,
                           exchange=EXCHANGE)
    eng.set_lengths([ctx] * batch)
    eng.fill_random_kv(seed + 17 * rank)
    eng.x.copy_(torch.randn_like(eng.x, dtype=torch.float32).to(torch.bfloat16))
    # gloo collectives are not capturable (the fused exchange is)
    if os.environ.get("FS_BENCH_SHARED_GPU") != "1" or eng.xchg is not None or group is None:
        eng.capture()
    return eng


def time_graph(fn, steps, warmup, stream=None):
    """Device time (ms per call) of ``fn`` with CUDA events on the current
    stream, synchronized on both sides."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def attention_op_graph(eng):
    """A CUDA graph of just the per-layer fs_decode_attention launches."""
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for layer in range(eng.model.num_layers):
            eng.cache.decode_layer_fused(layer, eng.qkv, eng.o)
    return g


def step_kv_bytes(eng):
    return sum(eng.cache.layer_kv_bytes(l) for l in range(eng.model.num_layers))


def ncu_traffic():
    """dram bytes per decode launch from the committed ncu --set full
    summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ------------------------------------------------------- failure states --
def failure_states(steps, warmup, config, batch=64, ctx=4096, fails=(7, 3, 5), mlp=True):
    import torch
    from paper_2511_14116_b200 import _native as N
    from paper_2511_14116_b200.placement import (make_placement, memory_footprint,
                                                 owner_array)
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    model = llama70b()
    peak, _ = measured_peaks()
    plan = make_placement("hybrid", model, range(8))
    alive = list(range(8))
    states = []
    chain = [None] + list(fails)
    for f in chain:
        if f is not None:
            alive = [g for g in alive if g != f]
            plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan(
                "hybrid", model)
        owner = owner_array(plan, model.num_kv_heads)
        routing = route(batch, alive, ctx)
        fp = memory_footprint(plan, model, {r: ctx for r in range(batch)}, routing)
        per_rank = []
        for g in alive:
            eng = build_rank(model, plan, g, routing, batch, ctx, None, config, mlp=mlp)
            ms = time_graph(eng.step, min(steps, 20), warmup)
            kb = step_kv_bytes(eng)
            att = attention_op_graph(eng)
            att_ms = time_graph(att.replay, min(steps, 20), 2)
            per_rank.append({"rank": g, "step_ms": round(ms, 4), "kv_bytes": kb,
                             "weight_bytes": eng.weight_bytes(),
                             "step_frac": round((kb + eng.weight_bytes()) / (ms / 1e3) / 1e9 /
                                                peak, 4),
                             "attn_ms": round(att_ms, 4),
                             "attn_gbs": round(kb / att_ms / 1e6, 1)})
            del eng, att
            torch.cuda.empty_cache()
        worst = max(per_rank, key=lambda r: r["step_ms"])
        states.append({
            "world": len(alive), "failed": f, "max_rank_step_ms": worst["step_ms"],
            "tok_s": round(batch / (worst["step_ms"] / 1e3), 1),
            "max_kv_bytes": max(fp.values()),
            "kv_roofline_frac": round(max(fp.values()) / (worst["step_ms"] / 1e3) / 1e9 / peak, 4),
            "attn_frac_min": round(min(r["attn_gbs"] for r in per_rank) / peak, 4),
            "step_frac_max_rank": worst["step_frac"],
            "ranks": per_rank})
    r8 = states[0]["tok_s"]
    out = {"workload": "C3 Llama-3-70B-shaped decode step (attention + TP MLP), B=64, "
                       "ctx 4096, hybrid(8) then "
                       "on-demand shrink after failures of GPU 7, 3, 5",
           "emulation": "every rank of every world timed on this one GPU (graph replay); "
                        "step = max over ranks; the NCCL exchange is excluded (1 GPU)",
           "states": states}
    for s in states[1:]:
        s["vs_8_scaled"] = round(s["tok_s"] / (r8 * s["world"] / 8), 4)
    return out


# --------------------------------------- failure chain (N>1, processes) --
def chain_reserve_pages(model, world, fails, batch, ctx):
    """KV pages every rank keeps free so the whole on-demand chain adopts
    in place: max over ranks and states of (pages then - pages at start)."""
    from paper_2511_14116_b200.failover import route_for
    from paper_2511_14116_b200.cluster import _decode_requests
    from paper_2511_14116_b200.kvcache import RankWork
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    plan = make_placement("hybrid", model, range(world))
    alive = list(range(world))
    routing = route(batch, alive, ctx)
    reqs = _decode_requests(batch, ctx, 1024)
    pages = (ctx + 15) // 16

    def items(plan, routing):
        owner = owner_array(plan, model.num_kv_heads)
        return {g: RankWork.build(owner, g, routing, batch).n_items for g in plan.alive}
    start = items(plan, routing)
    need = 0
    for f in fails:
        alive = [g for g in alive if g != f]
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
        routing = route_for(sorted(reqs), reqs, routing, alive)
        now = items(plan, routing)
        need = max(need, max(now[g] - start[g] for g in alive))
    return need * pages


def failure_chain(args, world, rank, local_rank):
    """BASELINE configs 3 + 4 on one process per GPU: the C3 decode step
    (Llama-3-70B shape, B=64, ctx 4096, attention + TP MLP, fused exchange)
    on hybrid(N), then for each GPU in ``--failures``: that rank's process
    EXITS, the survivors recover in place (cluster.ClusterRank.recover:
    regroup, K7 weights from the host store + peers, adoption, K6 KV from
    the dead rank's mirror, exchange rebuilt, graph, first step) and are
    timed again.  Per world: max-rank step time INCLUDING the exchange,
    tok/s, KV-roofline fraction, N/(8 scaled) ratio; per failure: recovery
    wall clock with its phases (max over survivors)."""
    import torch
    from paper_2511_14116_b200.cluster import ClusterRank, shm_cleanup
    from paper_2511_14116_b200.hostmirror import SharedHostRegion, WeightLayout
    from paper_2511_14116_b200.placement import make_placement, memory_footprint
    from paper_2511_14116_b200.core import ModelSpec
    fails = [int(f) for f in args.failures.split(",") if f != ""]
    model = llama70b()
    if args.chain_layers:  # testing on a shared GPU only: NOT the C3 measurement
        model = ModelSpec(num_layers=args.chain_layers, num_kv_heads=8, num_q_heads=64,
                          head_dim=128, hidden_dim=8192, ffn_intermediate_dim=28672)
    batch, ctx = 64, 4096
    peak, _ = measured_peaks()
    import torch.distributed as dist
    store = dist.TCPStore(os.environ.get("MASTER_ADDR", "127.0.0.1"),
                          int(os.environ["MASTER_PORT"]), None, False)
    # one job name for all ranks (rank 0 picks it); stale regions of earlier
    # runs on a reused box are removed first (they would pin host memory)
    if rank == 0:
        shm_cleanup("fsb")
        store.set("fs/job", f"fsb{os.getpid()}x{int(time.time())}")
    job = store.get("fs/job").decode()
    reserve = chain_reserve_pages(model, world, fails, batch, ctx)
    # host memory: weight store + every rank's mirror (pool incl. reserve)
    lay = WeightLayout(model, model.default_num_shards())
    plan0 = make_placement("hybrid", model, range(world))
    fp0 = memory_footprint(plan0, model, {r: ctx for r in range(batch)}, route(batch, range(world),
                                                                             ctx))
    need_host = lay.total + world * (max(fp0.values()) + reserve * 8192) * 1.05
    free = SharedHostRegion.free_bytes()
    if need_host > free:
        return {"skipped": f"/dev/shm has {free / 1e9:.0f} GB free, the weight store + KV "
                           f"mirrors need {need_host / 1e9:.0f} GB"}
    t0 = time.perf_counter()
    cr = ClusterRank(model, rank, range(world), store, job, batch, ctx, seed=0, mlp=True,
                     reserve_pages=reserve, device=torch.device("cuda", local_rank),
                     config=args.kernel_config)
    cr.eng.fill_random_kv(17 + rank)
    cr.backup_all()
    cr.eng.x.copy_(torch.randn_like(cr.eng.x, dtype=torch.float32).to(torch.bfloat16))
    cr.eng.capture()
    setup_s = time.perf_counter() - t0

    def timed_world():
        for _ in range(args.warmup):
            cr.step()
        torch.cuda.synchronize()
        cr.ctl.barrier()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        for _ in range(args.steps):
            cr.step()
        e_.record()
        torch.cuda.synchronize()
        ms = s_.elapsed_time(e_) / args.steps
        c = cr.eng.cache
        kv = int(c.item_len.sum().item()) * KV_UNIT
        every = cr.ctl.all_gather_object((rank, ms, kv, cr.eng.weight_bytes()))
        worst = max(every, key=lambda t: t[1])
        return {"world": cr.ctl.world, "alive": list(cr.ctl.alive),
                "max_rank_step_ms": round(worst[1], 4),
                "tok_s": round(batch / (worst[1] / 1e3), 1),
                "max_kv_bytes": max(t[2] for t in every),
                "kv_roofline_frac": round(max(t[2] for t in every) / (worst[1] / 1e3) / 1e9 /
                                          peak, 4),
                "step_frac_max_rank": round((worst[2] + worst[3]) / (worst[1] / 1e3) / 1e9 / peak,
                                            4),
                "rank_step_ms": {t[0]: round(t[1], 4) for t in every}}

    states = [timed_world()]
    states[0]["failed"] = None
    recoveries = []
    for f in fails:
        cr.mark_backed()
        if rank == f:
            cr.die()                      # the process exits here
        rep = cr.recover(f)
        every = cr.ctl.all_gather_object(rep.__dict__)
        worst = max(every, key=lambda d: d["recovery_ms"])
        recoveries.append({"failed": f, "world_after": rep.world_after,
                           "recovery_ms_max": worst["recovery_ms"],
                           "phases_ms_of_max": worst["phases_ms"],
                           "kv_restore_bytes_max": max(d["kv_restore_bytes"] for d in every),
                           "weight_pcie_bytes_max": max(d["weight_pcie_bytes"] for d in every),
                           "weight_nvlink_bytes_max": max(d["weight_nvlink_bytes"] for d in every),
                           "plan_bytes_match": all(
                               d["weight_pcie_bytes"] == d["planned_weight_pcie_bytes"] and
                               d["weight_nvlink_bytes"] == d["planned_weight_nvlink_bytes"]
                               for d in every)})
        st = timed_world()
        st["failed"] = f
        states.append(st)
    r8 = states[0]["tok_s"]
    for st in states[1:]:
        st["vs_first_scaled"] = round(st["tok_s"] / (r8 * st["world"] / states[0]["world"]), 4)
    cr.ctl.barrier()
    if cr.ctl.index == 0:
        shm_cleanup(job)
    return {"workload": f"C3 Llama-3-70B-shaped decode step ({model.num_layers} layers, attention"
                        " + TP MLP, fused exchange), B=64, ctx 4096, hybrid(" + str(world) +
                        ") then on-demand shrink after failures of GPU " +
                        ", ".join(map(str, fails)) + "; one process per GPU, victims exit",
            "setup_s": round(setup_s, 1), "states": states, "recoveries": recoveries,
            "test_only": bool(args.chain_layers)}


# ------------------------------------------------- mixed trace (config 5) --
def sharegpt_trace(n=120, seed=20240701, n_long=2, long_len=32768):
    """ShareGPT-shaped lognormal lengths (the reference's synth_trace
    recipe, traces.py:66-84: median 256 / sigma 1.0 inputs, median 192 /
    sigma 0.8 outputs) with ``n_long`` injected 32k-token prompts."""
    import math
    import random
    rng = random.Random(seed)

    def ln(median, sigma, mx):
        return max(1, min(int(round(math.exp(math.log(median) + sigma * rng.gauss(0, 1)))), mx))

    rows = [(ln(256.0, 1.0, 8192), ln(192.0, 0.8, 2048)) for _ in range(n)]
    for i in range(n_long):
        rows.insert((i + 1) * n // (n_long + 1), (long_len, ln(192.0, 0.8, 2048)))
    return rows


def mixed_iterations(inputs, ranks, budget, skip, n_iter):
    """Router + Alg. 1 batcher over the trace (all requests queued at t=0);
    the first ``skip`` iterations only advance the host state (their KV is
    random-filled), the next ``n_iter`` are returned as StepBatches."""
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.scheduler import (SchedulerState, build_prefill_batch,
                                                 route_request)
    from paper_2511_14116_b200.serving import StepBatch
    st = SchedulerState(token_budget=budget, rank_set=tuple(ranks))
    reqs = [Request(id=i, arrival_time=0.0, input_len=a, output_len=o)
            for i, (a, o) in enumerate(inputs)]
    routing = {r.id: route_request(st, r) for r in reqs}
    steps = []
    for it in range(skip + n_iter):
        b = build_prefill_batch(st)
        dec = [(r.id, r.input_len + r.tokens_decoded - 1) for r in reqs
               if r.tokens_prefilled == r.input_len and 1 <= r.tokens_decoded < r.output_len]
        if it >= skip:
            steps.append(StepBatch(prefill=list(b.entries), decode=dec))
        for rid, _, n in b.entries:
            reqs[rid].tokens_prefilled += n
        for rid, _ in dec:
            reqs[rid].tokens_decoded += 1
            st.note_decode_token(reqs[rid], routing[rid])
        for r in reqs:
            if r.tokens_prefilled == r.input_len and r.tokens_decoded == 0:
                r.tokens_decoded = 1
    caps = [a + o - 1 for a, o in inputs]
    return routing, steps, caps


def mixed_trace(skip=24, n_iter=3, budget=2048, fail=7):
    """BASELINE config 5: Llama-3-70B-shaped mixed prefill/decode iterations
    of a ShareGPT-shaped trace with two 32k prompts, load-aware routing and
    Alg. 1 chunked prefill on the 7 survivors of hybrid(8) after losing GPU
    ``fail`` (on-demand target).  Every rank timed on this GPU."""
    import torch
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    from paper_2511_14116_b200.serving import HybridServingRank
    model = llama70b()
    plan = make_placement("hybrid", model, range(8))
    alive = [g for g in range(8) if g != fail]
    plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
    owner = owner_array(plan, model.num_kv_heads)
    shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
    inputs = sharegpt_trace()
    routing, steps, caps = mixed_iterations(inputs, alive, budget, skip, n_iter)
    max_tokens = max(s.num_tokens for s in steps)
    per_rank = []
    for g in alive:
        eng = HybridServingRank(model, owner, g, routing, caps, max_tokens, seed=0,
                                shard_owner=shards)
        eng.fill_random_kv(100 + g)
        t0 = time.perf_counter()
        plans = [eng.plan(s) for s in steps]
        plan_ms = (time.perf_counter() - t0) * 1e3 / len(plans)
        xs = [torch.randn((s.num_tokens, model.hidden_dim), device="cuda").to(torch.bfloat16)
              for s in steps]
        eng.serve(plans[0], xs[0])  # warm-up (cuBLAS heuristics, attributes)
        torch.cuda.synchronize()
        times = []
        for p, x in zip(plans, xs):
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            eng.serve(p, x)
            e_.record()
            torch.cuda.synchronize()
            times.append(s_.elapsed_time(e_))
        pipe = None
        if g == alive[0]:
            # wall clock per iteration with the host plan of iteration k+1
            # built while the device runs iteration k, against plan-then-serve
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for s, x in zip(steps, xs):
                eng.serve(eng.plan(s), x)
                torch.cuda.synchronize()
            serial = (time.perf_counter() - t0) * 1e3 / len(steps)
            t0 = time.perf_counter()
            nxt = eng.plan(steps[0])
            for k, x in enumerate(xs):
                cur = nxt
                eng.serve(cur, x)
                if k + 1 < len(steps):
                    nxt = eng.plan(steps[k + 1])
                torch.cuda.synchronize()
            piped = (time.perf_counter() - t0) * 1e3 / len(steps)
            pipe = {"serial_wall_ms": round(serial, 3), "pipelined_wall_ms": round(piped, 3)}
        per_rank.append({"rank": g, "iter_ms": [round(t, 3) for t in times],
                         "host_plan_ms": round(plan_ms, 2),
                         **({"host_overlap": pipe} if pipe else {}),
                         "kv_read_gb": [round(p.kv_read_bytes / 1e9, 3) for p in plans],
                         "prefill_attn_tflop": [round(p.attn_flops / 1e12, 3) for p in plans],
                         "launches": [eng.serve_launches(p) for p in plans]})
        del eng, plans
        torch.cuda.empty_cache()
    it_ms = [max(r["iter_ms"][i] for r in per_rank) for i in range(len(steps))]
    toks = [s.num_tokens for s in steps]
    return {"workload": "C5 Llama-3-70B-shaped mixed prefill/decode iterations (attention + TP "
                        "MLP), ShareGPT-shaped trace (120 requests) + two 32k prompts, "
                        f"load-aware routing + Alg. 1 chunked prefill (budget {budget}) on 7 "
                        f"survivors (hybrid(8), GPU {fail} lost, on-demand target)",
            "emulation": "every rank timed on this one GPU; iteration = max over ranks; NCCL "
                         "exchange excluded (1 GPU)",
            "iterations": [{"prefill_tokens": sum(n for _, _, n in s.prefill),
                            "prefill_chunks": len(s.prefill), "decode_tokens": len(s.decode),
                            "max_rank_ms": round(t, 3)} for s, t in zip(steps, it_ms)],
            "tok_s": round(sum(toks) / (sum(it_ms) / 1e3), 1),
            "ranks": per_rank}


# ------------------------------------------------- cost-model calibration --
def cost_calibration(fstates, mixed, batch=64, ctx=4096, fails=(7, 3, 5), budget=2048):
    """Fit the reference's iteration-time model (costmodel.py) to the
    per-rank times measured above (C3 decode states, C5 mixed iterations):
    SURVEY 8f rank 4.  Reports the B200 constants (seconds per unit), the
    fit's RMS relative error per regime, and the error of the reference's
    own FLOP constants at their default throughput for contrast."""
    from paper_2511_14116_b200.core import load_config
    from paper_2511_14116_b200.costmodel import (BatchWork, ChunkWork, CostParams, PlanCost,
                                                 calibrate)
    from paper_2511_14116_b200.placement import make_placement
    from paper_2511_14116_b200.recovery import plan_weight_recovery
    model, cluster = load_config(os.path.join(ROOT, "paper_2511_14116_b200", "data",
                                              "llama70b.toml"))
    ref = CostParams.from_model(model)
    groups = {"decode": [], "mixed": []}
    plan = make_placement("hybrid", model, range(8))
    alive = list(range(8))
    plans = {8: (plan, list(alive))}
    for f in fails:
        alive = [g for g in alive if g != f]
        plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan("hybrid", model)
        plans[len(alive)] = (plan, list(alive))
    for st in fstates["states"]:
        plan, al = plans[st["world"]]
        routing = route(batch, al, ctx)
        work = BatchWork([ChunkWork.decode(r, routing[r], ctx - 1) for r in range(batch)])
        groups["decode"].append((PlanCost(plan, model, ref, cluster), work,
                                 {r["rank"]: r["step_ms"] / 1e3 for r in st["ranks"]}))
    plan, al = plans[7]
    routing, steps, _ = mixed_iterations(sharegpt_trace(), al, budget, 24, 3)
    for i, stb in enumerate(steps):
        work = BatchWork([ChunkWork.prefill(r, routing[r], s0, n) for r, s0, n in stb.prefill] +
                         [ChunkWork.decode(r, routing[r], pos) for r, pos in stb.decode])
        groups["mixed"].append((PlanCost(plan, model, ref, cluster), work,
                                {r["rank"]: r["iter_ms"][i] / 1e3 for r in mixed["ranks"]}))

    from paper_2511_14116_b200.costmodel import calibrate_b200, rms_error

    def ref_form(params):
        return lambda pc, work: PlanCost(pc.plan, model, params, cluster).per_gpu_compute_time(work)

    dec = groups["decode"]
    train_dec = [s_ for s_, st in zip(dec, fstates["states"]) if st["world"] >= 7]
    test_dec = [s_ for s_, st in zip(dec, fstates["states"]) if st["world"] < 7]
    out = {"model": "reference costmodel.py features (attention per head-token and per "
                    "head-context-token, FFN per token-shard; per-GPU compute time), fitted by "
                    "NNLS on relative error (gpu_throughput = 1, constants in seconds); "
                    "'b200' adds the two terms a B200 decode step has and the FLOP model lacks: "
                    "seconds per resident weight byte and a fixed per-iteration cost",
           "reference_flop_constants_rms_rel_err": {
               "decode": round(rms_error(ref_form(ref), dec), 4),
               "mixed": round(rms_error(ref_form(ref), groups["mixed"]), 4)}}
    for name, train, test in (("decode_8_7_predicts_6_5", train_dec, test_dec),
                              ("decode_predicts_mixed_c5", dec, groups["mixed"]),
                              ("joint_in_sample", dec + groups["mixed"], [])):
        fit3, err3 = calibrate(train)
        fit5, err5 = calibrate_b200(train)
        out[name] = {
            "reference_form": {"attn_s_per_head_token": fit3.attn_flop_per_head_token,
                               "attn_s_per_head_ctx_token": fit3.attn_flop_per_head_ctx_token,
                               "ffn_s_per_token_shard": fit3.ffn_flop_per_token_per_shard,
                               "train_rms_rel_err": round(err3, 4),
                               "heldout_rms_rel_err": round(rms_error(ref_form(fit3), test), 4)
                               if test else None},
            "b200": {"coef": [float(c) for c in fit5.coef],
                     "terms": ["attn_s_per_head_token", "attn_s_per_head_ctx_token",
                               "ffn_s_per_token_shard", "s_per_weight_byte", "fixed_s"],
                     "train_rms_rel_err": round(err5, 4),
                     "heldout_rms_rel_err": round(rms_error(fit5.per_gpu_time, test), 4)
                     if test else None},
            "train_samples": sum(len(m) for _, _, m in train),
            "test_samples": sum(len(m) for _, _, m in test)}
    return out


# ------------------------------------------------------------ CPU oracle --
C2_SHAPE = dict(hidden=4096, kv_heads=8, qpk=4, hd=128, ffn=14336, batch=64, ctx=4096, layers=32)


def cpu_decode_step(layer_samples):
    """The reference's CPU path for the hot path, like for like with the GPU
    step: the float64 oracle restatement of one hybrid decode step
    (oracle/decode_step.py: refexec.py:249-308 decode form -- QKV
    projection, KV append + GQA attention per (request, KV head), output
    projection, gated MLP, residuals) at C2 (B=64, ctx 4096) on every host
    core.  Bounded sample: one full layer is timed ``layer_samples`` times
    (median) and the step is 32 x that (the 32 layers are identical).
    Imports nothing from the product package.  Returns (step_s, info)."""
    from oracle.decode_step import DecodeLayerF64, host_info, time_layers
    c = C2_SHAPE
    t0 = time.perf_counter()
    layer = DecodeLayerF64(c["hidden"], c["kv_heads"], c["qpk"], c["hd"], c["ffn"], c["batch"],
                           c["ctx"])
    setup_s = time.perf_counter() - t0
    per_layer, times, cores = time_layers(layer, layer_samples)
    del layer
    info = host_info()
    info.update({"setup_s": round(setup_s, 1), "layer_s": [round(t, 4) for t in times]})
    return per_layer * c["layers"], info


# ---------------------------------------------------------------- drivers --
def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation of the path
    (the float64 oracle port of refexec.py's decode step; the reference is
    pure Python and cannot travel to the GPU box) on all host cores, rank 0
    only; the other ranks exit without work.  Nothing from the product
    package is imported (no product .so is loaded)."""
    if rank != 0:
        return
    c = C2_SHAPE
    step_s, info = cpu_decode_step(args.warmup + args.steps)
    value = c["batch"] / step_s
    sample = (f"each step = 32 x one float64 C2 decode layer (QKV, KV append + attention, "
              f"O, gated MLP; B=64, ctx 4096), layer timed {args.warmup + args.steps} times "
              f"(median) on {info['cores']} cores")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(world),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": info["cores"],
                             "kind": "port", "sample": sample, "host": info},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(world, batch=64, ctx=4096):
    c = C2_SHAPE
    return {"workload": "C2 Llama-3-8B-shaped hybrid-attention decode step, all 32 layers: "
                        "QKV GEMM, fused KV-append + paged GQA decode, O GEMM, TP MLP "
                        "partial (gate/up GEMM with fused SwiGLU, down GEMM); when N>1 the "
                        "attention and MLP "
                        "partials are exchanged by fs_ar_residual (ordered sum + residual in one "
                        "kernel over IPC-mapped peer buffers; --exchange nccl: NCCL all-reduce)",
            "layers": c["layers"], "q_heads": c["kv_heads"] * c["qpk"],
            "kv_heads": c["kv_heads"], "head_dim": c["hd"], "hidden": c["hidden"],
            "ffn": c["ffn"], "batch": batch, "ctx": ctx, "world": world,
            "placement": "hybrid", "page_tokens": 16, "parallelism": f"hybrid-tp{world}",
            "l2": "no flush: KV working set >> 126 MB L2 (34 GB at N=1)"}


def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    group = dist.group.WORLD if world > 1 else None
    model = llama8b()
    batch, ctx = 64, 4096
    from paper_2511_14116_b200.placement import make_placement, owner_array
    plan = make_placement("hybrid", model, range(world))
    owner = owner_array(plan, model.num_kv_heads)
    routing = route(batch, range(world), ctx)
    eng = build_rank(model, plan, rank, routing, batch, ctx, group, args.kernel_config,
                     mlp=not args.no_mlp)
    peak, peak_src = measured_peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: resident inputs, graph replay, CUDA events ----
    for _ in range(args.warmup):
        eng.step()
    barrier()
    with ClockSampler(local_rank) as clk:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            eng.step()
        e.record()
        barrier()
        ms = s.elapsed_time(e) / args.steps
    ms = max_over_ranks(ms)
    value = batch / (ms / 1e3)

    # ---- e2e: public API, pinned host x in, result back to host ----
    x_host = torch.randn((batch, model.hidden_dim)).to(torch.bfloat16).pin_memory()
    y_host = torch.empty_like(x_host).pin_memory()
    io = os.environ.get("FS_E2E_IO", "graph") == "graph" and eng.group is None
    for _ in range(2):
        if io:
            eng.step_io(x_host, y_host)
        else:
            y_host.copy_(eng.step(x_host))
        torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if io:  # H2D, the step and the D2H of the result: one graph launch
            eng.step_io(x_host, y_host)
        else:
            y_host.copy_(eng.step(x_host))   # H2D inside step(), D2H read of the result
        torch.cuda.current_stream().synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
    nbytes = x_host.numel() * 2

    # ---- roofline: the fused decode launches alone ----
    att = attention_op_graph(eng)
    att_ms = time_graph(att.replay, max(3, args.steps), 3)
    kv_step = step_kv_bytes(eng)
    per_launch_bytes = kv_step / model.num_layers
    per_launch_ms = att_ms / model.num_layers
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    traffic, _ = ncu_traffic() if world == 1 else (None, None)  # capture is of the N=1 config
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "frac_of_nominal_8tbs": round(achieved / 8000.0, 4),
                "kernel": KERNEL_NAMES.get(args.kernel_config, f"config {args.kernel_config}") +
                          " (fs_decode_attention: fused KV append + paged GQA decode + "
                          "in-kernel split merge), one launch per layer",
                "bytes_per_launch": int(per_launch_bytes),
                "launch_ms": round(per_launch_ms, 5), "peak_source": peak_src,
                "step_kv_frac": round(kv_step / (ms / 1e3) / 1e9 / peak, 4),
                "step_bytes": kv_step + eng.weight_bytes(),
                "step_frac": round((kv_step + eng.weight_bytes()) / (ms / 1e3) / 1e9 / peak, 4)}
    del att

    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded random weights and KV)",
            "config": workload_config(world, batch, ctx),
            "e2e": {"value": round(batch / (e2e_ms / 1e3), 1), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "ms_per_step": round(e2e_ms, 4),
                    "api": ("HybridDecodeRank.step_io(x_pinned_host, y_pinned_host): H2D, step, "
                            "D2H in one graph launch" if io else
                            "HybridDecodeRank.step(x_pinned_host) + D2H of x")},
            "roofline": roofline, "clocks": clk.summary(),
            "gpu_launches": eng.launches_per_step() * args.steps}
    del eng
    torch.cuda.empty_cache()

    if world > 1 and args.failures:
        try:
            chain = failure_chain(args, world, rank, local_rank)
            torch.cuda.synchronize()
        except Exception as exc:  # report, never lose the main line
            import traceback
            traceback.print_exc()
            chain = {"error": f"rank {rank}: {type(exc).__name__}: {exc}"}
        if rank == min(r for r in range(world) if str(r) not in args.failures.split(",")):
            line["failure_chain"] = chain
            print(json.dumps(line), flush=True)
        sys.stdout.flush()
        os._exit(0)  # dead peers: skip communicator teardown
    if world == 1 and rank == 0:
        if not args.skip_failure_states:
            line["failure_states"] = failure_states(args.steps, args.warmup, args.kernel_config,
                                                    mlp=not args.no_mlp)
        if not args.skip_mixed:
            line["mixed_trace"] = mixed_trace()
            if "failure_states" in line:
                line["cost_calibration"] = cost_calibration(line["failure_states"],
                                                            line["mixed_trace"])
        if not args.skip_recovery:
            try:
                from paper_2511_14116_b200.recovery_exec import recovery_microbench
                line["recovery"] = recovery_microbench()
            except ImportError:
                pass
        if not args.skip_cpu:
            step_s, info = cpu_decode_step(args.cpu_layers)
            line["cpu_baseline"] = {
                "value": round(batch / step_s, 4), "unit": UNIT, "cores": info["cores"],
                "kind": "port", "host": info,
                "sample": f"32 x one float64 C2 decode layer (oracle/decode_step.py: QKV, KV "
                          f"append + attention, O, gated MLP; B=64, ctx 4096), median of "
                          f"{args.cpu_layers} on {info['cores']} cores"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--kernel-config", type=int, default=0)
    ap.add_argument("--skip-failure-states", action="store_true")
    ap.add_argument("--skip-recovery", action="store_true")
    ap.add_argument("--skip-mixed", action="store_true",
                    help="skip the config-5 mixed prefill/decode trace section")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--gemm", default="tcgen05", choices=("tcgen05", "cublas"))
    ap.add_argument("--exchange", default="fused", choices=("fused", "nccl"),
                    help="N>1 exchange: one fs_ar_residual kernel over IPC-mapped peer "
                         "buffers (default) or an NCCL all-reduce + add")
    ap.add_argument("--no-mlp", action="store_true",
                    help="attention sublayer only (no TP MLP partial / MLP all-reduce)")
    ap.add_argument("--failures", default=None,
                    help="N>1: GPUs lost one after another in the C3 failure chain "
                         "(default 7,3,5 at N=8; '' disables)")
    ap.add_argument("--chain-layers", type=int, default=0,
                    help="testing only (shared GPU): C3 chain with this many layers")
    ap.add_argument("--cpu-layers", type=int, default=3,
                    help="cpu_baseline sample: float64 C2 layers timed (median)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    global GEMM_BACKEND, EXCHANGE
    GEMM_BACKEND = args.gemm
    EXCHANGE = args.exchange
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.failures is None:
        args.failures = "7,3,5" if world == 8 else ""
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            ap.error("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    # FS_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 with the gloo
    # backend, to exercise the multi-rank path on a one-GPU box
    shared = os.environ.get("FS_BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        if not shared and local_rank >= torch.cuda.device_count():
            raise SystemExit(f"bench.py: rank {rank} needs GPU {local_rank} but only "
                             f"{torch.cuda.device_count()} visible (one process per GPU; "
                             f"FS_BENCH_SHARED_GPU=1 runs every rank on cuda:0 for testing)")
        torch.cuda.set_device(local_rank)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
