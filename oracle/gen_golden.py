"""Generate golden vectors from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Imports the unmodified reference package ``failsafe`` (read-only at
``/root/reference``) and writes JSON fixtures under ``tests/golden/``.  The
fixtures travel with the repo; ``/root/reference`` never does, so nothing on
the GPU box reads the reference at run time.  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import failsafe  # noqa: E402
from failsafe.core import ClusterSpec, ModelSpec, Request, load_config  # noqa: E402
from failsafe.placement import make_placement, memory_footprint  # noqa: E402
from failsafe.recovery import (BackupState, advance_backup,  # noqa: E402
                               plan_kv_recovery, plan_weight_recovery)
from failsafe.refexec import (ToyLayerWeights, ToyModelWeights,  # noqa: E402
                              _head_attention, _segments, parallel_forward,
                              reference_forward)
from failsafe.scheduler import (SchedulerState, build_prefill_batch,  # noqa: E402
                                fifo_chunked_prefill, round_robin_route, route_request)

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")
DATA = "/root/reference/pkg/src/failsafe/data"


def spec(L, H, qpk=1, hd=8, hidden=32, ffn=2520, shards=None):
    return ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H * qpk, head_dim=hd,
                     hidden_dim=hidden, ffn_intermediate_dim=ffn, ffn_num_shards=shards)


def owner_table(plan, H):
    tab = []
    for a in plan.per_layer:
        row = [None] * H
        for h in range(H):
            o = a.owner_of(h)
            row[h] = -1 if o is None else o
        tab.append(row)
    return tab


def shard_table(ffn):
    return [ffn.owner[s] for s in range(ffn.num_shards)]


def xfer(t):
    return [t.dest_gpu, t.num_bytes, t.medium, t.content, list(t.detail)]


# ---------------------------------------------------------------------------

def gen_placement():
    rng = random.Random(20251114)
    cases = []
    grid = [(4, 8, list(range(8))), (4, 8, list(range(7))), (14, 8, list(range(7))),
            (3, 4, list(range(3))), (80, 8, list(range(8))), (80, 8, list(range(7))),
            (80, 8, list(range(6))), (80, 8, list(range(5))), (32, 8, [0, 1]),
            (32, 8, [0, 1, 2, 3]), (6, 8, [0, 2, 3, 5, 7]), (24, 8, list(range(7)))]
    for _ in range(40):
        H = rng.randint(1, 16)
        n = rng.randint(1, min(H, 9))
        alive = sorted(rng.sample(range(12), n))
        grid.append((rng.randint(1, 12), H, alive))
    for L, H, alive in grid:
        m = spec(L, H, ffn=2520, shards=None)  # 36 shards divide 2520
        for mode in ("naive", "cyclic", "hybrid"):
            plan = make_placement(mode, m, alive, 36)
            cases.append({"mode": mode, "L": L, "H": H, "alive": alive, "num_shards": 36,
                          "owner": owner_table(plan, H), "shard_owner": shard_table(plan.ffn)})
    # on-demand shrink chains, incl. the Llama-70B 8->7->6->5 sequence
    chains = []
    llama, _ = load_config(os.path.join(DATA, "llama70b.toml"))
    for mode, fails in (("hybrid", [7, 3, 5]), ("cyclic", [7, 3, 5]), ("hybrid", [0, 1, 2]),
                        ("naive", [3, 6, 1])):
        plan = make_placement(mode, llama, range(8))
        alive = list(range(8))
        steps = []
        for f in fails:
            alive = [g for g in alive if g != f]
            rp = plan_weight_recovery(llama, plan, alive, "on_demand")
            plan = rp.target_plan(mode, llama)
            pc = rp.pcie_bytes_by_gpu()
            nv = rp.nvlink_bytes_by_gpu()
            steps.append({"fail": f, "owner": owner_table(plan, 8),
                          "shard_owner": shard_table(plan.ffn),
                          "pcie_by_gpu": {str(k): v for k, v in pc.items()},
                          "nvlink_by_gpu": {str(k): v for k, v in nv.items()},
                          "total_pcie": rp.total_pcie_bytes()})
        chains.append({"model": "llama70b", "mode": mode, "steps": steps,
                       "initial": owner_table(make_placement(mode, llama, range(8)), 8),
                       "initial_shards": shard_table(make_placement(mode, llama, range(8)).ffn)})
    # footprints
    fps = []
    for _ in range(30):
        H = rng.randint(1, 10)
        n = rng.randint(1, min(H, 6))
        L = rng.randint(1, 6)
        m = spec(L, H, ffn=2520)
        tokens = {i: rng.randint(0, 500) for i in range(rng.randint(0, 6))}
        routing = {i: rng.randrange(n) for i in tokens}
        for mode in ("naive", "cyclic", "hybrid"):
            plan = make_placement(mode, m, range(n))
            fp = memory_footprint(plan, m, tokens, routing)
            fps.append({"mode": mode, "L": L, "H": H, "n": n, "unit": m.kv_bytes_per_head_token(),
                        "tokens": {str(k): v for k, v in tokens.items()},
                        "routing": {str(k): v for k, v in routing.items()},
                        "footprint": {str(k): v for k, v in fp.items()}})
    # Llama-70B footprint at hybrid 7 (SURVEY a4 figure)
    return {"cases": cases, "chains": chains, "footprints": fps}


def gen_routing():
    rng = random.Random(7)
    cases = []
    for _ in range(60):
        n = rng.randint(1, 8)
        reqs = [(rng.randint(1, 3000), rng.randint(1, 600)) for _ in range(rng.randint(1, 40))]
        include = rng.random() < 0.8
        st = SchedulerState(token_budget=2048, rank_set=tuple(range(n)),
                            include_decode_in_workload=include)
        ranks = []
        for i, (a, b) in enumerate(reqs):
            ranks.append(route_request(st, Request(id=i, arrival_time=0.0, input_len=a,
                                                   output_len=b)))
        cases.append({"n": n, "include_decode": include, "requests": reqs, "ranks": ranks,
                      "workload": [st.workload[r] for r in range(n)]})
    # decode accounting interleaved with routing
    st = SchedulerState(token_budget=64, rank_set=(0, 1, 2))
    reqs = [Request(id=i, arrival_time=0.0, input_len=100 + 37 * i, output_len=20 + i)
            for i in range(9)]
    events = []
    for i, r in enumerate(reqs):
        rank = route_request(st, r)
        events.append(["route", i, rank])
        if i % 2 == 1:
            for rr in reqs[:i]:
                if rr.tokens_decoded < rr.output_len:
                    rr.tokens_decoded += 1
                    st.note_decode_token(rr, rr.dp_rank)
                    events.append(["decode", rr.id, rr.dp_rank])
    interleaved = {"requests": [[r.input_len, r.output_len] for r in reqs], "events": events,
                   "workload": [st.workload[r] for r in range(3)]}
    return {"cases": cases, "interleaved": interleaved}


def gen_batches():
    """Adaptive (Alg. 1) and FIFO chunked-prefill batches: random backlogs
    routed by the load-aware or round-robin router, then batches drained
    until the queues are empty, with arrivals and decode accounting
    interleaved (scheduler.py:139-281)."""
    rng = random.Random(2024)
    cases = []
    for ci in range(80):
        n = rng.randint(1, 8)
        budget = rng.choice([1, 2, 3, 7, 16, 64, 256, 2048])
        max_in = 900 if budget >= 64 else 40
        kappa = rng.choice([1.0 / 512.0, 1.0 / 512.0, 1.0, 0.25])
        sched = "fifo" if ci % 4 == 3 else "load_aware"
        st = SchedulerState(token_budget=budget, rank_set=tuple(range(n)), kappa=kappa,
                            include_decode_in_workload=rng.random() < 0.8)
        reqs, events = [], []
        waves = rng.randint(1, 3)
        for wave in range(waves):
            for _ in range(rng.randint(0 if wave else 1, 10)):
                i = len(reqs)
                r = Request(id=i, arrival_time=0.0, input_len=rng.randint(1, max_in),
                            output_len=rng.randint(1, 50))
                reqs.append(r)
                rank = (route_request if sched == "load_aware" else round_robin_route)(st, r)
                events.append({"route": [i, r.input_len, r.output_len], "rank": rank})
            for _ in range(rng.randint(1, 4)):
                b = (build_prefill_batch if sched == "load_aware" else fifo_chunked_prefill)(st)
                for rid, start, length in b.entries:
                    reqs[rid].tokens_prefilled += length
                events.append({"batch": [list(e) for e in b.entries],
                               "per_rank_load": [b.per_rank_load[g] for g in range(n)],
                               "workload": [st.workload[g] for g in range(n)]})
                # one decode token for finished prefills
                for r in reqs:
                    if r.tokens_prefilled == r.input_len and r.tokens_decoded < r.output_len:
                        r.tokens_decoded += 1
                        st.note_decode_token(r, r.dp_rank)
                        events.append({"decode": [r.id, r.dp_rank]})
        for _ in range(12):  # drain (bounded: keeps the fixture small)
            if not st.has_prefill_work():
                break
            b = (build_prefill_batch if sched == "load_aware" else fifo_chunked_prefill)(st)
            if not b.entries:
                break
            events.append({"batch": [list(e) for e in b.entries],
                           "per_rank_load": [b.per_rank_load[g] for g in range(n)],
                           "workload": [st.workload[g] for g in range(n)]})
        cases.append({"n": n, "budget": budget, "kappa": kappa, "scheduler": sched,
                      "include_decode": st.include_decode_in_workload, "events": events})
    return {"cases": cases}


def gen_prefill():
    """Chunked-prefill rows of ``_head_attention`` (refexec.py:85-103): the
    rows [start, start+n) of each request attend causally (including self)
    to the request's prefix; GQA by tied identity K/V weights, bf16-exact
    inputs (as gen_decode)."""
    rng = np.random.default_rng(777)
    hd = 128
    cases = []
    for qpk, seq_lens, chunks in ((1, [40, 17], [(8, 32), (0, 17)]),
                                  (4, [64, 33, 5], [(16, 20), (1, 31), (0, 5)]),
                                  (8, [90, 24], [(60, 30), (0, 24)]),
                                  (2, [160], [(100, 60)])):
        x = bf16_round(rng.standard_normal((sum(seq_lens), hd)))
        eye = np.eye(hd)
        diags = [np.diag(rng.choice([-2.0, -1.0, -0.5, 0.5, 1.0, 2.0], size=hd))
                 for _ in range(qpk)]
        lw = ToyLayerWeights(wq=np.stack(diags), wk=np.stack([eye] * qpk),
                             wv=np.stack([eye] * qpk), wo=np.stack([eye] * qpk),
                             w_up=np.zeros((2, hd)), w_down=np.zeros((hd, 2)))
        segs = _segments(x.shape[0], seq_lens)
        rows = np.zeros(x.shape[0], dtype=bool)
        for (s, e), (c0, cn) in zip(segs, chunks):
            rows[s + c0:s + c0 + cn] = True
        outs = [_head_attention(lw, h, x, segs, rows=rows) for h in range(qpk)]
        sel = np.flatnonzero(rows)
        cases.append({"qpk": qpk, "seq_lens": seq_lens, "chunks": chunks, "x": x.tolist(),
                      "diag": [np.diag(d).tolist() for d in diags],
                      "out": [[outs[h][t].tolist() for h in range(qpk)] for t in sel]})
    return {"head_dim": hd, "cases": cases}


def gen_metrics():
    """A small live-reference simulation (Llama-70B config, bundled
    mooncake_small trace head, one GPU failure): its JSONL records and
    report.summarize() of them -- the wire format the B200 runs emit."""
    import tempfile
    from failsafe.recovery import load_failure_trace
    from failsafe.report import summarize
    from failsafe.simulation import MetricsLog, run_simulation
    from failsafe.traces import load_request_trace
    model, cluster = load_config(os.path.join(DATA, "llama70b.toml"))
    with open(os.path.join(DATA, "traces", "mooncake_small.csv")) as fh:
        rows = load_request_trace(fh.read())[:24]
    fails = load_failure_trace("ts_s,event,gpu_id\n6.0,fail,7\n")
    log = run_simulation(model, cluster, "hybrid", "load_aware", rows, fails,
                         record_iterations=True, max_time=60.0)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.jsonl")
        log.write_jsonl(path)
        text = open(path).read()
        summ = summarize(MetricsLog.read_jsonl(path))
    return {"jsonl": text, "summary": summ}


def gen_costmodel():
    """iteration_time / per_gpu_compute_time of the live cost model for
    mixed batches on hybrid / cyclic / on-demand plans (costmodel.py)."""
    from failsafe.costmodel import BatchWork, ChunkWork, CostParams, PlanCost
    rng = random.Random(31)
    model, cluster = load_config(os.path.join(DATA, "llama70b.toml"))
    params = CostParams.from_model(model)
    cases = []
    for mode, world, fail in (("hybrid", 8, None), ("hybrid", 8, 7), ("cyclic", 7, None),
                              ("hybrid", 6, None), ("naive", 5, None)):
        plan = make_placement(mode, model, range(world))
        alive = list(range(world))
        if fail is not None:
            alive.remove(fail)
            plan = plan_weight_recovery(model, plan, alive, "on_demand").target_plan(mode, model)
        for _ in range(4):
            chunks = []
            for r in range(rng.randint(1, 40)):
                g = rng.choice(alive)
                if rng.random() < 0.3:
                    chunks.append(["prefill", r, g, rng.randint(0, 5000), rng.randint(1, 512)])
                else:
                    chunks.append(["decode", r, g, rng.randint(1, 8000)])
            work = BatchWork([ChunkWork.prefill(*c[1:]) if c[0] == "prefill"
                              else ChunkWork.decode(*c[1:]) for c in chunks])
            pc = PlanCost(plan, model, params, cluster)
            cases.append({"mode": mode, "world": world, "fail": fail, "chunks": chunks,
                          "iteration_time": pc.iteration_time(work),
                          "per_gpu": {str(g): t for g, t in pc.per_gpu_compute_time(work).items()}})
    p = params
    return {"params": [p.attn_flop_per_head_token, p.attn_flop_per_head_ctx_token,
                       p.ffn_flop_per_token_per_shard, p.gpu_throughput],
            "allreduce": [cluster.allreduce_alpha, cluster.allreduce_beta], "cases": cases}


def toy_model(L, H, shards, qpk=1):
    return ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H * qpk, head_dim=8,
                     hidden_dim=32, ffn_intermediate_dim=96, ffn_num_shards=shards)


def gen_recovery():
    rng = random.Random(99)
    weight = []
    for _ in range(60):
        H = rng.randint(2, 10)
        n = rng.randint(2, min(H, 8))
        L = rng.randint(1, 5)
        shards = rng.choice([d for d in range(n, 25) if 96 % d == 0] or [96])
        m = toy_model(L, H, shards)
        mode = rng.choice(("naive", "cyclic", "hybrid"))
        old = make_placement(mode, m, range(n), shards)
        if rng.random() < 0.15:
            new_alive = list(range(n + 1)) if n + 1 <= H else list(range(n))
        else:
            k = rng.randint(1, min(3, n - 1))
            dead = set(rng.sample(range(n), k))
            new_alive = [g for g in range(n) if g not in dead]
        for wmode in ("on_demand", "naive_reshard"):
            rp = plan_weight_recovery(m, old, new_alive, wmode)
            weight.append({
                "H": H, "L": L, "n": n, "num_shards": shards, "mode": mode, "wmode": wmode,
                "new_alive": new_alive, "owner": owner_table(old, H),
                "shard_owner": shard_table(old.ffn),
                "shard_bytes": m.num_layers * m.ffn_weight_bytes_per_layer() // shards,
                "head_bytes": m.attn_weight_bytes_per_head_layer(),
                "transfers": [xfer(t) for t in rp.transfers],
                "target_owner": [[(-1 if a.owner_of(h) is None else a.owner_of(h))
                                  for h in range(H)] for a in rp.target_heads],
                "target_shards": [rp.target_ffn.owner[s] for s in range(shards)]})
    kv = []
    for _ in range(40):
        H = rng.randint(2, 8)
        n = rng.randint(2, min(H, 6))
        L = rng.randint(1, 6)
        m = toy_model(L, H, 12)
        mode = rng.choice(("naive", "cyclic", "hybrid"))
        old = make_placement(mode, m, range(n), 12)
        dead = rng.randrange(n)
        surv = [g for g in range(n) if g != dead]
        new = plan_weight_recovery(m, old, surv, "on_demand").target_plan(mode, m) \
            if rng.random() < 0.5 else make_placement(mode, m, surv, 12)
        backup = BackupState(host_memory_bytes=10 ** 12, kv_bytes_per_token=m.kv_bytes_per_token())
        contexts, backed = {}, {}
        for req in range(rng.randint(1, 6)):
            produced = rng.randint(0, 60)
            w = rng.randint(0, produced)
            backup.register(req)
            backup.backed[req] = w
            backup.lag[req] = produced - w
            contexts[req] = produced
            backed[req] = w
        old_routing = {r: rng.randrange(n) for r in contexts}
        new_routing = {r: rng.choice(surv) for r in contexts}
        kmode = rng.choice(("recompute", "host_restore"))
        rp = plan_kv_recovery(backup, old, new, m, contexts, old_routing, new_routing, kmode)
        kv.append({"mode": kmode, "H": H, "L": L, "n": n, "surv": surv,
                   "old_owner": owner_table(old, H), "new_owner": owner_table(new, H),
                   "contexts": {str(k): v for k, v in contexts.items()},
                   "backed": {str(k): v for k, v in backed.items()},
                   "old_routing": {str(k): v for k, v in old_routing.items()},
                   "new_routing": {str(k): v for k, v in new_routing.items()},
                   "unit": m.kv_bytes_per_head_token(),
                   "transfers": [xfer(t) for t in rp.transfers],
                   "recompute_tokens": {str(k): v for k, v in rp.recompute_tokens.items()},
                   "recompute_start": {str(k): v for k, v in rp.recompute_start.items()}})
    backup_cases = []
    for case in range(25):
        host = rng.choice([10 ** 9, 5 * 384, 3 * 384, 40 * 384, 200 * 384])
        bk = BackupState(host_memory_bytes=host, kv_bytes_per_token=384)
        cl = ClusterSpec(num_gpus=8, hbm_bytes_per_gpu=10 ** 9,
                         pcie_bw_per_gpu=rng.choice([3840.0, 38400.0, 1e9]),
                         nvlink_bw_per_gpu=1e12, allreduce_alpha=0.0, allreduce_beta=0.0,
                         host_memory_bytes=host)
        frac = rng.choice([0.1, 0.2, 0.5, 1.0])
        steps = []
        for _ in range(rng.randint(3, 15)):
            elapsed = rng.choice([0.0, 0.5, 1.0, 2.0, 4.0, 10.0])
            new = {r: rng.randint(0, 12) for r in rng.sample(range(6), rng.randint(0, 3))}
            finish = [r for r in list(bk.backed) if rng.random() < 0.2]
            for r in finish:
                bk.mark_finished(r)
            advance_backup(bk, elapsed, new, cl, frac)
            steps.append({"elapsed": elapsed, "new": {str(k): v for k, v in new.items()},
                          "finish": finish,
                          "backed": {str(k): v for k, v in bk.backed.items()},
                          "lag": {str(k): v for k, v in bk.lag.items()},
                          "used": bk.host_bytes_used, "carry": bk.carry_bytes,
                          "evictions": list(bk.evictions)})
        backup_cases.append({"host": host, "unit": 384, "pcie": cl.pcie_bw_per_gpu, "frac": frac,
                             "steps": steps})
    return {"weight": weight, "kv": kv, "backup": backup_cases}


def bf16_round(a):
    """Round float64 -> nearest-even bfloat16 value, returned as float64."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def gen_forward():
    """Toy float64 forward outputs from the live reference (for the GPU
    ``parallel_forward`` drop-in and the oracle restatement)."""
    rng = np.random.default_rng(1234)
    cases = []
    for i in range(12):
        H = int(rng.integers(2, 9))
        world = int(rng.integers(1, min(H, 6) + 1))
        L = int(rng.integers(1, 4))
        shards = int(rng.integers(world, 13))
        weights = ToyModelWeights.random(500 + i, num_layers=L, num_heads=H, head_dim=4,
                                         hidden=12, intermediate=shards * 2)
        m = ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H, head_dim=4, hidden_dim=12,
                      ffn_intermediate_dim=shards * 2, ffn_num_shards=shards)
        seq_lens = [int(rng.integers(1, 7)) for _ in range(int(rng.integers(1, 4)))]
        x = rng.standard_normal((sum(seq_lens), 12))
        mode = ("naive", "cyclic", "hybrid")[i % 3]
        plan = make_placement(mode, m, range(world))
        routing = {idx: int(rng.integers(0, world)) for idx in range(len(seq_lens))}
        out = parallel_forward(weights, plan, routing, x, seq_lens)
        ref = reference_forward(weights, x, seq_lens)
        cases.append({
            "mode": mode, "world": world, "H": H, "L": L, "num_shards": shards,
            "seq_lens": seq_lens, "routing": {str(k): v for k, v in routing.items()},
            "x": x.tolist(), "owner": owner_table(plan, H), "shard_owner": shard_table(plan.ffn),
            "layers": [{k: getattr(lw, k).tolist() for k in
                        ("wq", "wk", "wv", "wo", "w_up", "w_down")} for lw in weights.layers],
            "parallel_out": out.tolist(), "reference_out": ref.tolist()})
    return {"cases": cases}


def gen_decode():
    """Decode rows of the reference ``_head_attention`` at head_dim 128 with
    bf16-exact inputs.  hidden == head_dim, wk = wv = wo = I and
    wq[h] = diag(d_h) with power-of-two entries, so q_h = x * d_h, K = V = x
    are exactly what the GPU sees.  The heads of one case share K/V, i.e.
    they form one GQA group (q_per_kv = number of heads)."""
    rng = np.random.default_rng(4242)
    hd = 128
    cases = []
    for qpk, seq_lens in ((1, [1, 17, 40]), (4, [16, 33, 64, 5]), (8, [128, 3, 97]),
                          (4, [300]), (2, [15, 16, 31, 32, 48])):
        x = bf16_round(rng.standard_normal((sum(seq_lens), hd)))
        eye = np.eye(hd)
        diags = [np.diag(rng.choice([-2.0, -1.0, -0.5, 0.5, 1.0, 2.0], size=hd))
                 for _ in range(qpk)]
        lw = ToyLayerWeights(wq=np.stack(diags), wk=np.stack([eye] * qpk),
                             wv=np.stack([eye] * qpk), wo=np.stack([eye] * qpk),
                             w_up=np.zeros((2, hd)), w_down=np.zeros((hd, 2)))
        segs = _segments(x.shape[0], seq_lens)
        rows = np.zeros(x.shape[0], dtype=bool)
        for s, e in segs:
            rows[e - 1] = True
        outs = [_head_attention(lw, h, x, segs, rows=rows) for h in range(qpk)]
        last = [e - 1 for s, e in segs]
        cases.append({"qpk": qpk, "seq_lens": seq_lens, "x": x.tolist(),
                      "diag": [np.diag(d).tolist() for d in diags],
                      "out": [[outs[h][t].tolist() for h in range(qpk)] for t in last]})
    return {"head_dim": hd, "cases": cases}


def gen_reconfig():
    """Reconfiguration decisions of the live reference's serving loop
    (simulation.py:198-397): a Simulation over the bundled mooncake_small
    trace with a fail / fail / recover failure CSV, and a small-HBM cluster
    whose second shrink preempts residents.  For every reconfiguration the
    inputs at ``_reconfigure`` (alive set, plan tables, residents with their
    progress, routing, backup watermarks) and the outcome after
    ``_handle_reconfig_done`` (serving world, target plan, routing, residents
    / waiting order, preempted ids, capacities, reservations, router
    workload) are recorded by wrapping the two methods on the instance (the
    reference code is not modified).  With preemption the reference's run
    stops at its next iteration (KeyError: the preempted request stays in
    the rebuilt router's prefill queue, simulation.py:255-262 vs 458-462);
    the recorded decisions precede that."""
    import dataclasses
    from failsafe.costmodel import CostParams
    from failsafe.recovery import load_failure_trace
    from failsafe.simulation import SimConfig, Simulation
    from failsafe.traces import load_request_trace
    model, cluster = load_config(os.path.join(DATA, "llama70b.toml"))
    with open(os.path.join(DATA, "traces", "mooncake_small.csv")) as fh:
        rows = load_request_trace(fh.read())[:40]
    H = model.num_kv_heads

    def req_state(sim, rid):
        r = sim.requests[rid]
        return [rid, r.arrival_time, r.input_len, r.output_len, r.tokens_prefilled,
                r.tokens_decoded]

    scenarios = []
    for name, hbm, csv in (("expand", 80_000_000_000,
                            "10.0,fail,7\n20.0,fail,3\n35.0,recover,7\n"),
                           ("preempt", 32_000_000_000,
                            "10.0,fail,7\n20.0,fail,3\n35.0,recover,7\n")):
        cl = dataclasses.replace(cluster, hbm_bytes_per_gpu=hbm, switch_latency=0.5)
        fails = load_failure_trace("ts_s,event,gpu_id\n" + csv)
        sim = Simulation(model, cl, CostParams.from_model(model), SimConfig(max_time=60.0),
                         rows, fails)
        events = []
        orig_reconf, orig_done, orig_preempt = (sim._reconfigure, sim._handle_reconfig_done,
                                                sim._preempt)
        preempted = []

        def reconf():
            if sim.plan is None or sim._desired_serving() is None:
                return orig_reconf()
            ev = {"t": sim.now, "alive": sorted(sim.alive), "serving": list(sim.serving),
                  "owner": owner_table(sim.plan, H), "shards": shard_table(sim.plan.ffn),
                  "plan_mode": sim.plan.mode,
                  "residents": [req_state(sim, rid) for rid in sim.residents],
                  "routing": [[rid, sim.routing[rid]] for rid in sim.residents],
                  "backed": [[rid, sim.backup.backed.get(rid, 0)] for rid in sim.residents]}
            gen0 = sim.reconf_gen
            orig_reconf()
            if sim.reconf_gen == gen0:
                return
            payload = [e[3] for e in sim.heap if e[3][0] == "reconfig_done"
                       and e[3][1] == sim.reconf_gen][0]
            _, _, desired, new_plan, new_routing, merged = payload
            ev["desired"] = list(desired)
            ev["new_owner"] = owner_table(new_plan, H)
            ev["new_shards"] = shard_table(new_plan.ffn)
            ev["new_routing"] = sorted([rid, g] for rid, g in new_routing.items())
            ev["recompute"] = sorted([rid, n] for rid, n in merged.recompute_tokens.items())
            ev["pcie_bytes"] = merged.total_pcie_bytes()
            ev["gen"] = sim.reconf_gen
            events.append(ev)

        def done(payload):
            preempted.clear()
            orig_done(payload)
            if payload[1] != sim.reconf_gen or not events or events[-1]["gen"] != payload[1]:
                return
            ev = events[-1]
            ev["after"] = {
                "serving": list(sim.serving),
                "routing": sorted([rid, g] for rid, g in sim.routing.items()),
                "residents": list(sim.residents), "waiting": list(sim.waiting),
                "preempted": list(preempted),
                "capacity": sorted([g, v] for g, v in sim.capacity.items()),
                "reserved": sorted([g, v] for g, v in sim.reserved.items()),
                "workload": sorted([g, v] for g, v in sim.sched.workload.items()),
                "waiting_state": [req_state(sim, rid) for rid in sim.waiting]}

        def preempt(rid):
            preempted.append(rid)
            orig_preempt(rid)

        sim._reconfigure, sim._handle_reconfig_done, sim._preempt = reconf, done, preempt
        try:
            sim.run()
            stopped = None
        except KeyError as exc:
            stopped = f"KeyError {exc} at t={sim.now}"
        scenarios.append({"name": name, "hbm_bytes_per_gpu": hbm, "failures": csv,
                          "switch_latency": 0.5, "events": events, "reference_stopped": stopped})
    return {"scenarios": scenarios, "model": "llama70b.toml",
            "trace": "mooncake_small.csv[:40]"}


def main():
    os.makedirs(OUT, exist_ok=True)
    gens = (("placement", gen_placement), ("routing", gen_routing),
            ("recovery", gen_recovery), ("forward", gen_forward), ("decode", gen_decode),
            ("batches", gen_batches), ("prefill", gen_prefill), ("metrics", gen_metrics),
            ("costmodel", gen_costmodel), ("reconfig", gen_reconfig))
    only = sys.argv[1:]
    for name, fn in gens:
        if only and name not in only:
            continue
        data = fn()
        data["_generated_by"] = ("oracle/gen_golden.py from the live reference "
                                 f"failsafe {getattr(failsafe, '__version__', '?')}")
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(OUT, f"{name}.json")))


if __name__ == "__main__":
    main()
