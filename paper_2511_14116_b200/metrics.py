"""Metrics wire format of measured runs.

The reference's simulator writes a JSONL log of ``kind``-discriminated
records (``MetricsLog``, simulation.py:84-132; schema pkg/README.md:124-141)
and its report tooling aggregates it (``report.summarize``,
report.py:39-72).  This module restates both, so that the B200 runs
(:class:`~.failover.EmulatedCluster` driven iterations, whose clock is the
MEASURED device time of every iteration and recovery) emit records the
reference's own ``report`` / ``MetricsLog.read_jsonl`` consume unchanged, and
B200 and simulated runs can be compared line for line.
"""

from __future__ import annotations

import json
import math

from .core import SimulationError, ValidationError


def percentile_nearest_rank(samples, q: float) -> float:
    """Nearest-rank percentile: the ceil(q/100 * N)-th smallest sample
    (simulation.py:39-47)."""
    if not 0 < q <= 100:
        raise ValidationError("percentile must be in (0, 100]")
    data = sorted(samples)
    if not data:
        return 0.0
    rank = max(1, math.ceil(q / 100.0 * len(data)))
    return float(data[rank - 1])


class MetricsLog:
    """Append-only event/interval records (simulation.py:84-132)."""

    def __init__(self):
        self.records = []

    def add(self, kind: str, **fields):
        rec = {"kind": kind}
        rec.update(fields)
        self.records.append(rec)

    def of_kind(self, kind: str) -> list:
        return [r for r in self.records if r["kind"] == kind]

    def request_records(self) -> list:
        return self.of_kind("request")

    def ttfts(self) -> list:
        return [r["ttft"] for r in self.request_records() if r.get("ttft") is not None]

    def tbt_samples(self) -> list:
        out = []
        for r in self.request_records():
            out.extend(r.get("tbt", []))
        return out

    def max_tbt_per_request(self) -> list:
        return [r["max_tbt"] for r in self.request_records() if r.get("max_tbt") is not None]

    def summary(self) -> dict:
        rows = self.of_kind("run_summary")
        if not rows:
            raise SimulationError("simulation produced no run summary")
        return rows[-1]

    def write_jsonl(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            for rec in self.records:
                fh.write(json.dumps(rec, sort_keys=True) + "\n")

    @classmethod
    def read_jsonl(cls, path) -> "MetricsLog":
        log = cls()
        with open(path, "r", encoding="utf-8") as fh:
            for line in fh:
                line = line.strip()
                if line:
                    log.records.append(json.loads(line))
        return log


def summarize(log: MetricsLog) -> dict:
    """Latency / throughput summary of one log (report.py:39-72):
    nearest-rank percentiles; max-TBT per request before aggregation."""
    ttfts = log.ttfts()
    tbts = log.tbt_samples()
    max_tbts = log.max_tbt_per_request()
    rows = log.of_kind("run_summary")
    run = rows[-1] if rows else {}

    def stats(samples):
        if not samples:
            return {"mean": 0.0, "median": 0.0, "p90": 0.0, "p99": 0.0, "max": 0.0}
        return {"mean": sum(samples) / len(samples),
                "median": percentile_nearest_rank(samples, 50),
                "p90": percentile_nearest_rank(samples, 90),
                "p99": percentile_nearest_rank(samples, 99),
                "max": max(samples)}

    return {
        "warning_empty": not (ttfts or tbts or run),
        "requests_completed": run.get("completed", 0),
        "prefill_tokens": run.get("prefill_tokens", 0),
        "decode_tokens": run.get("decode_tokens", 0),
        "prefill_throughput": run.get("prefill_throughput", 0.0),
        "decode_throughput": run.get("decode_throughput", 0.0),
        "recomputed_tokens": run.get("recomputed_tokens", 0),
        "ttft": stats(ttfts),
        "tbt": stats(tbts),
        "max_tbt_per_request": stats(max_tbts),
    }


class RunRecorder:
    """Emits the reference's records for a measured serving run: the clock
    advances by each iteration's measured duration (seconds), so ``t``,
    ``ttft`` and ``tbt`` are real B200 times (requests arrive at t=0 here:
    the driver admits the whole window at once)."""

    def __init__(self, requests, world: int, interval: float = 10.0, record_tbt: bool = True):
        self.log = MetricsLog()
        self.requests = requests
        self.now = 0.0
        self.interval = interval
        self.record_tbt = record_tbt
        self.last_token = {}
        self.tbt = {r.id: [] for r in requests}
        self.ttft = {}
        self.busy = {g: 0.0 for g in range(world)}
        self.buckets = {}
        self.prefill_tokens = self.decode_tokens = self.recomputed = 0
        self.completed = 0
        self.preempted = 0
        self.done = set()

    def iteration(self, batch, duration_s: float, per_rank_s=None, finished_prefill=()):
        """Account one executed iteration: ``batch`` (StepBatch) took
        ``duration_s``; ``finished_prefill`` = requests whose prompt
        completed in it (their first output token is emitted now,
        simulation.py:536-549)."""
        self.now += duration_s
        pf = sum(n for _, _, n in batch.prefill)
        dc = len(batch.decode)
        for rid in finished_prefill:
            req = self.requests[rid]
            self.ttft.setdefault(rid, self.now - req.arrival_time)
            self.last_token[rid] = self.now
            dc += 1
        for rid, _ in batch.decode:
            self.tbt[rid].append(self.now - self.last_token.get(rid, self.now - duration_s))
            self.last_token[rid] = self.now
        self.prefill_tokens += pf
        self.decode_tokens += dc
        b = int(self.now // self.interval)
        acc = self.buckets.setdefault(b, [0, 0])
        acc[0] += pf
        acc[1] += dc
        ratio = None
        if per_rank_s:
            for g, t in per_rank_s.items():
                self.busy[g] = self.busy.get(g, 0.0) + t
            vals = list(per_rank_s.values())
            if len(vals) > 1 and min(vals) > 0:
                ratio = max(vals) / min(vals)
        self.log.add("iteration", t=round(self.now, 9), duration=round(duration_s, 9),
                     prefill_tokens=pf, decode_tokens=dc,
                     batch_requests=len(batch.prefill) + len(batch.decode),
                     compute_ratio=round(ratio, 6) if ratio else None)
        for req in self.requests:
            if req.id not in self.done and req.tokens_decoded >= req.output_len \
                    and req.tokens_prefilled >= req.input_len:
                self._finish(req)

    def _finish(self, req):
        self.done.add(req.id)
        self.completed += 1
        samples = self.tbt[req.id]
        rec = {"t": round(self.now, 9), "id": req.id, "arrival": req.arrival_time,
               "input_len": req.input_len, "output_len": req.output_len,
               "ttft": self.ttft.get(req.id), "n_tbt": len(samples),
               "max_tbt": max(samples) if samples else None}
        if self.record_tbt:
            rec["tbt"] = [round(x, 9) for x in samples]
        self.log.add("request", **rec)

    def failure(self, gpu: int, alive: int):
        self.log.add("failure", t=round(self.now, 9), gpu=gpu, alive=alive)

    def recovery(self, gpu: int, alive: int):
        """A GPU rejoined (simulation.py:626-633)."""
        self.log.add("recovery", t=round(self.now, 9), gpu=gpu, alive=alive)

    def preemption(self, rid: int):
        """A resident preempted over KV capacity (simulation.py:283-310)."""
        self.preempted += 1
        self.log.add("preemption", t=round(self.now, 9), request=rid)

    def reconfig(self, world: int, recovery_s: float, recomputed_tokens: int, pcie_bytes: int):
        """A measured reconfiguration: the world stalls for ``recovery_s``."""
        self.log.add("reconfig_start", t=round(self.now, 9), world=world,
                     recovery_latency=recovery_s, recomputed_tokens=recomputed_tokens,
                     pcie_bytes=pcie_bytes)
        self.now += recovery_s
        self.recomputed += recomputed_tokens
        self.log.add("reconfig_done", t=round(self.now, 9), world=world)

    def finish(self, unserved: int = 0) -> MetricsLog:
        end = self.now
        for b in range(max(self.buckets, default=-1) + 1):
            pf, dc = self.buckets.get(b, (0, 0))
            self.log.add("interval", t0=b * self.interval, t1=(b + 1) * self.interval,
                         prefill_tokens=pf, decode_tokens=dc)
        iters = [r["compute_ratio"] for r in self.log.of_kind("iteration")
                 if r["compute_ratio"] is not None]
        self.log.add(
            "run_summary", t=round(end, 9), completed=self.completed, rejected=0,
            preempted=self.preempted,
            prefill_tokens=self.prefill_tokens, decode_tokens=self.decode_tokens,
            recomputed_tokens=self.recomputed,
            prefill_throughput=round(self.prefill_tokens / end, 6) if end > 0 else 0.0,
            decode_throughput=round(self.decode_tokens / end, 6) if end > 0 else 0.0,
            busy_fraction={str(g): round(t / end, 6) if end > 0 else 0.0
                           for g, t in sorted(self.busy.items())},
            compute_ratio_mean=round(sum(iters) / len(iters), 6) if iters else None,
            compute_ratio_max=round(max(iters), 6) if iters else None,
            unserved=unserved)
        return self.log
