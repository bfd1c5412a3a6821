"""Oracle: load-aware DP routing (TEST INFRASTRUCTURE ONLY).

Restates the router of ``/root/reference/pkg/src/failsafe/scheduler.py``:

* pending cost of a request = sum over unprocessed prefill tokens i of
  ``1 + kappa*i`` plus (optionally) over undecoded output tokens j of
  ``1 + kappa*(input_len + j)`` (scheduler.py:38-47);
* a request goes to ``argmin (workload[r], r)`` and that rank's workload
  grows by the pending cost (scheduler.py:139-145, 160-164);
* a generated token retires ``1 + kappa*(input_len + decoded - 1)`` from
  its rank, clamped at zero (scheduler.py:147-151).

kappa = 1/512 is dyadic, so every sum is exact in float64 and decisions are
bit-exact with the reference.
"""

from __future__ import annotations

KAPPA = 1.0 / 512.0


def pending_cost(input_len, output_len, prefilled=0, decoded=0, kappa=KAPPA,
                 include_decode=True):
    total = 0.0
    for i in range(prefilled, input_len):
        total += 1.0 + kappa * i
    if include_decode:
        for j in range(decoded, output_len):
            total += 1.0 + kappa * (input_len + j)
    return total


class Router:
    """Minimal restatement of the routing half of ``SchedulerState``."""

    def __init__(self, ranks, kappa=KAPPA, include_decode=True):
        self.ranks = sorted(set(ranks))
        self.kappa = kappa
        self.include_decode = include_decode
        self.load = {r: 0.0 for r in self.ranks}

    def route(self, input_len, output_len, prefilled=0, decoded=0):
        best = self.ranks[0]
        for r in self.ranks[1:]:
            if self.load[r] < self.load[best]:
                best = r
        self.load[best] += pending_cost(input_len, output_len, prefilled, decoded,
                                        self.kappa, self.include_decode)
        return best

    def decode_token(self, rank, input_len, decoded_after):
        if self.include_decode:
            cost = 1.0 + self.kappa * (input_len + decoded_after - 1)
            self.load[rank] = max(0.0, self.load[rank] - cost)


def route_sequence(requests, ranks, kappa=KAPPA, include_decode=True):
    """Route ``[(input_len, output_len), ...]`` in order; returns the rank
    list and the final per-rank workload."""
    r = Router(ranks, kappa, include_decode)
    out = [r.route(i, o) for i, o in requests]
    return out, dict(r.load)


def prefill_schedule(queues, budget, kappa=KAPPA, workload=None):
    """Alg. 1 adaptive chunked prefill, restated literally
    (scheduler.py:189-245): ``queues`` maps rank -> list of
    ``[request, next token, end]`` spans (mutated); each step feeds ONE token
    to ``argmin (load, rank)`` over ranks with queued tokens; a token at
    prompt index i costs ``1 + kappa*i`` (scheduler.py:24-35).  Returns
    (entries, per-rank load) with entries in first-scheduled order;
    ``workload`` (rank -> pending cost) is decremented per token, clamped
    at zero, as the reference does."""
    ranks = sorted(queues)
    loads = {r: 0.0 for r in ranks}
    chunks = {}
    taken = 0
    while taken < budget:
        live = [r for r in ranks if queues[r]]
        if not live:
            break
        r = min(live, key=lambda g: (loads[g], g))
        span = queues[r][0]
        rid, idx = span[0], span[1]
        span[1] += 1
        if span[1] >= span[2]:
            queues[r].pop(0)
        cost = 1.0 + kappa * idx
        loads[r] = loads[r] + cost
        if workload is not None:
            workload[r] = max(0.0, workload[r] - cost)
        if rid in chunks:
            chunks[rid][1] += 1
        else:
            chunks[rid] = [idx, 1]
        taken += 1
    return [(rid, s, n) for rid, (s, n) in chunks.items()], loads
