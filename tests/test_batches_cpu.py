"""Adaptive chunked-prefill batching (Alg. 1, scheduler.py:160-281) against
golden batches produced by the live reference (tests/golden/batches.json),
the reference's own acceptance scenario (test_acceptance.py:87-117) and the
oracle's literal restatement (oracle/routing.py)."""

import random

import pytest

from oracle.routing import prefill_schedule
from paper_2511_14116_b200.core import Request, ValidationError
from paper_2511_14116_b200.scheduler import (PrefillBatch, SchedulerState, build_prefill_batch,
                                             choose_best_batch, fifo_chunked_prefill,
                                             round_robin_route, route_request)


def _req(i, a, b=1):
    return Request(id=i, arrival_time=0.0, input_len=a, output_len=b)


def test_batches_golden(golden):
    """Every batch (entries, per-rank loads, residual workloads) bit-exact."""
    cases = golden("batches")["cases"]
    n_batches = 0
    for case in cases:
        n = case["n"]
        st = SchedulerState(token_budget=case["budget"], rank_set=tuple(range(n)),
                            kappa=case["kappa"],
                            include_decode_in_workload=case["include_decode"])
        load_aware = case["scheduler"] == "load_aware"
        build = build_prefill_batch if load_aware else fifo_chunked_prefill
        route = route_request if load_aware else round_robin_route
        reqs = []
        for ev in case["events"]:
            if "route" in ev:
                i, a, b = ev["route"]
                reqs.append(_req(i, a, b))
                assert route(st, reqs[-1]) == ev["rank"]
            elif "decode" in ev:
                rid, rank = ev["decode"]
                reqs[rid].tokens_decoded += 1
                st.note_decode_token(reqs[rid], rank)
            else:
                b = build(st)
                n_batches += 1
                assert [list(e) for e in b.entries] == ev["batch"]
                assert [b.per_rank_load[g] for g in range(n)] == ev["per_rank_load"]
                assert [st.workload[g] for g in range(n)] == ev["workload"]
                assert b.num_tokens <= case["budget"]
                for rid, _, length in b.entries:
                    reqs[rid].tokens_prefilled += length
    assert n_batches > 100


def test_skewed_backlog_acceptance():
    """The reference's criterion 4 (test_acceptance.py:87-117, scenario
    data/scenarios/skewed_backlog.json): requests 0..2 pinned one per rank
    (input 4 / 1 / 1), request 3 routed -> rank 1, budget 3."""
    st = SchedulerState(token_budget=3, rank_set=(0, 1, 2))
    for i, (a, g) in enumerate(((4, 0), (1, 1), (1, 2))):
        st.pin_request(_req(i, a), g)
    assert route_request(st, _req(3, 1)) == 1
    golden = [(((0, 0, 1), (1, 0, 1), (2, 0, 1)), [1.0, 1.0, 1.0]),
              (((0, 1, 2), (3, 0, 1)), [2.005859, 1.0, 0.0]),
              ((((0, 3, 1)),), [1.005859, 0.0, 0.0])]
    for entries, loads in golden:
        b = build_prefill_batch(st)
        assert b.entries == entries
        assert [round(b.per_rank_load[g], 6) for g in range(3)] == loads
    assert build_prefill_batch(st).entries == ()
    # FIFO baseline: one request, whole budget (test_acceptance.py:115-117)
    st = SchedulerState(token_budget=3, rank_set=(0, 1, 2))
    for i, (a, g) in enumerate(((4, 0), (1, 1), (1, 2))):
        st.pin_request(_req(i, a), g)
    round_robin_route(st, _req(3, 1))
    b = fifo_chunked_prefill(st)
    assert b.entries == ((0, 0, 3),)
    assert round(b.per_rank_load[0], 6) == 3.005859


def test_matches_oracle_restatement():
    """Heap-based product schedule == the literal per-token argmin scan."""
    rng = random.Random(5)
    for _ in range(200):
        n = rng.randint(1, 8)
        budget = rng.randint(1, 300)
        kappa = rng.choice([1 / 512, 1.0, 0.0])
        st = SchedulerState(token_budget=budget, rank_set=tuple(range(n)), kappa=kappa)
        for i in range(rng.randint(0, 12)):
            st.pin_request(_req(i, rng.randint(1, 200)), rng.randrange(n))
        queues = {r: [list(s) for s in st.schedulable[r].spans] for r in range(n)}
        work = dict(st.workload)
        want, loads = prefill_schedule(queues, budget, kappa, work)
        b = build_prefill_batch(st)
        assert list(b.entries) == want
        assert b.per_rank_load == loads
        assert st.workload == work
        assert {r: [list(s) for s in st.schedulable[r].spans] for r in range(n)} == queues


def test_budget_and_chunk_invariants():
    rng = random.Random(11)
    for _ in range(100):
        budget = rng.randint(1, 64)
        st = SchedulerState(token_budget=budget, rank_set=tuple(range(rng.randint(1, 5))))
        reqs = [_req(i, rng.randint(1, 40)) for i in range(rng.randint(1, 8))]
        for r in reqs:
            route_request(st, r)
        while st.has_prefill_work():
            b = build_prefill_batch(st)
            assert 0 < b.num_tokens <= budget
            assert len({e[0] for e in b.entries}) == len(b.entries)
            for rid, start, length in b.entries:
                assert start == reqs[rid].tokens_prefilled   # contiguous, in order
                reqs[rid].tokens_prefilled += length
        assert all(r.tokens_prefilled == r.input_len for r in reqs)


def test_choose_best_batch():
    a = PrefillBatch(entries=((0, 0, 2),), per_rank_load={0: 2.0, 1: 0.0})
    b = PrefillBatch(entries=((0, 0, 1), (1, 0, 1)), per_rank_load={0: 1.0, 1: 1.0})
    c = PrefillBatch(entries=((0, 0, 1),), per_rank_load={0: 1.0, 1: 0.0})
    assert choose_best_batch([a, b, c]) is b
    assert choose_best_batch([c]) is c
    with pytest.raises(ValidationError):
        choose_best_batch([])
