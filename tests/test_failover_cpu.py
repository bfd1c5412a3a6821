"""Host logic of the failover orchestration (no GPU)."""


def test_route_for_matches_reference_semantics():
    """simulation.py:358-371: a request keeps a surviving rank; an orphan
    goes to argmin (load, rank) where load accumulates the remaining tokens
    of the residents placed so far, in resident order."""
    from paper_2511_14116_b200.core import Request
    from paper_2511_14116_b200.failover import route_for
    reqs = [Request(id=i, arrival_time=0.0, input_len=a, output_len=o)
            for i, (a, o) in enumerate([(10, 5), (20, 5), (30, 5), (5, 1), (7, 2)])]
    reqs[0].tokens_prefilled = 10
    old = {0: 3, 1: 0, 2: 3, 3: 1, 4: 3}
    # r0 -> 0 (all loads 0; cost 5), r1 stays 0 (30), r2 -> 1 (35),
    # r3 stays 1 (41), r4 -> 2
    assert route_for([0, 1, 2, 3, 4], reqs, old, [0, 1, 2]) == {0: 0, 1: 0, 2: 1, 3: 1, 4: 2}
    # nobody orphaned: identity
    assert route_for([1, 3], reqs, old, [0, 1]) == {1: 0, 3: 1}
