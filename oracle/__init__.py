"""CPU oracle for the FailSafe hybrid-attention decode hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2511_14116_b200/`` imports
this package; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
there only as the checker (or as the timed CPU baseline), never as the thing
that is measured or shipped.

Each module restates one part of the reference algorithm (FailSafe,
arXiv 2511.14116, ``/root/reference/pkg/src/failsafe``) in a table-oriented
form and cites the reference ``file:line`` it follows:

* :mod:`oracle.placement` -- head/shard ownership tables, footprints
  (``placement.py:76-251``) and the on-demand shrink target
  (``recovery.py:323-427``).
* :mod:`oracle.routing`   -- greedy least-loaded routing (``scheduler.py:21-164``).
* :mod:`oracle.recovery`  -- backup watermarks, weight/KV recovery plans
  (``recovery.py:143-504``).
* :mod:`oracle.attention` -- float64 paged GQA decode and the hybrid
  ``parallel_forward`` reduce structure (``refexec.py:85-308``).

Parity is PINNED: ``oracle/gen_golden.py`` imports the live reference (in the
build container only) and writes ``tests/golden/*.json``; the CPU test-suite
checks every oracle function against those vectors.
"""
