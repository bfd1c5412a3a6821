"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/failsafe_b200.h declares, and its host planners are bit-exact with
the oracle / reference golden vectors.  No GPU needed."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "failsafe_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2511_14116_b200 import _native as N
    declared = _declared()
    assert len(declared) >= 15
    assert sorted(N.EXPORTS) == declared
    for name in declared:
        assert hasattr(N.lib, name)
    assert N.lib.fs_abi_version() == 1


def test_library_exports_nothing_undeclared():
    """Every fs_* symbol the .so exports is declared in the header."""
    import shutil
    import subprocess
    from paper_2511_14116_b200 import _native as N
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines()
                       if ln.split() and ln.split()[-1].startswith("fs_")})
    assert exported == _declared()


def test_native_placement_matches_golden(golden):
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.core import ModelSpec
    for c in golden("placement")["cases"]:
        m = ModelSpec(num_layers=c["L"], num_kv_heads=c["H"], num_q_heads=c["H"], head_dim=8,
                      hidden_dim=32, ffn_intermediate_dim=2520)
        plan = make_placement(c["mode"], m, c["alive"], c["num_shards"])
        assert owner_array(plan, c["H"]).tolist() == c["owner"]
        assert [plan.ffn.owner[s] for s in range(c["num_shards"])] == c["shard_owner"]
        assert plan.alive == tuple(sorted(c["alive"]))


def test_native_on_demand_chain(golden):
    from paper_2511_14116_b200 import _native as N
    for chain in golden("placement")["chains"]:
        owner = np.array(chain["initial"], dtype=np.int32)
        shards = np.array(chain["initial_shards"], dtype=np.int32)
        alive = list(range(8))
        for step in chain["steps"]:
            alive = [g for g in alive if g != step["fail"]]
            surv, n = N.i32_array(alive)
            new_o = np.zeros_like(owner)
            new_s = np.zeros_like(shards)
            N.check(N.lib.fs_plan_on_demand(owner.shape[0], owner.shape[1],
                                            owner.ctypes.data_as(N._i32p), len(shards),
                                            shards.ctypes.data_as(N._i32p), surv, n,
                                            new_o.ctypes.data_as(N._i32p),
                                            new_s.ctypes.data_as(N._i32p)))
            assert new_o.tolist() == step["owner"]
            assert new_s.tolist() == step["shard_owner"]
            owner, shards = new_o, new_s


def test_native_footprint_matches_golden(golden):
    from paper_2511_14116_b200.core import ModelSpec
    from paper_2511_14116_b200.placement import make_placement, memory_footprint
    for c in golden("placement")["footprints"]:
        m = ModelSpec(num_layers=c["L"], num_kv_heads=c["H"], num_q_heads=c["H"], head_dim=8,
                      hidden_dim=32, ffn_intermediate_dim=2520)
        plan = make_placement(c["mode"], m, range(c["n"]))
        tokens = {int(k): v for k, v in c["tokens"].items()}
        routing = {int(k): v for k, v in c["routing"].items()}
        fp = memory_footprint(plan, m, tokens, routing)
        assert fp == {int(k): v for k, v in c["footprint"].items()}


def test_errors_map_to_reference_classes():
    from paper_2511_14116_b200 import ValidationError, make_placement
    from paper_2511_14116_b200.core import ModelSpec
    m = ModelSpec(num_layers=2, num_kv_heads=4, num_q_heads=4, head_dim=8, hidden_dim=32,
                  ffn_intermediate_dim=96)
    with pytest.raises(ValidationError, match="unsupported"):
        make_placement("naive", m, range(5))
    with pytest.raises(ValidationError):
        make_placement("bogus", m, range(2))
    with pytest.raises(ValidationError):
        make_placement("hybrid", m, [])


def test_prefill_tile_planner():
    """fs_plan_prefill_tiles (host code, no GPU): every chunk token lies in
    exactly one token tile, each tile's page splits tile its causal range
    [0, ceil((start + last + 1) / 16)) exactly once, slots are unique, and
    tiles come heaviest first."""
    import ctypes as C
    from paper_2511_14116_b200 import _native as N
    rng = np.random.default_rng(0)
    for qpk, variant in ((1, 0), (3, 1), (4, 0), (8, 1), (8, 0), (5, 0), (3, 2)):
        tpt = N.lib.fs_prefill_tokens_per_tile(qpk, variant)
        assert tpt == {0: 256, 1: 64, 2: 128}[variant] // qpk
        starts = rng.integers(0, 5000, size=12).astype(np.int32)
        lens = rng.integers(0, 300, size=12).astype(np.int32)
        for target in (1, 600, 100000):
            cap = 20000
            arr = {k: (C.c_int32 * cap)() for k in ("i", "t", "a", "b", "s", "ci", "ct", "c0", "cn")}
            nt, nc, ns = C.c_int32(), C.c_int32(), C.c_int32()
            P = C.POINTER(C.c_int32)
            rc = N.lib.fs_plan_prefill_tiles(
                12, starts.ctypes.data_as(P), lens.ctypes.data_as(P), qpk, variant, target, cap,
                arr["i"], arr["t"], arr["a"], arr["b"], arr["s"], C.byref(nt), cap, arr["ci"],
                arr["ct"], arr["c0"], arr["cn"], C.byref(nc), C.byref(ns))
            assert rc == 0
            tiles = [tuple(arr[k][j] for k in "itabs") for j in range(nt.value)]
            widths = [b - a for _, _, a, b, _ in tiles]
            assert widths == sorted(widths, reverse=True)
            cover = {}
            for i, t0, a, b, s in tiles:
                cover.setdefault((i, t0), []).append((a, b, s))
            want = {(i, t0) for i in range(12) for t0 in range(0, lens[i], tpt)}
            assert set(cover) == want
            slots = [s for *_, s in tiles if s >= 0]
            assert len(slots) == len(set(slots)) == ns.value
            for (i, t0), parts in cover.items():
                last = min(t0 + tpt, lens[i]) - 1
                pages = (starts[i] + last + 1 + 15) // 16
                parts.sort()
                assert parts[0][0] == 0 and parts[-1][1] == pages
                assert all(p[1] == q[0] for p, q in zip(parts, parts[1:]))
                assert (len(parts) == 1) == (parts[0][2] < 0)
            assert nc.value == sum(1 for p in cover.values() if len(p) > 1)
        # too small an output array is a ValidationError-class status
        one = (C.c_int32 * 1)()
        rc = N.lib.fs_plan_prefill_tiles(12, starts.ctypes.data_as(P), lens.ctypes.data_as(P),
                                         qpk, variant, 1, 1, one, one, one, one, one, C.byref(nt), 1,
                                         one, one, one, one, C.byref(nc), C.byref(ns))
        assert rc == N.FS_EVALIDATION


def test_prefill_tile_planner_makespan():
    """The split size minimises the list-scheduling makespan on target_units
    slots: one slot -> no split at all (every token tile whole); many slots
    -> the minimum 32-page splits; 148 slots on one long chunk -> more tiles
    than slots would idle fewer SMs than one wave of 64 unsplit tiles."""
    from paper_2511_14116_b200.prefill import PrefillTilePlan
    one = PrefillTilePlan([8192], [2048], 8, 1, 3)
    assert one.n_comb == 0 and one.n_tiles == 2048 // 32
    many = PrefillTilePlan([8192], [2048], 8, 100000, 3)
    widths = many.tiles[3] - many.tiles[2]
    assert widths.max() <= 2 * 32 and many.n_comb == 2048 // 32
    sm = PrefillTilePlan([8192], [2048], 8, 148, 3)
    assert sm.n_tiles > 148 and sm.n_comb == 64
    # every variant of the same rows plans the same tiles
    v0 = PrefillTilePlan([8192], [2048], 8, 148, 0)
    assert (v0.tiles == sm.tiles).all()
