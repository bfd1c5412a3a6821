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
