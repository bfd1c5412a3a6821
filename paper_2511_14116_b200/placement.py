"""Placement planner of the drop-in API, computed by the native planner.

Same public names and return types as the reference ``failsafe.placement``
(``/root/reference/pkg/src/failsafe/placement.py:25-251``).  The head and
shard tables themselves come from ``libfailsafe_b200`` (``fs_plan_placement``,
``fs_plan_ffn``; ``csrc/planner.cpp``) as flat int32 owner tables; this module
only wraps them in the reference's frozen dataclasses.  :func:`owner_array`
goes the other way and is what the device page / work tables are built
from (see :mod:`paper_2511_14116_b200.kvcache`).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Mapping, Optional

import numpy as np

from . import _native as N
from .core import ModelSpec, ValidationError


@dataclass(frozen=True)
class HeadAssignment:
    """Per-layer ownership of KV heads (placement.py:25-40)."""

    layer: int
    tp_heads: dict  # gpu -> frozenset of heads
    dp_heads: frozenset  # replicated on every alive GPU

    def owner_of(self, head: int) -> Optional[int]:
        if head in self.dp_heads:
            return None
        for gpu, heads in self.tp_heads.items():
            if head in heads:
                return gpu
        raise ValidationError(f"head {head} is not assigned in layer {self.layer}")


@dataclass(frozen=True)
class ShardAssignment:
    """FFN shard ownership (placement.py:43-57)."""

    num_shards: int
    owner: dict  # shard -> gpu

    def shards_of(self, gpu: int) -> frozenset:
        return frozenset(s for s, g in self.owner.items() if g == gpu)

    def counts(self) -> dict:
        out: dict = {}
        for g in self.owner.values():
            out[g] = out.get(g, 0) + 1
        return out


@dataclass(frozen=True)
class PlacementPlan:
    mode: str
    world_size: int
    alive: tuple
    per_layer: tuple
    ffn: ShardAssignment


def _ranks(alive: Iterable[int]) -> list:
    ranks = sorted(set(int(g) for g in alive))
    if not ranks:
        raise ValidationError("alive GPU set must be nonempty")
    return ranks


def _assignments(table: np.ndarray, ranks) -> tuple:
    out = []
    for layer, row in enumerate(table):
        tp = {g: frozenset(int(h) for h in np.flatnonzero(row == g)) for g in ranks}
        dp = frozenset(int(h) for h in np.flatnonzero(row == N.REPLICATED))
        out.append(HeadAssignment(layer=layer, tp_heads=tp, dp_heads=dp))
    return tuple(out)


def native_owner_table(mode: str, num_layers: int, num_heads: int, alive) -> np.ndarray:
    """int32 [L, H] owner table from the native planner (-1 = replicated)."""
    if mode not in N.MODES:
        raise ValidationError(f"unknown placement mode {mode!r}")
    arr, n = N.i32_array(_ranks(alive))
    out = (N.C.c_int32 * (num_layers * num_heads))()
    N.check(N.lib.fs_plan_placement(N.MODES[mode], num_layers, num_heads, arr, n, out),
            "placement")
    return np.frombuffer(out, dtype=np.int32).reshape(num_layers, num_heads).copy()


def ffn_assignment(model: ModelSpec, alive: Iterable[int],
                   num_shards: Optional[int] = None) -> ShardAssignment:
    ranks = _ranks(alive)
    if num_shards is None:
        num_shards = model.default_num_shards()
    if num_shards < len(ranks):
        raise ValidationError(f"num_shards ({num_shards}) must be >= world size ({len(ranks)})")
    if model.ffn_intermediate_dim % num_shards:
        raise ValidationError(f"num_shards ({num_shards}) must divide ffn_intermediate_dim "
                              f"({model.ffn_intermediate_dim}) evenly")
    arr, n = N.i32_array(ranks)
    out = (N.C.c_int32 * num_shards)()
    N.check(N.lib.fs_plan_ffn(num_shards, arr, n, out), "ffn_assignment")
    return ShardAssignment(num_shards=num_shards, owner={s: int(out[s]) for s in range(num_shards)})


def _plan(mode: str, model: ModelSpec, alive, num_shards) -> PlacementPlan:
    ranks = _ranks(alive)
    if len(ranks) > model.num_kv_heads:
        raise ValidationError(f"unsupported configuration: {len(ranks)} GPUs exceed "
                              f"{model.num_kv_heads} KV heads (cannot give each GPU a head)")
    table = native_owner_table(mode, model.num_layers, model.num_kv_heads, ranks)
    return PlacementPlan(mode=mode, world_size=len(ranks), alive=tuple(ranks),
                         per_layer=_assignments(table, ranks),
                         ffn=ffn_assignment(model, ranks, num_shards))


def naive_placement(model, alive, num_shards=None) -> PlacementPlan:
    return _plan("naive", model, alive, num_shards)


def cyclic_placement(model, alive, num_shards=None) -> PlacementPlan:
    return _plan("cyclic", model, alive, num_shards)


def hybrid_placement(model, alive, num_shards=None) -> PlacementPlan:
    return _plan("hybrid", model, alive, num_shards)


def make_placement(mode: str, model: ModelSpec, alive: Iterable[int],
                   num_shards: Optional[int] = None) -> PlacementPlan:
    if mode not in N.MODES:
        raise ValidationError(f"unknown placement mode {mode!r}")
    return _plan(mode, model, alive, num_shards)


def owner_array(plan: PlacementPlan, num_heads: int) -> np.ndarray:
    """int32 [L, H]: owning GPU of each (layer, head), -1 if replicated."""
    t = np.full((len(plan.per_layer), num_heads), -2, dtype=np.int32)
    for layer, a in enumerate(plan.per_layer):
        for g, heads in a.tp_heads.items():
            for h in heads:
                t[layer, h] = g
        for h in a.dp_heads:
            t[layer, h] = N.REPLICATED
    if (t == -2).any():
        raise ValidationError("plan leaves a head unassigned")
    return t


def plan_from_tables(mode: str, owner: np.ndarray, shard_owner, alive) -> PlacementPlan:
    ranks = _ranks(alive)
    shards = [int(x) for x in shard_owner]
    return PlacementPlan(mode=mode, world_size=len(ranks), alive=tuple(ranks),
                         per_layer=_assignments(np.asarray(owner), ranks),
                         ffn=ShardAssignment(num_shards=len(shards),
                                             owner={s: g for s, g in enumerate(shards)}))


# ---------------------------------------------------------------------------
# footprint accounting (placement.py:189-251)
# ---------------------------------------------------------------------------

def head_layer_counts(plan: PlacementPlan) -> dict:
    counts = {g: 0 for g in plan.alive}
    for a in plan.per_layer:
        for g, heads in a.tp_heads.items():
            counts[g] += len(heads)
    return counts


def dp_head_layer_count(plan: PlacementPlan) -> int:
    return sum(len(a.dp_heads) for a in plan.per_layer)


def memory_footprint(plan: PlacementPlan, model: ModelSpec,
                     per_request_tokens: Mapping[int, int],
                     routing: Optional[Mapping[int, int]] = None) -> dict:
    """Per-GPU KV bytes (native ``fs_kv_footprint``); this is also the
    algorithmic byte count of one decode step on each GPU."""
    has_dp = any(a.dp_heads for a in plan.per_layer)
    reqs = list(per_request_tokens)
    route = None
    if has_dp:
        if routing is None:
            raise ValidationError("routing is required for plans with replicated heads")
        for r in reqs:
            if r not in routing:
                raise ValidationError(f"missing routing entry for request {r}")
            if routing[r] not in plan.alive:
                raise ValidationError(f"request {r} routed to GPU {routing[r]} outside the plan")
        route, _ = N.i32_array(routing[r] for r in reqs)
    owner = owner_array(plan, model.num_kv_heads)
    o_arr = owner.ravel().ctypes.data_as(N._i32p)
    alive, n = N.i32_array(plan.alive)
    toks, nr = N.i64_array(per_request_tokens[r] for r in reqs)
    out = (N.C.c_int64 * n)()
    N.check(N.lib.fs_kv_footprint(owner.shape[0], owner.shape[1], o_arr, alive, n, toks,
                                  route, nr, model.kv_bytes_per_head_token(), out),
            "memory_footprint")
    return {g: int(out[i]) for i, g in enumerate(plan.alive)}


def weight_bytes_per_gpu(plan: PlacementPlan, model: ModelSpec) -> dict:
    shard_bytes = model.num_layers * model.ffn_weight_bytes_per_layer() // plan.ffn.num_shards
    head_bytes = model.attn_weight_bytes_per_head_layer()
    counts = plan.ffn.counts()
    hl = head_layer_counts(plan)
    dp = dp_head_layer_count(plan)
    return {g: counts.get(g, 0) * shard_bytes + (hl[g] + dp) * head_bytes for g in plan.alive}
