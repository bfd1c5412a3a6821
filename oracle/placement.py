"""Oracle: KV-head / FFN-shard ownership tables (TEST INFRASTRUCTURE ONLY).

Restates ``/root/reference/pkg/src/failsafe/placement.py`` as plain integer
tables instead of frozen dataclasses:

* ``owner[layer][head]`` -- GPU id owning a partitioned (TP) head, or ``-1``
  when the head is replicated (data-parallel, "DP") on every alive GPU.
* ``shard_owner[shard]`` -- GPU id owning an FFN shard.

The product computes the same tables in native code
(``paper_2511_14116_b200/csrc/planner.cpp``); tests compare the two
bit-exactly and pin this module against golden vectors produced by the live
reference (``tests/golden/placement.json``).
"""

from __future__ import annotations

REPLICATED = -1


def _sorted_alive(alive):
    """Rank order = ascending distinct GPU ids (placement.py:69-73)."""
    ranks = sorted(set(int(g) for g in alive))
    if not ranks:
        raise ValueError("alive GPU set must be nonempty")
    return ranks


def block_sizes(num_heads, n):
    """Contiguous blocks, the ``num_heads % n`` heavy blocks first
    (placement.py:76-84)."""
    q, r = divmod(num_heads, n)
    return [q + (1 if b < r else 0) for b in range(n)]


def owner_table(mode, num_layers, num_heads, alive):
    """Per-layer head -> GPU table for naive / cyclic / hybrid placement.

    naive/cyclic follow ``_block_plan`` (placement.py:117-135): block ``b``
    of the contiguous split lands on rank ``(b + shift) % n`` where shift is
    0 (naive) or the layer index (cyclic).  hybrid follows
    ``hybrid_placement`` (placement.py:148-170): ``H % n`` heads starting at
    ``(layer * rem) % H`` are replicated; the rest, in rotated order, are
    dealt ``H // n`` per rank with the rank rotating by the layer index.
    """
    ranks = _sorted_alive(alive)
    n = len(ranks)
    if n > num_heads:
        raise ValueError("unsupported configuration: more GPUs than KV heads")
    table = []
    if mode in ("naive", "cyclic"):
        sizes = block_sizes(num_heads, n)
        for layer in range(num_layers):
            row = [None] * num_heads
            shift = layer if mode == "cyclic" else 0
            head = 0
            for b, size in enumerate(sizes):
                g = ranks[(b + shift) % n]
                for _ in range(size):
                    row[head] = g
                    head += 1
            table.append(row)
    elif mode == "hybrid":
        base, rem = divmod(num_heads, n)
        for layer in range(num_layers):
            row = [None] * num_heads
            first = (layer * rem) % num_heads
            for j in range(rem):
                row[(first + j) % num_heads] = REPLICATED
            rest = [(first + rem + i) % num_heads for i in range(num_heads - rem)]
            for b in range(n):
                g = ranks[(b + layer) % n]
                for h in rest[b * base:(b + 1) * base]:
                    row[h] = g
            table.append(row)
    else:
        raise ValueError(f"unknown placement mode {mode!r}")
    return table


def shard_owner_table(num_shards, alive):
    """FFN shards in contiguous blocks, sizes differ by <= 1, larger blocks
    on lower ranks (placement.py:94-114)."""
    ranks = _sorted_alive(alive)
    if num_shards < len(ranks):
        raise ValueError("num_shards must be >= world size")
    out = []
    for i, size in enumerate(block_sizes(num_shards, len(ranks))):
        out.extend([ranks[i]] * size)
    return out


def on_demand_target(owner, shard_owner, survivors):
    """Shrink target of on-demand weight recovery.

    Survivors keep their TP heads; heads of departed GPUs join the
    replicated set (recovery.py:405-413).  Lost FFN shards go, in ascending
    shard order, to the survivor with the fewest shards, lowest id on ties
    (recovery.py:323-340).
    """
    surv = set(int(g) for g in survivors)
    new_owner = [[(g if (g == REPLICATED or g in surv) else REPLICATED)
                  for g in row] for row in owner]
    counts = {g: 0 for g in sorted(surv)}
    new_shards = list(shard_owner)
    lost = []
    for s, g in enumerate(shard_owner):
        if g in counts:
            counts[g] += 1
        else:
            lost.append(s)
    for s in lost:
        g = min(counts, key=lambda k: (counts[k], k))
        new_shards[s] = g
        counts[g] += 1
    return new_owner, new_shards


def kv_footprint(owner, alive, tokens, routing, unit):
    """Per-GPU KV bytes (placement.py:206-236): a TP head stores every
    request's tokens on its owner; a replicated head stores a request's
    tokens only on the GPU the request is routed to."""
    ranks = _sorted_alive(alive)
    total = sum(tokens.values())
    routed = {g: 0 for g in ranks}
    has_dp = any(g == REPLICATED for row in owner for g in row)
    if has_dp:
        if routing is None:
            raise ValueError("routing is required for plans with replicated heads")
        for req, t in tokens.items():
            routed[routing[req]] += t
    out = {g: 0 for g in ranks}
    for row in owner:
        n_dp = sum(1 for g in row if g == REPLICATED)
        for g in ranks:
            out[g] += sum(1 for x in row if x == g) * total + n_dp * routed[g]
    return {g: v * unit for g, v in out.items()}
