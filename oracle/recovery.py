"""Oracle: KV backup watermarks and recovery plans (TEST INFRASTRUCTURE ONLY).

Restates ``/root/reference/pkg/src/failsafe/recovery.py`` on the integer
tables of :mod:`oracle.placement`:

* :func:`backup_step`     -- ``advance_backup`` (recovery.py:193-247)
* :func:`weight_plan`     -- ``plan_weight_recovery`` (recovery.py:343-427)
* :func:`kv_plan`         -- ``plan_kv_recovery`` (recovery.py:430-504)

Transfers are tuples ``(dest_gpu, num_bytes, medium, content, detail)`` in
the order the reference emits them.
"""

from __future__ import annotations

from . import placement as P


# ---------------------------------------------------------------------------
# backup (recovery.py:143-247)
# ---------------------------------------------------------------------------

def new_backup(host_bytes, bytes_per_token, enabled=True):
    return {"host": host_bytes, "unit": bytes_per_token, "enabled": enabled,
            "backed": {}, "lag": {}, "order": [], "finished": [],
            "used": 0, "carry": 0.0, "evictions": []}


def _register(st, req):
    if req not in st["backed"]:
        st["backed"][req] = 0
        st["lag"][req] = 0
        st["order"].append(req)


def _make_room(st):
    """Evict oldest finished backups until one token fits; returns whether
    anything was evicted (recovery.py:215-229)."""
    unit, host = st["unit"], st["host"]
    evicted = False
    while st["finished"] and st["used"] + unit > host:
        victim = st["finished"].pop(0)
        held = st["backed"].get(victim, 0)
        if held == 0:
            continue
        st["used"] -= held * unit
        st["backed"][victim] = 0
        st["evictions"].append(victim)
        evicted = True
    return evicted


def backup_step(st, elapsed, new_tokens, pcie_bw, fraction):
    """Drain lag oldest-request-first with ``fraction * pcie_bw * elapsed``
    bytes (plus carried budget), then append this iteration's tokens."""
    if not (0.0 < fraction <= 1.0) or elapsed < 0:
        raise ValueError("bad backup arguments")
    if not st["enabled"]:
        return st
    unit, host = st["unit"], st["host"]
    budget = st["carry"] + fraction * pcie_bw * elapsed
    for req in st["order"]:
        remaining = st["lag"].get(req, 0)
        if remaining <= 0:
            continue
        while remaining > 0 and budget >= unit:
            if st["used"] + unit > host:
                if not _make_room(st) and st["used"] + unit > host:
                    budget = 0.0
                    break
            take = min(remaining, int(budget // unit), (host - st["used"]) // unit)
            if take <= 0:
                break
            st["lag"][req] -= take
            st["backed"][req] += take
            st["used"] += take * unit
            budget -= take * unit
            remaining -= take
        if budget < unit:
            break
    st["carry"] = budget if sum(st["lag"].values()) > 0 else 0.0
    for req in sorted(new_tokens):
        _register(st, req)
        st["lag"][req] += new_tokens[req]
    return st


# ---------------------------------------------------------------------------
# weight recovery (recovery.py:343-427)
# ---------------------------------------------------------------------------

def split_bytes(total, parts):
    q, r = divmod(total, parts)
    return [q + (1 if i < r else 0) for i in range(parts)]


def _held_heads(row, g):
    return {h for h, o in enumerate(row) if o == g or o == P.REPLICATED}


def weight_plan(mode, place_mode, owner, shard_owner, old_alive, new_alive,
                shard_bytes, head_bytes):
    """Returns ``(transfers, target_owner, target_shard_owner)``."""
    surv = sorted(set(new_alive))
    old = sorted(set(old_alive))
    if set(surv) == set(old):
        return [], owner, shard_owner
    num_layers, num_heads = len(owner), len(owner[0])
    xfers = []
    if mode == "naive_reshard" or set(surv) - set(old):
        tgt = P.owner_table(place_mode, num_layers, num_heads, surv)
        tgt_shards = P.shard_owner_table(len(shard_owner), surv)
        for g in surv:
            for s, og in enumerate(tgt_shards):
                if og == g and shard_owner[s] != g:
                    xfers.append((g, shard_bytes, "pcie_host", "ffn_shard", (s,)))
        for layer in range(num_layers):
            for g in surv:
                have = _held_heads(owner[layer], g) if g in old else set()
                need = _held_heads(tgt[layer], g)
                for h in sorted(need - have):
                    xfers.append((g, head_bytes, "pcie_host", "attn_head_slice", (layer, h)))
        return xfers, tgt, tgt_shards
    if mode != "on_demand":
        raise ValueError(mode)
    tgt, tgt_shards = P.on_demand_target(owner, shard_owner, surv)
    for s in range(len(shard_owner)):
        if tgt_shards[s] != shard_owner[s]:
            xfers.append((tgt_shards[s], shard_bytes, "pcie_host", "ffn_shard", (s,)))
    slices = split_bytes(head_bytes, len(surv))
    for layer, row in enumerate(owner):
        lost = [h for h, g in enumerate(row) if g != P.REPLICATED and g not in surv]
        for h in lost:
            for i, g in enumerate(surv):
                if slices[i]:
                    xfers.append((g, slices[i], "pcie_host", "attn_head_slice", (layer, h, i)))
                if head_bytes - slices[i]:
                    xfers.append((g, head_bytes - slices[i], "nvlink_peer",
                                  "attn_head_slice", (layer, h, i)))
    return xfers, tgt, tgt_shards


# ---------------------------------------------------------------------------
# KV recovery (recovery.py:430-504)
# ---------------------------------------------------------------------------

def kv_plan(mode, old_owner, new_owner, new_alive, contexts, backed,
            old_routing, new_routing, unit):
    """Returns ``(transfers, recompute_tokens, recompute_start)``.

    A (layer, head, request) slice whose location is unchanged on a survivor
    stays; one that moves between survivors is an NVLink peer move; one
    that lived on a departed GPU is restored from host up to the request's
    backup watermark and the remainder recomputed.
    """
    surv = set(new_alive)
    reqs = sorted(r for r, t in contexts.items() if t > 0)
    lost, moves, restores = set(), {}, {}
    rc_tok, rc_start = {}, {}
    for layer in range(len(old_owner)):
        for h in range(len(old_owner[layer])):
            o_old, o_new = old_owner[layer][h], new_owner[layer][h]
            old_dp, new_dp = o_old == P.REPLICATED, o_new == P.REPLICATED
            if not old_dp and not new_dp and o_old == o_new and o_old in surv:
                continue
            for req in reqs:
                tok = contexts[req]
                src = old_routing.get(req) if old_dp else o_old
                dst = new_routing.get(req) if new_dp else o_new
                if dst is None:
                    raise ValueError("no destination")
                if src == dst and src in surv:
                    continue
                if src in surv:
                    moves[(req, dst)] = moves.get((req, dst), 0) + tok
                elif mode == "recompute":
                    lost.add(req)
                else:
                    saved = min(tok, backed.get(req, 0))
                    if saved:
                        key = (req, dst, layer, h)
                        restores[key] = restores.get(key, 0) + saved
                    if tok > saved:
                        rc_tok[req] = max(rc_tok.get(req, 0), tok - saved)
                        rc_start[req] = saved
    for req in sorted(lost):
        rc_tok[req] = contexts[req]
        rc_start[req] = 0
    xfers = []
    for (req, dst) in sorted(moves):
        if req not in lost:
            xfers.append((dst, moves[(req, dst)] * unit, "nvlink_peer", "kv_slice", (req,)))
    for (req, dst, layer, h) in sorted(restores):
        xfers.append((dst, restores[(req, dst, layer, h)] * unit, "pcie_host",
                      "kv_slice", (req, layer, h)))
    return xfers, rc_tok, rc_start
