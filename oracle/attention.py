"""Oracle: float64 GQA decode attention and the hybrid reduce structure
(TEST INFRASTRUCTURE ONLY).

Restates the numerical semantics of
``/root/reference/pkg/src/failsafe/refexec.py``:

* :func:`head_decode` -- one decode row of ``_head_attention``
  (refexec.py:85-103): scores over the request's own prefix *including the
  current token*, scaled by ``1/sqrt(head_dim)``, max-subtracted softmax,
  weighted sum of values.  GQA: the ``q_per_kv`` query heads of KV head
  ``j`` are ``j*q_per_kv .. (j+1)*q_per_kv-1`` (core.py:71-72).
* :func:`paged_decode` -- the same over a paged KV pool addressed through a
  block table (the layout the CUDA kernel reads).
* :func:`parallel_forward` / :func:`reference_forward` -- the toy float64
  forward (refexec.py:111-125, 249-308) on owner tables: TP heads computed
  by their owner for all rows, replicated heads only for rows routed to the
  rank, partial sums accumulated in ascending rank order, residual, then the
  FFN partial of each rank's shard columns in ascending rank order.
"""

from __future__ import annotations

import numpy as np

REPLICATED = -1


def head_decode(q, k, v, scale):
    """q: [qpk, hd]; k, v: [len, hd] -> [qpk, hd] (float64)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    s = (q @ k.T) * scale                       # [qpk, len]
    s = s - s.max(axis=1, keepdims=True)
    w = np.exp(s)
    w = w / w.sum(axis=1, keepdims=True)
    return w @ v


def head_prefill(q, k, v, start, scale):
    """Chunked-prefill rows of ``_head_attention`` (refexec.py:85-103):
    q: [n, qpk, hd] for prompt positions start..start+n-1; k, v: [>= start+n,
    hd].  Row t attends to positions 0..start+t (causal, including self).
    Returns [n, qpk, hd] float64."""
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[0]
    out = np.empty(q.shape, dtype=np.float64)
    for t in range(n):
        out[t] = head_decode(q[t], k[:start + t + 1], v[:start + t + 1], scale)
    return out


def paged_decode(q_rows, k_pool, v_pool, block_table, item_seq, item_len,
                 item_qrow, n_out_rows, scale, page_size=16):
    """Paged GQA decode over work items.

    q_rows: [n_q_rows, qpk, hd]; k_pool/v_pool: [num_pages, page_size, hd]
    (dense, unswizzled); block_table: [n_seq, max_pages]; one work item
    attends ``item_len[i]`` tokens of sequence ``item_seq[i]`` with query
    row ``item_qrow[i]`` and writes output row ``item_qrow[i]``.
    Rows without an item stay zero.
    """
    qpk, hd = q_rows.shape[1], q_rows.shape[2]
    out = np.zeros((n_out_rows, qpk, hd), dtype=np.float64)
    for seq, length, row in zip(item_seq, item_len, item_qrow):
        if length <= 0:
            continue
        n_pages = (length + page_size - 1) // page_size
        pages = block_table[seq][:n_pages]
        k = k_pool[pages].reshape(-1, hd)[:length]
        v = v_pool[pages].reshape(-1, hd)[:length]
        out[row] = head_decode(q_rows[row], k, v, scale)
    return out


# ---------------------------------------------------------------------------
# toy float64 forward on owner tables (refexec.py:69-125, 249-308)
# ---------------------------------------------------------------------------

def _silu(x):
    return x / (1.0 + np.exp(-x))


def _segments(n_tokens, seq_lens):
    if seq_lens is None:
        return [(0, n_tokens)]
    out, s = [], 0
    for length in seq_lens:
        out.append((s, s + length))
        s += length
    return out


def bf16_round(a):
    """Round to the nearest-even bfloat16 value (returned as float64): the
    rounding the GPU path applies to q/K/V ("identical inputs")."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def causal_head(lw, head, x, segs, rows=None, qkv_round=None):
    """Causal attention of one (MHA) head restricted to ``rows``;
    ``qkv_round`` optionally rounds the projections (e.g. ``bf16_round``)."""
    q = x @ lw["wq"][head].T
    k = x @ lw["wk"][head].T
    v = x @ lw["wv"][head].T
    if qkv_round is not None:
        q, k, v = qkv_round(q), qkv_round(k), qkv_round(v)
    scale = 1.0 / np.sqrt(lw["wq"].shape[1])
    out = np.zeros_like(x)
    for s, e in segs:
        for t in range(s, e):
            if rows is not None and not rows[t]:
                continue
            attn = head_decode(q[t][None], k[s:t + 1], v[s:t + 1], scale)[0]
            out[t] = lw["wo"][head] @ attn
    return out


def ffn_partial(lw, x, cols):
    return _silu(x @ lw["w_up"][cols].T) @ lw["w_down"][:, cols].T


def reference_forward(layers, x, seq_lens=None):
    x = np.asarray(x, dtype=np.float64)
    segs = _segments(x.shape[0], seq_lens)
    for lw in layers:
        attn = np.zeros_like(x)
        for h in range(lw["wq"].shape[0]):
            attn += causal_head(lw, h, x, segs)
        x = x + attn
        x = x + ffn_partial(lw, x, np.arange(lw["w_up"].shape[0]))
    return x


def parallel_forward(layers, owner, shard_owner, alive, routing, x, seq_lens=None, qkv_round=None):
    """Hybrid forward on owner tables; ``routing`` maps request index ->
    GPU and only matters for replicated heads."""
    x = np.asarray(x, dtype=np.float64)
    segs = _segments(x.shape[0], seq_lens)
    ranks = sorted(alive)
    n_shards = len(shard_owner)
    width = layers[0]["w_up"].shape[0] // n_shards
    rows_of = {}
    for g in ranks:
        rows = np.zeros(x.shape[0], dtype=bool)
        for idx, (s, e) in enumerate(segs):
            if routing is not None and routing.get(idx) == g:
                rows[s:e] = True
        rows_of[g] = rows
    for layer, lw in enumerate(layers):
        row = owner[layer]
        dp = sorted(h for h, o in enumerate(row) if o == REPLICATED)
        attn = np.zeros_like(x)
        for g in ranks:
            for h in sorted(h for h, o in enumerate(row) if o == g):
                attn += causal_head(lw, h, x, segs, qkv_round=qkv_round)
            if dp and rows_of[g].any():
                for h in dp:
                    attn += causal_head(lw, h, x, segs, rows=rows_of[g], qkv_round=qkv_round)
        x = x + attn
        ffn = np.zeros_like(x)
        for g in ranks:
            shards = [s for s, o in enumerate(shard_owner) if o == g]
            cols = np.array([c for s in shards for c in range(s * width, (s + 1) * width)],
                            dtype=np.intp)
            if len(cols):
                ffn += ffn_partial(lw, x, cols)
        x = x + ffn
    return x
