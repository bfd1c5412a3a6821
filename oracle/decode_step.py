"""Oracle: one float64 decode step of the hybrid-attention forward at a GQA
shape (TEST / BASELINE INFRASTRUCTURE ONLY -- never on the product path).

The decode form of the reference's ``parallel_forward``
(``/root/reference/pkg/src/failsafe/refexec.py:249-308``) on one rank that
owns every head and every FFN shard (N = 1, so the ordered sum over ranks is
the identity):

* per layer, the q/k/v projections of the new token (``refexec.py:88-90``,
  fused here into one matrix ``[q heads | k heads | v heads]``);
* the new token's K/V join the request's cache and every q-head attends its
  KV head's prefix including itself (``_head_attention``'s decode row,
  ``refexec.py:91-101``; GQA grouping ``core.py:71-72``), 1/sqrt(hd) scale,
  max-subtracted softmax;
* the output projection summed into the residual (``refexec.py:298``);
* the FFN over all shards, gated form (the 3-matrix byte accounting of
  ``core.py:93-95``: ``silu(x Wg) * (x Wu) @ Wd``), added to the residual
  (``refexec.py:299-307``).

This is what ``bench.py --impl reference`` and the ``cpu_baseline`` leg time
(numpy float64 on all host cores: BLAS threads for the projections, one
thread per (request, KV head) item for the attention).  It does not import
the product package.
"""

from __future__ import annotations

import os
import platform
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def _silu(x):
    return x / (1.0 + np.exp(-x))


class DecodeLayerF64:
    """Weights and KV cache of ONE layer (float64) at a GQA shape."""

    def __init__(self, hidden, kv_heads, qpk, hd, ffn, batch, ctx, seed=0):
        rng = np.random.default_rng(seed)

        def rand(*shape, scale=1.0):
            return rng.standard_normal(shape, dtype=np.float32).astype(np.float64) * scale

        self.H, self.qpk, self.hd, self.batch, self.ctx = kv_heads, qpk, hd, batch, ctx
        qw = kv_heads * qpk * hd
        self.wqkv = rand(hidden, qw + 2 * kv_heads * hd, scale=hidden ** -0.5)
        self.wo = rand(qw, hidden, scale=0.5 * qw ** -0.5)
        self.wgu = rand(hidden, 2 * ffn, scale=hidden ** -0.5)
        self.wd = rand(ffn, hidden, scale=0.5 * ffn ** -0.5)
        # [head, request, position, dim]; positions < ctx-1 hold the history
        self.k = rand(kv_heads, batch, ctx, hd)
        self.v = rand(kv_heads, batch, ctx, hd)
        self.scale = 1.0 / np.sqrt(hd)

    def step(self, x, pos, pool):
        """x [B, hidden] float64; the new token sits at ``pos`` (attends
        positions 0..pos).  Returns the updated x."""
        H, qpk, hd, B = self.H, self.qpk, self.hd, self.batch
        qw = H * qpk * hd
        qkv = x @ self.wqkv                                   # refexec.py:88-90
        q = qkv[:, :qw].reshape(B, H, qpk, hd)
        self.k[:, :, pos] = qkv[:, qw:qw + H * hd].reshape(B, H, hd).transpose(1, 0, 2)
        self.v[:, :, pos] = qkv[:, qw + H * hd:].reshape(B, H, hd).transpose(1, 0, 2)
        o = np.empty((B, H, qpk, hd))

        def item(idx):                                        # refexec.py:91-101
            r, h = divmod(idx, H)
            k = self.k[h, r, :pos + 1]
            s = (q[r, h] @ k.T) * self.scale
            s -= s.max(axis=1, keepdims=True)
            w = np.exp(s)
            w /= w.sum(axis=1, keepdims=True)
            o[r, h] = w @ self.v[h, r, :pos + 1]

        with _one_blas_thread():  # one worker per item, BLAS single-threaded inside
            list(pool.map(item, range(B * H)))
        x = x + o.reshape(B, qw) @ self.wo                    # refexec.py:298
        hgu = x @ self.wgu
        C = hgu.shape[1] // 2
        return x + (_silu(hgu[:, :C]) * hgu[:, C:]) @ self.wd  # refexec.py:299-307


class MixedIterationF64:
    """Float64 restatement of one serving iteration over all layers
    (TEST INFRASTRUCTURE): the token rows of a mixed batch -- prefill-chunk
    tokens and decode tokens, each a (request, position) pair
    (simulation.py:413-443) -- are projected to q/k/v (refexec.py:88-90),
    every row's K/V joins its request's cache at its position, and every row
    attends its request's positions 0..pos, causal including itself (the
    multi-row ``rows`` mask of ``_head_attention``, refexec.py:91-101), with
    q-head j reading KV head j // qpk (core.py:71-72); then the output
    projection and residual (refexec.py:298) and the gated MLP and residual
    (refexec.py:299-307).  The cache persists across calls, as the
    iterations of a trace do.

    ``layers``: per layer (wqkv [hidden, (H*qpk + 2H)*hd] as [q heads | k
    heads | v heads], wo [H*qpk*hd, hidden], wgu [hidden, 2C] as [gate | up],
    wd [C, hidden]), float64."""

    def __init__(self, H, qpk, hd, layers):
        self.H, self.qpk, self.hd, self.layers = H, qpk, hd, layers
        self.kv = {}  # (layer, head, request) -> {position: (k, v)}

    def step(self, rows, x):
        H, qpk, hd = self.H, self.qpk, self.hd
        qw = H * qpk * hd
        scale = 1.0 / np.sqrt(hd)
        for layer, (wqkv, wo, wgu, wd) in enumerate(self.layers):
            qkv = x @ wqkv
            for t, (r, pos) in enumerate(rows):
                for h in range(H):
                    self.kv.setdefault((layer, h, r), {})[pos] = (
                        qkv[t, qw + h * hd:qw + (h + 1) * hd],
                        qkv[t, qw + (H + h) * hd:qw + (H + h + 1) * hd])
            o = np.zeros((len(rows), qw))
            for t, (r, pos) in enumerate(rows):
                for h in range(H):
                    cache = self.kv[(layer, h, r)]
                    k = np.stack([cache[p][0] for p in range(pos + 1)])
                    v = np.stack([cache[p][1] for p in range(pos + 1)])
                    q = qkv[t, h * qpk * hd:(h + 1) * qpk * hd].reshape(qpk, hd)
                    s = (q @ k.T) * scale
                    s -= s.max(axis=1, keepdims=True)
                    w = np.exp(s)
                    w /= w.sum(axis=1, keepdims=True)
                    o[t, h * qpk * hd:(h + 1) * qpk * hd] = (w @ v).reshape(-1)
            x = x + o @ wo
            hgu = x @ wgu
            C = hgu.shape[1] // 2
            x = x + (_silu(hgu[:, :C]) * hgu[:, C:]) @ wd
        return x


class _one_blas_thread:
    def __enter__(self):
        try:
            from threadpoolctl import threadpool_limits
            self._c = threadpool_limits(1)
        except Exception:  # pragma: no cover
            self._c = None
        return self

    def __exit__(self, *exc):
        if self._c is not None:
            self._c.restore_original_limits()


def host_info():
    """lscpu model, usable cores, BLAS backend / threads."""
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads"),
                 "version": d.get("version")} for d in threadpool_info()
                if d.get("user_api") == "blas"]
    except Exception:
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "blas": blas}


def time_layers(layer: DecodeLayerF64, n: int):
    """Seconds per decode layer (median of ``n`` after one warm-up), with
    all host cores: BLAS threads for the GEMMs, one worker per attention
    item (BLAS limited to 1 thread inside the workers)."""
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(1)
    x = rng.standard_normal((layer.batch, layer.wqkv.shape[0]))
    times = []
    with ThreadPoolExecutor(cores) as pool:
        for i in range(n + 1):
            t0 = time.perf_counter()
            layer.step(x, layer.ctx - 1, pool)
            if i:
                times.append(time.perf_counter() - t0)
    times.sort()
    return times[len(times) // 2], times, cores
