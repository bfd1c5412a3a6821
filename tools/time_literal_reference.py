"""Time the LITERAL reference decode path once (build container only: it
imports /root/reference, which does not exist on the GPU box).

refexec._head_attention (refexec.py:85-103) with a last-token ``rows`` mask
is how the reference's parallel_forward evaluates a decode row: it
recomputes q/k/v of the whole segment for every call.  One call = one
(q-head, request) at the C2 shape (hidden 4096, head_dim 128, ctx 4096);
a C2 decode step is 32 layers x 32 q-heads x 64 requests such calls (+ the
FFN, not counted).  Writes profiles/r02_literal_reference_cpu.json.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from failsafe.refexec import ToyLayerWeights, _head_attention  # noqa: E402
from oracle.decode_step import host_info  # noqa: E402

hidden, hd, ctx = 4096, 128, 4096
rng = np.random.default_rng(0)
lw = ToyLayerWeights(wq=rng.standard_normal((1, hd, hidden)) / 64,
                     wk=rng.standard_normal((1, hd, hidden)) / 64,
                     wv=rng.standard_normal((1, hd, hidden)) / 64,
                     wo=rng.standard_normal((1, hidden, hd)) / 64,
                     w_up=np.zeros((1, hidden)), w_down=np.zeros((hidden, 1)))
x = rng.standard_normal((ctx, hidden))
rows = np.zeros(ctx, dtype=bool)
rows[-1] = True
_head_attention(lw, 0, x, [(0, ctx)], rows)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    _head_attention(lw, 0, x, [(0, ctx)], rows)
    ts.append(time.perf_counter() - t0)
per_call = sorted(ts)[1]
calls = 32 * 32 * 64
step_s = per_call * calls
out = {"what": "literal reference refexec._head_attention, one decode row (last-token rows "
               "mask) per call, C2 shape (hidden 4096, hd 128, ctx 4096), float64 numpy",
       "per_call_s": round(per_call, 4), "calls_per_c2_step": calls,
       "step_s_attention_only": round(step_s, 1), "tok_s": round(64 / step_s, 5),
       "host": host_info(), "where": "build container (no GPU), not the GPU box"}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r02_literal_reference_cpu.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
