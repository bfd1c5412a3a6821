"""The tuning knobs change timing only: a ragged
two-layer decode step with the MLP, through the captured ``step_io`` graph,
gives the same bits with the K1 / GEMM pre-wait L2 prefetches at their
defaults, off, or deeper.  The knobs are read once per process, so every
setting runs in its own subprocess."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib
import torch
from paper_2511_14116_b200.core import ModelSpec
from paper_2511_14116_b200.hybrid import HybridDecodeRank
from paper_2511_14116_b200.placement import make_placement, owner_array
m = ModelSpec(num_layers=2, num_kv_heads=8, num_q_heads=32, head_dim=128, hidden_dim=4096,
              ffn_intermediate_dim=14336)
plan = make_placement("hybrid", m, [0])
shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
B, ctx = 16, 2048
e = HybridDecodeRank(m, owner_array(plan, 8), 0, {r: 0 for r in range(B)}, B, ctx, seed=4,
                     page_order="shuffled", mlp=True, shard_owner=shards)
e.set_lengths([ctx - 37 * r for r in range(B)])
e.fill_random_kv(5)
e.capture()
x = torch.randn((B, 4096), generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
xh, yh = x.pin_memory(), torch.empty_like(x).pin_memory()
e.step_io(xh, yh)
torch.cuda.synchronize()
print("SHA", hashlib.sha256(yh.view(torch.int16).numpy().tobytes()).hexdigest())
"""


def _run(env_extra):
    env = dict(os.environ)
    for k in ("FS_K1_L2_PREFETCH", "FS_GEMM_L2_PREFETCH"):
        env.pop(k, None)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [ln.split()[1] for ln in out.stdout.splitlines() if ln.startswith("SHA ")][0]


def test_prefetch_knobs_do_not_change_bits():
    ref = _run({})
    for extra in ({"FS_K1_L2_PREFETCH": "0"}, {"FS_GEMM_L2_PREFETCH": "0"},
                  {"FS_K1_L2_PREFETCH": "0", "FS_GEMM_L2_PREFETCH": "0"},
                  {"FS_K1_L2_PREFETCH": "8", "FS_GEMM_L2_PREFETCH": "8"}):
        assert _run(extra) == ref, extra
