"""A GPU failure handled end to end on the emulated world (failover.py):
serve with incremental KV backup, lose a GPU, adopt the on-demand target,
restore the lost GPU's KV from its pinned-host mirror (K6), recompute the
tails past the backup watermark, resume -- and the served outputs keep
matching a world-1 run of the same iterations that never failed.  Restored
pages are checked byte for byte against the lost GPU's pages."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _model():
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=2, num_kv_heads=8, num_q_heads=32, head_dim=128,
                     hidden_dim=512, ffn_intermediate_dim=1024, ffn_num_shards=16)


def _close(got, ref, tol=3e-2):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    assert err.max().item() <= tol * max(1.0, ref.abs().max().item()), err.max().item()
    assert (err.mean() / ref.abs().mean()).item() <= 1e-2


@pytest.mark.parametrize("world,fails", [(4, [3]), (8, [7, 3])])
def test_failover_resumes_with_identical_outputs(world, fails):
    from paper_2511_14116_b200.failover import EmulatedCluster
    model = _model()
    inputs = [(40, 8), (100, 6), (17, 10), (64, 7), (33, 9), (90, 5)]
    cl = EmulatedCluster(model, world, inputs, token_budget=64, seed=5)
    ref = EmulatedCluster(model, 1, inputs, token_budget=64, seed=5)
    gen = torch.Generator().manual_seed(1)

    def run(n):
        for _ in range(n):
            b = cl.next_batch()
            if not b.num_tokens:
                return
            x = torch.randn((b.num_tokens, model.hidden_dim), generator=gen).to(torch.bfloat16)
            _close(cl.step(b, x), ref.step(b, x))

    run(3)
    for g in fails:
        rep = cl.fail(g)
        assert rep.world_after == len(cl.alive)
        assert rep.restored_exact
        assert rep.kv_restore_bytes > 0
        # the lost GPU's slices that were not yet on the host (partial pages)
        # are recomputed, everything else restored
        assert rep.recompute_tokens >= 0
        run(3)
    # every request finishes on the shrunk world
    run(40)
    assert all(r.tokens_decoded == r.output_len for r in cl.requests)
    # the measured run in the reference's metrics wire format
    from paper_2511_14116_b200.metrics import summarize
    log = cl.metrics()
    kinds = [r["kind"] for r in log.records]
    assert kinds.count("request") == len(inputs) and kinds.count("failure") == len(fails)
    assert kinds.count("reconfig_done") == len(fails) and kinds[-1] == "run_summary"
    s = summarize(log)
    assert s["requests_completed"] == len(inputs)
    assert s["prefill_tokens"] == sum(a for a, _ in inputs)
    assert s["decode_tokens"] == sum(o for _, o in inputs)
    assert s["ttft"]["max"] > 0 and s["tbt"]["max"] > 0
