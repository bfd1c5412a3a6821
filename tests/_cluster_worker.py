"""Worker process of tests/test_cluster_gpu.py (one rank of a world whose
processes share cuda:0): serve, lose ranks on schedule, recover in place."""

import json
import os
import sys
from datetime import timedelta

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def tiny_model(L=2, H=8, qpk=4, hidden=256, ffn=1024):
    from paper_2511_14116_b200.core import ModelSpec
    return ModelSpec(num_layers=L, num_kv_heads=H, num_q_heads=H * qpk, head_dim=128,
                     hidden_dim=hidden, ffn_intermediate_dim=ffn)


def kv_history(layer, head, req, n):
    g = torch.Generator().manual_seed(1_000_003 * layer + 10_007 * head + req)
    return (torch.randn((n, 128), generator=g).to(torch.bfloat16),
            torch.randn((n, 128), generator=g).to(torch.bfloat16))


def x0(batch, hidden):
    g = torch.Generator().manual_seed(77)
    return torch.randn((batch, hidden), generator=g).to(torch.bfloat16)


def fill_kv(eng, ctx):
    """History tokens 0..ctx-2 of every item (keyed by layer, head, request)."""
    import numpy as np
    w = eng.work
    seqs, poss, ks, vs = [], [], [], []
    for i in range(w.n_items):
        layer = int(np.searchsorted(w.seg_items, i, side="right") - 1)
        k, v = kv_history(layer, int(w.item_head[i]), int(w.item_req[i]), ctx - 1)
        seqs.append(np.full(ctx - 1, i))
        poss.append(np.arange(ctx - 1))
        ks.append(k)
        vs.append(v)
    if seqs:
        eng.cache.write_tokens(np.concatenate(seqs), np.concatenate(poss),
                               torch.cat(ks).to(eng.device), torch.cat(vs).to(eng.device))


def main(rank, world, port, job, out_dir, steps_before, fails, batch, ctx, reserve):
    torch.cuda.set_device(0)
    from paper_2511_14116_b200.cluster import ClusterRank
    store = torch.distributed.TCPStore("127.0.0.1", port, None, False,
                                       timeout=timedelta(seconds=120))
    model = tiny_model()
    cr = ClusterRank(model, rank, range(world), store, job, batch, ctx, seed=3, mlp=True,
                     reserve_pages=reserve, page_order="shuffled",
                     kv_fill=lambda e: fill_kv(e, ctx))
    cr.eng.x.copy_(x0(batch, model.hidden_dim).to(cr.eng.device))
    cr.eng.capture()
    for _ in range(steps_before):
        cr.step()
    torch.cuda.synchronize()
    torch.save(cr.eng.x.cpu(), os.path.join(out_dir, f"x_pre_r{rank}.pt"))
    for k, f in enumerate(fails):
        cr.mark_backed()
        if rank == f:
            cr.die()
        rep = cr.recover(f)
        torch.cuda.synchronize()
        torch.save(cr.eng.x.cpu(), os.path.join(out_dir, f"x_fail{k}_r{rank}.pt"))
        with open(os.path.join(out_dir, f"rep_fail{k}_r{rank}.json"), "w") as fh:
            json.dump(rep.__dict__, fh)
    cr.ctl.barrier()
    cr.close(unlink=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]), int(a[1]), int(a[2]), a[3], a[4], int(a[5]),
         [int(x) for x in a[6].split(",") if x], int(a[7]), int(a[8]), int(a[9]))
