"""The fused exchange (fs_ar_residual over CUDA-IPC-mapped peer buffers) with
real separate processes: two ranks share one B200 here (IPC works within a
device; the kernel is the same one that reads peers over NVLink), the
handles are swapped over gloo.  Checked: x += bf16(ordered sum) exactly,
bit-identical on both ranks, across alternating buffers; and a whole
hybrid decode step with exchange="fused" equals the single-process
emulation of the same partition."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    torch.cuda.set_device(0)
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    return dist


def _exchange_worker(rank, world, port, q, mode=0, n=64 * 512):
    try:
        dist = _init(rank, world, port)
        from paper_2511_14116_b200.collective import FusedExchange
        xc = FusedExchange(dist.group.WORLD, n, "cuda:0")
        xc.mode = mode
        x = torch.randn(n, generator=torch.Generator().manual_seed(7)).to(torch.bfloat16)
        want = x.clone()
        xd = x.cuda()
        for k in range(6):
            parts = [torch.randn(n, generator=torch.Generator().manual_seed(100 * r + k))
                     .to(torch.bfloat16) for r in range(world)]
            xc.partial(k % 2, (n,)).copy_(parts[rank].cuda())
            xc.reduce_residual(k % 2, xd)
            tot = torch.zeros(n)
            for p in parts:
                tot += p.float()
            want = (want.float() + tot.to(torch.bfloat16).float()).to(torch.bfloat16)
        got = xd.cpu()
        ok = torch.equal(got, want)
        allx = [torch.empty_like(got) for _ in range(world)]
        dist.all_gather(allx, got)
        same = all(torch.equal(a, allx[0]) for a in allx)
        xc.close()
        dist.destroy_process_group()
        q.put((rank, ok, same, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, False, repr(e)))


def _run(worker, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=worker, args=(r, world, port, q) + args) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    return sorted(res)


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_ordered_sum(world):
    res = _run(_exchange_worker, world)
    for rank, ok, same, err in res:
        assert err is None, err
        assert ok and same, (rank, ok, same)


@pytest.mark.parametrize("world,mode,n", [(2, 2, 64 * 512), (3, 2, 64 * 512), (3, 1, 64 * 8192),
                                          (3, 2, 64 * 8192), (3, 2, 8 * 1001), (4, 2, 8)])
def test_fused_exchange_two_shot(world, mode, n):
    """The two-shot form (slice sums, then gather) gives the one-shot's exact
    ordered sums, also for slices of unequal length and fewer elements than
    ranks' slices (n = 8: three empty slices)."""
    res = _run(_exchange_worker, world, mode, n)
    for rank, ok, same, err in res:
        assert err is None, err
        assert ok and same, (rank, ok, same)


def _step_worker(rank, world, port, q, gemm="cublas"):
    try:
        dist = _init(rank, world, port)
        from paper_2511_14116_b200.core import ModelSpec
        from paper_2511_14116_b200.hybrid import HybridDecodeRank, emulated_parallel_step
        from paper_2511_14116_b200.placement import make_placement, owner_array
        model = ModelSpec(num_layers=2, num_kv_heads=8, num_q_heads=32, head_dim=128,
                          hidden_dim=512, ffn_intermediate_dim=1024, ffn_num_shards=16)
        plan = make_placement("hybrid", model, range(world))
        owner = owner_array(plan, 8)
        shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
        lens = [40, 7, 64, 19]
        routing = {r: r % world for r in range(len(lens))}

        def engine(g, group, exchange):
            e = HybridDecodeRank(model, owner, g, routing, len(lens), 64, seed=3, group=group,
                                 mlp=True, shard_owner=shards, exchange=exchange, gemm=gemm)
            e.set_lengths(lens)
            e.fill_random_kv(11 + g)
            return e
        x0 = torch.randn((len(lens), 512), generator=torch.Generator().manual_seed(5))
        x0 = x0.to(torch.bfloat16)
        mine = engine(rank, dist.group.WORLD, "fused")
        y = mine.step(x0.cuda()).clone()
        # the same partition emulated in this process (fresh engines, same KV)
        emu = [engine(g, None, "nccl") for g in range(world)]
        ref = emulated_parallel_step(emu, x0.cuda())
        ok = torch.equal(y, ref)
        mine.capture()  # the fused exchange inside a CUDA graph
        for e in emu:
            e.set_lengths(lens)
        y2 = mine.step(x0.cuda()).clone()
        ok2 = torch.equal(y2, ref)
        mine.xchg.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, ok2, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, False, repr(e)))


@pytest.mark.parametrize("gemm", ["cublas", "tcgen05"])
def test_fused_exchange_decode_step_matches_emulation(gemm):
    """Eager and graph-captured 2-rank steps with the fused exchange equal
    the single-process emulation bit for bit, with the cuBLAS projections
    and with the tcgen05 skinny GEMM writing straight into the exchange
    buffers."""
    for rank, ok, ok2, err in _run(_step_worker, 2, gemm):
        assert err is None, err
        assert ok and ok2, (rank, ok, ok2)


def _serve_worker(rank, world, port, q):
    try:
        dist = _init(rank, world, port)
        from paper_2511_14116_b200.core import ModelSpec
        from paper_2511_14116_b200.placement import make_placement, owner_array
        from paper_2511_14116_b200.serving import (HybridServingRank, StepBatch,
                                                   emulated_serving_step)
        model = ModelSpec(num_layers=2, num_kv_heads=8, num_q_heads=64, head_dim=128,
                          hidden_dim=512, ffn_intermediate_dim=1024, ffn_num_shards=16)
        plan = make_placement("hybrid", model, range(world))
        owner = owner_array(plan, 8)
        shards = [plan.ffn.owner[s] for s in range(plan.ffn.num_shards)]
        caps = [80, 40, 120]
        routing = {r: r % world for r in range(3)}
        batch = StepBatch(prefill=[(0, 0, 30), (2, 64, 40)], decode=[(1, 20)])

        def engine(g, group, exchange):
            e = HybridServingRank(model, owner, g, routing, caps, 96, seed=3, group=group,
                                  shard_owner=shards, exchange=exchange)
            e.fill_random_kv(5 + g)
            return e
        x = torch.randn((batch.num_tokens, 512), generator=torch.Generator().manual_seed(9))
        x = x.to(torch.bfloat16).cuda()
        mine = engine(rank, dist.group.WORLD, "fused")
        y = mine.serve(mine.plan(batch), x).clone()
        emu = [engine(g, None, "nccl") for g in range(world)]
        ref = emulated_serving_step(emu, [e.plan(batch) for e in emu], x)
        ok = torch.equal(y, ref)
        mine.xchg.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, True, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, False, repr(e)))


def test_fused_exchange_serving_iteration_matches_emulation():
    """A mixed prefill/decode iteration (K8 + K1) on 2 real ranks with the
    fused exchange == the single-process emulation, bit for bit."""
    for rank, ok, _, err in _run(_serve_worker, 2):
        assert err is None, err
        assert ok, rank
