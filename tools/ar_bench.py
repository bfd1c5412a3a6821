"""fs_ar_residual latency per exchange (CUDA events, graph of back-to-back
exchanges alternating the two buffers), one-shot vs two-shot.
Shared-GPU test form (every rank on cuda:0, IPC within one device -- NOT
NVLink numbers):
  FS_BENCH_SHARED_GPU=1 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 \\
      --master-port 29511 tools/ar_bench.py
On a multi-GPU node run it without FS_BENCH_SHARED_GPU (rank r on GPU r)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

shared = os.environ.get("FS_BENCH_SHARED_GPU") == "1"
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
dev = 0 if shared else int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(dev)
if world > 1:
    dist.init_process_group("gloo")
from paper_2511_14116_b200.collective import FusedExchange

out = []
for nbytes in (128 << 10, 512 << 10, 1 << 20):
    n = nbytes // 2
    if world == 1:
        break
    xc = FusedExchange(dist.group.WORLD, n, f"cuda:{dev}")
    x = torch.zeros(n, dtype=torch.bfloat16, device=f"cuda:{dev}")
    for mode in (1, 2):
        for i in range(2):
            xc.partial(i, (n,)).normal_()
        reps = 20
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(2):  # warm
            for k in range(2):
                xc.reduce_residual(k, x, mode)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for k in range(reps):
            xc.reduce_residual(k % 2, x, mode)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / reps
        t = torch.tensor([us])
        allt = [torch.zeros(1) for _ in range(world)]
        dist.all_gather(allt, t)
        if rank == 0:
            out.append({"bytes": nbytes, "mode": "one-shot" if mode == 1 else "two-shot",
                        "us_max_over_ranks": round(max(float(v) for v in allt), 2)})
    xc.close()
if rank == 0:
    print(json.dumps({"world": world, "shared_gpu": shared, "exchanges": out}))
if world > 1:
    dist.destroy_process_group()
