"""Where the e2e step's extra time goes (C2, N=1): graph replays back to back
(device events), replays with a host sync per step, step_io (H2D + step + D2H
in one graph) with a sync per step, and the sync round trip of an empty
stream.  python tools/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2511_14116_b200.placement import make_placement  # noqa: E402


def main(layers=None):
    import dataclasses
    model = bench.llama8b()
    if layers:
        model = dataclasses.replace(model, num_layers=layers)
    print(f"== {model.num_layers} layers")
    plan = make_placement("hybrid", model, [0])
    eng = bench.build_rank(model, plan, 0, {r: 0 for r in range(64)}, 64, 4096, None, 0)
    steps = 30
    for _ in range(5):
        eng.step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        eng.step()
    e.record()
    torch.cuda.synchronize()
    print(f"back to back (events): {s.elapsed_time(e) / steps:.4f} ms")
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.step()
        torch.cuda.current_stream().synchronize()
    print(f"replay + sync per step: {(time.perf_counter() - t0) * 1e3 / steps:.4f} ms")
    dev = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.step()
        b.record()
        b.synchronize()
        dev.append(a.elapsed_time(b))
    dev.sort()
    print(f"replay + sync per step, device events: median {dev[len(dev) // 2]:.4f} ms, "
          f"min {dev[0]:.4f}")
    t0 = time.perf_counter()
    for _ in range(steps // 2):
        eng.step()
        eng.step()
        torch.cuda.current_stream().synchronize()
    print(f"two replays + sync: {(time.perf_counter() - t0) * 1e3 / (steps // 2 * 2):.4f} ms per step")
    xh = torch.randn((64, model.hidden_dim)).to(torch.bfloat16).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    for _ in range(3):
        eng.step_io(xh, yh)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.step_io(xh, yh)
        torch.cuda.current_stream().synchronize()
    print(f"step_io + sync per step: {(time.perf_counter() - t0) * 1e3 / steps:.4f} ms")
    done = torch.cuda.Event()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.step_io(xh, yh)
        done.record()
        while not done.query():
            pass
    print(f"step_io + spin-wait per step: {(time.perf_counter() - t0) * 1e3 / steps:.4f} ms")
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.step()
        done.record()
        while not done.query():
            pass
    print(f"replay + spin-wait per step: {(time.perf_counter() - t0) * 1e3 / steps:.4f} ms")
    t0 = time.perf_counter()
    for _ in range(steps):
        eng._io[0].replay()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"step_io graph launch CPU cost: {(t1 - t0) * 1e6 / steps:.1f} us")
    t0 = time.perf_counter()
    for _ in range(200):
        torch.cuda.current_stream().synchronize()
    print(f"empty sync: {(time.perf_counter() - t0) * 1e6 / 200:.1f} us")
    ev = torch.cuda.Event(enable_timing=True)
    ev2 = torch.cuda.Event(enable_timing=True)
    ev.record()
    eng.step_io(xh, yh)
    ev2.record()
    torch.cuda.synchronize()
    print(f"step_io device time (events): {ev.elapsed_time(ev2):.4f} ms")


if __name__ == "__main__":
    for n in ([int(a) for a in sys.argv[1:]] or [None]):
        main(n)
        torch.cuda.empty_cache()
