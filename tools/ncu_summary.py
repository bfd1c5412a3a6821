"""Summarise the ncu outputs of tools/profile.sh into profiles/ (run here,
after gpurun brought gpurun_out/ back).

    python tools/ncu_summary.py --round 1 [--src gpurun_out]

Writes
  profiles/r{NN}_launch_summary.txt   per-kernel launch counts / time shares
  profiles/r{NN}_launches_bench.csv.gz the raw launch list (ncu --metrics
                                       gpu__time_duration.sum)
  profiles/ncu_decode_summary.json    the --set full capture of decode_kernel
                                       (dram traffic per launch etc.; read by
                                       bench.py for roofline.traffic)
  profiles/r{NN}_decode_full.ncu-rep  the capture itself
"""

import argparse
import collections
import csv
import gzip
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEP_KERNELS = ("decode", "nvjet", "gemm", "cutlass", "bfloat16_copy", "plan_pages", "swiglu")


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0}.get(r[ui], 1.0)
        c, t = tot.get(r[ki], (0, 0.0))
        tot[r[ki]] = (c + 1, t + v)
    return tot


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--bytes-per-launch", type=float, default=32 * 8 * 64 * 4096 * 512 / 32,
                    help="algorithmic KV bytes per decode launch of the bench config")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    tag = f"r{a.round:02d}"
    lst = os.path.join(a.src, "launches.csv")
    if os.path.exists(lst):
        tot = launch_table(lst)
        step = {k: v for k, v in tot.items() if any(s in k for s in STEP_KERNELS)}
        all_t = sum(t for _, t in tot.values())
        step_t = sum(t for _, t in step.values())
        lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache,"
                 f" serialised) of: python bench.py --steps 3 --warmup 3 --skip-failure-states"
                 f" --skip-recovery --skip-cpu --skip-mixed", "",
                 "## step kernels (share of the decode-step kernels)",
                 f"{'launches':>8} {'total_us':>12} {'avg_us':>10} {'share':>7}  kernel"]
        for k, (c, t) in sorted(step.items(), key=lambda x: -x[1][1]):
            lines.append(f"{c:8d} {t:12.1f} {t / c:10.2f} {100 * t / step_t:6.1f}%  {k[:110]}")
        lines += ["", "## all kernels incl. setup (random init of weights / KV)",
                  f"{'launches':>8} {'total_us':>12} {'share':>7}  kernel"]
        for k, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
            lines.append(f"{c:8d} {t:12.1f} {100 * t / all_t:6.1f}%  {k[:110]}")
        with open(os.path.join(prof, f"{tag}_launch_summary.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        with open(lst, "rb") as src, gzip.open(os.path.join(prof, f"{tag}_launches_bench.csv.gz"),
                                               "wb") as dst:
            shutil.copyfileobj(src, dst)
    rep = os.path.join(a.src, "decode_full.ncu-rep")
    if os.path.exists(rep):
        m = raw_metrics(rep)

        def num(k, scale=1.0):
            v, u = m[k]
            f = float(v.replace(",", ""))
            mul = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3,
                   "ns": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1.0)
            return f * mul * scale
        dur = num("gpu__time_duration.sum")
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
                  for k, (v, u) in m.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
        tot_st = sum(stalls.values()) or 1.0
        summ = {
            "source": f"profiles/{tag}_decode_full.ncu-rep (ncu --set full --clock-control none"
                      " -k regex:decode -s 40 -c 1, bench.py C2 config)",
            "kernel": m.get("Kernel Name", ("decode_kernel", ""))[0],
            "duration_us": dur * 1e6,
            "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch": rd + wr,
            "algorithmic_bytes_per_launch": a.bytes_per_launch,
            "traffic_over_algorithmic": (rd + wr) / a.bytes_per_launch,
            "achieved_gbs_under_ncu": a.bytes_per_launch / dur / 1e9,
            "dram_throughput_pct_of_peak": float(
                m["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "registers_per_thread": int(float(m["launch__registers_per_thread"][0])),
            "grid": int(float(m["launch__grid_size"][0])),
            "block": int(float(m["launch__block_size"][0])),
            "tensor_pipe_pct": float(
                m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][0]),
            "sm_active_over_elapsed": num("sm__cycles_active.avg") / num("sm__cycles_elapsed.avg"),
            "stall_share_top": {k: round(v / tot_st, 3) for k, v in
                                sorted(stalls.items(), key=lambda t: -t[1])[:6]},
        }
        with open(os.path.join(prof, "ncu_decode_summary.json"), "w") as fh:
            json.dump(summ, fh, indent=1)
        shutil.copy(rep, os.path.join(prof, f"{tag}_decode_full.ncu-rep"))
        print(json.dumps(summ, indent=1))
    rep = os.path.join(a.src, "prefill_full.ncu-rep")
    if os.path.exists(rep):
        m = raw_metrics(rep)

        def num2(k):
            v, u = m[k]
            f = float(v.replace(",", ""))
            return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "us": 1e-6, "ms": 1e-3,
                        "ns": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1.0)
        dur = num2("gpu__time_duration.sum")
        # tools/prefill_bench.py --cases 1x2048@8192 (q_per_kv 8): 2048 chunk
        # tokens behind an 8192-token prefix, 4*hd FLOP per (q head, key)
        vis = 8192 * 2048 + 2048 * 2049 // 2
        flops = 4 * 128 * 8 * vis
        summ = {
            "source": f"profiles/{tag}_prefill_full.ncu-rep (ncu --set full --clock-control none "
                      "-k regex:prefill_tc -s 3 -c 1, tools/prefill_bench.py --variant 3 --cases "
                      "1x2048@8192)",
            "kernel": m.get("Kernel Name", ("prefill_kernel", ""))[0],
            "duration_us": dur * 1e6,
            "algorithmic_flop": flops,
            "achieved_tflops_under_ncu": flops / dur / 1e12,
            "dram_bytes": num2("dram__bytes_read.sum") + num2("dram__bytes_write.sum"),
            "registers_per_thread": int(float(m["launch__registers_per_thread"][0])),
            "grid": int(float(m["launch__grid_size"][0])),
            "block": int(float(m["launch__block_size"][0])),
            "tensor_pipe_pct": float(
                m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][0]),
            "sm_active_over_elapsed": num2("sm__cycles_active.avg") / num2("sm__cycles_elapsed.avg"),
        }
        with open(os.path.join(prof, "ncu_prefill_summary.json"), "w") as fh:
            json.dump(summ, fh, indent=1)
        shutil.copy(rep, os.path.join(prof, f"{tag}_prefill_full.ncu-rep"))
        print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
