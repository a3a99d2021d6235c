#!/usr/bin/env python
"""Summaries of the ncu evidence for profiles/ (runs here, no GPU needed).

  python scripts/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
  python scripts/summarize_ncu.py full gpurun_out/prof_force.ncu-rep --n 262144 --nloc 262144 \
      > profiles/rNN_force_ncu.txt   (also writes profiles/force_traffic.json with --traffic-out)
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    per = collections.OrderedDict()
    for r in rows:
        name = re.sub(r"\(.*", "", r[4]).replace("nb::<unnamed>::", "")
        t = float(r[14])
        d = per.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += t
    tot = sum(v[1] for v in per.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none, cold-cache, serialised")
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {t / 1e6:10.3f} {t / n / 1e3:10.1f} {t / tot:7.2%}")


WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.per_cycle_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
]


def full(path, n, nloc, flops_per_int, traffic_out, config, n_gpus):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({path})")
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"\n## {d.get('Kernel Name', '?')}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k in WANT:
            if k in d:
                print(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
        stalls = {k: float(v) for k, v in d.items()
                  if re.match(r"smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio$", k)
                  and v not in ("", "n/a")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        print("  top stall reasons (warps per issue-active cycle):")
        for k, v in top:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:6.3f}")
        def num(k, scale=1.0):
            try:
                s = float(d[k].replace(",", ""))
            except Exception:
                return None
            un = u.get(k, "")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
                    "ns": 1e-9, "s": 1.0}.get(un, 1.0)
            return s * mult * scale
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        t = num("gpu__time_duration.sum")
        if n and nloc and t:
            fl = flops_per_int * n * nloc
            print(f"  algorithmic: {flops_per_int} flops x {nloc} i x {n} j = {fl:.4e} flops -> "
                  f"{fl / t / 1e12:.2f} TFLOP/s at ncu's (cold, serialised) duration {t * 1e3:.3f} ms")
        if traffic_out and rd is not None and wr is not None and "force_kernel" in d.get("Kernel Name", ""):
            json.dump({"config": config, "n_gpus": n_gpus, "dram_bytes_per_launch": rd + wr,
                       "dram_read": rd, "dram_write": wr, "source": path}, open(traffic_out, "w"))
            print(f"  traffic (dram read + write) per launch: {rd + wr:.4e} B -> {traffic_out}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nloc", type=int, default=0)
    ap.add_argument("--flops", type=int, default=40)
    ap.add_argument("--traffic-out", default=None)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n-gpus", type=int, default=1)
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.path)
    else:
        full(a.path, a.n, a.nloc, a.flops, a.traffic_out, a.config, a.n_gpus)
