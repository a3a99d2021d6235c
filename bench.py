#!/usr/bin/env python
"""Benchmark: pairwise interactions/s (and FP32 TFLOP/s vs peak) of the
direct-summation Hermite step on 1..8 B200s (BASELINE.json metric).

One "step" = one pass of the whole hot path over the whole system:
predict+pack (fp64) -> all-gather of j packets (N > 1) -> force pass
(FP32, all i x all j) -> fold + correct (fp64).  Default workload: config C4
(N = 262144 two-cluster Plummer, log-normal masses, eps = 1e-3, dt = 1/1024),
the largest single-GPU config of BASELINE.json carrying the >= 60 %-of-peak
target (N >= 262144) and run at 1/2/4/8 GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints one JSON line.  `--impl reference` times the fp64 oracle (the
only reference this paper-only run has) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# executed FP32 flops per interaction, FFMA = 2 (R#20; ncu-checked)
FLOPS = {"hermite": 40, "leapfrog": 18, "block": 40}
FP32_LANES_PER_SM = 128      # FP32 FMA lanes per SM (4 SMSP x 32)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C4")
    p.add_argument("--integrator", default="hermite", choices=["hermite", "leapfrog", "block"])
    p.add_argument("--dt-max", type=float, default=1.0 / 128,
                   help="block time steps: largest step dt_max (one bench step = dt_max of time)")
    p.add_argument("--eta", type=float, default=0.02, help="block time steps: Aarseth eta")
    p.add_argument("--hilo", default="auto", choices=["auto", "on", "off"],
                   help="two-float positions (NEXT f2); auto = on for block time steps only")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-flush", action="store_true")
    p.add_argument("--nccl1", action="store_true",
                   help="with one GPU: run the multi-rank code path through a 1-rank NCCL communicator "
                        "(all-gather on the comm stream, local-first + concurrent remote force launches)")
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [s.strip() for s in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


class EnergyMeter:
    """GPU energy over a region from NVML's total-energy counter (mJ), the B200 form
    of the paper's energy-to-solution measurement (NEXT f3); host-package
    energy from RAPL sysfs when the box exposes it."""

    def __init__(self, index):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.h = None
        self.rapl = [os.path.join(r, "energy_uj") for r in
                     sorted(__import__("glob").glob("/sys/class/powercap/intel-rapl:[0-9]*"))
                     if os.path.exists(os.path.join(r, "energy_uj"))]

    def _read(self):
        g = self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) / 1e3 if self.h else None
        c = None
        try:
            c = sum(int(open(f).read()) for f in self.rapl) / 1e6 if self.rapl else None
        except Exception:
            c = None
        return g, c

    def start(self):
        self.t0 = time.perf_counter()
        self.e0 = self._read()

    def stop(self):
        t = time.perf_counter() - self.t0
        e1 = self._read()
        g = (e1[0] - self.e0[0]) if e1[0] is not None and self.e0[0] is not None else None
        if g is not None and (t < 0.25 or g <= 0):   # below the counter's update granularity
            return {"gpu_joules": None, "host_cpu_joules": None, "seconds": t, "gpu_avg_w": None,
                    "note": "region shorter than the NVML energy counter resolution"}
        c = (e1[1] - self.e0[1]) if e1[1] is not None and self.e0[1] is not None else None
        return {"gpu_joules": g, "host_cpu_joules": c, "seconds": t,
                "gpu_avg_w": g / t if g is not None and t > 0 else None}


def cpu_baseline(m, x, v, eps2, budget_s):
    """The fp64 oracle as it stands, timed on the host cores on a bounded
    sample of the same workload: forces on n_s strided i against all N j."""
    import numpy as np
    import oracle
    n = m.shape[0]
    ns = 512
    oracle.forces(m, x, v, eps2, idx=np.arange(64))      # thread-pool start-up
    t0 = time.perf_counter()
    oracle.forces(m, x, v, eps2, idx=np.arange(ns))
    dt = max(time.perf_counter() - t0, 1e-4)
    ns = int(min(n, max(ns, ns * budget_s / dt)))
    idx = np.linspace(0, n - 1, ns).astype(np.int64)
    t0 = time.perf_counter()
    oracle.forces(m, x, v, eps2, idx=idx)
    el = time.perf_counter() - t0
    cores = oracle.threads()
    # the same oracle on one core, on an eighth of the time budget
    n1 = max(16, int(ns * (budget_s / 8) / max(el * cores, 1e-4)))
    idx1 = np.linspace(0, n - 1, min(n, n1)).astype(np.int64)
    oracle.set_threads(1)
    try:
        t0 = time.perf_counter()
        oracle.forces(m, x, v, eps2, idx=idx1)
        el1 = time.perf_counter() - t0
    finally:
        oracle.set_threads(cores)
    return {"value": ns * n / el, "unit": "interactions/s", "cores": cores,
            "kind": "oracle",
            "sample": f"acc+jerk of {ns} evenly strided i against all {n} j (fp64, OpenMP over i); "
                      f"{el:.1f} s",
            "value_1core": len(idx1) * n / el1,
            "sample_1core": f"{len(idx1)} strided i against all {n} j on 1 thread; {el1:.1f} s"}


def run_reference(args):
    """--impl reference: the fp64 oracle, rank 0 only, each step a bounded sample."""
    import numpy as np
    import oracle
    from paper_2509_19294_b200 import inputs
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = inputs.CONFIGS[args.config]
    m, x, v = inputs.make(args.config)
    eps2 = float(np.float32(c.eps * c.eps))
    n = c.n
    total_budget = 120.0
    per_step = total_budget / max(1, args.steps + args.warmup)
    ns = 256
    oracle.forces(m, x, v, eps2, idx=np.arange(64))      # thread-pool start-up
    t0 = time.perf_counter()
    oracle.forces(m, x, v, eps2, idx=np.arange(ns))
    ns = int(min(n, max(ns, ns * per_step / max(time.perf_counter() - t0, 1e-4))))
    times = []
    for s in range(args.warmup + args.steps):
        idx = (np.arange(ns, dtype=np.int64) * (n // ns) + s) % n
        t0 = time.perf_counter()
        oracle.forces(m, x, v, eps2, idx=idx)
        el = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(el)
    tot = sum(times)
    value = args.steps * ns * n / tot
    line = {
        "impl": "reference", "metric": "pairwise interactions/s", "value": value,
        "unit": "interactions/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {c.kind} N={n} eps={c.eps} dt=1/1024 Hermite-4",
                   "n": n, "sample_i_per_step": ns},
        "cpu_baseline": {"value": value, "unit": "interactions/s", "cores": oracle.threads(),
                         "kind": "oracle",
                         "sample": f"each step: acc+jerk of {ns} strided i x all {n} j (fp64)"},
        "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_19294_b200 import binding, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.cuda.set_stream(torch.cuda.Stream(dev))   # one explicit stream for every launch
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    c = inputs.CONFIGS[args.config]
    m, x, v = inputs.make(args.config)          # fp32-representable fp64 (R#9)
    n = c.n
    eps2 = float(np.float32(c.eps * c.eps))
    mt = torch.from_numpy(m).to(dev)
    xt = torch.from_numpy(x).to(dev)
    vt = torch.from_numpy(v).to(dev)

    nccl_id = None
    if world > 1:
        obj = [binding.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    elif args.nccl1:
        nccl_id = binding.nccl_unique_id()

    block = args.integrator == "block"
    hilo = args.hilo == "on" or (args.hilo == "auto" and block)
    sim = binding.NBody(mt, xt, vt, eps=c.eps, dt=args.dt_max if block else c.dt, rank=rank,
                        world=world, nccl_id=nccl_id, device=local, integrator=args.integrator,
                        eta=args.eta, hilo=hilo)

    def active_sum():
        """Block time steps: force evaluations so far, summed over ranks (each active
        particle costs N interactions); None for the shared-dt integrators."""
        if not block:
            return None
        a = torch.tensor([float(sim.block_stats()[1])], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(a, op=dist.ReduceOp.SUM)
        return a.item()
    # hi/lo positions add 6 FADD per interaction (d = (xj_hi - xi_hi) + (xj_lo - xi_lo))
    FLOPS_PER_INTERACTION = FLOPS[args.integrator] + (6 if hilo else 0)
    stream = torch.cuda.current_stream(dev)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    # warm-up (includes the t = 0 force evaluation a0, j0)
    sim.step(args.warmup)
    sim.sync()
    sim.prof_read(reset=True)            # zero the launch counters

    # ---- pass A (the headline): K steps as a user runs them (CUDA-graph replay when
    #      the stream allows it), one CUDA-event pair per step, L2 flushed in between
    clocks = ClockSampler(local)
    meter = EnergyMeter(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier()
    act0 = active_sum()
    bs0 = sim.block_stats()[0] if block else None
    clocks.start()
    meter.start()
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()                     # L2 flush between steps, outside the step events
        ev[k][0].record(stream)
        sim.step(1)
        ev[k][1].record(stream)
    barrier()
    energy = meter.stop()
    clk = clocks.stop()
    sim.sync()
    ms_steps = sum(a.elapsed_time(b) for a, b in ev)
    act_a = (active_sum() - act0) if block else None
    block_steps_a = (sim.block_stats()[0] - bs0) if block else None
    if world > 1:   # whole-job GPU energy: sum over ranks (NaN marks a rank without a reading)
        ej = torch.tensor([energy["gpu_joules"] if energy["gpu_joules"] is not None else float("nan")],
                          dtype=torch.float64, device=dev)
        dist.all_reduce(ej, op=dist.ReduceOp.SUM)
        energy["gpu_joules"] = None if ej.isnan().item() else ej.item()
    _, _, launches = sim.prof_read(reset=True)

    # ---- pass B (roofline of the force kernel): the library brackets every force
    #      launch with CUDA events on the stream that launches it
    sim.prof_enable(True)
    barrier()
    act1 = active_sum()
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        sim.step(1)
    barrier()
    force_ms, force_launches, _ = sim.prof_read(reset=True)
    sim.prof_enable(False)
    act_b = (active_sum() - act1) if block else None
    t_local = torch.tensor([ms_steps, force_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_total, force_ms_max = t_local.tolist()
    ms_per_step = ms_total / args.steps
    # interactions per pass: N^2 per shared step; block steps: N per active particle
    interactions = float(n) * act_a if block else float(n) * float(n) * args.steps
    value = interactions / (ms_total * 1e-3)

    # ---- roofline of the dominant kernel (force pass): FP32 FMA pipe
    peaks = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = peaks.get("sm_max_mhz") or clk.get("sm_max_mhz") or 1965.0
    peak_tflops = sm_count * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    n_loc = sim.n_loc
    plan_info = binding.plan(n, world, rank)
    plan_info["items"] = -(-n_loc // 1024) * plan_info["n_chunks"]
    force_launch_ms = force_ms / max(1, force_launches)
    i_evals_b = (act_b / world) if block else float(n_loc) * args.steps   # this rank's i per pass
    flops_per_launch = FLOPS_PER_INTERACTION * i_evals_b * float(n) / max(1, force_launches)
    achieved = flops_per_launch / (force_launch_ms * 1e-3) / 1e12 if force_launch_ms > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "force_traffic.json")) as f:
            tr = json.load(f)
            if (tr.get("config") == args.config and tr.get("n_gpus", 1) == world
                    and tr.get("integrator", "hermite") == args.integrator):
                traffic = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---- e2e through the C-ABI with pinned host buffers (paper's offload model:
    #      state H2D, step, state D2H every step)
    e2e = None
    if not args.no_e2e:
        i0, i1 = sim.i0, sim.i1
        hx = torch.from_numpy(np.ascontiguousarray(x[:, i0:i1])).pin_memory()
        hv = torch.from_numpy(np.ascontiguousarray(v[:, i0:i1])).pin_memory()
        sim_h = sim
        lib = binding.lib()
        binding._check(lib.nbody_get_state(sim_h._ctx, hx.data_ptr(), hv.data_ptr()), sim_h._ctx)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        act2 = active_sum()
        t0.record(stream)
        for k in range(args.steps):
            binding._check(lib.nbody_set_state(sim_h._ctx, hx.data_ptr(), hv.data_ptr(), 1), sim_h._ctx)
            sim_h.step(1)
            binding._check(lib.nbody_get_state(sim_h._ctx, hx.data_ptr(), hv.data_ptr()), sim_h._ctx)
        t1.record(stream)
        barrier()
        e_ms = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        inter_e = float(n) * (active_sum() - act2) if block else interactions
        e2e = {"value": inter_e / (e_ms.item() * 1e-3), "unit": "interactions/s",
               "h2d_bytes_per_step": int(2 * 3 * 8 * (i1 - i0)) * world,
               "d2h_bytes_per_step": int(2 * 3 * 8 * (i1 - i0)) * world}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(m, x, v, eps2, args.cpu_seconds)

    sim.close()
    if rank == 0:
        line = {
            "metric": "pairwise interactions/s",
            "value": value,
            "unit": "interactions/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {
                "workload": f"{args.config}: {c.kind} N={n} eps={c.eps} " + (
                    "dt=1/1024, Hermite-4 P(EC)^1 step (predict, all-gather, acc+jerk force, correct)"
                    if args.integrator == "hermite" else
                    "dt=1/1024, kick-drift-kick leapfrog step (kick+drift, all-gather, acc force, kick)"
                    if args.integrator == "leapfrog" else
                    f"block time steps, one step = dt_max = {args.dt_max:g} of individual Hermite-4 "
                    f"steps (eta = {args.eta:g}, eta_s = 0.01): t_next, active set, predict all, "
                    f"all-gather, force on the active set, correct + new levels")
                + (", hi/lo positions" if hilo else ""),
                "integrator": args.integrator,
                "n": n, "flops_per_interaction": FLOPS_PER_INTERACTION,
                "l2": "flushed between steps (256 MiB memset outside the per-step events)"
                      if flush is not None else "not flushed",
                "parallelism": f"i-shard x{world}",
                "exchange": ("ncclAllGather (1-rank communicator, --nccl1)" if world == 1 and args.nccl1
                             else "ncclAllGather" if world > 1 else "none (one GPU holds every packet)"),
                "j_split": {k: plan_info[k] for k in ("chunk", "n_chunks")} | {
                    "i_per_cta": 1024, "work_items_per_gpu": plan_info["items"],
                    "note": "canonical (i-block x j-chunk) work items; results bit-identical for any P"},
                **({"block_steps_per_step": block_steps_a / args.steps,
                    "mean_active": act_a / max(1, block_steps_a),
                    "force_evaluations_per_step": act_a / args.steps} if block else {}),
            },
            "tflops": value * FLOPS_PER_INTERACTION / 1e12,
            "frac_fp32_peak": value * FLOPS_PER_INTERACTION / 1e12 / peak_tflops,
            "roofline": {
                "bound": "alu", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": (achieved / peak_tflops) if achieved else None, "traffic": traffic,
                "kernel": "force_kernel", "launches": force_launches,
                "ms_per_launch": force_launch_ms,
                "force_share_of_step": force_ms_max / ms_total if ms_total else None,
                "peak_basis": f"{sm_count} SM x 128 FP32 lanes x 2 x {sm_max:.0f} MHz "
                              f"({'MEASURED_PEAKS.json sm_max_mhz' if peaks.get('sm_max_mhz') else 'nvidia-smi max clock'})",
            },
            "clocks": clk,
            "energy": dict(energy, joules_per_step=(energy["gpu_joules"] / args.steps
                                                    if energy["gpu_joules"] is not None else None),
                           interactions_per_joule=(interactions / energy["gpu_joules"]
                                                   if energy["gpu_joules"] else None),
                           scope=f"{world} GPU(s), NVML total-energy counter, summed over ranks, timed region"),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
