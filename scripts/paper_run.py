#!/usr/bin/env python
"""NEXT f4 (+ f3): the paper-shaped run on one B200 -- Plummer N = 102 400, ten Hermite
steps ("ten time cycles", R#4, R#24) -- with the paper's two metrics measured per
simulation:

* time-to-solution: the simulation only, as the paper's MPI_Wtime brackets it:
  the t = 0 force evaluation, ten steps and the final state's device-to-host copy.  The
  set-up (context creation, host-to-device copy and validation of the ICs) is timed and
  reported separately.
* energy-to-solution (R#25): GPU energy of each simulation from NVML's total
  energy counter (mJ).  The counter advances in discrete updates (the script measures
  their interval first), so each simulation starts on a counter update and the reading
  is taken at the first update after it ends; the idle power measured in the pad before
  it, times the overhang past the end, is subtracted.  Each repeat is preceded by an idle
  pad (120 s) that also gives the idle baseline.  The paper adds the host
  processor's energy; host package energy (RAPL, /sys/class/powercap) is read
  when the box exposes it and otherwise reported as unavailable.

Median and interquartile range over the repeats.  The paper's numbers are quoted as
context only (other hardware, unstated ICs, softening and dt).

  python scripts/paper_run.py [--repeats 5] [--pad 120] [--trace power.csv]
"""
import argparse
import glob
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def quartiles(v):
    v = sorted(v)
    if len(v) < 2:
        return {"median": v[0] if v else None, "q1": None, "q3": None, "iqr": None, "n": len(v)}
    q = statistics.quantiles(v, n=4, method="inclusive")
    return {"median": statistics.median(v), "q1": q[0], "q3": q[2], "iqr": q[2] - q[0],
            "min": v[0], "max": v[-1], "n": len(v)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--pad", type=float, default=120.0)
    ap.add_argument("--integrator", default="hermite")
    ap.add_argument("--trace", default=None)
    a = ap.parse_args()
    import numpy as np
    import pynvml
    import torch
    from paper_2509_19294_b200 import binding, inputs
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    energy_mj = lambda: pynvml.nvmlDeviceGetTotalEnergyConsumption(h)   # noqa: E731
    rapl = [f for f in sorted(glob.glob("/sys/class/powercap/intel-rapl:[0-9]*/energy_uj"))
            if os.access(f, os.R_OK)]

    def rapl_uj():
        try:
            return sum(int(open(f).read()) for f in rapl) if rapl else None
        except OSError:
            return None

    c = inputs.CONFIGS["PAPER"]
    m, x, v = inputs.make("PAPER")
    hm, hx, hv = (torch.from_numpy(t).pin_memory() for t in (m, x, v))
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    xo = torch.empty((3, c.n), dtype=torch.float64).pin_memory()
    vo = torch.empty((3, c.n), dtype=torch.float64).pin_memory()

    def setup():
        return binding.NBody(hm, hx, hv, eps=c.eps, dt=c.dt, integrator=a.integrator, stream=st)

    def simulate(s):
        s.step(c.steps)                    # the t = 0 force evaluation, then c.steps steps
        binding._check(binding.lib().nbody_get_state(s._ctx, xo.data_ptr(), vo.data_ptr()), s._ctx)

    # warm-up (module load, graph capture code paths, clocks)
    for _ in range(2):
        with setup() as s:
            simulate(s)

    # NVML energy counter update interval (idle)
    ticks, e_prev, t_end = [], energy_mj(), time.perf_counter() + 3.0
    while time.perf_counter() < t_end:
        e = energy_mj()
        if e != e_prev:
            ticks.append(time.perf_counter())
            e_prev = e
    tick_s = statistics.median(np.diff(ticks)) if len(ticks) > 2 else None

    def wait_tick():
        e0 = energy_mj()
        while True:
            e = energy_mj()
            if e != e0:
                return e, time.perf_counter()

    trace, phase, stop = [], ["idle"], [False]

    def sampler():   # NVML power every 50 ms (the paper samples at ~1 Hz)
        t0 = time.perf_counter()
        while not stop[0]:
            try:
                trace.append((time.perf_counter() - t0, pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0, phase[0]))
            except pynvml.NVMLError:
                pass
            time.sleep(0.05)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    runs = []
    for r in range(a.repeats):
        phase[0] = "idle"
        e_a, t_a = wait_tick()
        time.sleep(a.pad)
        e_b, t_b = wait_tick()
        p_idle = (e_b - e_a) * 1e-3 / (t_b - t_a)
        phase[0] = "setup"
        t0 = time.perf_counter()
        s = setup()
        st.synchronize()
        t_setup = time.perf_counter() - t0
        phase[0] = "idle"
        e0, t0 = wait_tick()
        c0 = rapl_uj()
        phase[0] = "run"
        t1 = time.perf_counter()
        simulate(s)                        # ends with the blocking D2H of the final state
        t2 = time.perf_counter()
        phase[0] = "idle"
        e1, t3 = wait_tick()
        c1 = rapl_uj()
        s.close()
        raw = (e1 - e0) * 1e-3
        runs.append({"time_to_solution_s": t2 - t1, "setup_s": t_setup,
                     "gpu_joules_window": raw, "window_s": t3 - t0,
                     "gpu_joules": raw - p_idle * (t3 - t2) - p_idle * (t1 - t0),
                     "idle_w": p_idle,
                     "host_cpu_joules": (c1 - c0) * 1e-6 if c0 is not None and c1 is not None else None})
    stop[0] = True
    th.join(timeout=1)
    if a.trace and trace:
        with open(a.trace, "w") as f:
            f.write("seconds,device,watts,phase\n")
            for t, w, ph in trace:
                f.write(f"{t:.3f},0,{w:.1f},{ph}\n")
    with setup() as s:                     # final-state energy check of the last run's system
        simulate(s)
        ke, pe = s.energy()
    pw = {ph: [w for _, w, p in trace if p == ph] for ph in ("idle", "run")}
    host = [r["host_cpu_joules"] for r in runs if r["host_cpu_joules"] is not None]
    out = {
        "workload": f"PAPER: Plummer N={c.n} eps={c.eps} dt=1/1024, {c.steps} {a.integrator} steps "
                    "(+ t=0 force evaluation and the final state's D2H); one B200",
        "repeats": a.repeats, "idle_pad_s": a.pad,
        "time_to_solution_s": quartiles([r["time_to_solution_s"] for r in runs]),
        "setup_s": quartiles([r["setup_s"] for r in runs]),
        "energy_to_solution_gpu_j": quartiles([r["gpu_joules"] for r in runs]),
        "energy_window_gpu_j": quartiles([r["gpu_joules_window"] for r in runs]),
        "host_cpu_energy_j": quartiles(host) if host else
            "unavailable: no readable RAPL counter under /sys/class/powercap on this box "
            "(the paper's total adds the host processor, P:234; this is GPU energy only)",
        "nvml_energy_counter_update_s": tick_s,
        "method": "per simulation: start on an NVML energy-counter update, read at the first update "
                  "after the end, minus idle power (from the pad before) x the time outside the "
                  "simulation in that window",
        "final_energy": ke + pe,
        "power_w": {ph: ({"mean": statistics.mean(v), "max": max(v), "samples": len(v)} if v else None)
                    for ph, v in pw.items()},
        "paper_context_other_hardware": {
            "wormhole_n300_plus_1_host_thread_s": "301.40 +- 0.24 (P:191)",
            "cpu_2x_epyc9124_32_threads_s": "672.90 +- 7.83 (P:191)",
            "energy_kJ": "71.56 +- 0.13 (Wormhole) vs 128.89 +- 1.52 (CPU) (P:236-237)",
            "note": "paper ICs, softening, dt and 'time cycle' unstated; not comparable targets",
        },
        "runs": runs,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
