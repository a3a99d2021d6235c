#!/usr/bin/env python
"""Accuracy per cost: shared-dt Hermite vs block time steps on the same system and time
span (energy drift by the oracle's fp64 energy, force evaluations, GPU time).  One GPU.
  python scripts/block_vs_shared.py [--config C2] [--t 0.25]"""
import argparse
import json
import sys

sys.path.insert(0, ".")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--t", type=float, default=0.25)
    a = ap.parse_args()
    import numpy as np
    import torch
    import oracle
    from paper_2509_19294_b200 import binding, inputs
    c = inputs.CONFIGS[a.config]
    m, x, v = inputs.make(a.config)
    e2 = float(np.float32(c.eps * c.eps))
    E0 = sum(oracle.energy(m, x, v, e2))
    st = torch.cuda.Stream()
    rows = []
    runs = [("hermite", 1 / 256, {}), ("hermite", 1 / 1024, {}), ("hermite", 1 / 4096, {}),
            ("block", 1 / 128, {"eta": 0.02}), ("block", 1 / 128, {"eta": 0.005})]
    for integ, dt, kw in runs:
        nsteps = int(round(a.t / dt))
        with binding.NBody(m, x, v, eps=c.eps, dt=dt, integrator=integ, stream=st, **kw) as s:
            s.forces()
            s.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.step(nsteps)
            e1.record(st)
            xs_t, vs_t = s.state()
            s.sync()                      # the copies run on `st`
            xs, vs = xs_t.cpu().numpy(), vs_t.cpu().numpy()
            ms = e0.elapsed_time(e1)
            evals = s.block_stats()[1] if integ == "block" else nsteps * c.n
        drift = abs(sum(oracle.energy(m, xs, vs, e2)) - E0) / abs(E0)
        rows.append({"integrator": integ, "dt_or_dt_max": dt, **kw, "steps": nsteps,
                     "force_evaluations": int(evals), "gpu_ms": ms, "energy_drift": drift})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
