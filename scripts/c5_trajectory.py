#!/usr/bin/env python
"""C5 trajectory and energy-drift parity (BASELINE.json configs[4]: Plummer N = 1 048 576,
eps = 5e-4, 5 Hermite steps at dt = 1/1024) -- the GPU path against the fp64 oracle.

Readings: R#14 (drift D = max_k |E_k - E_0| / |E_0| with BOTH energies from the oracle's
fp64 function, checkpoints at the end for C4/C5; pass if D_gpu <= 2 max(D_orc, 1e-11)),
R#15 (trajectory deltas from the same fp32-representable IC).  PAPER.md:161 (§3): device
results are validated against "a naive, double-precision brute-force implementation".

The oracle trajectory is ~6.6e12 fp64 pair evaluations (about 40 min on 16 host cores), so
the three phases may run on different machines:

  python scripts/c5_trajectory.py gpu      # on the B200: 5 steps, final state -> npz
  python scripts/c5_trajectory.py oracle   # any host: oracle 5 steps -> npz
  python scripts/c5_trajectory.py compare  # any host: oracle energies, deltas -> JSON

Files go to gpurun_out/ (scratch); `compare` writes profiles/r02_c5_trajectory.json with
the SHA-256 of both state files.
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")


def sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for b in iter(lambda: f.read(1 << 20), b""):
            h.update(b)
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("phase", choices=["gpu", "oracle", "compare"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--threads", type=int, default=0, help="oracle OpenMP threads (0: all)")
    a = ap.parse_args()
    import numpy as np
    from paper_2509_19294_b200 import inputs
    c = inputs.CONFIGS[a.config]
    m, x, v = inputs.make(a.config)
    eps2 = float(np.float32(c.eps * c.eps))   # R#18
    os.makedirs(OUT, exist_ok=True)
    gpu_f = os.path.join(OUT, f"{a.config.lower()}_gpu_state.npz")
    orc_f = os.path.join(OUT, f"{a.config.lower()}_oracle_state.npz")
    if a.phase == "gpu":
        import torch
        from paper_2509_19294_b200 import binding
        st = torch.cuda.Stream()
        t0 = time.perf_counter()
        with binding.NBody(m, x, v, eps=c.eps, dt=c.dt, stream=st) as s:
            s.step(c.steps)
            xs, vs = s.state()
            ke, pe = s.energy()
            s.sync()
            st.synchronize()
            xs, vs = xs.cpu().numpy(), vs.cpu().numpy()
        np.savez(gpu_f, x=xs, v=vs, gpu_energy=np.array([ke, pe]))
        print(json.dumps({"phase": "gpu", "seconds": time.perf_counter() - t0, "file": gpu_f,
                          "sha256": sha(gpu_f)}))
        return 0
    import oracle
    if a.threads:
        oracle.set_threads(a.threads)
    if a.phase == "oracle":
        t0 = time.perf_counter()
        xo, vo, _, _ = oracle.hermite(m, x, v, eps2, c.dt, c.steps)
        np.savez(orc_f, x=xo, v=vo)
        print(json.dumps({"phase": "oracle", "seconds": time.perf_counter() - t0,
                          "threads": oracle.threads(), "file": orc_f, "sha256": sha(orc_f)}))
        return 0
    g = np.load(gpu_f)
    o = np.load(orc_f)
    t0 = time.perf_counter()
    E0 = sum(oracle.energy(m, x, v, eps2))
    Eg = sum(oracle.energy(m, g["x"], g["v"], eps2))
    Eo = sum(oracle.energy(m, o["x"], o["v"], eps2))
    Dg, Do = abs(Eg - E0) / abs(E0), abs(Eo - E0) / abs(E0)
    dx = np.linalg.norm(g["x"] - o["x"], axis=0)
    dv = np.linalg.norm(g["v"] - o["v"], axis=0)
    gE = float(g["gpu_energy"].sum())
    rec = {
        "config": a.config, "n": c.n, "eps": c.eps, "dt": c.dt, "steps": c.steps,
        "what": "GPU Hermite-4 P(EC)^1 trajectory vs the fp64 oracle from the same fp32-representable IC "
                "(R#9); energies by the oracle's fp64 O(N^2) function (R#14)",
        "E0": E0, "E_gpu": Eg, "E_oracle": Eo, "D_gpu": Dg, "D_oracle": Do,
        "drift_ratio": Dg / Do if Do else None, "drift_bar": 2 * max(Do, 1e-11),
        "drift_pass": Dg <= 2 * max(Do, 1e-11),
        "gpu_energy_kernel_vs_oracle_rel": abs(gE - Eg) / abs(Eg),
        "max_dx": float(dx.max()), "median_dx": float(np.median(dx)),
        "max_dv": float(dv.max()), "median_dv": float(np.median(dv)),
        "dx_bar": 1e-6, "dv_bar": 1e-4,
        "trajectory_pass": bool(dx.max() <= 1e-6 and dv.max() <= 1e-4),
        "all_particles": True,
        "gpu_state_sha256": sha(gpu_f), "oracle_state_sha256": sha(orc_f),
        "oracle_threads": oracle.threads(), "energy_seconds": time.perf_counter() - t0,
    }
    path = os.path.join(ROOT, "profiles", f"r02_{a.config.lower()}_trajectory.json")
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))
    return 0 if rec["drift_pass"] and rec["trajectory_pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
