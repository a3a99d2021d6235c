#!/usr/bin/env python
"""the fp64 oracle timed on the GPU box's host cores -- one full force
evaluation at C1..C4 (all cores and one core for C1/C2), full oracle trajectories (t = 0
evaluation + the config's Hermite steps) at C1..C3, and C5 as 8192 strided i x N,
extrapolated and labelled as such.  Prints one JSON line per measurement.
  python scripts/oracle_timing.py > profiles/r01_oracle_timing.jsonl"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2509_19294_b200 import inputs  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    cores = oracle.threads()
    for cfg in ("C1", "C2", "C3", "C4"):
        c = inputs.CONFIGS[cfg]
        m, x, v = inputs.make(cfg)
        e2 = float(np.float32(c.eps * c.eps))
        t0 = time.perf_counter()
        oracle.forces(m, x, v, e2)
        el = time.perf_counter() - t0
        emit(config=cfg, what="one force evaluation", cores=cores, seconds=el,
             interactions_per_s=c.n * c.n / el)
        if cfg in ("C1", "C2"):
            oracle.set_threads(1)
            t0 = time.perf_counter()
            oracle.forces(m, x, v, e2)
            el1 = time.perf_counter() - t0
            oracle.set_threads(cores)
            emit(config=cfg, what="one force evaluation", cores=1, seconds=el1,
                 interactions_per_s=c.n * c.n / el1)
        if cfg in ("C1", "C2", "C3"):
            t0 = time.perf_counter()
            oracle.hermite(m, x, v, e2, c.dt, c.steps)
            el = time.perf_counter() - t0
            emit(config=cfg, what=f"full trajectory: t = 0 evaluation + {c.steps} Hermite steps",
                 cores=cores, seconds=el, interactions_per_s=(c.steps + 1) * c.n * c.n / el)
    c = inputs.CONFIGS["C5"]
    m, x, v = inputs.make("C5")
    idx = np.linspace(0, c.n - 1, 8192).astype(np.int64)
    t0 = time.perf_counter()
    oracle.forces(m, x, v, float(np.float32(c.eps * c.eps)), idx=idx)
    el = time.perf_counter() - t0
    emit(config="C5", what="8192 strided i x N, extrapolated x N/8192 (EXTRAPOLATED)", cores=cores,
         seconds=el * c.n / 8192, interactions_per_s=8192 * c.n / el)


if __name__ == "__main__":
    main()
