#!/usr/bin/env python
"""Projected strong scaling at P = 1/2/4/8 from ONE GPU (this environment has one B200).

Loopback mode runs the P shards' force passes one after another on one GPU with the
same kernels, chunk order and launch shapes a P-GPU run uses per rank; the per-shard
CUDA-event times are the per-GPU compute times.  The exchange is added from the
measured peer bandwidth in /opt/skills/guides/B200_PROFILING.md (770 GB/s per
direction) without crediting its overlap, so the projection is pessimistic for
communication.  It is a projection, labelled as such -- not a bench value.

  python scripts/project_scaling.py [--configs C3,C4,C5] [--steps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--integrator", default="hermite")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2509_19294_b200 import binding, inputs
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    for name in a.configs.split(","):
        c = inputs.CONFIGS[name]
        m, x, v = inputs.make(name)
        mt, xt, vt = (torch.from_numpy(t).to(dev) for t in (m, x, v))
        rows = []
        t1 = None
        for P in (1, 2, 4, 8):
            with binding.NBody(mt, xt, vt, eps=c.eps, dt=c.dt, world=P, loopback=P > 1,
                               stream=st, integrator=a.integrator) as s:
                s.step(2)
                s.sync()
                s.prof_enable(True)
                s.prof_read(reset=True)
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(st)
                s.step(a.steps)
                ev1.record(st)
                times = s.prof_launch_times()
                s.prof_read(reset=True)
                st.synchronize()
                wall = ev0.elapsed_time(ev1) / a.steps
            per_shard = times.reshape(a.steps, -1)          # [step][shard] (one launch per shard)
            force_per_gpu = per_shard.max(axis=1).mean()    # the slowest rank sets the step
            other = (wall - per_shard.sum(axis=1).mean()) / P   # predict/correct kernels, per rank
            comm = (P - 1) / P * c.n * 32 / 770e9 * 1e3 if P > 1 else 0.0
            t = force_per_gpu + other + comm
            if P == 1:
                t1 = t
            rows.append({"P": P, "force_ms_per_gpu": float(force_per_gpu), "other_ms": float(other),
                         "allgather_ms_est": comm, "step_ms": float(t),
                         "interactions_per_s": c.n * c.n / (t * 1e-3),
                         "efficiency": t1 / (P * t)})
        print(json.dumps({"config": name, "n": c.n, "integrator": a.integrator,
                          "kind": "projection from 1 GPU (loopback shards + modeled all-gather)",
                          "rows": rows}), flush=True)


if __name__ == "__main__":
    main()
