#!/usr/bin/env python
"""Projected strong scaling at P = 1/2/4/8 from ONE GPU (this environment has one B200).

Loopback mode runs the P shards one after another on one GPU with exactly the launch
sequence an NCCL rank issues per step (nbody.cu exchange_and_force): the local-first
force launch (1024-i CTAs, one wave of work items inside the shard's own slice), the
exchange (here: one device copy per remote slice into the shard's own buffer), the
remote-chunk launch, and the fused corrector.  Kernel timing brackets every force
launch with CUDA events, so each shard's two launch times are its per-GPU force time.
The corrector share is the P = 1 step time minus its force time, divided by P (it is
HBM-bound over the shard's own particles).  The NCCL all-gather is modelled from the
measured peer bandwidth in /opt/skills/guides/B200_PROFILING.md (770 GB/s per
direction) and overlapped with the local-first launch only: its exposed part is
max(0, t_gather - t_local).  A projection, labelled as such -- not a bench value.

  python scripts/project_scaling.py [--configs C3,C4,C5] [--steps 3] [--out FILE]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PEER_GBS = 770.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--integrator", default="hermite")
    ap.add_argument("--out", default=None, help="append JSON lines here as well")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2509_19294_b200 import binding, inputs
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name in a.configs.split(","):
        c = inputs.CONFIGS[name]
        m, x, v = inputs.make(name)
        mt, xt, vt = (torch.from_numpy(t).to(dev) for t in (m, x, v))
        rows = []
        t1 = other1 = None
        for P in (1, 2, 4, 8):
            with binding.NBody(mt, xt, vt, eps=c.eps, dt=c.dt, world=P, loopback=P > 1,
                               stream=st, integrator=a.integrator) as s:
                s.step(2)
                s.sync()
                # pass 1: graph replay, CUDA events around each step (L2 flushed between)
                walls = []
                for _ in range(a.steps):
                    with torch.cuda.stream(st):
                        flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    s.step(1)
                    e1.record(st)
                    st.synchronize()
                    walls.append(e0.elapsed_time(e1))
                # pass 2: eager with per-launch events
                s.prof_enable(True)
                s.prof_read(reset=True)
                for _ in range(a.steps):
                    with torch.cuda.stream(st):
                        flush.zero_()
                    s.step(1)
                times = s.prof_launch_times()
                ni, nj = s.prof_launch_sizes()
                s.prof_read(reset=True)
                plan = [binding.plan(c.n, P, r) for r in range(P)]
            per_step = times.reshape(a.steps, -1)
            ni_s, nj_s = ni.reshape(a.steps, -1)[0], nj.reshape(a.steps, -1)[0]
            # attribute launches to shards in order: each shard's launches cover n_loc x n
            shards, k = [], 0
            for r in range(P):
                n_loc = plan[r]["i1"] - plan[r]["i0"]
                if n_loc <= 0:
                    continue
                idx, cov = [], 0
                while cov < c.n:
                    assert ni_s[k] == n_loc
                    idx.append(k)
                    cov += int(nj_s[k])
                    k += 1
                shards.append(idx)
            wall = float(np.median(walls))
            local = [float(per_step[:, idx[0]].mean()) if len(idx) > 1 else 0.0 for idx in shards]
            force = [float(per_step[:, idx].sum(axis=1).mean()) for idx in shards]
            if P == 1:
                other1 = max(0.0, wall - force[0])
            other = other1 / P
            gather = (P - 1) / P * c.n * 32 / (PEER_GBS * 1e9) * 1e3 if P > 1 else 0.0
            exposed = max(0.0, gather - min(local)) if P > 1 else 0.0
            t = max(force) + other + exposed
            if P == 1:
                t1 = wall
                t = wall
            rows.append({"P": P, "force_ms_per_gpu_max": max(force), "force_ms_per_gpu_min": min(force),
                         "local_first_ms": min(local) if P > 1 else None,
                         "corrector_ms": other, "allgather_ms_model": gather,
                         "allgather_exposed_ms": exposed, "step_ms": t,
                         "launches_per_shard": [len(i) for i in shards],
                         "interactions_per_s": c.n * c.n / (t * 1e-3),
                         "efficiency": t1 / (P * t)})
        rec = {"config": name, "n": c.n, "integrator": a.integrator,
               "kind": "projection from 1 GPU: loopback shards running the NCCL rank's launch "
                       "sequence (local-first 1024-i launch, per-slice copies, remote launch, "
                       "corrector); all-gather modelled at 770 GB/s, overlapped with the "
                       "local-first launch",
               "rows": rows}
        line = json.dumps(rec)
        print(line, flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(line + "\n")


if __name__ == "__main__":
    main()
