#!/usr/bin/env python
"""Projected strong scaling at P = 1/2/4/8 from ONE GPU (this environment has one B200).

Loopback mode with NBODY_LOOPBACK_CONCURRENT=1 runs the P shards one after another on one
GPU, each with exactly the stream structure an NCCL rank uses per step (nbody.cu
exchange_and_force): the local-first force launch (1024-i CTAs, one wave of work items
inside the shard's own slice) on the compute stream; the exchange (here one device copy
per remote slice into the shard's own buffer) and the remote-chunk launch on the comm
stream, concurrent with it; the join; the fused corrector.  Shards are equal (N / P is a
multiple of the 1024-i block at C3-C5), so one rank's step time is the loopback step time
divided by P.  The NCCL all-gather is modelled from the measured peer bandwidth in
/opt/skills/guides/B200_PROFILING.md (770 GB/s per direction) and overlapped with the
local-first launch only: its exposed part is max(0, t_gather - t_local).  A projection,
labelled as such -- not a bench value.

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
    os.environ["NBODY_LOOPBACK_CONCURRENT"] = "1"   # read by nbody_init
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
                # pass 2: eager with per-launch events (the local-first launch's duration)
                s.prof_enable(True)
                s.prof_read(reset=True)
                for _ in range(a.steps):
                    with torch.cuda.stream(st):
                        flush.zero_()
                    s.step(1)
                times = s.prof_launch_times()
                ni, nj = s.prof_launch_sizes()
                s.prof_read(reset=True)
            wall = float(np.median(walls))
            per_step = times.reshape(a.steps, -1)
            n_launch = per_step.shape[1]
            # launch order per shard: local-first, remote (2 per shard when P > 1)
            local = float(per_step[:, 0::2].mean()) if P > 1 else None
            gather = (P - 1) / P * c.n * 32 / (PEER_GBS * 1e9) * 1e3 if P > 1 else 0.0
            exposed = max(0.0, gather - local) if P > 1 else 0.0
            t = wall / P + exposed
            if P == 1:
                t1 = t
            rows.append({"P": P, "loopback_step_ms": wall, "rank_step_ms": t,
                         "local_first_ms": local, "launches_per_step": n_launch,
                         "allgather_ms_model": gather, "allgather_exposed_ms": exposed,
                         "interactions_per_s": c.n * c.n / (t * 1e-3),
                         "efficiency": t1 / (P * t)})
        rec = {"config": name, "n": c.n, "integrator": a.integrator,
               "kind": "projection from 1 GPU: loopback shards in the NCCL rank's stream form "
                       "(local-first 1024-i launch; per-slice copies and the remote launch on the "
                       "comm stream, concurrent with it; corrector), rank step = loopback step / P; "
                       "all-gather modelled at 770 GB/s, overlapped with the local-first launch",
               "rows": rows}
        line = json.dumps(rec)
        print(line, flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(line + "\n")


if __name__ == "__main__":
    main()
