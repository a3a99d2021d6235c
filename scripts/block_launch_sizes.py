#!/usr/bin/env python
"""Force-pass efficiency of block time steps by active-set size (one GPU).

Runs `--cycles` dt_max of block steps with kernel timing on (the host-driven loop), then
pairs every force launch's CUDA-event time with its size (nbody_prof_launch_sizes) and
reports, per bucket of active counts, the launches, the interactions and the achieved rate
against the shared-step rate of the same N -- where the block-step force time goes.

  python scripts/block_launch_sizes.py [--config C4] [--dt-max 0.0078125] [--cycles 1]
"""
import argparse
import json
import sys

sys.path.insert(0, ".")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--dt-max", type=float, default=1 / 128)
    ap.add_argument("--cycles", type=int, default=1)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2509_19294_b200 import binding, inputs
    c = inputs.CONFIGS[a.config]
    m, x, v = inputs.make(a.config)
    dev = torch.device("cuda", 0)
    mt, xt, vt = (torch.from_numpy(t).to(dev) for t in (m, x, v))
    with binding.NBody(mt, xt, vt, eps=c.eps, dt=c.dt, hilo=True) as s:   # shared-step reference
        s.forces()
        s.prof_enable(True)
        s.prof_read(reset=True)
        for _ in range(3):
            s.forces()
        ms, nf, _ = s.prof_read(reset=True)
        shared_rate = c.n * c.n * nf / (ms * 1e-3)
    with binding.NBody(mt, xt, vt, eps=c.eps, dt=a.dt_max, integrator="block") as s:
        s.step(1)                       # warm-up cycle (levels settle, graph-free path)
        s.prof_enable(True)
        s.prof_read(reset=True)
        s.step(a.cycles)
        t = s.prof_launch_times()
        ni, nj = s.prof_launch_sizes()
    inter = ni.astype(np.float64) * nj
    edges = [1, 64, 256, 1024, 4096, 16384, 65536, 1 << 40]
    print(f"# {a.config} N={c.n} block steps dt_max={a.dt_max:g}, {len(t)} force launches over "
          f"{a.cycles} dt_max; shared-step force rate (hi/lo) {shared_rate:.4g} int/s")
    print(f"# {'active':>15} {'launches':>8} {'share of time':>13} {'share of int.':>13} "
          f"{'int/s':>10} {'vs shared':>9} {'ms/launch':>9}")
    rows = []
    for lo, hi in zip(edges, edges[1:]):
        k = (ni >= lo) & (ni < hi)
        if not k.any():
            continue
        tt, ii = t[k].sum(), inter[k].sum()
        r = dict(active_lo=lo, active_hi=hi, launches=int(k.sum()), time_share=float(tt / t.sum()),
                 inter_share=float(ii / inter.sum()), rate=float(ii / (tt * 1e-3)),
                 ms_per_launch=float(tt / k.sum()))
        rows.append(r)
        print(f"  [{lo:>6}, {min(hi, c.n + 1):>6}) {r['launches']:>8} {r['time_share']:>13.3f} "
              f"{r['inter_share']:>13.3f} {r['rate']:>10.3e} {r['rate'] / shared_rate:>9.3f} "
              f"{r['ms_per_launch']:>9.4f}")
    tot = inter.sum() / (t.sum() * 1e-3)
    print(f"  all {len(t):>23} {1:>13.3f} {1:>13.3f} {tot:>10.3e} {tot / shared_rate:>9.3f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(dict(config=a.config, dt_max=a.dt_max, shared_rate=shared_rate, rows=rows,
                           total_rate=tot, launches=len(t)), f)


if __name__ == "__main__":
    main()
