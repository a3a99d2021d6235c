#!/usr/bin/env python
"""Force-kernel tuning sweep.  `build` (CPU): compile variants into scripts/sweep/;
`run` (GPU): time each variant's force pass at a config in a subprocess.

  python scripts/sweep_force.py build
  python scripts/sweep_force.py run [--config C4] [--reps 3]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "scripts", "sweep")

VARIANTS = {
    # round-1 variants (3-stage ring, 3 CTAs/SM, 64/96/160 threads, 2/3/5 pairs, ptxas -O1/-O2,
    # 1 CTA/SM with unroll 3/4, constant-memory j, register prefetch) are recorded in
    # profiles/r01_sweep_force.txt; round 2's software-pipelined j loop, register-copy squares
    # and 5 pairs per thread in profiles/r02_sweep_force.txt (all slower; code removed)
    "base":      dict(),
    "p3b3":      dict(FK_PAIRS=3, FK_MINB=3),
}
if os.environ.get("SWEEP_ONLY"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SWEEP_ONLY"].split(",")}


def build():
    from concurrent.futures import ThreadPoolExecutor
    from paper_2509_19294_b200 import _build
    os.makedirs(OUT, exist_ok=True)

    def one(item):
        name, d = item
        path = os.path.join(OUT, f"lib_{name}.so")
        try:
            _build.build(defines=[f"{k}={v}" for k, v in d.items() if k != "_FLAGS"], out=path,
                         extra_flags=d.get("_FLAGS", ()))
            r = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
            regs = [ln for ln in r.splitlines() if "force_kernelILb0" in ln]
            return name, "ok", regs
        except Exception as e:  # noqa: BLE001
            return name, f"FAILED {e}", []
    with ThreadPoolExecutor(4) as ex:
        for name, st, regs in ex.map(one, VARIANTS.items()):
            print(name, st)


def time_one(config, reps):
    import numpy as np
    import torch
    from paper_2509_19294_b200 import binding, inputs
    c = inputs.CONFIGS[config]
    m, x, v = inputs.make(config)
    dev = torch.device("cuda", 0)
    sim = binding.NBody(torch.from_numpy(m).to(dev), torch.from_numpy(x).to(dev),
                        torch.from_numpy(v).to(dev), eps=c.eps, dt=c.dt,
                        integrator=os.environ.get("SWEEP_INTEGRATOR", "hermite"))
    sim.forces()
    sim.sync()
    sim.prof_enable(True)
    sim.prof_read(reset=True)
    for _ in range(reps):
        sim.forces()
    ms, nf, _ = sim.prof_read(reset=True)
    a, j = sim.forces()
    sim.sync()
    chk = float(a.abs().sum().item() + j.abs().sum().item())
    import oracle
    idx = np.linspace(0, c.n - 1, 2048).astype(np.int64)
    idx = np.unique(np.concatenate([idx, np.arange(1024, 1280), np.arange(768, 1024)]))
    ao, jo = oracle.forces(m, x, v, float(np.float32(c.eps * c.eps)), idx=idx)
    an, jn = a.cpu().numpy()[:, idx], j.cpu().numpy()[:, idx]
    ea = float(np.max(np.linalg.norm(an - ao, axis=0) / np.linalg.norm(ao, axis=0)))
    ej = float(np.max(np.linalg.norm(jn - jo, axis=0) / np.linalg.norm(jo, axis=0)))
    t = ms / max(nf, 1)
    fl = 40 if os.environ.get("SWEEP_INTEGRATOR", "hermite") == "hermite" else 18
    return {"ms": t, "interactions_per_s": c.n * c.n / (t * 1e-3),
            "tflops": fl * c.n * c.n / (t * 1e-3) / 1e12, "checksum": chk, "err_a": ea, "err_j": ej}


def run(config, reps):
    for name in VARIANTS:
        path = os.path.join(OUT, f"lib_{name}.so")
        if not os.path.exists(path):
            continue
        env = dict(os.environ, NBODY_LIB=path)
        r = subprocess.run([sys.executable, __file__, "one", config, str(reps)], env=env,
                           capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
        print(json.dumps({"variant": name, **VARIANTS[name], "result": line}), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        build()
    elif cmd == "one":
        print(json.dumps(time_one(sys.argv[2], int(sys.argv[3]))))
    elif cmd == "run":
        cfg = "C4"
        reps = 3
        if "--config" in sys.argv:
            cfg = sys.argv[sys.argv.index("--config") + 1]
        if "--reps" in sys.argv:
            reps = int(sys.argv[sys.argv.index("--reps") + 1])
        run(cfg, reps)
