import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import os, numpy as np, torch
from paper_2509_19294_b200 import binding, inputs
os.environ["NBODY_DEBUG"] = "1"
for cfg in ("C2", "C4"):
    m, x, v = inputs.make(cfg)
    c = inputs.CONFIGS[cfg]
    with binding.NBody(m, x, v, eps=c.eps, dt=1/128, integrator="block") as s:
        s.step(1); s.sync()
        s.prof_enable(True); s.prof_read(reset=True)
        s.step(1)
        t = s.prof_launch_times()
        st = s.block_stats()
        print(cfg, "force launches", len(t), "mean ms", t.mean(), "max", t.max(), "stats", st, flush=True)
