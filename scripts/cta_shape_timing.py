#!/usr/bin/env python
"""Force-pass time per evaluation for the two CTA shapes (NBODY_FORCE_CTA=big|small)
over N, to place the automatic switch (force.cu use_small_cta).  One GPU.
  python scripts/cta_shape_timing.py > profiles/r01_cta_shapes.txt"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(n, reps):
    import numpy as np
    import torch  # noqa: F401
    from paper_2509_19294_b200 import binding, inputs
    m, x, v = inputs.parity_round(*inputs.plummer(n, 3))
    with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024, hilo=False) as s:
        s.forces()
        s.sync()
        s.prof_enable(True)
        s.prof_read(reset=True)
        for _ in range(reps):
            s.forces()
        ms, nf, _ = s.prof_read(reset=True)
    t = ms / max(nf, 1)
    return t, n * n / (t * 1e-3)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        t, r = one(int(sys.argv[2]), int(sys.argv[3]))
        print(f"{t:.5f} {r:.4e}")
        sys.exit(0)
    print("# force pass per evaluation (ms) and interactions/s, Plummer N, eps = 1e-3, 1 B200")
    print("# shape: big = 1024 i/CTA (2 CTAs/SM), small = 256 i/CTA (6 CTAs/SM), auto = library choice")
    for n in (1024, 4096, 16384, 32768, 65536, 131072):
        row = [f"N={n:7d}"]
        for shape in ("big", "small", "auto"):
            env = dict(os.environ, NBODY_FORCE_CTA=shape)
            reps = max(3, int(2e9 / (n * n)))
            out = subprocess.run([sys.executable, __file__, "one", str(n), str(min(reps, 2000))],
                                 env=env, capture_output=True, text=True).stdout.split()
            row.append(f"{shape} {out[0]} ms {out[1]} int/s" if len(out) == 2 else f"{shape} FAILED")
        print("  ".join(row), flush=True)
