#!/usr/bin/env python
"""Write the tests/golden/ fixtures that hold computed values.

This script calls only `oracle/` (plus the seeded input generators, which hold none of
the method's arithmetic), so no stored expected value comes from the CUDA path.  The
fixtures it writes are pinned independently of the oracle in tests/test_golden.py
(40-digit mpmath evaluation of the force definition; the Kepler closed form).  The
paper prints no per-particle worked example; its printed numbers are
stored by hand in tests/golden/paper_numbers.json with their line citations.

  python scripts/make_golden.py
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")


def main():
    import numpy as np
    import oracle
    from paper_2509_19294_b200 import inputs
    os.makedirs(OUT, exist_ok=True)

    # (1) forces of a small seeded system, eps > 0, fp32-representable inputs (R#9)
    m, x, v = inputs.parity_round(*inputs.uniform_cube(6, 7))
    eps2 = float(np.float32(1e-2 * 1e-2))   # R#18: eps^2 := fp32(eps * eps)
    a, j = oracle.forces(m, x, v, eps2)
    rec = {
        "what": "acceleration and jerk of every particle, softened direct sum (P:134-138, R#1, R#2), "
                "fp64 oracle (oracle_forces), G = 1",
        "cite": "PAPER.md:134-138 (Sec. 3 force equation; jerk: 'first time derivative'), :161 (fp64 golden reference)",
        "written_by": "scripts/make_golden.py (oracle/ only)",
        "n": 6, "G": 1.0, "eps2": eps2,
        "m": m.tolist(), "x": x.tolist(), "v": v.tolist(),
        "acc": a.tolist(), "jerk": j.tolist(),
    }
    with open(os.path.join(OUT, "forces_cube6.json"), "w") as f:
        json.dump(rec, f, indent=1)

    # (2) Hermite-4 P(EC)^1 (R#3) on a Kepler orbit, e = 0.5, one period in 6434 steps
    m, x, v = inputs.kepler(0.5)
    nsteps = 6434
    dt = 2 * math.pi / nsteps
    x1, v1, _, _ = oracle.hermite(m, x, v, 0.0, dt, nsteps)
    rec = {
        "what": "two bodies m = 1/2 each, a = 1, e = 0.5, eps = 0, started at pericentre; state after "
                "one period (2 pi) of 6434 Hermite-4 P(EC)^1 steps with the Makino-Aarseth corrector (R#3)",
        "cite": "PAPER.md:158 (fp64 host-side integrator); SPEC.md:458-459 (Kepler check); DESIGN.md R#3",
        "written_by": "scripts/make_golden.py (oracle/ only)",
        "m": m.tolist(), "x0": x.tolist(), "v0": v.tolist(), "dt": dt, "nsteps": nsteps,
        "x": x1.tolist(), "v": v1.tolist(),
        "closed_form_relative_position": [1.0 - 0.5, 0.0, 0.0],
    }
    with open(os.path.join(OUT, "kepler_e05_period.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
