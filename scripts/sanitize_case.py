#!/usr/bin/env python
"""Small end-to-end case for compute-sanitizer (racecheck / memcheck / synccheck):
every force-kernel instantiation (eps > 0 and eps = 0 guard, Hermite and
leapfrog, hi/lo, block-step active lists), loopback shards, graph replay and the
energy kernel, N = 3000; block steps at N = 70 001 (tile-split force kernel).  Also run against the NB_DEBUG_CHECKS=1 library
(tests/test_gpu_debug_checks.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19294_b200 import binding, inputs  # noqa: E402

m, x, v = inputs.parity_round(*inputs.plummer(3000, 3))
st = torch.cuda.Stream()
for kw in (dict(), dict(integrator="leapfrog"), dict(hilo=True), dict(world=3, loopback=True),
           dict(eps=0.0), dict(eps=0.0, integrator="leapfrog", hilo=True),
           dict(integrator="block"), dict(integrator="block", world=3, loopback=True),
           dict(integrator="block", eps=0.0)):
    eps = kw.pop("eps", 1e-3)
    with binding.NBody(m, x, v, eps=eps, dt=1 / 1024, stream=st, **kw) as s:
        s.forces()
        s.step(3)
        s.energy()
        s.sync()
# block steps with >= 2 tiles per chunk: the tile-split force kernel (small active sets)
# and the list kernel; eps > 0 and the eps = 0 guard
m2, x2, v2 = inputs.parity_round(*inputs.plummer(70001, 4))
for kw in (dict(integrator="block"), dict(integrator="block", eps=0.0, hilo=False),
           dict(integrator="block", listbig=True)):
    eps = kw.pop("eps", 1e-3)
    # every list launch in 1024-i CTAs (NBODY_LISTBIG_MIN is read per launch)
    os.environ["NBODY_LISTBIG_MIN"] = "1" if kw.pop("listbig", False) else ""
    os.environ["NBODY_TSPLIT1_MAX"] = "0" if os.environ["NBODY_LISTBIG_MIN"] else ""
    os.environ["NBODY_TSPLIT_MAX"] = "0" if os.environ["NBODY_LISTBIG_MIN"] else ""
    with binding.NBody(m2, x2, v2, eps=eps, dt=1 / 256, stream=st, **kw) as s:
        s.step(1)
        assert s.block_stats()[0] > 1
        s.sync()
print("sanitize case ok")
