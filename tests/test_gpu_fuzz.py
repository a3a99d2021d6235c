"""Randomised GPU parity sweep through the C-ABI: seeded random system sizes, softenings,
shard counts, position modes and integrators, each checked against the fp64 oracle and
against the unsharded run.  The seeds are fixed, so a failure is reproducible."""
import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import binding, inputs
from metrics import TOL_ACC, TOL_JERK, max_rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = list(range(24))


def _case(k):
    rng = np.random.default_rng(9000 + k)
    n = int(rng.choice([2, 3, 17, 255, 256, 257, 700, 1500, 2049, 3333]))
    kind = rng.choice(["cube", "plummer"])
    eps = float(rng.choice([0.0, 1e-3, 1e-2, 0.1]))
    world = int(rng.integers(1, 6))
    hilo = bool(rng.integers(0, 2))
    integrator = str(rng.choice(["hermite", "leapfrog", "block"]))
    if kind == "cube":
        m, x, v = inputs.uniform_cube(n, 100 + k, scale=float(rng.uniform(0.5, 5.0)))
    else:
        m, x, v = inputs.plummer(max(n, 2), 100 + k)
    m, x, v = inputs.parity_round(m, x, v)
    return n, m, x, v, eps, min(world, n), hilo, integrator


@pytest.mark.parametrize("k", CASES)
def test_random_case(k):
    n, m, x, v, eps, world, hilo, integrator = _case(k)
    out = {}
    for w in sorted({1, world}):
        with binding.NBody(m, x, v, eps=eps, dt=1 / 256, integrator=integrator, world=w,
                           loopback=w > 1, hilo=hilo) as s:
            a, j = (t.cpu().numpy() for t in s.forces())
            s.step(2)
            xs, vs = (t.cpu().numpy() for t in s.state())
            s.sync()
        out[w] = (a, j, xs, vs)
    a, j = out[1][0], out[1][1]
    ao, jo = oracle.forces(m, x, v, float(np.float32(eps * eps)))
    assert max_rel(a, ao) <= TOL_ACC, (k, n, eps, max_rel(a, ao))
    if integrator != "leapfrog":
        assert max_rel(j, jo) <= TOL_JERK, (k, n, eps, max_rel(j, jo))
    for arr_w, arr_1 in zip(out[world], out[1]):
        assert np.array_equal(arr_w, arr_1), (k, world)
    assert all(np.isfinite(t).all() for t in out[1])
