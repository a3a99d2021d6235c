"""GPU parity of SURVEY 8(f) row f2: two-float (hi/lo) position differencing.

Inputs here are the raw fp64 ICs (NOT rounded to fp32), i.e. positions off the
fp32 grid like any mid-trajectory state.  The oracle sees those exact values;
with hilo the GPU's differences carry ~48 bits, so the 1e-5 acceleration bar is
met without the R#9 fp32-rounding of the inputs.
"""
import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import binding, inputs
from metrics import TOL_ACC, TOL_JERK, TOL_PAPER_ACC, TOL_PAPER_JERK, max_rel, paper_norm, sample_indices

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def eps2_of(eps):
    return float(np.float32(eps * eps))


def forces(m, x, v, eps, **kw):
    with binding.NBody(m, x, v, eps=eps, dt=1 / 1024, **kw) as s:
        a, j = s.forces()
        s.sync()
        return a.cpu().numpy(), j.cpu().numpy()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_hilo_parity_on_fp64_inputs(cfg):
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg, parity=False)
    m = m.astype(np.float32).astype(np.float64)    # masses stay fp32 (G m is an fp32 operand)
    idx = None if c.n <= 16384 else sample_indices(x, n_stride=4096)
    a, j = forces(m, x, v, c.eps, hilo=True)
    ao, jo = oracle.forces(m, x, v, eps2_of(c.eps), idx=idx)
    if idx is not None:
        a, j = a[:, idx], j[:, idx]
    assert max_rel(a, ao) <= TOL_ACC, max_rel(a, ao)
    assert max_rel(j, jo) <= TOL_JERK and paper_norm(a, ao) <= TOL_PAPER_ACC
    assert paper_norm(j, jo) <= TOL_PAPER_JERK


def test_hilo_equals_plain_on_fp32_inputs():
    """On fp32-representable positions every lo part is 0, so hi/lo is the same arithmetic."""
    m, x, v = inputs.make("C2")
    a0, j0 = forces(m, x, v, 1e-3)
    a1, j1 = forces(m, x, v, 1e-3, hilo=True)
    assert np.array_equal(a0, a1) and np.array_equal(j0, j1)


def test_hilo_leapfrog_and_loopback():
    m, x, v = inputs.plummer(6000, 12)
    m = m.astype(np.float32).astype(np.float64)
    ref = None
    for world in (1, 3):
        with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024, hilo=True, integrator="leapfrog",
                           world=world, loopback=world > 1) as s:
            a, _ = s.forces()
            s.step(2)
            got = [t.cpu().numpy() for t in (a, *s.state())]
        if ref is None:
            ref = got
        else:
            assert all(np.array_equal(g, r) for g, r in zip(got, ref))
    ao, _ = oracle.forces(m, x, v, eps2_of(1e-3))
    assert max_rel(ref[0], ao) <= TOL_ACC


def test_hilo_trajectory_c2():
    c = inputs.CONFIGS["C2"]
    m, x, v = inputs.make("C2", parity=False)
    m = m.astype(np.float32).astype(np.float64)
    e2 = eps2_of(c.eps)
    with binding.NBody(m, x, v, eps=c.eps, dt=c.dt, hilo=True) as s:
        s.step(c.steps)
        xs, vs = (t.cpu().numpy() for t in s.state())
    xo, vo, _, _ = oracle.hermite(m, x, v, e2, c.dt, c.steps)
    E0 = sum(oracle.energy(m, x, v, e2))
    Dg = abs(sum(oracle.energy(m, xs, vs, e2)) - E0) / abs(E0)
    Do = abs(sum(oracle.energy(m, xo, vo, e2)) - E0) / abs(E0)
    assert Dg <= 2 * max(Do, 1e-11), (Dg, Do)
    assert np.linalg.norm(xs - xo, axis=0).max() <= 1e-6
