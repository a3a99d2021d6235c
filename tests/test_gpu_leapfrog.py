"""GPU parity of SURVEY 8(f) row f1: acceleration-only force kernel + kick-drift-kick
leapfrog (NBODY_LEAPFROG_KDK) against the oracle's leapfrog."""
import math

import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import binding, inputs
from metrics import TOL_ACC, TOL_PAPER_ACC, max_rel, paper_norm, sample_indices

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def eps2_of(eps):
    return float(np.float32(eps * eps))


def lf_forces(m, x, v, eps, **kw):
    with binding.NBody(m, x, v, eps=eps, dt=1 / 1024, integrator="leapfrog", **kw) as s:
        a, j = s.forces()
        s.sync()
        return a.cpu().numpy(), j.cpu().numpy()


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_accel_only_parity(cfg):
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    a, j = lf_forces(m, x, v, c.eps)
    ao, _ = oracle.forces(m, x, v, eps2_of(c.eps))
    assert max_rel(a, ao) <= TOL_ACC and paper_norm(a, ao) <= TOL_PAPER_ACC
    assert not j.any()                       # jerk is not computed (zero-filled)


def test_accel_only_matches_hermite_kernel_bitwise():
    """The acceleration of the accel-only kernel is the same arithmetic as the
    accel+jerk kernel's (same operation order), so the results are bit-identical."""
    m, x, v = inputs.make("C2")
    a_lf, _ = lf_forces(m, x, v, 1e-3)
    with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024) as s:
        a_h, _ = s.forces()
        a_h = a_h.cpu().numpy()
    assert np.array_equal(a_lf, a_h)


@pytest.mark.parametrize("cfg", ["C4"])
def test_accel_only_parity_sampled(cfg):
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    idx = sample_indices(x, n_stride=4096)
    a, _ = lf_forces(m, x, v, c.eps)
    ao, _ = oracle.forces(m, x, v, eps2_of(c.eps), idx=idx)
    assert max_rel(a[:, idx], ao) <= TOL_ACC


@pytest.mark.parametrize("cfg,every", [("C1", 1), ("C2", 20)])
def test_leapfrog_trajectory_and_drift(cfg, every):
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    e2 = eps2_of(c.eps)
    g = [(x, v)]
    with binding.NBody(m, x, v, eps=c.eps, dt=c.dt, integrator="leapfrog") as s:
        done = 0
        while done < c.steps:
            s.step(every)
            done += every
            xs, vs = s.state()
            g.append((xs.cpu().numpy(), vs.cpu().numpy()))
    o = [(x, v)]
    acc = None
    xo, vo = x, v
    for _ in range(c.steps // every):
        xo, vo, acc = oracle.leapfrog(m, xo, vo, e2, c.dt, every, acc=acc)
        o.append((xo, vo))
    Eg = [sum(oracle.energy(m, a, b, e2)) for a, b in g]
    Eo = [sum(oracle.energy(m, a, b, e2)) for a, b in o]
    Dg = max(abs(e - Eg[0]) / abs(Eg[0]) for e in Eg)
    Do = max(abs(e - Eo[0]) / abs(Eo[0]) for e in Eo)
    assert Dg <= 2 * max(Do, 1e-11), (Dg, Do)
    dx = np.linalg.norm(g[-1][0] - o[-1][0], axis=0).max()
    dv = np.linalg.norm(g[-1][1] - o[-1][1], axis=0).max()
    assert dx <= (1e-9 if cfg == "C1" else 1e-6) and dv <= (1e-6 if cfg == "C1" else 1e-4), (dx, dv)


def test_leapfrog_kepler_gpu():
    """fp32 accelerations, fp64 KDK, eps = 0 guarded path: one period of e = 0.5 at dt ~ 1/1024,
    within 2x of the oracle's own (2nd-order) error against the closed form."""
    m, x, v = inputs.kepler(0.5)
    nsteps = 6434
    dt = 2 * math.pi / nsteps
    with binding.NBody(m, x, v, eps=0.0, dt=dt, integrator="leapfrog") as s:
        s.step(nsteps)
        xs = s.state()[0].cpu().numpy()
    xo, _, _ = oracle.leapfrog(m, x, v, 0.0, dt, nsteps)
    target = np.array([0.5, 0.0, 0.0])
    eg = np.linalg.norm((xs[:, 1] - xs[:, 0]) - target)
    eo = np.linalg.norm((xo[:, 1] - xo[:, 0]) - target)
    assert eg <= 2 * eo + 1e-6, (eg, eo)


def test_leapfrog_loopback_bit_identical():
    m, x, v = inputs.parity_round(*inputs.plummer(9000, 31))
    out = []
    for world in (1, 4):
        with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024, integrator="leapfrog", world=world,
                           loopback=world > 1) as s:
            s.step(3)
            out.append([t.cpu().numpy() for t in s.state()])
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
