"""Pins for the fp64 oracle against things other than itself.

Each test cites what fixes the expected value: a closed form, an invariant,
an independent high-precision definition (mpmath derivative of the softened
potential / of the acceleration along the trajectory), or a convergence law.
Together they are chosen so that a dropped term, a wrong sign, a wrong power
of r or a transposed operand in oracle.c fails at least one of them.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import inputs


# ---------------------------------------------------------------- closed forms

def test_two_body_unit_case():
    """SPEC S:313-314 two-body case: a1 = (+1,0,0), a2 = (-1,0,0), jerk 0; with
    v2 = (0,1,0) the jerk is j1 = m2 w / r^3 = (0,1,0) since d.w = 0."""
    m = np.array([1.0, 1.0])
    x = np.array([[0.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    v = np.zeros((3, 2))
    a, j = oracle.forces(m, x, v, eps2=0.0)
    assert np.array_equal(a, np.array([[1.0, -1.0], [0.0, 0.0], [0.0, 0.0]]))
    assert np.array_equal(j, np.zeros((3, 2)))
    v[1, 1] = 1.0
    a, j = oracle.forces(m, x, v, eps2=0.0)
    assert np.array_equal(j[:, 0], [0.0, 1.0, 0.0])
    assert np.array_equal(j[:, 1], [0.0, -1.0, 0.0])


def test_equilateral_triangle():
    """side 1, unit masses -> |a_i| = sqrt(3), pointing at the centroid."""
    m = np.ones(3)
    pts = np.array([[0.0, 1.0, 0.5], [0.0, 0.0, math.sqrt(3) / 2], [0.0, 0.0, 0.0]])
    a, _ = oracle.forces(m, pts, np.zeros((3, 3)), eps2=0.0)
    c = pts.mean(axis=1)
    for i in range(3):
        assert abs(np.linalg.norm(a[:, i]) - math.sqrt(3)) < 1e-14
        u = (c - pts[:, i]) / np.linalg.norm(c - pts[:, i])
        assert np.dot(a[:, i], u) / np.linalg.norm(a[:, i]) > 1 - 1e-14


def test_kepler_energy_closed_form():
    """Two-body energy: E = -G m1 m2 / (2a), PE = -G m1 m2 / r_p (softening 0)."""
    for e in (0.0, 0.5, 0.9):
        m, x, v = inputs.kepler(e)
        ke, pe = oracle.energy(m, x, v, eps2=0.0)
        assert abs(pe - (-0.25 / (1.0 - e))) < 1e-15
        assert abs((ke + pe) - (-0.125)) < 1e-14


def test_softened_pair_energy_closed_form():
    """PE of one softened pair = -G m1 m2 / sqrt(r^2 + eps^2)."""
    m = np.array([2.0, 3.0])
    x = np.array([[0.0, 3.0], [0.0, 4.0], [0.0, 0.0]])
    ke, pe = oracle.energy(m, x, np.zeros((3, 2)), eps2=11.0, G=0.5)
    assert ke == 0.0
    assert abs(pe - (-0.5 * 6.0 / 6.0)) < 1e-15


# ------------------------------------------- independent high-precision definitions

def _mp_potential_grad(m, x, i, eps2, G=1.0):
    """a_i = -grad_i Phi, Phi_i = -sum_j G m_j / sqrt(|x_j - x_i|^2 + eps^2) (mpmath diff)."""
    n = len(m)

    def phi(c, t):
        xi = [mp.mpf(x[k][i]) for k in range(3)]
        xi[c] += t
        s = mp.mpf(0)
        for j in range(n):
            if j == i:
                continue
            r2 = sum((mp.mpf(x[k][j]) - xi[k]) ** 2 for k in range(3)) + mp.mpf(eps2)
            s -= G * mp.mpf(m[j]) / mp.sqrt(r2)
        return s

    return [-mp.diff(lambda t: phi(c, t), 0) for c in range(3)]


def _mp_accel(m, x, v, i, eps2, t, G=1.0):
    n = len(m)
    out = [mp.mpf(0)] * 3
    xi = [mp.mpf(x[k][i]) + t * mp.mpf(v[k][i]) for k in range(3)]
    for j in range(n):
        if j == i:
            continue
        d = [mp.mpf(x[k][j]) + t * mp.mpf(v[k][j]) - xi[k] for k in range(3)]
        s = sum(dk * dk for dk in d) + mp.mpf(eps2)
        f = G * mp.mpf(m[j]) / s ** mp.mpf(1.5)
        out = [out[k] + f * d[k] for k in range(3)]
    return out


@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_vs_mpmath_small_n(seed):
    """N <= 8: oracle a vs -grad of the softened potential and jerk vs d a/dt
    along x + v t, both by mpmath numerical differentiation at 40 digits."""
    mp.mp.dps = 40
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 9))
    eps2 = 0.0 if seed % 2 == 0 else 1e-2
    m = rng.random(n) + 0.1
    x = rng.standard_normal((3, n))
    v = rng.standard_normal((3, n))
    a, j = oracle.forces(m, x, v, eps2=eps2)
    for i in range(n):
        ga = np.array([float(t) for t in _mp_potential_grad(m, x, i, eps2)])
        assert np.linalg.norm(a[:, i] - ga) <= 1e-14 * np.linalg.norm(ga)
        gj = np.array([float(mp.diff(lambda t: _mp_accel(m, x, v, i, eps2, t)[c], 0))
                       for c in range(3)])
        assert np.linalg.norm(j[:, i] - gj) <= 1e-13 * np.linalg.norm(gj)


def test_jerk_finite_difference():
    """jerk = central difference of a along x + v t, h = 1e-6 (rel 1e-7)."""
    m, x, v = inputs.plummer(64, 7)
    eps2 = 1e-4
    _, j = oracle.forces(m, x, v, eps2)
    h = 1e-6
    ap, _ = oracle.forces(m, x + h * v, v, eps2)
    am, _ = oracle.forces(m, x - h * v, v, eps2)
    fd = (ap - am) / (2 * h)
    rel = np.linalg.norm(j - fd, axis=0) / np.linalg.norm(j, axis=0)
    assert rel.max() < 1e-7


# ------------------------------------------------------------------- invariants

def test_momentum_conservation():
    """Newton's third law: sum_i m_i a_i = 0 (and sum m_i j_i = 0) to round-off."""
    m, x, v = inputs.make("C1")
    a, j = oracle.forces(m, x, v, eps2=np.float32(1e-4))
    for q in (a, j):
        res = np.linalg.norm(q @ m) / np.sum(m * np.linalg.norm(q, axis=0))
        assert res < 1e-13


def test_momentum_two_cluster_mass_spectrum():
    m, x, v = inputs.two_cluster(2048, 11)
    m, x, v = inputs.parity_round(m, x, v)
    a, _ = oracle.forces(m, x, v, eps2=1e-6)
    res = np.linalg.norm(a @ m) / np.sum(m * np.linalg.norm(a, axis=0))
    assert res < 1e-13


def test_translation_invariance_bitexact():
    """SPEC S:413 (corrected): on fp32-representable inputs x + 0.5 is exact in fp64,
    so all differences, and hence a and j, are bit-identical."""
    m, x, v = inputs.parity_round(*inputs.plummer(512, 3))
    assert np.all((np.abs(x) >= 2.0 ** -29) | (x == 0))
    a0, j0 = oracle.forces(m, x, v, 1e-4)
    a1, j1 = oracle.forces(m, x + 0.5, v, 1e-4)
    assert np.array_equal(a0, a1) and np.array_equal(j0, j1)


def test_scaling_law():
    """x -> s x, eps -> s eps, v = 0 gives a -> a / s^2, j = 0 (exact for s = 2)."""
    m, x, v = inputs.plummer(256, 5)
    v = np.zeros_like(v)
    a0, j0 = oracle.forces(m, x, v, 1e-4)
    a2, j2 = oracle.forces(m, 2 * x, v, 4e-4)
    assert np.array_equal(a2, a0 / 4) and not j2.any() and not j0.any()
    a3, _ = oracle.forces(m, 3 * x, v, 9e-4)
    assert np.max(np.abs(a3 * 9 - a0)) <= 1e-14 * np.max(np.abs(a0))


def test_shell_theorem_plummer():
    """Spherical symmetry: shell-averaged radial acceleration of a Plummer sphere
    equals G M(<r) / r^2 with the empirical enclosed mass (<= 1% per shell)."""
    m, x, v = inputs.make("C2")
    a, _ = oracle.forces(m, x, v, np.float32(1e-6))
    r = np.linalg.norm(x, axis=0)
    ar = -np.sum(a * x, axis=0) / r
    order = np.argsort(r)
    menc = np.empty_like(r)
    menc[order] = np.cumsum(m[order]) - m[order]
    newton = menc / r ** 2
    shells = np.array_split(order[200:-200], 18)
    for s in shells:
        assert abs(ar[s].mean() / newton[s].mean() - 1) < 0.01


def test_thread_count_invariance():
    """results do not depend on the thread count (bit-identical)."""
    m, x, v = inputs.make("C1")
    nt = oracle.threads()
    try:
        oracle.set_threads(1)
        a1, j1 = oracle.forces(m, x, v, 1e-4)
        e1 = oracle.energy(m, x, v, 1e-4)
        oracle.set_threads(max(nt, 4))
        a4, j4 = oracle.forces(m, x, v, 1e-4)
        e4 = oracle.energy(m, x, v, 1e-4)
    finally:
        oracle.set_threads(nt)
    assert np.array_equal(a1, a4) and np.array_equal(j1, j4) and e1 == e4


def test_index_subset_matches_full():
    m, x, v = inputs.plummer(300, 9)
    a, j = oracle.forces(m, x, v, 1e-4)
    idx = np.array([299, 0, 17, 17, 150])
    a_s, j_s = oracle.forces(m, x, v, 1e-4, idx=idx)
    assert np.array_equal(a_s, a[:, idx]) and np.array_equal(j_s, j[:, idx])


def test_coincident_pair_is_an_error():
    """eps = 0 with two coincident distinct particles is refused, naming the pair."""
    m = np.ones(3)
    x = np.array([[0.0, 1.0, 1.0], [0.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    with pytest.raises(oracle.OracleError, match=r"\(1, 2\)"):
        oracle.forces(m, x, np.zeros((3, 3)), 0.0)
    a, _ = oracle.forces(m, x, np.zeros((3, 3)), 1e-6)  # softened: fine
    assert np.all(np.isfinite(a))


# ------------------------------------------------------------------- integrator

def _kepler_rel(e, t, a=1.0):
    """Closed-form relative position of a Kepler orbit from pericentre (G M = 1)."""
    n_mean = 1.0 / a ** 1.5
    M = n_mean * t
    E = M if e < 0.8 else math.pi
    for _ in range(100):
        E -= (E - e * math.sin(E) - M) / (1 - e * math.cos(E))
    return np.array([a * (math.cos(E) - e), a * math.sqrt(1 - e * e) * math.sin(E), 0.0])


def _kepler_err(e, nsteps, frac=1.0):
    m, x, v = inputs.kepler(e)
    T = 2 * math.pi
    dt = T / nsteps
    k = int(round(frac * nsteps))
    x1, v1, _, _ = oracle.hermite(m, x, v, 0.0, dt, k)
    rel = x1[:, 1] - x1[:, 0]
    return np.linalg.norm(rel - _kepler_rel(e, k * dt)), (m, x, v, x1, v1)


def test_kepler_closed_form_one_period():
    """X7 / SPEC S:458: after one period the Hermite orbit returns to the closed form."""
    err0, _ = _kepler_err(0.0, 6434)   # dt ~ 1/1024
    err5, _ = _kepler_err(0.5, 6434)
    err9, _ = _kepler_err(0.9, 6434)
    assert err0 < 1e-11
    assert err5 < 1e-9
    assert err9 < 1e-4


def test_kepler_mid_orbit_closed_form():
    err, _ = _kepler_err(0.5, 6434, frac=0.37)
    assert err < 1e-9


def test_hermite_fourth_order_convergence():
    """Halving dt reduces the one-period error by ~2^4 (accept [12, 20])."""
    for e in (0.0, 0.5):
        e1, _ = _kepler_err(e, 1600)
        e2, _ = _kepler_err(e, 3200)
        assert 12.0 <= e1 / e2 <= 20.0, (e, e1, e2)


def test_hermite_energy_conservation_kepler():
    _, (m, x, v, x1, v1) = _kepler_err(0.5, 6434)
    E0 = sum(oracle.energy(m, x, v, 0.0))
    E1 = sum(oracle.energy(m, x1, v1, 0.0))
    assert abs((E1 - E0) / E0) < 1e-9


def test_free_particle():
    """with a negligible partner mass, r(t) = r0 + v0 t to fp64 rounding."""
    m = np.array([1.0, 1e-300])
    x = np.array([[0.0, 5.0], [0.0, 0.0], [0.0, 0.0]])
    v = np.array([[0.3, 0.0], [-0.2, 0.0], [0.1, 0.0]])
    x1, v1, _, _ = oracle.hermite(m, x, v, 0.0, 1.0 / 64, 64)
    assert np.max(np.abs(x1[:, 0] - (x[:, 0] + v[:, 0]))) < 1e-14
    assert np.array_equal(v1[:, 0], v[:, 0])


def test_hermite_chaining():
    """k steps then k more (passing a0, j0 through) equals 2k steps bit-for-bit."""
    m, x, v = inputs.make("C1")
    xa, va, aa, ja = oracle.hermite(m, x, v, 1e-4, 1 / 1024, 4)
    xb, vb, ab, jb = oracle.hermite(m, xa, va, 1e-4, 1 / 1024, 4, acc=aa, jerk=ja)
    xc, vc, ac, jc = oracle.hermite(m, x, v, 1e-4, 1 / 1024, 8)
    assert np.array_equal(xb, xc) and np.array_equal(vb, vc) and np.array_equal(ab, ac)


def _kepler_state(e, t):
    """Closed-form relative position and velocity (G M = 1, a = 1) at time t after pericentre."""
    E = t
    for _ in range(100):
        E -= (E - e * math.sin(E) - t) / (1 - e * math.cos(E))
    Ed = 1.0 / (1 - e * math.cos(E))
    r = np.array([math.cos(E) - e, math.sqrt(1 - e * e) * math.sin(E), 0.0])
    w = np.array([-math.sin(E) * Ed, math.sqrt(1 - e * e) * math.cos(E) * Ed, 0.0])
    return r, w


@pytest.mark.parametrize("e,t0", [(0.0, 0.3), (0.5, 1.0), (0.5, 2.5)])
def test_hermite_local_error_orders(e, t0):
    """One step from an exact Kepler state.  The corrector is the double / single
    integral of the cubic Hermite interpolant of a(t) through (a0, j0, a1, j1), whose
    error is a''''(xi) s^2 (s - dt)^2 / 4!; integrating gives a local position error
    O(dt^6) and a local velocity error O(dt^5) (ratios 64 and 32 per halving of dt).
    A wrong coefficient on any corrector term drops the position order to dt^5."""
    def step_err(dt):
        r, w = _kepler_state(e, t0)
        m = np.array([0.5, 0.5])
        x = np.stack([-r / 2, r / 2], 1)
        v = np.stack([-w / 2, w / 2], 1)
        x1, v1, _, _ = oracle.hermite(m, x, v, 0.0, dt, 1)
        r1, w1 = _kepler_state(e, t0 + dt)
        return (np.linalg.norm((x1[:, 1] - x1[:, 0]) - r1),
                np.linalg.norm((v1[:, 1] - v1[:, 0]) - w1))
    ex1, ev1 = step_err(1 / 16)
    ex2, ev2 = step_err(1 / 32)
    assert 50 <= ex1 / ex2 <= 80, ex1 / ex2
    assert 26 <= ev1 / ev2 <= 38, ev1 / ev2


# ------------------------------------------------------- leapfrog (NEXT f1)

def _kepler_lf_err(e, nsteps):
    m, x, v = inputs.kepler(e)
    dt = 2 * math.pi / nsteps
    x1, v1, _ = oracle.leapfrog(m, x, v, 0.0, dt, nsteps)
    rel = x1[:, 1] - x1[:, 0]
    return np.linalg.norm(rel - _kepler_rel(e, nsteps * dt)), (m, x, v, x1, v1)


def test_leapfrog_second_order_convergence():
    """KDK is 2nd order: halving dt divides the one-period Kepler error by ~4."""
    for e in (0.0, 0.5):
        e1, _ = _kepler_lf_err(e, 2000)
        e2, _ = _kepler_lf_err(e, 4000)
        assert 3.5 <= e1 / e2 <= 4.5, (e, e1, e2)


def test_leapfrog_time_reversible():
    """KDK is time-symmetric: n steps with +dt then n with -dt return to the start."""
    m, x, v = inputs.make("C1")
    x1, v1, a1 = oracle.leapfrog(m, x, v, 1e-4, 1 / 512, 20)
    x2, v2, _ = oracle.leapfrog(m, x1, v1, 1e-4, -1 / 512, 20, acc=a1)
    assert np.max(np.abs(x2 - x)) < 1e-12 and np.max(np.abs(v2 - v)) < 1e-11


def test_leapfrog_local_error_order():
    """One KDK step from an exact Kepler state: local position error O(dt^3) (ratio 8)."""
    def err(dt):
        r, w = _kepler_state(0.5, 1.0)
        m = np.array([0.5, 0.5])
        x = np.stack([-r / 2, r / 2], 1)
        v = np.stack([-w / 2, w / 2], 1)
        x1, _, _ = oracle.leapfrog(m, x, v, 0.0, dt, 1)
        r1, _ = _kepler_state(0.5, 1.0 + dt)
        return np.linalg.norm((x1[:, 1] - x1[:, 0]) - r1)
    ratio = err(1 / 32) / err(1 / 64)
    assert 7.0 <= ratio <= 9.0, ratio


def test_leapfrog_free_particle_and_energy():
    m = np.array([1.0, 1e-300])
    x = np.array([[0.0, 5.0], [0.0, 0.0], [0.0, 0.0]])
    v = np.array([[0.3, 0.0], [-0.2, 0.0], [0.1, 0.0]])
    x1, v1, _ = oracle.leapfrog(m, x, v, 0.0, 1.0 / 64, 64)
    assert np.max(np.abs(x1[:, 0] - (x[:, 0] + v[:, 0]))) < 1e-14
    _, (m, x, v, x1, v1) = _kepler_lf_err(0.5, 6434)
    E0 = sum(oracle.energy(m, x, v, 0.0))
    E1 = sum(oracle.energy(m, x1, v1, 0.0))
    assert abs((E1 - E0) / E0) < 1e-5      # symplectic: bounded, O(dt^2) energy error


# ------------------------------------------------------- block time steps (R#28)

def _kep_rel_e(e, t):
    E = t if e < 0.8 else math.pi
    for _ in range(100):
        E -= (E - e * math.sin(E) - t) / (1 - e * math.cos(E))
    return np.array([math.cos(E) - e, math.sqrt(1 - e * e) * math.sin(E), 0.0])


def test_block_reduces_to_shared_step_bitwise():
    """With eta, eta_s -> infinity every particle stays on level 0 (dt = dt_max), and the
    block scheme is the shared-dt Hermite scheme of R#3 operation for operation."""
    m, x, v = inputs.make("C1")
    xs, vs, as_, js = oracle.hermite(m, x, v, 1e-4, 1 / 1024, 4)
    xb, vb, ab, jb, lev, st, _ = oracle.hermite_block(m, x, v, 1e-4, 1 / 1024, 4, eta=1e30,
                                                      eta_s=1e30)
    assert np.array_equal(xs, xb) and np.array_equal(vs, vb)
    assert np.array_equal(as_, ab) and np.array_equal(js, jb)
    assert lev.max() == 0 and st == (4, 4 * 1024)


def test_block_startup_level_closed_form():
    """Circular binary (omega = 1): |a| / |j| = 1 / omega, so eta_s |a|/|j| = eta_s and the
    startup level is the largest 2^-k <= eta_s: k = 7 for eta_s = 0.01, dt_max = 1."""
    m, x, v = inputs.kepler(0.0)
    a, j = oracle.forces(m, x, v, 0.0)
    lev, crit = oracle.block_init_levels(a, j, 1.0, 30, 0.01)
    assert np.allclose(crit, 0.01, rtol=1e-14, atol=0)
    assert list(lev) == [7, 7]
    lev, _ = oracle.block_init_levels(a, j, 1.0, 5, 0.01)     # capped at kmax
    assert list(lev) == [5, 5]


def test_block_aarseth_criterion_circular_orbit():
    """Aarseth criterion on a circular orbit: |a^(n)| = A omega^n, so
    dt = sqrt(eta (2 A^2 omega^2) / (2 A^2 omega^4)) = sqrt(eta) / omega (closed form).
    The oracle's value (from Hermite-interpolated a^(2), a^(3)) must match to O(dt^2)."""
    m, x, v = inputs.kepler(0.0)
    for eta in (0.01, 0.0025):
        _, _, _, _, lev, _, crit = oracle.hermite_block(m, x, v, 0.0, 1.0, 1, eta=eta,
                                                        eta_s=0.01, kmax=30)
        assert np.allclose(crit, math.sqrt(eta), rtol=1e-2, atol=0), (eta, crit)
        # the level that the criterion selects: largest 2^-k <= sqrt(eta)
        assert list(lev) == [int(math.ceil(-math.log2(math.sqrt(eta))))] * 2


@pytest.mark.parametrize("e", [0.5, 0.9])
def test_block_kepler_fourth_order_in_sqrt_eta(e):
    """Adaptive Hermite: dt ~ sqrt(eta), error ~ dt^4 ~ eta^2: eta / 4 halves every step
    and divides the one-period error (vs the Kepler closed form) by ~16 (accept [10, 24])."""
    errs, steps = [], []
    for eta in (0.004, 0.001):
        m, x, v = inputs.kepler(e)
        xb, _, _, _, _, st, _ = oracle.hermite_block(m, x, v, 0.0, 2 * math.pi / 16, 16, eta=eta,
                                                     eta_s=0.01, kmax=30)
        errs.append(np.linalg.norm((xb[:, 1] - xb[:, 0]) - _kep_rel_e(e, 2 * math.pi)))
        steps.append(st[0])
    assert 10.0 <= errs[0] / errs[1] <= 24.0, errs
    assert 1.8 <= steps[1] / steps[0] <= 2.2, steps
    assert errs[1] < (3e-7 if e == 0.5 else 3e-6)


def test_block_plummer_converges_to_small_shared_step():
    """N = 32 Plummer with a spread of levels (particles predicted to each other's block
    times): the block solution converges at 4th order in dt ~ sqrt(eta) to a shared-dt
    reference at dt = 2^-14 (a wrong predictor or corrector for unsynchronised particles
    breaks the ratio)."""
    m, x, v = inputs.plummer(32, 11)
    xr, _, _, _ = oracle.hermite(m, x, v, 1e-4, 2.0 ** -14, 2 ** 12)
    errs = []
    for eta in (0.02, 0.005):
        xb, _, _, _, lev, _, _ = oracle.hermite_block(m, x, v, 1e-4, 1 / 16, 4, eta=eta,
                                                      eta_s=0.01, kmax=30)
        assert lev.max() - lev.min() >= 3        # genuinely individual steps
        errs.append(np.max(np.abs(xb - xr)))
    assert 10.0 <= errs[0] / errs[1] <= 24.0, errs
    assert errs[1] < 1e-8


def test_block_chaining_and_energy():
    """k cycles then k more (passing acc, jerk, level) equals 2k cycles bit for bit (call
    boundaries are multiples of dt_max); energy conserved to ~eta^2."""
    m, x, v = inputs.plummer(256, 12)
    kw = dict(eta=0.02, eta_s=0.01, kmax=30)
    xa, va, aa, ja, la, sa, _ = oracle.hermite_block(m, x, v, 1e-4, 1 / 32, 3, **kw)
    xb, vb, _, _, lb, sb, _ = oracle.hermite_block(m, xa, va, 1e-4, 1 / 32, 3, acc=aa, jerk=ja,
                                                   level=la, **kw)
    xc, vc, _, _, lc, sc, _ = oracle.hermite_block(m, x, v, 1e-4, 1 / 32, 6, **kw)
    assert np.array_equal(xb, xc) and np.array_equal(vb, vc) and np.array_equal(lb, lc)
    assert (sa[0] + sb[0], sa[1] + sb[1]) == sc
    E0 = sum(oracle.energy(m, x, v, 1e-4))
    E1 = sum(oracle.energy(m, xc, vc, 1e-4))
    assert abs((E1 - E0) / E0) < 5e-8      # measured 1.3e-8


def _kepler_body_accel_derivs(e, t, orders):
    """Exact d^k a/dt^k of body 1 of inputs.kepler(e) (m = 1/2 each, G = 1): body 1 feels
    -(1/2) r / |r|^3 with r the closed-form relative orbit; 40-digit mpmath derivatives."""
    mp.mp.dps = 40

    def acc1(s, c):
        E = mp.mpf(s)
        for _ in range(80):
            E -= (E - e * mp.sin(E) - s) / (1 - e * mp.cos(E))
        r = [mp.cos(E) - e, mp.sqrt(1 - e * e) * mp.sin(E)]
        rn = mp.sqrt(r[0] ** 2 + r[1] ** 2)
        return -r[c] / rn ** 3 * 0.5
    return [np.array([float(mp.diff(lambda s: acc1(s, c), t, k)) for c in range(2)])
            for k in orders]


def test_block_interpolated_derivatives_converge():
    """The criterion's a^(2)(t_next) = a2 + dt a3 and a^(3) = a3 are the 2nd and 3rd
    derivatives of the Hermite cubic through (a0, j0, a1, j1): against the exact Kepler
    derivatives at t_next they converge as dt^2 and dt (halving dt: ratios 4 and 2).
    Using a2 (the value at the start of the step) instead would converge only as dt."""
    ex2, ex3 = _kepler_body_accel_derivs(0.5, 1.0, (2, 3))
    e2, e3 = [], []
    for eta in (1e-3, 2.5e-4):      # eta / 4 -> one level finer (dt / 2)
        m, x, v = inputs.kepler(0.5)
        out = oracle.hermite_block(m, x, v, 0.0, 1.0, 1, eta=eta, eta_s=0.01, kmax=30,
                                   derivs=True)
        d2, d3 = out[7], out[8]
        e2.append(np.linalg.norm(d2[:2, 1] - ex2) / np.linalg.norm(ex2))
        e3.append(np.linalg.norm(d3[:2, 1] - ex3) / np.linalg.norm(ex3))
        assert abs(d2[2, 1]) < 1e-12 and abs(d3[2, 1]) < 1e-9      # planar orbit
    assert 3.2 <= e2[0] / e2[1] <= 4.8, e2
    assert 1.6 <= e3[0] / e3[1] <= 2.4, e3
    assert e2[1] < 2e-5 and e3[1] < 1e-2


def test_block_level_drops_several_levels_at_once():
    """eta_s = 1 starts the circular binary at dt = dt_max = 1; after that one step the
    Aarseth value is ~sqrt(eta) = 0.01 and the block rule halves repeatedly (not once):
    level 7 (dt = 2^-7 <= 0.013 < 2^-6)."""
    m, x, v = inputs.kepler(0.0)
    _, _, _, _, lev, st, crit = oracle.hermite_block(m, x, v, 0.0, 1.0, 1, eta=1e-4, eta_s=1.0,
                                                     kmax=30)
    assert st == (1, 2)
    assert 2.0 ** -7 <= crit[0] < 2.0 ** -6
    assert list(lev) == [7, 7]
