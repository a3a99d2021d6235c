"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

All inputs are seeded and synthetic (paper_2509_19294_b200.inputs) and, for
force parity, fp32-representable (R#9), so both sides see identical values.
Bars: max per-particle relative acceleration error 1e-5 (BASELINE.json), jerk
1e-4 (R#12), the paper's 0.05 % / 0.2 % of the typical magnitude,
energy drift within 2x the oracle's own drift (BASELINE.json, R#14).
"""
import math

import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import binding, inputs
from metrics import (TOL_ACC, TOL_JERK, TOL_PAPER_ACC, TOL_PAPER_JERK, max_rel,
                     momentum_residual, paper_norm, sample_indices)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def eps2_of(eps):
    return float(np.float32(eps * eps))   # R#18: both paths use fp32(eps^2)


def gpu_forces(m, x, v, eps, **kw):
    with binding.NBody(m, x, v, eps=eps, dt=1.0 / 1024, **kw) as sim:
        a, j = sim.forces()
        sim.sync()
        return a.cpu().numpy(), j.cpu().numpy()


def check_forces(m, x, v, eps, idx=None, return_all=False, **kw):
    a_all, j_all = gpu_forces(m, x, v, eps, **kw)
    ao, jo = oracle.forces(m, x, v, eps2_of(eps), idx=idx)
    a, j = (a_all[:, idx], j_all[:, idx]) if idx is not None else (a_all, j_all)
    ea, ej = max_rel(a, ao), max_rel(j, jo)
    pa, pj = paper_norm(a, ao), paper_norm(j, jo)
    assert ea <= TOL_ACC, ea
    assert ej <= TOL_JERK, ej
    assert pa <= TOL_PAPER_ACC and pj <= TOL_PAPER_JERK, (pa, pj)
    return (a_all, j_all) if return_all else (ea, ej)


# --------------------------------------------------------------- closed forms

def test_two_body_closed_form_eps0():
    """SPEC S:313-314 with eps = 0 (guarded j == i path): a = (+-1, 0, 0), j1 = (0, 1, 0)."""
    m = np.array([1.0, 1.0])
    x = np.array([[0.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    v = np.array([[0.0, 0.0], [0.0, 1.0], [0.0, 0.0]])
    a, j = gpu_forces(m, x, v, 0.0)
    assert np.allclose(a, [[1, -1], [0, 0], [0, 0]], atol=1e-6, rtol=0)
    assert np.allclose(j, [[0, 0], [1, -1], [0, 0]], atol=1e-6, rtol=0)


def test_equilateral_triangle():
    m = np.ones(3)
    pts = np.array([[0.0, 1.0, 0.5], [0.0, 0.0, math.sqrt(3) / 2], [0.0, 0.0, 0.0]])
    a, _ = gpu_forces(m, pts, np.zeros((3, 3)), 0.0)
    assert np.allclose(np.linalg.norm(a, axis=0), math.sqrt(3), rtol=1e-6)


# ------------------------------------------------------------ force parity

@pytest.mark.parametrize("n", [2, 3, 255, 256, 257, 511, 1000, 1025, 3000, 4097])
def test_ragged_sizes(n):
    m, x, v = inputs.parity_round(*inputs.uniform_cube(n, 1000 + n))
    check_forces(m, x, v, 1e-2)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_forces_all_particles(cfg):
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    check_forces(m, x, v, c.eps)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_config_forces_sampled(cfg):
    """Full-size configs in the bench's launch configuration, R#11 sample of i."""
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    idx = sample_indices(x, n_stride=4096 if cfg == "C5" else 8192)
    check_forces(m, x, v, c.eps, idx=idx)


def test_max_size_n4m_sampled():
    """Beyond the largest config: N = 4 194 304 (2^22, 4x C5; 26 GB of device state, the
    canonical chunk 32 768 j = 128 tiles) in the bench's launch configuration, one force
    evaluation (1.76e13 interactions, ~14 s), R#11 sample against the oracle at the 1e-5 /
    1e-4 bars, and momentum conservation over every particle."""
    n = 1 << 22
    m, x, v = inputs.parity_round(*inputs.plummer(n, 222))
    idx = sample_indices(x, n_stride=1024, n_special=128)
    a, j = check_forces(m, x, v, 5e-4, idx=idx, return_all=True)
    assert momentum_residual(m, a) < 1e-6 and momentum_residual(m, j) < 1e-5


def test_large_ragged_n_sampled_and_sharded():
    """N = 300 001 (odd; chunk = 2560 j, the last chunk ragged; padding packets in the last
    tile): R#11 sample against the oracle, and loopback world = 3 (ragged shards) equal to
    world = 1 bit for bit."""
    n = 300001
    m, x, v = inputs.parity_round(*inputs.plummer(n, 41))
    idx = sample_indices(x, n_stride=2048, n_special=128)
    check_forces(m, x, v, 1e-3, idx=idx)
    a1, j1 = gpu_forces(m, x, v, 1e-3)
    a3, j3 = gpu_forces(m, x, v, 1e-3, world=3, loopback=True)
    assert np.array_equal(a1, a3) and np.array_equal(j1, j3)


def test_two_cluster_small_all_particles():
    m, x, v = inputs.parity_round(*inputs.two_cluster(8192, 4))
    check_forces(m, x, v, 1e-3)


def test_momentum_conservation_gpu():
    m, x, v = inputs.make("C2")
    a, j = gpu_forces(m, x, v, 1e-3)
    assert momentum_residual(m, a) < 1e-6
    assert momentum_residual(m, j) < 1e-5


@pytest.mark.parametrize("jchunks", [1, 7, 128])
def test_jchunk_counts(jchunks):
    m, x, v = inputs.parity_round(*inputs.plummer(5000, 8))
    check_forces(m, x, v, 1e-3, jchunks=jchunks)


# ----------------------------------------------------- determinism / sharding

def test_loopback_shards_bit_identical():
    """Results do not depend on the number of i-shards: loopback
    world = 2, 3, 8 (ragged, with an empty tail rank) equals world = 1 bit-for-bit."""
    n = 20000
    m, x, v = inputs.parity_round(*inputs.plummer(n, 21))
    ref = None
    for world in (1, 2, 3, 8):
        with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024, world=world, loopback=world > 1) as s:
            a, j = s.forces()
            s.step(3)
            xs, vs = s.state()
            got = [t.cpu().numpy() for t in (a, j, xs, vs)]
        if ref is None:
            ref = got
        else:
            for g, r in zip(got, ref):
                assert np.array_equal(g, r), world


def test_tiny_n_many_shards():
    m, x, v = inputs.parity_round(*inputs.uniform_cube(300, 5))
    a1, j1 = gpu_forces(m, x, v, 1e-2)
    a3, j3 = gpu_forces(m, x, v, 1e-2, world=3, loopback=True)   # rank 2 owns nothing
    assert np.array_equal(a1, a3) and np.array_equal(j1, j3)


def test_nccl_single_rank_communicator():
    """world = 1 with an NCCL communicator exercises the exchange path on one GPU."""
    m, x, v = inputs.make("C1")
    ref = gpu_forces(m, x, v, 1e-2)
    got = gpu_forces(m, x, v, 1e-2, nccl_id=binding.nccl_unique_id())
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_repeat_runs_bit_identical():
    m, x, v = inputs.make("C1")
    r1 = gpu_forces(m, x, v, 1e-2)
    r2 = gpu_forces(m, x, v, 1e-2)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])


# ------------------------------------------------------------------ energy

@pytest.mark.parametrize("which", ["C1", "C2", "cluster"])
def test_energy_matches_oracle(which):
    if which == "cluster":
        m, x, v = inputs.parity_round(*inputs.two_cluster(4096, 9))
        eps = 1e-3
    else:
        m, x, v = inputs.make(which)
        eps = inputs.CONFIGS[which].eps
    with binding.NBody(m, x, v, eps=eps, dt=1 / 1024) as s:
        ke, pe = s.energy()
    ko, po = oracle.energy(m, x, v, eps2_of(eps))
    assert abs(ke - ko) <= 1e-13 * abs(ko)
    assert abs(pe - po) <= 1e-12 * abs(po)


# ------------------------------------------------------------- trajectories

def _drift(E):
    return max(abs(e - E[0]) / abs(E[0]) for e in E)


def run_gpu_traj(m, x, v, eps, dt, nsteps, every):
    states = [(x, v)]
    with binding.NBody(m, x, v, eps=eps, dt=dt) as s:
        done = 0
        while done < nsteps:
            k = min(every, nsteps - done)
            s.step(k)
            done += k
            xs, vs = s.state()
            s.sync()
            states.append((xs.cpu().numpy(), vs.cpu().numpy()))
    return states


def run_oracle_traj(m, x, v, eps, dt, nsteps, every):
    states = [(x, v)]
    acc = jerk = None
    done = 0
    while done < nsteps:
        k = min(every, nsteps - done)
        x, v, acc, jerk = oracle.hermite(m, x, v, eps2_of(eps), dt, k, acc=acc, jerk=jerk)
        done += k
        states.append((x, v))
    return states


@pytest.mark.parametrize("cfg,every,dx_tol,dv_tol", [("C1", 1, 1e-9, 1e-6), ("C2", 10, 1e-6, 1e-4),
                                                    ("C3", 5, 1e-6, 1e-4), ("C4", 10, 1e-6, 1e-4)])
def test_trajectory_and_energy_drift(cfg, every, dx_tol, dv_tol):
    """R#14/R#15: same fp32 IC, Hermite P(EC)^1 on both sides; trajectory deltas and
    drift D = max_k |E_k - E_0| / |E_0| with both energies from the oracle.  C4 is the
    bench workload (BASELINE.json configs[3]: 10 steps, every particle compared, the
    oracle trajectory ~5 min on the GPU box's host cores; C5 runs through
    scripts/c5_trajectory.py, profiles/r02_c5_trajectory.json)."""
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    g = run_gpu_traj(m, x, v, c.eps, c.dt, c.steps, every)
    o = run_oracle_traj(m, x, v, c.eps, c.dt, c.steps, every)
    e2 = eps2_of(c.eps)
    Eg = [sum(oracle.energy(m, xs, vs, e2)) for xs, vs in g]
    Eo = [sum(oracle.energy(m, xs, vs, e2)) for xs, vs in o]
    Dg, Do = _drift(Eg), _drift(Eo)
    assert Dg <= 2 * max(Do, 1e-11), (Dg, Do)
    dx = np.linalg.norm(g[-1][0] - o[-1][0], axis=0)
    dv = np.linalg.norm(g[-1][1] - o[-1][1], axis=0)
    assert dx.max() <= dx_tol and dv.max() <= dv_tol, (dx.max(), dv.max())
    print(f"{cfg}: D_gpu {Dg:.3e} D_orc {Do:.3e} ratio {Dg / Do if Do else float('nan'):.3f} "
          f"max dx {dx.max():.3e} median dx {np.median(dx):.3e} max dv {dv.max():.3e}")
    if cfg != "C1":
        assert np.median(dx) <= 1e-9
    # momentum: sum m v stays at its initial value
    p0 = v @ m
    p1 = g[-1][1] @ m
    assert np.max(np.abs(p1 - p0)) < 1e-9


def test_gpu_energy_tracks_oracle_energy_along_trajectory():
    c = inputs.CONFIGS["C1"]
    m, x, v = inputs.make("C1")
    with binding.NBody(m, x, v, eps=c.eps, dt=c.dt) as s:
        s.step(10)
        ke, pe = s.energy()
        xs, vs = s.state()
    ko, po = oracle.energy(m, xs.cpu().numpy(), vs.cpu().numpy(), eps2_of(c.eps))
    assert abs((ke + pe) - (ko + po)) <= 1e-12 * abs(ko + po)


@pytest.mark.parametrize("e,tol", [(0.0, 1e-5), (0.5, 1e-5)])
def test_kepler_one_period_gpu(e, tol):
    """X7: fp32 forces, fp64 Hermite, eps = 0 guarded path; one period at dt ~ 1/1024."""
    m, x, v = inputs.kepler(e)
    nsteps = 6434
    dt = 2 * math.pi / nsteps
    with binding.NBody(m, x, v, eps=0.0, dt=dt) as s:
        s.step(nsteps)
        xs, _ = s.state()
        xs = xs.cpu().numpy()
    rel = xs[:, 1] - xs[:, 0]
    target = np.array([1.0 - e, 0.0, 0.0])
    assert np.linalg.norm(rel - target) < tol


def test_state_round_trip_keeps_trajectory():
    """set_state(get_state(), keep_forces) through host memory is transparent."""
    m, x, v = inputs.make("C1")
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        s.step(4)
        ref = [t.cpu().numpy() for t in s.state()]
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        s.step(2)
        hx = np.empty((3, 1024))
        hv = np.empty((3, 1024))
        binding._check(binding.lib().nbody_get_state(s._ctx, hx.ctypes.data, hv.ctypes.data), s._ctx)
        s.set_state(hx, hv, keep_forces=True)
        s.step(2)
        got = [t.cpu().numpy() for t in s.state()]
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_host_pointer_inputs_and_outputs():
    m, x, v = inputs.make("C1")
    a_dev, j_dev = gpu_forces(m, x, v, 1e-2)
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        ha = np.empty((3, 1024))
        hj = np.empty((3, 1024))
        binding._check(binding.lib().nbody_compute_forces(s._ctx, ha.ctypes.data, hj.ctypes.data),
                       s._ctx)
    assert np.array_equal(ha, a_dev) and np.array_equal(hj, j_dev)


# ------------------------------------------------------------------- errors

def test_invalid_inputs_name_the_particle():
    m, x, v = inputs.make("C1")
    xb = x.copy()
    xb[1, 77] = np.nan
    with pytest.raises(binding.NBodyError, match="particle 77") as e:
        binding.NBody(m, xb, v, eps=1e-2, dt=1 / 1024)
    assert e.value.code == binding.NBODY_EINVAL
    mb = m.copy()
    mb[5] = 0.0
    with pytest.raises(binding.NBodyError, match="particle 5"):
        binding.NBody(mb, x, v, eps=1e-2, dt=1 / 1024)


def test_coincident_pair_eps0_is_reported_and_sticky():
    m = np.ones(4)
    x = np.array([[0.0, 1.0, 1.0, 3.0], [0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0]])
    s = binding.NBody(m, x, np.zeros((3, 4)), eps=0.0, dt=1 / 1024)
    s.forces()
    with pytest.raises(binding.NBodyError) as e:
        s.sync()
    assert e.value.code == binding.NBODY_ENONFINITE and "coincident" in str(e.value)
    with pytest.raises(binding.NBodyError) as e2:
        s.step(1)
    assert e2.value.code == binding.NBODY_ESTATE
    s.close()


def test_cuda_graph_replay_bit_identical(monkeypatch):
    """Steady-state steps replay a captured CUDA graph on a non-default stream; the
    result equals eager launches (NBODY_NO_GRAPH=1) bit for bit."""
    m, x, v = inputs.make("C1")
    out = []
    for no_graph in ("0", "1"):
        monkeypatch.setenv("NBODY_NO_GRAPH", no_graph)
        st = torch.cuda.Stream()
        with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024, stream=st) as s:
            s.step(5)
            s.step(5)
            xs, vs = s.state()
            s.sync()
            st.synchronize()
            out.append((xs.cpu().numpy(), vs.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("integrator", ["hermite", "leapfrog", "block"])
def test_runtime_non_finite_state_is_reported_and_sticky(integrator):
    """Fault injection through the step size: dt = 1e200 is a valid argument, but the
    predictor's dt^3 term overflows, so the fp64 update kernels flag a non-finite state;
    the next blocking call returns NBODY_ENONFINITE naming a particle, and every later
    call on the context NBODY_ESTATE."""
    m, x, v = inputs.make("C1")
    with binding.NBody(m, x, v, eps=1e-2, dt=1e200, integrator=integrator) as s:
        with pytest.raises(binding.NBodyError) as e:
            s.step(1)
            s.sync()
        assert e.value.code == binding.NBODY_ENONFINITE and "non-finite state at particle" in str(e.value)
        with pytest.raises(binding.NBodyError) as e2:
            s.forces()
        assert e2.value.code == binding.NBODY_ESTATE


def test_c_abi_argument_errors():
    """EINVAL paths of the C-ABI with a live context (messages name the problem)."""
    m, x, v = inputs.make("C1")
    L = binding.lib()
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        assert L.nbody_step(s._ctx, 0) == binding.NBODY_EINVAL
        assert "nsteps" in L.nbody_last_error(s._ctx).decode()
        xb = np.ascontiguousarray(x.copy())
        xb[2, 900] = np.inf
        with pytest.raises(binding.NBodyError, match="particle 900"):
            s.set_state(xb, v)
        # the context stays usable after a rejected set_state (not sticky)
        s.set_state(x, v)
        a, _ = s.forces()
        s.sync()
        ao, _ = oracle.forces(m, x, v, eps2_of(1e-2))
        assert max_rel(a.cpu().numpy(), ao) <= TOL_ACC
    L.nbody_destroy(None)   # no-op


def test_binding_rejects_wrong_shapes_before_the_c_abi():
    """The C-ABI trusts array sizes; the binding checks shapes before passing pointers."""
    m, x, v = inputs.make("C1")
    with pytest.raises(ValueError, match="x must have shape"):
        binding.NBody(m, x[:, :512], v, eps=1e-2, dt=1 / 1024)
    with pytest.raises(ValueError, match="m must be one-dimensional"):
        binding.NBody(m[None, :], x, v, eps=1e-2, dt=1 / 1024)
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        with pytest.raises(ValueError, match="acc must have shape"):
            s.forces(acc=np.empty((3, 100)))
        with pytest.raises(ValueError, match="v must have shape"):
            s.state(v=np.empty((1024, 3)))
        with pytest.raises(ValueError, match="x must have shape"):
            s.set_state(np.empty(3 * 1024), None)
        a, _ = s.forces()   # still usable
        ao, _ = oracle.forces(m, x, v, eps2_of(1e-2))
        assert max_rel(a.cpu().numpy(), ao) <= TOL_ACC


def test_get_state_partial_outputs_and_energy_consistency():
    m, x, v = inputs.make("C1")
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        xs = np.empty((3, 1024))
        binding._check(binding.lib().nbody_get_state(s._ctx, xs.ctypes.data, None), s._ctx)
        assert np.array_equal(xs, x)       # init copies the state losslessly
        ke1, pe1 = s.energy()
        ke2, pe2 = s.energy()
        assert (ke1, pe1) == (ke2, pe2)    # deterministic reduction


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_size_properties_all_particles(cfg):
    """Properties that hold at any size, checked on every particle of the full-size
    configs in the bench's launch configuration (the oracle samples the rest): momentum
    conservation (central pair forces, Sigma m a = 0) and permutation equivariance (a
    seeded permutation of the particles permutes the forces; the j order changes, so
    agreement is to fp32 rounding, not bitwise)."""
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    a, j = gpu_forces(m, x, v, c.eps)
    assert momentum_residual(m, a) < 1e-6, momentum_residual(m, a)
    assert momentum_residual(m, j) < 1e-5, momentum_residual(m, j)
    perm = np.random.default_rng(77).permutation(c.n)
    ap, jp = gpu_forces(m[perm], x[:, perm], v[:, perm], c.eps)
    assert max_rel(ap, a[:, perm]) <= 2 * TOL_ACC, max_rel(ap, a[:, perm])
    assert max_rel(jp, j[:, perm]) <= 2 * TOL_JERK, max_rel(jp, j[:, perm])
    assert paper_norm(ap, a[:, perm]) <= TOL_PAPER_ACC
