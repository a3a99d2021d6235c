"""GPU tests of the exchange: the multi-rank step path.

The paper's parallelisation gives every core "the complete set of particle data"
(Sec. 3) and names "MPI with multiple accelerators" as future work
(Sec. 5); here i-shards all-gather their j-packets every step.  Only one
GPU is available, so the path is exercised in the two ways it can run on one device:

* world = 1 with an NCCL communicator: the exact code an NCCL rank runs -- the in-place
  ncclAllGather on the comm stream, the fork/join events, the local-chunk launch in the
  1024-i shape overlapping it and the remote-chunk launch after it -- captured into the
  step's CUDA graph on a non-default stream, and eagerly with kernel timing on;
* loopback shards: every shard packs into its own exchange buffer and receives every
  other shard's slice by one device copy per slice, between the same two launches, so a
  wrong slice offset or a local launch that reads a remote chunk changes the result.

Both are compared bit for bit with the communicator-free single-shard run and, through
it, with the fp64 oracle (R#14, R#15 bars).  Mutation builds (NB_TEST_MUTATE) show the
loopback comparison detects a wrong slice offset and a wrong local-chunk range.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2509_19294_b200 import _build, binding, inputs
from metrics import TOL_ACC, TOL_JERK, max_rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def eps2_of(eps):
    return float(np.float32(eps * eps))


def run(m, x, v, eps, dt, nsteps, stream=None, prof=False, **kw):
    """forces at t = 0, nsteps steps, final state; (arrays, exec_stats, launch sizes)."""
    with binding.NBody(m, x, v, eps=eps, dt=dt, stream=stream, **kw) as s:
        if prof:
            s.prof_enable(True)
        a, j = s.forces()
        s.step(nsteps)
        xs, vs = s.state()
        s.sync()
        stats = s.exec_stats()
        sizes = s.prof_launch_sizes() if prof else None
        out = [t.cpu().numpy() for t in (a, j, xs, vs)]
    return out, stats, sizes


def same(a, b):
    return all(np.array_equal(p, q) for p, q in zip(a, b))


@pytest.mark.parametrize("cfg,nsteps", [("C1", 10), ("C2", 100)])
def test_nccl_step_path_graph_and_eager(cfg, nsteps):
    """world = 1 + NCCL communicator on a non-default stream: the captured step graph
    (all-gather fork/join + both force launches) and the eager path with kernel timing
    equal the communicator-free run bit for bit; the trajectory meets R#15's bars against
    the oracle."""
    c = inputs.CONFIGS[cfg]
    m, x, v = inputs.make(cfg)
    st = torch.cuda.Stream()
    ref, (g0, e0), _ = run(m, x, v, c.eps, c.dt, nsteps, stream=st)
    assert g0 == nsteps and e0 == 0          # the plain run replayed its step graph
    got, (g1, e1), _ = run(m, x, v, c.eps, c.dt, nsteps, stream=st, nccl_id=binding.nccl_unique_id())
    assert g1 == nsteps and e1 == 0          # ... and so did the NCCL run (capture succeeded)
    assert same(got, ref)
    got_e, (g2, e2), sizes = run(m, x, v, c.eps, c.dt, nsteps, stream=st, prof=True,
                                 nccl_id=binding.nccl_unique_id())
    assert g2 == 0 and e2 == nsteps          # kernel timing forces the eager path
    assert same(got_e, ref)
    # every evaluation (t = 0 and each step) is the local-first + remote launch pair, and
    # together they cover every j of every local i exactly once
    ni, nj = sizes
    assert np.all(ni == c.n) and (ni * nj).sum() == c.n * c.n * (nsteps + 1)
    if cfg == "C2":   # 64 chunks: 18 local-first (one wave of 16 i-blocks) + 46 after
        assert len(ni) == 2 * (nsteps + 1) and np.all(nj.reshape(-1, 2) == [18 * 256, 46 * 256])
    # the oracle: forces at t = 0 and the trajectory (R#15)
    ao, jo = oracle.forces(m, x, v, eps2_of(c.eps))
    assert max_rel(ref[0], ao) <= TOL_ACC and max_rel(ref[1], jo) <= TOL_JERK
    xo, vo, _, _ = oracle.hermite(m, x, v, eps2_of(c.eps), c.dt, nsteps)
    dx_tol, dv_tol = (1e-9, 1e-6) if cfg == "C1" else (1e-6, 1e-4)
    assert np.linalg.norm(ref[2] - xo, axis=0).max() <= dx_tol
    assert np.linalg.norm(ref[3] - vo, axis=0).max() <= dv_tol


@pytest.mark.parametrize("integrator,hilo,eps", [("leapfrog", False, 1e-3), ("hermite", True, 1e-3),
                                                 ("hermite", False, 0.0)])
def test_nccl_step_path_other_modes(integrator, hilo, eps):
    """The rank code path (1-rank NCCL communicator, graph-captured, two concurrent force
    launches) for the acceleration-only leapfrog kernel, hi/lo position tails (a second
    all-gather) and the eps = 0 guarded kernel: bit-identical to the communicator-free run."""
    m, x, v = inputs.parity_round(*inputs.plummer(20000, 57))
    st = torch.cuda.Stream()
    kw = dict(integrator=integrator, hilo=hilo)
    ref, _, _ = run(m, x, v, eps, 1 / 1024, 5, stream=st, **kw)
    got, (g, e), _ = run(m, x, v, eps, 1 / 1024, 5, stream=st, nccl_id=binding.nccl_unique_id(), **kw)
    assert g == 5 and e == 0 and same(got, ref)


@pytest.mark.parametrize("concurrent", ["0", "1"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_exchange_graph_and_eager(world, concurrent, monkeypatch):
    """Loopback shards with their own exchange buffers and per-slice copies equal the
    single-shard run bit for bit (graph replay and eager), with per shard one local-first
    launch over chunks inside its own slice and one launch over the rest -- in the checking
    form (copies between the launches on one stream) and in the NCCL rank's stream form
    (copies and remote launch on the comm stream, concurrent with the local launch;
    NBODY_LOOPBACK_CONCURRENT=1, the form scripts/project_scaling.py times)."""
    monkeypatch.setenv("NBODY_LOOPBACK_CONCURRENT", concurrent)
    n = 20000 if world != 8 else 16384 + 1000   # ragged: the last shard is short or empty
    m, x, v = inputs.parity_round(*inputs.plummer(n, 31 + world))
    st = torch.cuda.Stream()
    ref, _, _ = run(m, x, v, 1e-3, 1 / 1024, 6, stream=st)
    got, (g, e), _ = run(m, x, v, 1e-3, 1 / 1024, 6, stream=st, world=world, loopback=True)
    assert g == 6 and e == 0 and same(got, ref)
    got_e, (g, e), sizes = run(m, x, v, 1e-3, 1 / 1024, 6, stream=st, prof=True, world=world,
                               loopback=True)
    assert g == 0 and e == 6 and same(got_e, ref)
    ni, nj = sizes
    # per evaluation and shard: the launches of that shard cover all n j once
    per_eval = ni.size // 7
    assert ni.size == 7 * per_eval
    inter = (ni * nj).reshape(7, per_eval).sum(axis=1)
    assert np.all(inter == n * n)


@pytest.mark.parametrize("integrator", ["leapfrog", "block"])
def test_loopback_exchange_other_integrators(integrator):
    """The exchange is shared by every integrator: leapfrog and block time steps (whose
    block-step graph now holds the per-slice copies) are bit-identical across shards."""
    m, x, v = inputs.parity_round(*inputs.plummer(12000, 5))
    st = torch.cuda.Stream()
    dt = 1 / 1024 if integrator == "leapfrog" else 1 / 256
    outs = []
    for world in (1, 3):
        with binding.NBody(m, x, v, eps=1e-3, dt=dt, stream=st, world=world, loopback=world > 1,
                           integrator=integrator) as s:
            s.step(2)
            xs, vs = s.state()
            s.sync()
            outs.append([t.cpu().numpy() for t in (xs, vs)])
    assert same(outs[0], outs[1])


_MUTANT_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2509_19294_b200 import binding, inputs
m, x, v = inputs.parity_round(*inputs.plummer(20000, 33))
st = torch.cuda.Stream()
res = []
for world in (1, 2):
    with binding.NBody(m, x, v, eps=1e-3, dt=1 / 1024, stream=st, world=world, loopback=world > 1) as s:
        a, j = s.forces()
        s.step(3)
        xs, vs = s.state()
        s.sync()
        res.append([t.cpu().numpy() for t in (a, j, xs, vs)])
print(json.dumps({{"identical": all(np.array_equal(p, q) for p, q in zip(*res))}}))
"""


@pytest.mark.parametrize("mutation", [1, 2])
def test_exchange_mutations_are_detected(tmp_path, mutation):
    """Build the library with a deliberately wrong exchange (1: slice offsets permuted in
    the helper both exchange back ends use; 2: the local-first launch starting at chunk 0)
    and check that the loopback comparison above fails for it, while the product build
    passes it."""
    lib = str(tmp_path / f"libnbody_mut{mutation}.so")
    _build.build(defines=[f"NB_TEST_MUTATE={mutation}"], out=lib)
    script = _MUTANT_SCRIPT.format(root=ROOT)
    env = dict(os.environ, NBODY_LIB=lib)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["identical"] is False
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["identical"] is True


_HANG_SCRIPT = r"""
import sys, time
sys.path.insert(0, {root!r})
import numpy as np
from paper_2509_19294_b200 import binding, inputs
m, x, v = inputs.make("C1")
t0 = time.time()
try:
    binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024, rank=0, world=2, nccl_id=binding.nccl_unique_id())
    print("INIT-RETURNED-OK")
except binding.NBodyError as e:
    print(f"CODE={{e.code}} after {{time.time() - t0:.1f}} s: {{e}}")
"""


def test_nccl_missing_peer_times_out_and_aborts():
    """Rank 0 of a 2-rank communicator whose rank 1 never arrives: the non-blocking init
    gives up after NBODY_NCCL_TIMEOUT_S with NBODY_ENCCL, the half-built communicator is
    aborted (ncclCommAbort) and the process exits normally instead of hanging."""
    env = dict(os.environ, NBODY_NCCL_TIMEOUT_S="5")
    r = subprocess.run([sys.executable, "-c", _HANG_SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=240)
    out = r.stdout
    assert r.returncode == 0, (out, r.stderr[-2000:])
    assert f"CODE={binding.NBODY_ENCCL}" in out and "NBODY_NCCL_TIMEOUT_S" in out, out


def test_output_tensors_ordered_after_library_stream():
    """Binding stream hygiene: with the library on a side stream, output tensors are made
    on it and torch's current stream waits on it, so consuming results on the current
    stream without an explicit synchronize sees the finished values."""
    c = inputs.CONFIGS["C3"]
    m, x, v = inputs.make("C3")
    side = torch.cuda.Stream()
    with binding.NBody(m, x, v, eps=c.eps, dt=c.dt, stream=side) as s:
        ref, _ = s.forces()
        side.synchronize()
        ref = ref.cpu()
        for _ in range(3):
            a, _ = s.forces()                  # ~15 ms of work queued on the side stream
            got = (a * 1.0).cpu()              # consumed on the current stream at once
            assert torch.equal(got, ref)


def test_denormal_softening_uses_guarded_pass():
    """eps whose fp32 square is subnormal (flushed to 0 by the FTZ force pass) takes the
    guarded pass that excludes s == 0, so the self term does not become 0 * inf: forces
    match the oracle (G = 1e-30 keeps G m / eps^3 inside the fp32 range)."""
    m, x, v = inputs.parity_round(*inputs.uniform_cube(2000, 3))
    G, eps = 1e-30, 2e-20
    assert 0.0 < np.float32(eps * eps) < np.finfo(np.float32).tiny
    with binding.NBody(m, x, v, eps=eps, dt=1 / 1024, G=G) as s:
        a, j = s.forces()
        s.sync()
        a, j = a.cpu().numpy(), j.cpu().numpy()
    ao, jo = oracle.forces(m, x, v, eps2_of(eps), G=G)
    assert max_rel(a, ao) <= TOL_ACC and max_rel(j, jo) <= TOL_JERK


def test_softening_outside_fp32_range_is_rejected():
    """G max(m) / eps^3 beyond the fp32 range of the pair terms is rejected at init
    (NBODY_EINVAL naming the limit) instead of producing a spurious non-finite force."""
    m, x, v = inputs.make("C1")
    with pytest.raises(binding.NBodyError, match="fp32 range") as e:
        binding.NBody(m, x, v, eps=1e-13, dt=1 / 1024)
    assert e.value.code == binding.NBODY_EINVAL


def test_multi_gpu_example_runs():
    """examples/multi_gpu.py (the user-facing multi-rank recipe) with 3 emulated ranks."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "multi_gpu.py"), "C1", "5",
                        "--loopback", "3"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ranks = 3" in r.stdout and "relative drift" in r.stdout, r.stdout
