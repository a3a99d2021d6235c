"""Checkpoint / exact resume through the C-ABI (nbody_get_derivs / nbody_set_derivs /
nbody_set_levels): a run saved at a call boundary and resumed in a fresh context continues
bit for bit as the uninterrupted run, for shared-step Hermite, leapfrog and block time
steps (including a resume into a differently sharded context)."""
import numpy as np
import pytest

from paper_2509_19294_b200 import binding, inputs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _np(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else t


@pytest.mark.parametrize("integrator", ["hermite", "leapfrog"])
def test_shared_step_resume_is_exact(integrator):
    m, x, v = inputs.make("C1")
    kw = dict(eps=1e-2, dt=1 / 1024, integrator=integrator)
    with binding.NBody(m, x, v, **kw) as s:
        s.step(6)
        xa, va = (_np(t) for t in s.state())
    with binding.NBody(m, x, v, **kw) as s:
        s.step(3)
        x3, v3 = (_np(t) for t in s.state())
        a3, j3 = (_np(t) for t in s.derivs())
    with binding.NBody(m, x3, v3, **kw) as s:
        s.set_derivs(a3, j3 if integrator == "hermite" else None)
        s.step(3)
        xc, vc = (_np(t) for t in s.state())
    assert np.array_equal(xc, xa) and np.array_equal(vc, va)


@pytest.mark.parametrize("world", [1, 2])
def test_block_resume_is_exact(world):
    m, x, v = inputs.parity_round(*inputs.plummer(6000, 17))
    kw = dict(eps=1e-3, dt=1 / 128, integrator="block")
    with binding.NBody(m, x, v, **kw) as s:
        s.step(4)
        xa, va = (_np(t) for t in s.state())
        sa = s.block_stats(levels=True)
    with binding.NBody(m, x, v, **kw) as s:
        s.step(2)
        x2, v2 = (_np(t) for t in s.state())
        a2, j2 = (_np(t) for t in s.derivs())
        s2 = s.block_stats(levels=True)
    with binding.NBody(m, x2, v2, world=world, loopback=world > 1, **kw) as s:
        s.set_derivs(a2, j2)
        s.set_levels(s2[2])
        s.step(2)
        xc, vc = (_np(t) for t in s.state())
        sc = s.block_stats(levels=True)
    assert np.array_equal(xc, xa) and np.array_equal(vc, va)
    assert np.array_equal(sc[2], sa[2])
    assert sc[0] == sa[0] - s2[0] and sc[1] == sa[1] - s2[1]


def test_checkpoint_argument_errors():
    m, x, v = inputs.make("C1")
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        a, j = (_np(t) for t in s.derivs())
        bad = a.copy()
        bad[1, 77] = np.nan
        with pytest.raises(binding.NBodyError, match="particle 77") as e:
            s.set_derivs(bad, j)
        assert e.value.code == binding.NBODY_EINVAL
        with pytest.raises(binding.NBodyError) as e:
            s.set_levels(np.zeros(1024, dtype=np.int32))
        assert e.value.code == binding.NBODY_EINVAL
        s.set_derivs(a, j)   # still usable
        s.step(1)
        s.sync()
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 64, integrator="block", kmax=5) as s:
        lev = np.zeros(1024, dtype=np.int32)
        lev[500] = 6
        with pytest.raises(binding.NBodyError, match="particle 500") as e:
            s.set_levels(lev)
        assert e.value.code == binding.NBODY_EINVAL
