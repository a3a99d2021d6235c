"""Initial-condition generator checks (closed forms of the Plummer model)."""
import math

import numpy as np

import oracle
from paper_2509_19294_b200 import inputs


def test_plummer_deterministic_and_centred():
    m1, x1, v1 = inputs.plummer(4096, 42)
    m2, x2, v2 = inputs.plummer(4096, 42)
    assert np.array_equal(x1, x2) and np.array_equal(v1, v2)
    assert abs(m1.sum() - 1) < 1e-14
    assert np.max(np.abs(x1 @ m1)) < 1e-15 and np.max(np.abs(v1 @ m1)) < 1e-15


def test_plummer_half_mass_radius_and_virial():
    """Henon units: r_half = 3 pi / 16 (2^{2/3} - 1)^{-1/2} = 0.7686; E ~= -1/4; Q ~= 1/2."""
    m, x, v = inputs.plummer(16384, 2)
    r = np.sort(np.linalg.norm(x, axis=0))
    r_half_closed = 3 * math.pi / 16 / math.sqrt(2 ** (2 / 3) - 1)
    assert abs(r_half_closed - 0.7686) < 1e-4
    assert abs(r[len(r) // 2] / r_half_closed - 1) < 0.03
    ke, pe = oracle.energy(m, x, v, 0.0)
    assert abs((ke + pe) / -0.25 - 1) < 0.05
    assert abs(-ke / pe - 0.5) < 0.03


def test_parity_round_is_fp32_exact():
    m, x, v = inputs.make("C1")
    for a in (m, x, v):
        assert a.dtype == np.float64
        assert np.array_equal(a.astype(np.float32).astype(np.float64), a)
    assert np.all(m == 1.0 / 1024)


def test_two_cluster_structure():
    m, x, v = inputs.two_cluster(8192, 4)
    assert abs(m.sum() - 1) < 1e-13
    assert abs(m[:4096].sum() - 0.5) < 1e-14
    assert np.max(np.abs(x @ m)) < 1e-12 and np.max(np.abs(v @ m)) < 1e-14
    ca = x[:, :4096] @ m[:4096] / 0.5
    cb = x[:, 4096:] @ m[4096:] / 0.5
    assert np.allclose(ca, [-5, 0, 0], atol=1e-12) and np.allclose(cb, [5, 0, 0], atol=1e-12)
    ratio = m.max() / m.min()
    assert 20 < ratio < 1000                       # log-normal sigma 0.5 spread
    ln = np.log(m[:4096])
    assert abs(ln.std() - 0.5) < 0.03
    # circular relative orbit of the two 0.5 point masses: v_rel = sqrt(G M / d)
    va = v[:, :4096] @ m[:4096] / 0.5
    vb = v[:, 4096:] @ m[4096:] / 0.5
    assert abs(np.linalg.norm(vb - va) - math.sqrt(0.1)) < 1e-12


def test_configs_match_baseline():
    c = inputs.CONFIGS
    assert [c[k].n for k in ("C1", "C2", "C3", "C4", "C5")] == [1024, 16384, 131072, 262144, 1048576]
    assert [c[k].eps for k in ("C1", "C2", "C3", "C4", "C5")] == [1e-2, 1e-3, 1e-3, 1e-3, 5e-4]
    assert [c[k].steps for k in ("C1", "C2", "C3", "C4", "C5")] == [10, 100, 20, 10, 5]
