"""tests/golden/ fixtures: what each stores, what pins it, and the GPU against it.

* paper_numbers.json -- numbers the paper prints (PAPER.md:161 validation tolerances,
  :178/:180 paper-shaped run, :191 timings), stored by hand with citations; the test
  metrics use exactly these tolerances.
* forces_cube6.json, kepler_e05_period.json -- written by scripts/make_golden.py, which
  calls only oracle/.  Pinned here independently of the oracle: the forces by 40-digit
  mpmath differentiation of the softened potential (a = -grad Phi) and of a along x + v t
  (jerk), the Kepler state by the closed-form orbit.  The oracle must still reproduce
  both fixtures bit for bit (a regression guard on its arithmetic), and the GPU path must
  match them within the parity bars.
"""
import json
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
from metrics import TOL_ACC, TOL_JERK, TOL_PAPER_ACC, TOL_PAPER_JERK, max_rel, paper_norm
from test_oracle import _mp_accel, _mp_potential_grad

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def arrays(rec, *keys):
    return [np.ascontiguousarray(np.array(rec[k], dtype=np.float64)) for k in keys]


def test_paper_tolerances_are_the_ones_the_tests_use():
    p = load("paper_numbers.json")["validation_tolerance"]
    assert TOL_PAPER_ACC == p["acceleration_component_frac_of_typical_force"] == 5e-4
    assert TOL_PAPER_JERK == p["jerk_component_frac_of_typical_force"] == 2e-3


def test_forces_fixture_pinned_by_mpmath_and_reproduced_by_oracle():
    rec = load("forces_cube6.json")
    m, x, v, acc, jerk = arrays(rec, "m", "x", "v", "acc", "jerk")
    eps2 = rec["eps2"]
    a, j = oracle.forces(m, x, v, eps2)
    assert np.array_equal(a, acc) and np.array_equal(j, jerk)     # regression: same bits
    mp.mp.dps = 40
    for i in range(rec["n"]):
        ga = np.array([float(t) for t in _mp_potential_grad(m, x, i, eps2)])
        assert np.linalg.norm(acc[:, i] - ga) <= 1e-14 * np.linalg.norm(ga)
        gj = np.array([float(mp.diff(lambda t: _mp_accel(m, x, v, i, eps2, t)[c], 0)) for c in range(3)])
        assert np.linalg.norm(jerk[:, i] - gj) <= 1e-13 * np.linalg.norm(gj)


def test_kepler_fixture_pinned_by_closed_form_and_reproduced_by_oracle():
    rec = load("kepler_e05_period.json")
    m, x0, v0, x1, v1 = arrays(rec, "m", "x0", "v0", "x", "v")
    xo, vo, _, _ = oracle.hermite(m, x0, v0, 0.0, rec["dt"], rec["nsteps"])
    assert np.array_equal(xo, x1) and np.array_equal(vo, v1)
    rel = x1[:, 1] - x1[:, 0]
    assert np.linalg.norm(rel - np.array(rec["closed_form_relative_position"])) < 1e-9


@pytest.mark.gpu
def test_gpu_forces_match_golden():
    torch = pytest.importorskip("torch")   # noqa: F841
    from paper_2509_19294_b200 import binding
    rec = load("forces_cube6.json")
    m, x, v, acc, jerk = arrays(rec, "m", "x", "v", "acc", "jerk")
    with binding.NBody(m, x, v, eps=1e-2, dt=1 / 1024) as s:
        a, j = s.forces()
        s.sync()
        a, j = a.cpu().numpy(), j.cpu().numpy()
    assert max_rel(a, acc) <= TOL_ACC and max_rel(j, jerk) <= TOL_JERK
    assert paper_norm(a, acc) <= TOL_PAPER_ACC and paper_norm(j, jerk) <= TOL_PAPER_JERK


@pytest.mark.gpu
def test_gpu_kepler_period_matches_golden():
    torch = pytest.importorskip("torch")   # noqa: F841
    from paper_2509_19294_b200 import binding
    rec = load("kepler_e05_period.json")
    m, x0, v0, x1, _ = arrays(rec, "m", "x0", "v0", "x", "v")
    with binding.NBody(m, x0, v0, eps=0.0, dt=rec["dt"]) as s:
        s.step(rec["nsteps"])
        xs, _ = s.state()
        s.sync()
        xs = xs.cpu().numpy()
    rel_g, rel_o = xs[:, 1] - xs[:, 0], x1[:, 1] - x1[:, 0]
    assert np.linalg.norm(rel_g - rel_o) < 1e-5    # fp32 forces, eps = 0 guarded pass (X7)
