"""Seeded synthetic initial conditions (shared by tests, smoke and bench).

This module holds NO arithmetic of the method (no forces, no integrator, no
energy): it only draws particle systems.  Both the CUDA path and the fp64
oracle consume its output; neither is imported here.

Recipes (SURVEY.md 8(c) readings R#7, R#8, R#9, R#16):

* Plummer sphere, Aarseth-Henon-Wielen (1974) sampling in G = M = a = 1
  units, mass cut X <= 0.999, then Henon scaling r *= 3 pi / 16,
  v *= sqrt(16 / (3 pi)) so that E ~= -1/4 and the virial radius ~= 1
  (virialised in expectation; no exact rescale, which would need the energy
  arithmetic of the method), then the mass-weighted centre of mass and
  momentum are removed.
* Two-cluster system (config C4): Plummer a = 1 at (-5, 0, 0) and a = 0.5 at
  (+5, 0, 0), 1:1 mass, log-normal masses (sigma = 0.5 in ln m) renormalised
  to 0.5 per cluster, clusters on the circular relative orbit of two point
  masses 10 apart.
* Two-body Kepler orbit at pericentre (m1 = m2 = 1/2, semi-major axis a).

``parity_round`` rounds a system once to fp32-representable values (R#9):
the GPU packs those values losslessly and the oracle widens them exactly.

PRNG: ``numpy.random.default_rng(seed)`` (PCG64), seeds C1..C5 = 1..5.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    kind: str          # "plummer" | "two_cluster"
    eps: float
    dt: float
    steps: int
    seed: int
    gpus: tuple


# BASELINE.json configs[0..4]; dt for C3-C5 is unstated there -> 1/1024 (R#5).
CONFIGS = {
    "C1": Config("C1", 1024, "plummer", 1e-2, 1.0 / 1024, 10, 1, (1,)),
    "C2": Config("C2", 16384, "plummer", 1e-3, 1.0 / 1024, 100, 2, (1,)),
    "C3": Config("C3", 131072, "plummer", 1e-3, 1.0 / 1024, 20, 3, (1, 2, 4, 8)),
    "C4": Config("C4", 262144, "two_cluster", 1e-3, 1.0 / 1024, 10, 4, (1, 2, 4, 8)),
    "C5": Config("C5", 1048576, "plummer", 5e-4, 1.0 / 1024, 5, 5, (1, 2, 4, 8)),
    # NEXT f4: the paper's own workload shape, 102400 particles over "ten time
    # cycles"; ICs, softening and dt unstated -> Plummer, eps 1e-3,
    # dt 1/1024, one cycle = one Hermite step (R#4, R#24).
    "PAPER": Config("PAPER", 102400, "plummer", 1e-3, 1.0 / 1024, 10, 6, (1,)),
}


def _isotropic(rng, n):
    """Unit vectors, uniform on the sphere (z = 1 - 2u, phi = 2 pi u')."""
    z = 1.0 - 2.0 * rng.random(n)
    phi = 2.0 * np.pi * rng.random(n)
    rxy = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([rxy * np.cos(phi), rxy * np.sin(phi), z])


def plummer_unit(n: int, rng) -> tuple[np.ndarray, np.ndarray]:
    """Positions and velocities (3, n) of a Plummer model, G = M = a = 1 (AHW74)."""
    # radius from the cumulative mass M(<r) = r^3 / (1 + r^2)^{3/2}, cut at 0.999
    X = 0.999 * (1.0 - rng.random(n))          # in (0, 0.999]
    r = 1.0 / np.sqrt(X ** (-2.0 / 3.0) - 1.0)
    x = r * _isotropic(rng, n)
    # speed by von Neumann rejection on g(q) = q^2 (1 - q^2)^{7/2}, max < 0.1
    q = np.empty(n)
    todo = np.arange(n)
    while todo.size:
        qq = rng.random(todo.size)
        uu = 0.1 * rng.random(todo.size)
        ok = uu < qq * qq * (1.0 - qq * qq) ** 3.5
        q[todo[ok]] = qq[ok]
        todo = todo[~ok]
    vesc = np.sqrt(2.0) * (1.0 + r * r) ** (-0.25)
    v = (q * vesc) * _isotropic(rng, n)
    return x, v


def _recentre(m, x, v):
    M = m.sum()
    x = x - (x @ m / M)[:, None]
    v = v - (v @ m / M)[:, None]
    return x, v


def plummer(n: int, seed: int):
    """Equal-mass Plummer sphere in Henon units (total mass 1); returns (m, x, v)."""
    rng = np.random.default_rng(seed)
    x, v = plummer_unit(n, rng)
    x = x * (3.0 * np.pi / 16.0)
    v = v * np.sqrt(16.0 / (3.0 * np.pi))
    m = np.full(n, 1.0 / n)
    x, v = _recentre(m, x, v)
    return m, np.ascontiguousarray(x), np.ascontiguousarray(v)


def two_cluster(n: int, seed: int, sep: float = 10.0, a_b: float = 0.5,
                sigma: float = 0.5):
    """Config C4: two Plummer clusters (a = 1 and a = a_b), sep apart on a circular orbit."""
    rng = np.random.default_rng(seed)
    na = n // 2
    nb = n - na
    ms, xs, vs = [], [], []
    for k, (nk, ak, cx, vy) in enumerate(((na, 1.0, -sep / 2, -1.0),
                                           (nb, a_b, +sep / 2, +1.0))):
        Mk = 0.5
        xk, vk = plummer_unit(nk, rng)
        xk = xk * ak
        vk = vk * np.sqrt(Mk / ak)          # G = 1 velocity scale of a (Mk, ak) Plummer model
        mk = np.exp(sigma * rng.standard_normal(nk))
        mk = mk * (Mk / mk.sum())
        xk, vk = _recentre(mk, xk, vk)
        vrel_half = 0.5 * np.sqrt(1.0 / sep)  # circular relative orbit of two 0.5 masses
        xk[0] += cx
        vk[1] += vy * vrel_half
        ms.append(mk)
        xs.append(xk)
        vs.append(vk)
    m = np.concatenate(ms)
    x = np.concatenate(xs, axis=1)
    v = np.concatenate(vs, axis=1)
    return m, np.ascontiguousarray(x), np.ascontiguousarray(v)


def kepler(e: float, a: float = 1.0):
    """Two bodies m = 1/2 each at pericentre of a relative orbit (G = 1, M = 1)."""
    m = np.array([0.5, 0.5])
    rp = a * (1.0 - e)
    vp = np.sqrt((1.0 + e) / (a * (1.0 - e)))
    x = np.zeros((3, 2))
    v = np.zeros((3, 2))
    x[0] = [-rp / 2, rp / 2]
    v[1] = [-vp / 2, vp / 2]
    return m, x, v


def uniform_cube(n: int, seed: int, scale: float = 1.0):
    """Uniform positions in [-scale, scale]^3, small random velocities, equal masses."""
    rng = np.random.default_rng(seed)
    x = scale * (2.0 * rng.random((3, n)) - 1.0)
    v = 0.1 * (2.0 * rng.random((3, n)) - 1.0)
    m = np.full(n, 1.0 / n)
    return m, x, v


def parity_round(m, x, v):
    """Round a system once to fp32-representable values, held as float64 (R#9)."""
    r = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float32).astype(np.float64))
    return r(m), r(x), r(v)


def make(config: str | Config, parity: bool = True):
    """(m, x, v) for a named config (C1..C5), fp32-rounded when parity=True."""
    c = CONFIGS[config] if isinstance(config, str) else config
    if c.kind == "plummer":
        sysm = plummer(c.n, c.seed)
    elif c.kind == "two_cluster":
        sysm = two_cluster(c.n, c.seed)
    else:
        raise ValueError(c.kind)
    return parity_round(*sysm) if parity else sysm
