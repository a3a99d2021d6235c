"""fp64 CPU oracle for the direct-summation N-body hot path (arXiv 2509.19294).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with ``paper_2509_19294_b200`` and never imports it.

The arithmetic lives in ``oracle.c`` (plain C, fp64, OpenMP over i only); this
file only marshals numpy arrays through ctypes.  See the header of
``oracle.c`` for the paper passages each function follows.

Layout convention: positions / velocities / accelerations / jerks are SoA
arrays of shape ``(3, n)`` (float64, C-contiguous).

Parity status: every function here is pinned by
``tests/test_oracle.py`` (closed forms, mpmath brute force, invariants,
Kepler convergence); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, fp64, no fast-math, no FMA contraction)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-std=c11", "-Wall", "-o", tmp, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(build())
    d = ctypes.c_double
    i64 = ctypes.c_int64
    p = ctypes.c_void_p
    lib.oracle_forces.argtypes = [i64, d, d, p, p, p, p, i64, p, p, p]
    lib.oracle_forces.restype = ctypes.c_int
    lib.oracle_energy.argtypes = [i64, d, d, p, p, p,
                                  ctypes.POINTER(d), ctypes.POINTER(d)]
    lib.oracle_energy.restype = ctypes.c_int
    lib.oracle_hermite.argtypes = [i64, d, d, d, i64, p, p, p, p, p, ctypes.c_int]
    lib.oracle_hermite.restype = ctypes.c_int
    lib.oracle_leapfrog.argtypes = [i64, d, d, d, i64, p, p, p, p, ctypes.c_int]
    lib.oracle_leapfrog.restype = ctypes.c_int
    i32 = ctypes.c_int
    lib.oracle_block_init_levels.argtypes = [i64, d, i32, d, p, p, p, p]
    lib.oracle_block_init_levels.restype = ctypes.c_int
    lib.oracle_hermite_block.argtypes = [i64, d, d, d, i32, d, d, i64, p, p, p, p, p, p, i32, p, p,
                                         p, p]
    lib.oracle_hermite_block.restype = ctypes.c_int
    lib.oracle_threads.argtypes = []
    lib.oracle_threads.restype = ctypes.c_int
    lib.oracle_set_threads.argtypes = [ctypes.c_int]
    lib.oracle_set_threads.restype = None
    _lib = lib
    return lib


class OracleError(RuntimeError):
    pass


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def threads() -> int:
    return _load().oracle_threads()


def set_threads(t: int) -> None:
    _load().oracle_set_threads(int(t))


def forces(m, x, v, eps2: float, G: float = 1.0, idx=None):
    """Accelerations and jerks (each (3, len(idx)) float64) on particles idx (default all).

    P:134-138 [Sec. 3] with softening eps2 (R#1) and jerk per R#2.
    """
    m = _f64(m)
    n = m.shape[0]
    x = _f64(x, (3, n))
    v = _f64(v, (3, n))
    if idx is None:
        idx_arr, k = None, n
    else:
        idx_arr = np.ascontiguousarray(idx, dtype=np.int64)
        k = idx_arr.shape[0]
        if k and (idx_arr.min() < 0 or idx_arr.max() >= n):
            raise ValueError("idx out of range")
    acc = np.zeros((3, k))
    jerk = np.zeros((3, k))
    bad = np.full(2, -1, dtype=np.int64)
    rc = _load().oracle_forces(n, float(G), float(eps2), _ptr(m), _ptr(x), _ptr(v),
                               _ptr(idx_arr), k, _ptr(acc), _ptr(jerk), _ptr(bad))
    if rc:
        raise OracleError(f"coincident pair ({bad[0]}, {bad[1]}) with eps = 0")
    return acc, jerk


def energy(m, x, v, eps2: float, G: float = 1.0):
    """(KE, PE) in fp64; PE softened, pairs i<j (R#1, R#14)."""
    m = _f64(m)
    n = m.shape[0]
    x = _f64(x, (3, n))
    v = _f64(v, (3, n))
    ke = ctypes.c_double()
    pe = ctypes.c_double()
    rc = _load().oracle_energy(n, float(G), float(eps2), _ptr(m), _ptr(x), _ptr(v),
                               ctypes.byref(ke), ctypes.byref(pe))
    if rc:
        raise OracleError("coincident pair with eps = 0")
    return ke.value, pe.value


def hermite(m, x, v, eps2: float, dt: float, nsteps: int, G: float = 1.0,
            acc=None, jerk=None):
    """Advance (x, v) by nsteps Hermite-4 P(EC)^1 steps (R#3).

    If acc/jerk (a0, j0 at the given state) are None they are evaluated first.
    Returns (x, v, acc, jerk) with acc/jerk evaluated at the last predicted
    state (the a0, j0 of the next step).
    """
    m = _f64(m)
    n = m.shape[0]
    x = _f64(x, (3, n)).copy()
    v = _f64(v, (3, n)).copy()
    init = acc is None or jerk is None
    acc = np.zeros((3, n)) if init else _f64(acc, (3, n)).copy()
    jerk = np.zeros((3, n)) if init else _f64(jerk, (3, n)).copy()
    rc = _load().oracle_hermite(n, float(G), float(eps2), float(dt), int(nsteps),
                                _ptr(m), _ptr(x), _ptr(v), _ptr(acc), _ptr(jerk),
                                1 if init else 0)
    if rc == 1:
        raise OracleError("coincident pair with eps = 0")
    if rc == 3:
        raise OracleError("non-finite state")
    if rc:
        raise OracleError(f"oracle_hermite failed rc={rc}")
    return x, v, acc, jerk


def leapfrog(m, x, v, eps2: float, dt: float, nsteps: int, G: float = 1.0, acc=None):
    """Advance (x, v) by nsteps kick-drift-kick steps.

    Returns (x, v, acc) with acc = a(x) at the final state.
    """
    m = _f64(m)
    n = m.shape[0]
    x = _f64(x, (3, n)).copy()
    v = _f64(v, (3, n)).copy()
    init = acc is None
    acc = np.zeros((3, n)) if init else _f64(acc, (3, n)).copy()
    rc = _load().oracle_leapfrog(n, float(G), float(eps2), float(dt), int(nsteps),
                                 _ptr(m), _ptr(x), _ptr(v), _ptr(acc), 1 if init else 0)
    if rc == 1:
        raise OracleError("coincident pair with eps = 0")
    if rc:
        raise OracleError(f"oracle_leapfrog failed rc={rc}")
    return x, v, acc


def block_init_levels(acc, jerk, dt_max: float, kmax: int, eta_s: float):
    """Initial block levels k (dt = dt_max / 2^k) from eta_s |a| / |j| (R#28).

    Returns (level int32 [n], criterion fp64 [n])."""
    acc = _f64(acc)
    n = acc.shape[1]
    jerk = _f64(jerk, (3, n))
    level = np.zeros(n, dtype=np.int32)
    crit = np.zeros(n)
    _load().oracle_block_init_levels(n, float(dt_max), int(kmax), float(eta_s), _ptr(acc),
                                     _ptr(jerk), _ptr(level), _ptr(crit))
    return level, crit


def hermite_block(m, x, v, eps2: float, dt_max: float, ncycles: int, eta: float,
                  eta_s: float = 0.01, kmax: int = 20, G: float = 1.0, acc=None, jerk=None,
                  level=None, derivs=False):
    """Advance (x, v) by ncycles * dt_max with block (individual) time steps (R#28).

    If acc/jerk/level are None, forces and initial levels are evaluated first.
    Returns (x, v, acc, jerk, level, stats, crit): stats = (block steps, sum of
    active counts), crit = the last Aarseth criterion value of every particle.
    With derivs=True two more arrays follow: the interpolated a^(2)(t) and a^(3) [3][n]
    each particle's last criterion used.
    """
    m = _f64(m)
    n = m.shape[0]
    x = _f64(x, (3, n)).copy()
    v = _f64(v, (3, n)).copy()
    init = acc is None or jerk is None or level is None
    acc = np.zeros((3, n)) if init else _f64(acc, (3, n)).copy()
    jerk = np.zeros((3, n)) if init else _f64(jerk, (3, n)).copy()
    level = (np.zeros(n, dtype=np.int32) if init
             else np.ascontiguousarray(level, dtype=np.int32).copy())
    stats = np.zeros(2, dtype=np.int64)
    crit = np.full(n, np.nan)
    d2 = np.full((3, n), np.nan) if derivs else None
    d3 = np.full((3, n), np.nan) if derivs else None
    rc = _load().oracle_hermite_block(n, float(G), float(eps2), float(dt_max), int(kmax),
                                      float(eta), float(eta_s), int(ncycles), _ptr(m), _ptr(x),
                                      _ptr(v), _ptr(acc), _ptr(jerk), _ptr(level),
                                      1 if init else 0, _ptr(stats), _ptr(crit), _ptr(d2),
                                      _ptr(d3))
    if rc == 1:
        raise OracleError("coincident pair with eps = 0")
    if rc == 3:
        raise OracleError("non-finite state")
    if rc:
        raise OracleError(f"oracle_hermite_block failed rc={rc}")
    out = (x, v, acc, jerk, level, (int(stats[0]), int(stats[1])), crit)
    return out + (d2, d3) if derivs else out
