"""Comparison metrics (readings R#11-R#13).  Plain numpy, no method arithmetic."""
import numpy as np


def max_rel(gpu, ref):
    """max_i |q_i^gpu - q_i^ref|_2 / |q_i^ref|_2 over particles (columns)."""
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    num = np.linalg.norm(gpu - ref, axis=0)
    den = np.linalg.norm(ref, axis=0)
    return float(np.max(num / den))


def paper_norm(gpu, ref):
    """max component error relative to the typical magnitude mean_i |q_i^ref| (R#13)."""
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    return float(np.max(np.abs(gpu - ref)) / np.mean(np.linalg.norm(ref, axis=0)))


def momentum_residual(m, q):
    return float(np.linalg.norm(q @ m) / np.sum(m * np.linalg.norm(q, axis=0)))


# Tolerances (BASELINE.json north_star; R#12)
TOL_ACC = 1e-5       # max per-particle relative acceleration error, fp32 vs fp64
TOL_JERK = 1e-4      # per-particle jerk (R#12)
TOL_PAPER_ACC = 5e-4  # 0.05 % of the typical magnitude
TOL_PAPER_JERK = 2e-3  # 0.2 %


def sample_indices(x, n_stride=8192, n_special=256, seed=0):
    """R#11 sample at C4/C5: evenly strided i, plus the most central, plus the nearest-neighbour pairs."""
    from scipy.spatial import cKDTree
    n = x.shape[1]
    strided = np.linspace(0, n - 1, min(n, n_stride)).astype(np.int64)
    r = np.linalg.norm(x, axis=0)
    central = np.argsort(r)[:n_special]
    d, _ = cKDTree(x.T).query(x.T, k=2)
    closest = np.argsort(d[:, 1])[:n_special]
    return np.unique(np.concatenate([strided, central, closest]))
