"""Thin ctypes binding over libnbody.so (include/nbody.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Tensors may be torch tensors (CUDA or CPU) or numpy arrays;
they are passed to the C-ABI as raw pointers.  There is no fallback: if the
library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

NBODY_OK, NBODY_EINVAL, NBODY_ENONFINITE, NBODY_ECUDA, NBODY_ENCCL, NBODY_ENOMEM, NBODY_ESTATE = range(7)
NBODY_HERMITE4, NBODY_LEAPFROG_KDK, NBODY_HERMITE4_BLOCK = 0, 1, 2
INTEGRATORS = {"hermite": NBODY_HERMITE4, "leapfrog": NBODY_LEAPFROG_KDK, "block": NBODY_HERMITE4_BLOCK}

EXPORTS = (
    "nbody_plan", "nbody_nccl_unique_id", "nbody_init", "nbody_local_range",
    "nbody_compute_forces", "nbody_step", "nbody_energy", "nbody_get_state",
    "nbody_set_state", "nbody_sync", "nbody_prof_enable", "nbody_prof_read",
    "nbody_prof_launch_times", "nbody_prof_launch_sizes", "nbody_block_stats",
    "nbody_get_derivs", "nbody_set_derivs", "nbody_set_levels", "nbody_exec_stats",
    "nbody_last_error", "nbody_destroy",
)


class NBodyError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[nbody status {code}] {msg}")
        self.code = code


class Config(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("G", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("integrator", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("loopback", ctypes.c_int32),
        ("jchunks", ctypes.c_int32),
        ("hilo", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("eta", ctypes.c_double),
        ("eta_s", ctypes.c_double),
        ("kmax", ctypes.c_int32),
    ]


_lib = None


def _set_nccl_path():
    if os.environ.get("NBODY_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        p = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["NBODY_NCCL_LIB"] = p   # the NCCL torch itself loads
    except Exception:
        pass


def lib():
    """Load (building first if missing or stale) libnbody.so."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("NBODY_LIB")    # tuning sweeps only (scripts/sweep_force.py)
    if not path:
        path = _build.build() if _build.stale() else _build.LIB
    _set_nccl_path()
    L = ctypes.CDLL(path)
    i32, i64, p, d = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
    P64 = ctypes.POINTER(i64)
    Pd = ctypes.POINTER(d)
    sig = {
        "nbody_plan": ([i64, i32, i32, i32, P64, P64, P64, P64, P64], ctypes.c_int),
        "nbody_nccl_unique_id": ([p], ctypes.c_int),
        "nbody_init": ([ctypes.POINTER(Config), p, p, p, ctypes.POINTER(p)], ctypes.c_int),
        "nbody_local_range": ([p, P64, P64], ctypes.c_int),
        "nbody_compute_forces": ([p, p, p], ctypes.c_int),
        "nbody_step": ([p, i32], ctypes.c_int),
        "nbody_energy": ([p, Pd, Pd], ctypes.c_int),
        "nbody_get_state": ([p, p, p], ctypes.c_int),
        "nbody_set_state": ([p, p, p, i32], ctypes.c_int),
        "nbody_sync": ([p], ctypes.c_int),
        "nbody_prof_enable": ([p, i32], ctypes.c_int),
        "nbody_prof_read": ([p, Pd, P64, P64, i32], ctypes.c_int),
        "nbody_prof_launch_times": ([p, p, i64, P64], ctypes.c_int),
        "nbody_prof_launch_sizes": ([p, p, p, i64, P64], ctypes.c_int),
        "nbody_block_stats": ([p, P64, P64, p], ctypes.c_int),
        "nbody_get_derivs": ([p, p, p], ctypes.c_int),
        "nbody_set_derivs": ([p, p, p], ctypes.c_int),
        "nbody_set_levels": ([p, p], ctypes.c_int),
        "nbody_exec_stats": ([p, P64, P64], ctypes.c_int),
        "nbody_last_error": ([p], ctypes.c_char_p),
        "nbody_destroy": ([p], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc, ctx=None):
    if rc != NBODY_OK:
        msg = lib().nbody_last_error(ctx).decode()
        raise NBodyError(rc, msg)


def plan(n, world=1, rank=0, jchunks=0):
    """Partition / reduction plan (host-only): dict(i0, i1, slot, chunk, n_chunks)."""
    out = [ctypes.c_int64() for _ in range(5)]
    _check(lib().nbody_plan(n, world, rank, jchunks, *[ctypes.byref(o) for o in out]))
    return dict(zip(("i0", "i1", "slot", "chunk", "n_chunks"), (o.value for o in out)))


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().nbody_nccl_unique_id(buf))
    return bytes(buf)


def _ptr(a):
    """Raw data pointer of a contiguous float64 torch tensor / numpy array."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("numpy arrays must be C-contiguous float64")
        return a.ctypes.data
    import torch
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("tensors must be contiguous float64")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _want(a, shape, name):
    """Shape check before a raw pointer crosses the C-ABI (which trusts sizes)."""
    if a is not None and tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(a.shape)}")


class NBody:
    """One rank's (or, with loopback=True, all ranks') view of an N-body system.

    m: (n,), x, v: (3, n) float64 of the FULL system (torch CUDA/CPU tensors or
    numpy).  Work is ordered on ``stream`` (a torch.cuda.Stream, a raw
    cudaStream_t int, or None for torch's current stream).

    Stream hygiene with a torch stream other than the current one: the library's
    stream first waits on the current stream (inputs produced there are complete
    before the library reads them); conversions and output tensors are made on the
    library's stream, torch tensors the library writes are recorded on it (the
    caching allocator will not hand their memory out while it is still in use), and
    the current stream waits on the library's stream after every call that writes
    tensors, so results are safe to consume in torch's current stream order.
    """

    def __init__(self, m, x, v, eps, dt, G=1.0, integrator="hermite", rank=0, world=1,
                 loopback=False, nccl_id=None, device=None, stream=None, jchunks=0, hilo=None,
                 eta=0.02, eta_s=0.01, kmax=20):
        import torch
        if not torch.cuda.is_available():
            raise NBodyError(NBODY_ECUDA, "no CUDA device: libnbody has no CPU path")
        if device is None:
            device = torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._tstream = stream if hasattr(stream, "cuda_stream") else None   # torch stream object
        raw_stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        if raw_stream == 0:
            raw_stream = 1   # cudaStreamLegacy: torch's default stream, not "library-created"
        self._keep = []
        self._enter()
        with self._on_stream():
            m, x, v = (self._prep(a) for a in (m, x, v))
        if m.ndim != 1:
            raise ValueError("m must be one-dimensional (n,)")
        n = int(m.shape[0])
        _want(x, (3, n), "x")
        _want(v, (3, n), "v")
        if hilo is None:
            # block time steps difference forces over dt^2..dt^3 for the Aarseth
            # criterion; fp32-rounded positions make it noisy (R#28), so
            # two-float positions are the default there
            hilo = integrator == "block"
        cfg = Config(n=n, G=float(G), eps=float(eps), dt=float(dt),
                     integrator=INTEGRATORS[integrator],
                     device=int(device), rank=int(rank), world=int(world),
                     loopback=1 if loopback else 0, jchunks=int(jchunks), hilo=1 if hilo else 0,
                     nccl_id=None, stream=raw_stream, eta=float(eta), eta_s=float(eta_s),
                     kmax=int(kmax))
        if nccl_id is not None:
            idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            self._keep.append(idbuf)
            cfg.nccl_id = ctypes.addressof(idbuf)
        self.cfg = cfg
        self.n = n
        self.device = torch.device("cuda", int(device))
        ctx = ctypes.c_void_p()
        _check(lib().nbody_init(ctypes.byref(cfg), _ptr(m), _ptr(x), _ptr(v), ctypes.byref(ctx)))
        self._ctx = ctx
        i0, i1 = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().nbody_local_range(ctx, ctypes.byref(i0), ctypes.byref(i1)), ctx)
        self.i0, self.i1 = i0.value, i1.value
        self.n_loc = self.i1 - self.i0

    def _cur(self):
        import torch
        return torch.cuda.current_stream(self._tstream.device) if self._tstream is not None else None

    def _enter(self):
        """The library's stream waits on the current one (inputs made there are ready)."""
        cur = self._cur()
        if cur is not None and cur.cuda_stream != self._tstream.cuda_stream:
            self._tstream.wait_stream(cur)

    def _on_stream(self):
        import contextlib
        import torch
        return torch.cuda.stream(self._tstream) if self._tstream is not None else contextlib.nullcontext()

    def _written(self, *ts):
        """Tensors the library wrote on its stream: keep their memory alive for it and
        order the current stream after it."""
        import torch
        if self._tstream is None:
            return
        for t in ts:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(self._tstream)
        cur = self._cur()
        if cur.cuda_stream != self._tstream.cuda_stream:
            cur.wait_stream(self._tstream)

    def _empty3(self):
        import torch
        with self._on_stream():
            return torch.empty((3, self.n_loc), dtype=torch.float64, device=self.device)

    @staticmethod
    def _prep(a):
        if isinstance(a, np.ndarray):
            return np.ascontiguousarray(a, dtype=np.float64)
        return a.contiguous().to(dtype=__import__("torch").float64)

    def _c(self, rc):
        _check(rc, self._ctx)

    def forces(self, acc=None, jerk=None):
        """(acc, jerk) of the local particles, (3, n_loc) float64 CUDA tensors."""
        acc = self._empty3() if acc is None else acc
        jerk = self._empty3() if jerk is None else jerk
        _want(acc, (3, self.n_loc), "acc")
        _want(jerk, (3, self.n_loc), "jerk")
        self._enter()
        self._c(lib().nbody_compute_forces(self._ctx, _ptr(acc), _ptr(jerk)))
        self._written(acc, jerk)
        return acc, jerk

    def step(self, nsteps=1):
        self._c(lib().nbody_step(self._ctx, int(nsteps)))
        self._written()

    def energy(self):
        ke, pe = ctypes.c_double(), ctypes.c_double()
        self._c(lib().nbody_energy(self._ctx, ctypes.byref(ke), ctypes.byref(pe)))
        return ke.value, pe.value

    def state(self, x=None, v=None):
        x = self._empty3() if x is None else x
        v = self._empty3() if v is None else v
        _want(x, (3, self.n_loc), "x")
        _want(v, (3, self.n_loc), "v")
        self._enter()
        self._c(lib().nbody_get_state(self._ctx, _ptr(x), _ptr(v)))
        self._written(x, v)
        return x, v

    def set_state(self, x, v, keep_forces=False):
        """Overwrite the local (3, n_loc) positions and/or velocities (None keeps them)."""
        _want(x, (3, self.n_loc), "x")
        _want(v, (3, self.n_loc), "v")
        self._enter()
        self._c(lib().nbody_set_state(self._ctx, _ptr(x), _ptr(v), 1 if keep_forces else 0))

    def derivs(self, acc=None, jerk=None):
        """(acc, jerk) the next step starts from, (3, n_loc) float64 (checkpointing)."""
        acc = self._empty3() if acc is None else acc
        jerk = self._empty3() if jerk is None else jerk
        _want(acc, (3, self.n_loc), "acc")
        _want(jerk, (3, self.n_loc), "jerk")
        self._enter()
        self._c(lib().nbody_get_derivs(self._ctx, _ptr(acc), _ptr(jerk)))
        self._written(acc, jerk)
        return acc, jerk

    def set_derivs(self, acc, jerk=None):
        """Restore saved derivatives (exact resume; jerk unused by leapfrog)."""
        _want(acc, (3, self.n_loc), "acc")
        _want(jerk, (3, self.n_loc), "jerk")
        self._enter()
        self._c(lib().nbody_set_derivs(self._ctx, _ptr(acc), _ptr(jerk)))

    def set_levels(self, level):
        """Block time steps: restore saved levels, int32 (n_loc,)."""
        lev = np.ascontiguousarray(level, dtype=np.int32)
        if lev.shape != (self.n_loc,):
            raise ValueError(f"level must have shape ({self.n_loc},), got {lev.shape}")
        self._c(lib().nbody_set_levels(self._ctx, lev.ctypes.data))

    def sync(self):
        self._c(lib().nbody_sync(self._ctx))

    def prof_enable(self, on=True):
        self._c(lib().nbody_prof_enable(self._ctx, 1 if on else 0))

    def prof_read(self, reset=True):
        ms, nf, nk = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        self._c(lib().nbody_prof_read(self._ctx, ctypes.byref(ms), ctypes.byref(nf),
                                      ctypes.byref(nk), 1 if reset else 0))
        return ms.value, nf.value, nk.value

    def prof_launch_times(self):
        """Per-launch force-kernel times (ms) since the last prof_read(reset=True)."""
        n = ctypes.c_int64()
        self._c(lib().nbody_prof_launch_times(self._ctx, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value)
        self._c(lib().nbody_prof_launch_times(self._ctx, out.ctypes.data, n.value, ctypes.byref(n)))
        return out

    def prof_launch_sizes(self):
        """(n_i, n_j) int64 arrays of the launches prof_launch_times() reports."""
        n = ctypes.c_int64()
        self._c(lib().nbody_prof_launch_sizes(self._ctx, None, None, 0, ctypes.byref(n)))
        ni, nj = np.zeros(n.value, dtype=np.int64), np.zeros(n.value, dtype=np.int64)
        self._c(lib().nbody_prof_launch_sizes(self._ctx, ni.ctypes.data, nj.ctypes.data, n.value,
                                              ctypes.byref(n)))
        return ni, nj

    def block_stats(self, levels=False):
        """Block time steps: (block steps, sum of active counts[, levels int32 (n_loc,)])."""
        bs, asum = ctypes.c_int64(), ctypes.c_int64()
        lev = np.zeros(self.n_loc, dtype=np.int32) if levels else None
        self._c(lib().nbody_block_stats(self._ctx, ctypes.byref(bs), ctypes.byref(asum),
                                        None if lev is None else lev.ctypes.data))
        return (bs.value, asum.value, lev) if levels else (bs.value, asum.value)

    def exec_stats(self):
        """(CUDA-graph launches, eagerly launched steps) since init."""
        g, e = ctypes.c_int64(), ctypes.c_int64()
        self._c(lib().nbody_exec_stats(self._ctx, ctypes.byref(g), ctypes.byref(e)))
        return g.value, e.value

    def close(self):
        if getattr(self, "_ctx", None):
            lib().nbody_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
