"""Build libnbody.so in-tree: nvcc, sm_100a only (no other targets, no JIT).

Called by ``__graft_entry__.build()`` and, when the library is missing or
stale, by :mod:`paper_2509_19294_b200.binding`.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnbody.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-ftz=true",              # FP32: MUFU.RSQ without the denormal guard
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + [os.path.join(INCLUDE, "nbody.h")])


def nccl_include() -> str:
    cands = []
    try:
        import nvidia.nccl  # noqa: F401  (torch's NCCL wheel; headers only are used)
        cands.append(os.path.join(list(nvidia.nccl.__path__)[0], "include"))
    except Exception:
        pass
    cands.append("/usr/include")
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (needed for NCCL type declarations)")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None,
          extra_flags=()) -> str:
    """Compile every csrc/*.cu into one shared library (default: the in-tree LIB).

    `defines` (e.g. ["FK_PAIRS=3"]), `extra_flags` and `out` build tuning variants
    elsewhere (scripts/sweep_force.py); the product library is always the default."""
    target = out or LIB
    if not force and not defines and not extra_flags and out is None and not stale():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *extra_flags, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC,
           "-I", nccl_include(), "-o", tmp, *sources(), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        print(r.stdout)
        print(r.stderr)
    if r.returncode:
        raise RuntimeError(f"nvcc failed ({r.returncode})")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
