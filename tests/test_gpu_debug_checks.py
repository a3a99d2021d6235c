"""The NB_DEBUG_CHECKS=1 build (device-side bounds asserts on every index the force and
block-step kernels derive from device data) runs every kernel instantiation on a small
case without tripping an assert -- the stand-in for compute-sanitizer memcheck, which
this GPU pool does not allow."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2509_19294_b200", "libnbody_debug.so")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("host_loop", [False, True])
def test_debug_checks_build_runs_clean(host_loop):
    """Both execution paths: CUDA graphs (default) and host-driven launches, where the
    block-step force launches carry the host's active count."""
    from paper_2509_19294_b200 import _build
    if not os.path.exists(DEBUG_LIB) or os.path.getmtime(DEBUG_LIB) < max(
            os.path.getmtime(p) for p in _build._deps()):
        _build.build(defines=["NB_DEBUG_CHECKS=1"], out=DEBUG_LIB)
    env = dict(os.environ, NBODY_LIB=DEBUG_LIB)
    if host_loop:
        env["NBODY_NO_GRAPH"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize case ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
