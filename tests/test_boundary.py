"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/nbody.h declares, its host-only plan logic is right, and compute
entry points fail loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2509_19294_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nbody.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nbody_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("nbody_init", "nbody_compute_forces", "nbody_step", "nbody_energy",
              "nbody_destroy", "nbody_last_error", "nbody_plan"):
        assert s in syms
    assert set(syms) == set(binding.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = binding.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_exports_are_c_linkage():
    import subprocess
    from paper_2509_19294_b200 import _build
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True, check=True).stdout
    names = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for s in declared_symbols():
        assert s in names, f"{s} not exported unmangled"


def test_library_is_sm100a_only():
    import subprocess
    from paper_2509_19294_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_force_kernel_uses_packed_fp32x2_and_bulk_tma():
    """SASS evidence: FFMA2/FADD2/FMUL2 in the hot loop, MUFU.RSQ, UBLKCP (cp.async.bulk)."""
    import subprocess
    from paper_2509_19294_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    force = [b for b in blocks if b.startswith("_ZN2nb") and "force_kernel" in b.split("\n")[0]]
    assert force
    for b in force:
        for op in ("FFMA2", "FADD2", "FMUL2", "MUFU.RSQ", "UBLKCP", "SYNCS"):
            assert op in b, op
        assert "HMMA" not in b and "UTCHMMA" not in b   # no tensor cores: not a contraction


def _sass_loops(block):
    """(opcode histogram, body) of every backward-branch loop in one SASS function."""
    import collections
    ins = []
    for ln in block.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    at = {a: k for k, (a, _) in enumerate(ins)}
    loops = []
    for k, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?(?:\.ANY)? (?:!?U?P\w+, )?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a and int(m.group(1), 16) in at:
            body = [x for _, x in ins[at[int(m.group(1), 16)]:k + 1]]
            ops = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0]
                                      for x in body)
            loops.append(ops)
    return loops


# FP32 instructions per packed i-pair and j (R#20): acceleration + jerk 26
# (7 FFMA2 + 3 FMUL2 + ... = 40 flops per interaction), acceleration only 12 (18 flops),
# hi/lo positions + 6 FADD2; 2 MUFU.RSQ (one per lane) in every form.
@pytest.mark.parametrize("jerk,hilo,packed", [(1, 0, 26), (0, 0, 12), (1, 1, 32), (0, 1, 18)])
def test_force_hot_loop_instruction_histogram(jerk, hilo, packed):
    """SASS opcode count of the 1024-i CTA shape's j loop: per i-pair and j
    exactly `packed` FFMA2/FADD2/FMUL2 and 2 MUFU.RSQ, no scalar FP32 arithmetic, no
    FP64 and no tensor-core instruction -- a regression that adds scalar FMULs, splits a
    packed op or leaves a conversion in the loop fails here."""
    import subprocess
    from paper_2509_19294_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    # force_kernel<guard = false, jerk, hilo, CfgBig (4 pairs x 128 threads), list = false>
    pat = re.compile(rf"force_kernelILb0ELb{jerk}ELb{hilo}ENS0_5FkCfgILi4ELi128E.*ELb0EEEvNS_9ForceArgsE")
    fn = [b for b in blocks if pat.search(b.split("\n")[0])]
    assert len(fn) == 1, [b.split("\n")[0] for b in fn]
    loops = _sass_loops(fn[0])
    hot = min((c for c in loops if c["MUFU"]), key=lambda c: sum(c.values()))   # innermost j loop
    pairs = 4
    nj = hot["MUFU"] / (2 * pairs)          # j interactions per loop iteration
    assert nj >= 1 and nj == int(nj), hot
    assert hot["FFMA2"] + hot["FADD2"] + hot["FMUL2"] == packed * pairs * nj, hot
    for op in ("FFMA", "FADD", "FMUL", "DFMA", "DADD", "DMUL", "F2F", "HMMA", "UTCHMMA"):
        assert hot[op] == 0, (op, hot)


@pytest.mark.parametrize("n,world", [(2, 1), (1000, 3), (1024, 4), (262144, 8), (1048576, 8),
                                     (131072, 2), (12345, 7)])
def test_plan_partition_covers_all_particles(n, world):
    """SPEC S:96 contiguous partition: ranks tile [0, n) in order, equal `slot`
    slices (padding at the tail only), chunks <= 128 and multiples of the 256-j tile."""
    ranges = [binding.plan(n, world, r) for r in range(world)]
    assert ranges[0]["i0"] == 0 and ranges[-1]["i1"] == n
    for a, b in zip(ranges, ranges[1:]):
        assert a["i1"] == b["i0"]
    p = ranges[0]
    assert p["slot"] == 1024 * -(-n // (1024 * world))   # smallest multiple of the i-block
    assert p["chunk"] % 256 == 0 and p["n_chunks"] <= 128
    assert (p["n_chunks"] - 1) * p["chunk"] < n <= p["n_chunks"] * p["chunk"]
    # chunking does not depend on world (bit-identity across P)
    assert all(r["chunk"] == binding.plan(n, 1, 0)["chunk"] for r in ranges)


def test_plan_rejects_bad_arguments():
    for args in [(1, 1, 0), (10, 0, 0), (10, 11, 0), (10, 2, 2), (10, 2, -1),
                 (2**31, 1, 0), (2**33, 2, 1)]:   # > 2^31 - 1 particles per shard
        with pytest.raises(binding.NBodyError) as e:
            binding.plan(*args)
        assert e.value.code == binding.NBODY_EINVAL


def test_init_validates_scalars_before_touching_the_device():
    L = binding.lib()
    m = np.ones(4)
    x = np.zeros((3, 4))
    for kw, frag in [(dict(eps=-1.0), "eps"), (dict(dt=0.0), "dt"), (dict(G=float("nan")), "G"),
                     (dict(world=2), "nccl_id")]:
        c = dict(n=4, G=1.0, eps=0.1, dt=0.01, world=1)
        c.update(kw)
        cfg = binding.Config(**c)
        ctx = ctypes.c_void_p()
        rc = L.nbody_init(ctypes.byref(cfg), m.ctypes.data, x.ctypes.data, x.ctypes.data,
                          ctypes.byref(ctx))
        assert rc == binding.NBODY_EINVAL and not ctx.value
        assert frag in L.nbody_last_error(None).decode()


def test_no_cpu_fallback():
    """Without a CUDA device the product refuses to run (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(binding.NBodyError):
        binding.NBody(np.ones(4), np.zeros((3, 4)), np.zeros((3, 4)), eps=0.1, dt=0.01)
    L = binding.lib()
    cfg = binding.Config(n=4, G=1.0, eps=0.1, dt=0.01, world=1)
    ctx = ctypes.c_void_p()
    m = np.ones(4)
    x = np.zeros((3, 4))
    rc = L.nbody_init(ctypes.byref(cfg), m.ctypes.data, x.ctypes.data, x.ctypes.data, ctypes.byref(ctx))
    assert rc == binding.NBODY_ECUDA


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (parity independence)."""
    pkg = os.path.join(ROOT, "paper_2509_19294_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src and "oracle_forces" not in src, f


def _build_c_demo(tmp_path):
    import subprocess
    exe = tmp_path / "c_api_demo"
    lib_dir = os.path.join(ROOT, "paper_2509_19294_b200")
    binding.lib()   # builds libnbody.so if missing
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-o", str(exe),
                    os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", lib_dir, "-lnbody",
                    f"-Wl,-rpath,{lib_dir}", "-lm"], check=True)
    return exe


def test_c_program_links_against_the_c_abi(tmp_path):
    """examples/c_api_demo.c compiles against include/nbody.h and links libnbody.so with a
    plain C compiler (no C++, no torch); the host-only nbody_plan runs without a GPU."""
    import subprocess
    exe = _build_c_demo(tmp_path)
    out = subprocess.run([str(exe), "1000", "plan"], capture_output=True, text=True, check=True).stdout
    assert "chunk=256 n_chunks=4" in out


@pytest.mark.gpu
def test_c_program_runs_the_hot_path(tmp_path):
    """The same C program on the GPU: forces into host arrays, 10 Hermite steps, energy,
    then checkpoint / resume in a second context, bit-identical after 5 more steps."""
    import re
    import subprocess
    exe = _build_c_demo(tmp_path)
    out = subprocess.run([str(exe), "4096"], capture_output=True, text=True, check=True).stdout
    rel = float(re.search(r"rel\. change ([0-9.e+-]+)", out).group(1))
    assert rel < 1e-6, out
    assert "resume: bit-identical" in out, out
