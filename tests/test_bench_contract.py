"""bench.py contract: one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_runs_on_cpu():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"], 300)
    assert d["impl"] == "reference" and KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "interactions/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_json_line():
    d = _run(["--config", "C2", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1"], 600)
    assert KEYS <= set(d) and {"roofline", "clocks", "gpu_launches", "energy"} <= set(d)
    assert d["value"] > 1e11 and d["n_gpus"] == 1 and d["scaling"] == "strong"
    rf = d["roofline"]
    assert rf["bound"] == "alu" and 0 < rf["frac"] < 1.0 and rf["unit"] == "TFLOP/s"
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert d["e2e"]["h2d_bytes_per_step"] == 48 * 16384 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
