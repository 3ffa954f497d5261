"""bench.py keeps the driver's JSON-line contract (reference arm on CPU, our arm on GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["unit"] == "zone-cycles/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["dtype"] == "f64" and d["scaling"] == "weak"
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1.2 and r["peak"] > 10
    assert d["gpu_launches"] >= 4 * 5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    job = d["e2e"]["job"]  # the whole C4 job through the API, state from / to pinned host
    assert job["cycles"] == 100 and job["value"] > 0 and job["h2d_bytes"] == d["e2e"]["h2d_bytes_per_step"]
    assert "workload" in d["config"]
