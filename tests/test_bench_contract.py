"""bench.py keeps the driver's JSON-line contract (both arms)."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference runs the reference's CPU kernels (oracle/_ref, else the port)."""
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "vectors/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line(cuda_dev):
    d = _run(["--steps", "3", "--warmup", "3", "--e2e-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["gpu_launches"] == 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == (1 << 30) * 24 and e["d2h_bytes_per_step"] == (1 << 30) * 32
    assert d["value"] > 50e9 and e["value"] > 0.5e9
    assert d["validation"]["rows_counted"] == 1 << 30
    assert d["clocks"]["samples"] >= 1 and d["clocks"]["sm_max_mhz"]
    oc = d["other_configs"]
    assert {1, 2, 3, 4} <= {c["config"] for c in oc} <= {1, 2, 3, 4, 5}
    assert all(c["frac"] > 0.2 for c in oc)
    sd = d["sharded_driver"]
    assert "error" not in sd and len(sd["devices"]) == 2 and sd["rows"] == 1 << 30
    assert sd["gpu_launches"] == 10 and sd["vectors_per_s"] > 50e9
