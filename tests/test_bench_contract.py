"""bench.py keeps the driver's contract: one JSON line with the required keys.
The reference arm runs on the CPU (here); the device arm on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line(ref):
    d = _run(["--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "3",
              "--cpu-seconds", "1"], 600)
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["metric"] == "green_fn_evals_per_s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert set(d["modes"]) == {"direct", "table"}


@pytest.mark.gpu
def test_device_arm_line():
    d = _run(["--config", "c2", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1",
              "--c1", "0", "--vs-n", "0"], 900)
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["value"] > 1e10 and d["higher_is_better"] is True and d["dtype"] == "f64"
    rf = d["roofline"]
    assert rf["bound"] == "fp64" and 0 < rf["frac"] < 1.2 and rf["peak"] > 20
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 1280 ** 2 * 16
    assert d["gpu_launches"] >= 3 and d["clocks"]["sm_max_mhz"]
    assert d["config"]["workload"].startswith("C2")
    # the reference's calls per step vs the evaluations the kernel performed
    assert 0 < d["evaluations_per_step"] <= 3 * 6 * 4 * 1280 * 1279
    assert d["value_definition"] and d["modes"]["direct"]["evaluations_per_step"] > 0
