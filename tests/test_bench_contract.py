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


def _run(args, timeout, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line(ref):
    d = _run(["--impl", "reference", "--config", "c2", "--steps", "2", "--warmup", "3",
              "--cpu-seconds", "1"], 600)
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["metric"] == "green_fn_evals_per_s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["single_thread"]["value"] > 0      # threads = 1 too
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert set(d["modes"]) == {"direct", "table"} and d["mode_used"] in d["modes"]
    # the reference arm runs the reference only: never this package's library
    assert d["repo_libs_loaded"] == ["oracle/_ref/libgkref.so"], d["repo_libs_loaded"]
    # a step is a bounded sample: ms_per_step is its wall time, not an extrapolation
    assert d["ms_per_step"] < 60e3 and d["full_fill_s_extrapolated"] > 0
    # the same `config` object as the GPU arm's line (bench.config_of)
    import bench
    assert d["config"] == bench.config_of(bench.CONFIGS["c2"], 10000)


def test_reference_arm_never_maps_the_product_library(ref):
    """in-process check of the rule the driver applies to the reference arm"""
    code = ("import bench, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c2',"
            " '--steps', '1', '--warmup', '3', '--cpu-seconds', '0.5', '--cpu-single', '0'];"
            " bench.main(); maps = open('/proc/self/maps').read();"
            " assert 'libgk.so' not in maps and 'libgkref.so' in maps, 'libgk mapped';"
            " assert 'paper_1901_04162_b200' not in sys.modules; print('CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       timeout=300)
    assert r.returncode == 0 and "CLEAN" in r.stdout, r.stderr[-2000:]


def test_cpu_baseline_subprocess_is_the_reference_arm_code(ref):
    """the GPU arm's cpu_baseline leg: a clean subprocess of oracle/cpu_bench
    (no torch, no libgk), summarised with both thread counts"""
    import bench
    res = bench.cpu_baseline_subprocess(bench.CONFIGS["c2"], 10000, 1.0, 0.5)
    cb = bench.cpu_summary(res, 10000)
    assert cb["kind"] == "reference" and cb["value"] > 0 and cb["cores"] >= 1
    assert set(cb["modes"]) == {"direct", "table"} and cb["single_thread"]["value"] > 0
    assert res["N"] == 1280 and res["total_evals_per_fill"] == 3 * 6 * 4 * 1280 * 1279


def test_cpu_bench_mesh_is_the_workload_mesh(ref, oracle):
    """oracle/cpu_bench builds the bench mesh from the reference's own
    generate_sphere_mesh + a numpy restatement of the seeded jitter:
    bit-identical to the C restatement (and to libgk's gk_jitter, whose
    host-only entry point needs no GPU)"""
    import numpy as np
    from oracle.cpu_bench import jitter
    v, t = ref.sphere_mesh(1.0, 3)
    assert np.array_equal(jitter(v), oracle.jitter(v.copy(), 1901, 1e-3))
    import paper_1901_04162_b200 as gk
    m = gk.jitter(gk.generate_sphere_mesh(1.0, 3), 1901, 1e-3)
    assert np.array_equal(m.vertices, jitter(v)) and np.array_equal(m.triangles, t)


def test_selftest_gloo_two_ranks(ref):
    """bench.py --gpus 2 self-launches 2 ranks (torch.distributed.run); the
    gloo self-test runs the orchestration: row blocks, barriers, MAX over
    ranks, one JSON line from rank 0"""
    d = _run(["--selftest", "gloo", "--gpus", "2", "--config", "c2", "--steps", "2",
              "--warmup", "3"], 600)
    assert d["n_gpus"] == 2 and d["impl"] == "selftest-gloo"
    assert len(d["per_rank_ms"]) == 2 and d["ms_per_step"] == max(d["per_rank_ms"])
    assert d["row_blocks"] == [[0, 640], [640, 1280]]


def test_gpus_must_match_world_size():
    """under torchrun, --gpus N must equal WORLD_SIZE (no silent 1-GPU line)"""
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


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
    assert d["config"]["workload"].startswith("C2") and d["mode_used"] in ("direct", "table")
    assert d["cpu_baseline"]["single_thread"]["value"] > 0
    # the reference's calls per step vs the evaluations the kernel performed
    assert 0 < d["evaluations_per_step"] <= 3 * 6 * 4 * 1280 * 1279
    assert d["value_definition"] and d["modes"]["direct"]["evaluations_per_step"] > 0
