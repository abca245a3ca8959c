"""Pin the C restatement (oracle/gk_oracle.c) bit for bit against the
unmodified reference compiled in place (oracle/_ref/libgkref.so), and run the
reference's own unit-test suite (oracle/_ref/unit_tests, GTest shim).
Skipped where the reference was not built (e.g. on the GPU box without a
prebuilt _ref)."""
import math
import os
import subprocess

import numpy as np
import pytest

from oracle.pyoracle import (DIRECT, EXP, GREEN, HERE, TABLE, SamplingConfig,
                             splitmix64_uniform)


def random_cfgs(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        lam = float(rng.uniform(0.3, 3.0))
        out.append((SamplingConfig(r_min=float(1e-4 * lam * rng.uniform(0.5, 50)),
                                   r_max=float(lam * rng.uniform(0.8, 2.5)),
                                   samples_per_wavelength=int(rng.integers(20, 20001)),
                                   refine_interval_divisor=int(rng.integers(2, 5)),
                                   refine_halfwidth_in_t=float(rng.uniform(1.0, 3.0)),
                                   dedup_fraction=float(rng.uniform(0.25, 1.0)),
                                   refine=bool(rng.uniform() < 0.9)),
                    (lam, float(rng.uniform(1, 4)), float(rng.uniform(1, 2)))))
    return out


@pytest.mark.parametrize("cfg,med", random_cfgs(40, 20261019))
def test_plan_hash_bitwise(oracle, ref, cfg, med):
    a = oracle.build_plan(cfg, *med)
    b = ref.build_plan(cfg, *med)
    assert np.array_equal(a.abscissae, b.abscissae)
    assert np.array_equal(a.zeros, b.zeros)
    assert a.t == b.t and a.dr_min == b.dr_min
    ha, hb = oracle.build_hash(a.abscissae, a.zeros), ref.build_hash(b.abscissae, b.zeros)
    assert np.array_equal(ha[0], hb[0]) and ha[1:] == hb[1:]


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_evaluator_bitwise(oracle, ref, degree):
    cfg = SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=3000)
    p = oracle.build_plan(cfg, 0.5)
    k = oracle.wavenumber(0.5)
    eo, er = oracle.evaluator(p, k, degree), ref.evaluator(p, k, degree)
    for x, y in zip(eo.tables(), er.tables()):
        assert np.array_equal(x, y)
    r = splitmix64_uniform(11, 100000, 1e-4, 2.0)
    for kind in (EXP, GREEN):
        assert np.array_equal(eo.eval_batch(kind, r), er.eval_batch(kind, r))
    assert eo.fallbacks == er.fallbacks > 0
    rr = splitmix64_uniform(12, 105, 1e-3, 2.0)
    w = splitmix64_uniform(13, 105, -1.0, 1.0)
    assert eo.accumulate_green(rr, w) == er.accumulate_green(rr, w)
    for x in splitmix64_uniform(14, 500, 1e-3, 2.0):
        for kind in (EXP, GREEN):
            for method in (0, 1):
                assert eo.pointwise_bound(kind, method, x) == er.pointwise_bound(kind, method, x)


@pytest.mark.parametrize("level,m,n,threads", [(0, 4, 3, 1), (1, 6, 4, 3), (1, 7, 5, 2),
                                               (2, 1, 1, 4)])
def test_fill_bitwise(oracle, ref, level, m, n, threads):
    v, t = ref.sphere_mesh(0.7, level)
    ov, ot = oracle.sphere_mesh(0.7, level)
    assert np.array_equal(v, ov) and np.array_equal(t, ot)
    v = oracle.jitter(v, 1901, 1e-3)
    po, pr = oracle.points(v, t, m, n), ref.points(v, t, m, n)
    assert np.array_equal(po[0], pr[0]) and np.array_equal(po[1], pr[1])
    k = 2 * math.pi
    za, ra = oracle.fill_rows(v, t, m, n, DIRECT, k, threads=threads)
    zb, rb = ref.fill_matrix(v, t, m, n, DIRECT, k, threads=1)
    assert np.array_equal(za, zb) and ra.actual_calls == rb.actual_calls
    lo, hi = oracle.distance_range(v, t, m, n)
    p = oracle.build_plan(SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=2000))
    eo, er = oracle.evaluator(p, k), ref.evaluator(p, k)
    za, ra = oracle.fill_rows(v, t, m, n, TABLE, k, ev=eo, threads=threads)
    zb, rb = ref.fill_matrix(v, t, m, n, TABLE, k, ev=er, threads=2)
    assert np.array_equal(za, zb) and ra.fallback_calls == rb.fallback_calls == 0


def test_fallback_counts_bitwise(oracle, ref):
    v, t = ref.sphere_mesh(0.5, 1)
    hi = ref.max_vertex_distance(v) * 1.01
    assert oracle.max_vertex_distance(v) * 1.01 == hi
    p = oracle.build_plan(SamplingConfig(r_min=0.3, r_max=hi))
    eo, er = oracle.evaluator(p, 2 * math.pi), ref.evaluator(p, 2 * math.pi)
    za, ra = oracle.fill_rows(v, t, 1, 1, TABLE, 2 * math.pi, ev=eo)
    zb, rb = ref.fill_matrix(v, t, 1, 1, TABLE, 2 * math.pi, ev=er)
    assert np.array_equal(za, zb)
    assert ra.fallback_calls == rb.fallback_calls > 0


def test_sampled_rows_match_full_fill(ref):
    v, t = ref.sphere_mesh(1.0, 1)
    z, _ = ref.fill_matrix(v, t, 4, 3, DIRECT, 2 * math.pi)
    rows = np.array([0, 13, 79], np.uint64)
    zs, calls, _ = ref.fill_sampled_rows(v, t, 4, 3, DIRECT, 2 * math.pi, rows, threads=2)
    assert np.array_equal(zs, z[rows.astype(int)]) and calls == 3 * 36 * 79


def test_reference_unit_suite_passes(ref):
    exe = os.path.join(HERE, "_ref", "unit_tests")
    if not os.path.exists(exe):
        pytest.skip("unit_tests not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "113 tests, 0 failed" in r.stdout
