"""Pin the C restatement (oracle/) against golden fixtures generated from the
reference itself (tests/golden/make_golden.py) and against the reference
tests' own known answers.  Runs without /root/reference and without a GPU.
"""
import math
import os

import numpy as np
import pytest

from oracle.pyoracle import DIRECT, EXP, GREEN, TABLE, OracleError, SamplingConfig

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
PLANS = {
    "default": (dict(), (1.0, 1.0, 1.0)),
    "refine_off": (dict(refine=False), (1.0, 1.0, 1.0)),
    "c1_s1e3": (dict(r_min=1e-3, r_max=2.0), (0.5, 1.0, 1.0)),
    "c2_s1e3": (dict(r_min=0.0118, r_max=1.9997), (1.0, 1.0, 1.0)),
    "dielectric": (dict(r_min=1e-3, r_max=1.3, samples_per_wavelength=700,
                        refine_interval_divisor=3, refine_halfwidth_in_t=2.5,
                        dedup_fraction=0.7), (0.8, 2.3, 1.7)),
    "overlap_small_S": (dict(samples_per_wavelength=20, refine_halfwidth_in_t=3.0),
                        (1.0, 1.0, 1.0)),
}


@pytest.mark.parametrize("name", sorted(PLANS))
def test_plan_and_hash_match_reference_fixture(oracle, name):
    kw, med = PLANS[name]
    p = oracle.build_plan(SamplingConfig(**kw), *med)
    assert np.array_equal(p.abscissae, GOLD[f"plan/{name}/abscissae"])
    assert np.array_equal(p.zeros, GOLD[f"plan/{name}/zeros"])
    t, dr, inv = GOLD[f"plan/{name}/t_dr"]
    assert p.t == t and p.dr_min == dr
    b, dr2, inv2 = oracle.build_hash(p.abscissae, p.zeros)
    assert np.array_equal(b, GOLD[f"plan/{name}/buckets"]) and inv2 == inv


def test_evaluator_matches_reference_fixture(oracle):
    p = oracle.build_plan(SamplingConfig())
    ev = oracle.evaluator(p, oracle.wavenumber())
    e, g = ev.tables()
    assert np.array_equal(e, GOLD["eval/exp_table"])
    assert np.array_equal(g, GOLD["eval/green_table"])
    r = GOLD["eval/radii"]
    assert np.array_equal(ev.eval_batch(EXP, r), GOLD["eval/exp"])
    assert np.array_equal(ev.eval_batch(GREEN, r), GOLD["eval/green"])
    assert ev.fallbacks == int(GOLD["eval/fallbacks"][0])
    acc = ev.accumulate_green(GOLD["acc/radii"], GOLD["acc/weights"])
    assert acc == complex(GOLD["acc/value"][0])


def test_fills_match_reference_fixture(oracle):
    v0, t0 = oracle.sphere_mesh(0.5, 0)
    z, rep = oracle.fill_rows(v0, t0, 4, 3, DIRECT, 2 * math.pi)
    assert np.array_equal(z, GOLD["fill/l0_direct"])
    assert [rep.actual_calls, rep.predicted_calls] == list(GOLD["fill/l0_direct_calls"])
    hi = oracle.max_vertex_distance(v0) * 1.01
    pt = oracle.build_plan(SamplingConfig(r_min=1e-4, r_max=hi, samples_per_wavelength=10000))
    assert np.array_equal(pt.abscissae, GOLD["fill/l0_table_plan"])
    ev = oracle.evaluator(pt, 2 * math.pi)
    zt, _ = oracle.fill_rows(v0, t0, 4, 3, TABLE, 2 * math.pi, ev=ev, threads=3)
    assert np.array_equal(zt, GOLD["fill/l0_table"])
    v1, t1 = oracle.sphere_mesh(1.0, 1)
    v1 = oracle.jitter(v1, 1901, 1e-3)
    assert np.array_equal(v1, GOLD["mesh/l1j/vertices"])
    assert np.array_equal(t1, GOLD["mesh/l1j/triangles"])
    z1, _ = oracle.fill_rows(v1, t1, 6, 4, DIRECT, 2 * math.pi, threads=4)
    assert np.array_equal(z1, GOLD["fill/l1j_direct_m6n4"])
    z2, _ = oracle.fill_rows(v1, t1, 3, 2, DIRECT, 2 * math.pi, kind=EXP)
    assert np.array_equal(z2, GOLD["fill/l1j_green_exp_m3n2"])


def test_quadrature_rules_match_reference_fixture(oracle):
    for m in (1, 3, 4, 6, 7):
        assert np.array_equal(oracle.triangle_rule(m), GOLD[f"quad/tri{m}"])
    for n in range(1, 8):
        assert np.array_equal(oracle.gauss_legendre_unit(n), GOLD[f"quad/gl{n}"])


# ---- the reference tests' own known answers (file:line in proj/tests/) ----

def test_kernel_hand_values(oracle):
    v = oracle.eval_analytic(EXP, 2 * math.pi, 0.25)           # test_kernel.cpp:32-36
    assert abs(v.real) <= 1e-15 and abs(v.imag + 1.0) <= 1e-15
    g = oracle.eval_analytic(GREEN, 2 * math.pi, 0.5)          # test_kernel.cpp:42-46
    assert abs(g.real + 2.0) <= 4e-15 and abs(g.imag) <= 1e-14
    assert oracle.eval_analytic(EXP, 7.3, 0.0) == 1.0          # test_kernel.cpp:38-40
    with pytest.raises(OracleError) as e:
        oracle.eval_analytic(GREEN, 1.0, 0.0)                  # domain_error
    assert e.value.status == 2
    with pytest.raises(OracleError) as e:
        oracle.eval_analytic(EXP, 1.0, -0.1)
    assert e.value.status == 1
    assert oracle.wavenumber(1.0, 4.0, 1.0) == 4 * math.pi     # test_kernel.cpp:19-21


def test_green_is_exp_over_r_bitwise(oracle):
    rng = np.random.default_rng(77)                            # test_kernel.cpp:71-81
    for _ in range(2000):
        k, r = rng.uniform(0, 30), rng.uniform(1e-6, 5.0)
        e, g = oracle.eval_analytic(EXP, k, r), oracle.eval_analytic(GREEN, k, r)
        assert g.real == e.real / r and g.imag == e.imag / r


def test_sampling_known_answers(oracle):
    z = oracle.zero_crossings(2 * math.pi, 1e-4, 1.0)          # test_sampling.cpp:42-49
    assert list(z) == [0.25, 0.5, 0.75, 1.0]
    assert oracle.zero_crossings(2 * math.pi, 0.3, 0.4).size == 0
    assert list(oracle.zero_crossings(math.pi, 0.1, 1.0)) == [0.5, 1.0]
    p = oracle.build_plan(SamplingConfig(refine=False))        # test_sampling.cpp:122-129
    assert p.abscissae.size == 1001 and p.zeros.size == 0
    p = oracle.build_plan(SamplingConfig())
    assert p.abscissae[0] == 1e-4 and p.abscissae[-1] == 1.0   # EndpointsExact
    assert abs(p.t - 1e-3) <= 1e-6
    with pytest.raises(OracleError):                           # RangeTooSmallIsAnError
        oracle.build_plan(SamplingConfig(r_min=0.1, r_max=0.1 + 1.5e-3))


def test_hash_known_answers(oracle):
    b, _, _ = oracle.build_hash([0.25, 0.75, 1.25])            # test_table.cpp:51-59
    assert list(b) == [0, 1, 2]
    p = oracle.make_plan([0.0001, 0.0006, 0.0008, 0.0011])     # test_table.cpp:86-93
    ev = oracle.evaluator(p, 0.0, degree=1)
    b, _, _ = oracle.build_hash(p.abscissae)
    assert b.size == int(math.ceil((0.0011 - 0.0001) / p.dr_min)) + 1


def test_predicted_calls(oracle):
    assert oracle.predicted_calls(100, 4, 3) == 360000         # test_matfill.cpp:17-21
    assert oracle.predicted_calls(320, 4, 3) == 3686400
    with pytest.raises(OracleError) as e:
        oracle.predicted_calls(1 << 32, 1 << 16, 1 << 16)
    assert e.value.status == 4


def test_cli_bench_row_prefix(oracle):
    """test_cli.cpp:176-189: bench-fill on the 20-triangle sphere, m=4, n=3 writes
    the row prefix "20,4,3,14400,13680,0," (N, m, n, predicted, actual, fallbacks)."""
    v, t = oracle.sphere_mesh(0.5, 0)
    p = oracle.build_plan(SamplingConfig(r_max=oracle.max_vertex_distance(v) * 1.01,
                                         samples_per_wavelength=1000))
    ev = oracle.evaluator(p, 2 * math.pi)
    _, rep = oracle.fill_rows(v, t, 4, 3, TABLE, 2 * math.pi, ev=ev)
    assert (rep.N, rep.m, rep.n, rep.predicted_calls, rep.actual_calls,
            rep.fallback_calls) == (20, 4, 3, 14400, 13680, 0)


def test_linear_bound_value(oracle):
    import ctypes as C
    out = C.c_double()
    assert oracle.L.go_linear_bound(C.c_double(1e-3), C.c_int(EXP), C.c_double(2 * math.pi),
                                    C.c_double(0.1), C.byref(out)) == 0
    assert out.value == pytest.approx(4.934802200544679e-6, rel=1e-15)  # test_bounds.cpp:71-75
