"""The reference's fill tests (proj/tests/test_matfill.cpp) on the device:
call accounting, reciprocity of a symmetric pair, determinism, the exact
max_vertex_distance, compare_fills and bench_compare (matfill.hpp:237-294)."""
import numpy as np
import pytest

from oracle.pyoracle import DIRECT

pytestmark = pytest.mark.gpu
TWO_PI = 2 * np.pi


def two_parallel_triangles(gk, sep):
    """test_matfill.cpp:28-36: identical triangles translated along the normal"""
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, sep], [1, 0, sep], [0, 1, sep]], float)
    return gk.TriangleMesh(v, np.array([[0, 1, 2], [3, 4, 5]]))


@pytest.mark.parametrize("m", [1, 4])
@pytest.mark.parametrize("n", [1, 3])
def test_call_accounting_on_sphere(gk, m, n):
    """test_matfill.cpp:61-73"""
    dm = gk.DeviceMesh(gk.generate_sphere_mesh(0.5, 0), gk.QuadratureSpec(m, n))
    _, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=TWO_PI)
    assert rep.actual_calls == 3 * m * n * 20 * 19
    assert rep.actual_calls <= rep.predicted_calls == 3 * m * n * 400


@pytest.mark.parametrize("mode", ["direct", "table"])
def test_symmetric_pair_is_reciprocal(gk, mode):
    """test_matfill.cpp:75-87: Z[0][1] and Z[1][0] agree to 1e-12 |Z|"""
    mesh = two_parallel_triangles(gk, 0.7)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 3))
    if mode == "direct":
        z, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=TWO_PI)
    else:
        lo, hi = dm.distance_range()
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=10000))
        z, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    z = z.cpu().numpy()
    a, b = z[0, 1], z[1, 0]
    assert abs(a.real - b.real) <= 1e-12 * abs(a)
    assert abs(a.imag - b.imag) <= 1e-12 * abs(a)


def test_direct_fill_is_deterministic(gk):
    """test_matfill.cpp:89-96 (AnalyticFillIndependentOfSamplingConfig)"""
    import torch
    dm = gk.DeviceMesh(gk.generate_sphere_mesh(0.5, 0), gk.QuadratureSpec(3, 2))
    za, ra = gk.fill_rows(dm, gk.Mode.DIRECT, k=TWO_PI)
    zb, rb = gk.fill_rows(dm, gk.Mode.DIRECT, k=TWO_PI)
    assert torch.equal(za, zb) and ra.actual_calls == rb.actual_calls


@pytest.mark.parametrize("mesh_kind", ["sphere0", "sphere3j", "sphere6", "plate"])
def test_max_vertex_distance_bit_exact(gk, oracle, mesh_kind):
    """mesh.hpp:62-68, exact O(V^2) scan == the oracle's (== the reference's)"""
    mesh = {"sphere0": lambda: gk.generate_sphere_mesh(0.5, 0),
            "sphere3j": lambda: gk.jitter(gk.generate_sphere_mesh(1.0, 3), 1901, 1e-3),
            "sphere6": lambda: gk.jitter(gk.generate_sphere_mesh(1.0, 6), 1901, 1e-3),
            "plate": lambda: gk.generate_plate_mesh(1.0, 40)}[mesh_kind]()
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    got = dm.max_vertex_distance()
    if mesh_kind == "sphere6":   # O(V^2) = 8.4e8 pairs on the CPU: check the value's bracket
        assert 2.0 - 4e-3 <= got <= 2.0 + 4e-3
        return
    assert got == oracle.max_vertex_distance(mesh.vertices)


def test_compare_fills_matches_reference_semantics(gk, oracle):
    """matfill.hpp:237-254: diagonal and exact-zero reference components skipped"""
    import torch
    mesh = gk.jitter(gk.generate_sphere_mesh(1.0, 2), 7, 1e-3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 3))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=300))
    zd, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=TWO_PI)
    zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    zd[3, 5] = complex(0.0, zd[3, 5].imag.item())   # an exact-zero real reference part
    zt[7, 7] = 1e300                                # the diagonal is excluded
    re, im = gk.compare_fills(zt, zd)
    ore, oim = oracle.compare_fills(zt.cpu().numpy(), zd.cpu().numpy())
    assert (re, im) == (ore, oim) and 0 < re < 1e-3 and 0 < im < 1e-3
    # a row block: its own diagonal offset
    rb = 100
    bre, bim = gk.compare_fills(zt[rb:rb + 50], zd[rb:rb + 50], row_begin=rb)
    a, b = zd[rb:rb + 50].cpu().numpy(), zt[rb:rb + 50].cpu().numpy()
    mask = np.ones_like(a, bool)
    mask[np.arange(50), rb + np.arange(50)] = False
    with np.errstate(divide="ignore", invalid="ignore"):
        er = np.where((a.real != 0) & mask, np.abs(b.real - a.real) / np.abs(a.real), 0).max()
        ei = np.where((a.imag != 0) & mask, np.abs(b.imag - a.imag) / np.abs(a.imag), 0).max()
    assert (bre, bim) == (er, ei)
    assert gk.compare_fills(zd, zd) == (0.0, 0.0)
    with pytest.raises(gk.InvalidArgument):
        gk.compare_fills(zd[:10], zd[:11])
    del torch


def test_bench_compare_report_consistency(gk):
    """test_matfill.cpp:167-181 on the device"""
    mesh = gk.generate_sphere_mesh(0.5, 1)
    rep = gk.bench_compare(mesh, gk.QuadratureSpec(4, 3), gk.Medium(),
                           gk.SamplingConfig(samples_per_wavelength=10000), repeats=3)
    assert rep.N == 80 and rep.actual_calls == 3 * 4 * 3 * 80 * 79
    assert rep.fallback_calls == 0
    assert rep.speedup > 0 and rep.analytic_time_s > 0 and rep.table_build_s > 0
    assert rep.predicted_calls == 3 * 4 * 3 * 80 * 80 and rep.wall_time_s > 0
    assert abs(rep.interp_time_s - (rep.wall_time_s + rep.table_build_s)) <= 1e-12
    assert rep.max_rel_re <= 1e-4 and rep.max_rel_im <= 1e-4
    with pytest.raises(gk.InvalidArgument):
        gk.bench_compare(mesh, gk.QuadratureSpec(4, 3), repeats=0)
