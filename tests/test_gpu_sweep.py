"""Table sweep K3s (csrc/fill_sweep.cuh) vs the oracle.

K3s is the paper's table fill (TableKernel::accumulate, evaluator.hpp:150-194,
237-272) on shared edges with the table held in shared memory: a CTA owns a
cluster of rows and walks the source blocks in distance bands, staging each
band's slice of the base-grid node values.  The bar is K3e's
(tests/test_gpu_edges.py::test_table_edge_fill_parity):
  |Z - Z_cpu_direct| <= B_t = sum |w_o w_i| (pointwise_bound + 64 u (1 + |k| r) / r)
  |Z - Z_cpu_table|  <= B_d = sum |w_o w_i| 64 u (1 + |k| r) / r   (same plan)
and the fallback counts are the reference's.  A radius takes the window or
the global records by its value alone, so the result does not depend on the
row partition or on the window size: those are compared bitwise.
"""
import numpy as np
import pytest

from oracle.pyoracle import DIRECT, EXP, GREEN, TABLE

pytestmark = pytest.mark.gpu

ULPS = 64.0


def sphere(gk, level, radius=1.0, seed=1901, amp=1e-3):
    return gk.jitter(gk.generate_sphere_mesh(radius, level), seed, amp)


@pytest.fixture
def ctx_edges(gk):
    """shared edges on small meshes too (the default needs >= 4096 triangles)"""
    ctx = gk.Context.get()
    ctx.set_fill_options(gk.FillOptions(shared_edges=1))
    yield ctx
    ctx.set_fill_options(None)


def sweep(gk, **kw):
    return gk.FillOptions(shared_edges=1, table_placement=gk.GK_TABLE_SWEEP, **kw)


def k3e(gk):
    return gk.FillOptions(shared_edges=1, table_placement=gk.GK_TABLE_GLOBAL)


def _table(gk, oracle, dm, k, S, r_min=None, medium=None):
    lo, hi = dm.distance_range()
    med = medium or gk.Medium(lambda0=2 * np.pi / k)
    t = gk.DeviceTable(gk.SamplingConfig(r_min=r_min or lo, r_max=hi, samples_per_wavelength=S),
                       med)
    d = t.download()
    kc = complex(t.k)
    return t, oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), kc.real,
                               k_im=kc.imag)


@pytest.mark.parametrize("m,n,S,chunks", [(6, 4, 10000, 1), (7, 5, 3000, 3), (6, 4, 1000, 2),
                                          (3, 1, 3000, 1)])
def test_sweep_fill_parity(gk, oracle, ctx_edges, m, n, S, chunks):
    mesh = sphere(gk, 3)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n), options=gk.MeshOptions(sweep_chunks=chunks))
    t, ev = _table(gk, oracle, dm, k, S)
    z, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    assert rep.path_name == "table_sweep"
    z = z.cpu().numpy()
    ref_d, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k, threads=8)
    ref_t, rep_t = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, TABLE, k, ev=ev, threads=8)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, ev, k, ULPS)
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, k, ULPS)
    assert np.all(np.abs(z - ref_d) <= B_t), float(np.max(np.abs(z - ref_d) / B_t))
    assert np.all(np.abs(z - ref_t) <= B_d), float(np.max(np.abs(z - ref_t) / B_d))
    assert rep.fallback_calls == rep_t.fallback_calls == 0
    assert rep.actual_calls == rep_t.actual_calls
    assert rep.evaluations < 0.85 * rep.actual_calls
    assert np.all(np.diag(z) == 0)
    # the same matrix as K3e (the global interval records) up to rounding
    z3, rep3 = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=k3e(gk))
    assert rep3.path_name == "table_edge"
    z3 = z3.cpu().numpy()
    assert np.max(np.abs(z - z3) / np.maximum(np.abs(z3), 1e-300)) < 1e-12


def test_sweep_window_size_and_row_blocks_bit_exact(gk, ctx_edges):
    """smaller windows (more, narrower bands) and any row partition give the
    same bits"""
    import torch
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=1))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=0.01, r_max=2.1, samples_per_wavelength=5000))
    full, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    assert rep.path_name == "table_sweep"
    ran = 0
    for budget in (128 * 1024, 100 * 1024, 64 * 1024):
        z, r = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk, smem_budget=budget))
        if r.path_name == "table_sweep":
            ran += 1
            assert torch.equal(z, full)
            assert r.evaluations == rep.evaluations
    assert ran >= 2
    parts, evals = [], 0
    N = dm.N
    for b, e in [(0, 333), (333, 334), (334, 1000), (1000, N)]:
        z, r = gk.fill_rows(dm, gk.Mode.TABLE, table=t, row_begin=b, row_end=e,
                            options=sweep(gk))
        assert r.path_name == "table_sweep"
        parts.append(z)
        evals += r.evaluations
    assert torch.equal(torch.cat(parts), full)
    assert evals == rep.evaluations


@pytest.mark.parametrize("r_min", [0.03, 0.08])
def test_sweep_fallback_counts_match_reference(gk, oracle, ctx_edges, r_min):
    """a table starting above the nearest pairs: near tiles fall back like the
    reference (evaluator.hpp:199-205), far tiles never do"""
    mesh = sphere(gk, 3)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=1))
    t, ev = _table(gk, oracle, dm, k, 10000, r_min=r_min)
    z, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    assert rep.path_name == "table_sweep"
    ref_t, rep_t = oracle.fill_rows(mesh.vertices, mesh.triangles, 6, 4, TABLE, k, ev=ev, threads=8)
    assert rep.fallback_calls == rep_t.fallback_calls > 0
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, 6, 4, None, k, ULPS)
    assert np.all(np.abs(z.cpu().numpy() - ref_t) <= B_d)


@pytest.mark.parametrize("S", [3000, 10000])
def test_sweep_exp_kind_and_fused_pair(gk, oracle, ctx_edges, S):
    """the linear Exp table (evaluator.hpp:22-30) through the window; the
    fused pair is bitwise the two separate sweeps -- in one pass where both
    windows fit (S = 3000), as two single-kind sweeps where they do not"""
    import torch
    mesh = sphere(gk, 3)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=1))
    t, ev = _table(gk, oracle, dm, k, S)
    ze, rep = gk.fill_rows(dm, gk.Mode.TABLE, kind=gk.KernelKind.PlainExp, table=t,
                           options=sweep(gk))
    assert rep.path_name == "table_sweep"
    ref_e, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 6, 4, TABLE, k, ev=ev, kind=EXP,
                                threads=8)
    assert np.max(np.abs(ze.cpu().numpy() - ref_e)) <= 1e-13 * np.abs(ref_e).max() * 80
    zg, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    pe, pg, prep = gk.fill_rows_pair(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    assert prep.path_name == "table_sweep"
    assert torch.equal(pe, ze) and torch.equal(pg, zg)


def test_sweep_lossy_plate(gk, oracle, ctx_edges):
    """C4's complex k on the open plate (no reference path: the oracle's
    restatement)"""
    mesh = gk.generate_plate_mesh(1.0, 20)
    med = gk.Medium(1.0, 4.0, 1.0, -0.4)
    kc = complex(gk.wavenumber(med))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=2))
    t, ev = _table(gk, oracle, dm, kc, 10000, medium=med)
    z, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk))
    assert rep.path_name == "table_sweep"
    ref_d, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 6, 4, DIRECT, kc.real,
                                k_im=kc.imag, threads=8)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, 6, 4, ev, abs(kc), ULPS)
    assert np.all(np.abs(z.cpu().numpy() - ref_d) <= B_t)


def test_sweep_declines_when_the_window_cannot_cover_a_block(gk, ctx_edges):
    """a window narrower than a block's radius spread: K3e runs instead"""
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=12))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=0.01, r_max=2.1, samples_per_wavelength=10000))
    z, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=sweep(gk, smem_budget=16384))
    assert rep.path_name == "table_edge"


def test_sweep_dispatch_by_table_density(gk, ctx_edges):
    """GK_AUTO: a dense table (S = 1e4 here) goes to the sweep, a table staged
    whole stays per triangle (S = 300); GK_TABLE_GLOBAL keeps K3e"""
    mesh = sphere(gk, 3)
    # one-chunk sweep blocks: the L3 sphere's two-chunk blocks (rho 0.6 m) are
    # too wide for a window at S = 1e4, lambda = 1 (the dispatch then takes K3e)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(sweep_chunks=1))
    dm2 = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=10000))
    assert gk.fill_rows(dm2, gk.Mode.TABLE, table=t)[1].path_name == "table_edge"
    for S, want in ((10000, "table_sweep"), (300, "table_staged")):
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S))
        _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
        assert rep.path_name == want, (S, rep.path_name)
    _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, options=k3e(gk))
    assert rep.path_name == "table_edge"
