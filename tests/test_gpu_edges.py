"""Shared-edge direct fill (K4e, csrc/edges.cu) vs the oracle.

The reference evaluates every source triangle's own edge points
(inner_points, matfill.hpp:132-144).  The shared-edge kernel evaluates each
distinct edge of a block of source triangles once, in the orientation of its
first triangle, for (row, block) tiles at least r_far = delta / (32 u) apart,
delta being the measured largest distance between a point and its
reversed-edge twin.  The bar is the same as every direct fill's
(tests/test_gpu_fill.py):
  |Z_gpu - Z_cpu_direct| <= B_pq = sum_{o,i} |w_o w_i| 64 2^-53 (1 + |k| r) / r
which the reversed-edge rounding uses at most half of per term.
"""
import numpy as np
import pytest

from oracle.pyoracle import DIRECT, EXP, GREEN

pytestmark = pytest.mark.gpu

ULPS = 64.0


def sphere(gk, level, radius=1.0, seed=1901, amp=1e-3):
    return gk.jitter(gk.generate_sphere_mesh(radius, level), seed, amp)


@pytest.fixture
def ctx_edges(gk):
    """the context's default kernel selection: shared edges on small meshes"""
    ctx = gk.Context.get()
    ctx.set_fill_options(gk.FillOptions(shared_edges=1))
    yield ctx
    ctx.set_fill_options(None)


@pytest.fixture
def forced(gk, ctx_edges):
    """shared edges on small meshes, with small blocks so that far tiles
    exist: the MeshOptions to create the meshes with"""
    return gk.MeshOptions(edge_chunks=4)


def per_tri(gk):
    """per-call options: the reference-order per-triangle kernels"""
    return gk.FillOptions(shared_edges=0)


def _check(gk, oracle, mesh, m, n, k, kind=None, mopts=None):
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n), options=mopts)
    info = dm.edge_info()
    kw = dict(k=k) if kind is None else dict(k=k, kind=kind)
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, **kw)
    kc = complex(k)
    ref, orep = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, kc.real,
                                 kind=EXP if kind == gk.KernelKind.PlainExp else GREEN,
                                 k_im=kc.imag, threads=8)
    err = np.abs(z.cpu().numpy() - ref)
    if kind == gk.KernelKind.PlainExp:  # the Exp bar of test_gpu_fill.test_fill_exp_kind
        assert np.max(err) <= 1e-13 * np.abs(ref).max() * 80
    else:
        B = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, abs(kc), ULPS)
        assert np.all(err <= B), float(np.max(err / np.maximum(B, 1e-300)))
    N = mesh.triangle_count()
    assert rep.actual_calls == orep.actual_calls == 3 * m * n * N * (N - 1)
    assert np.all(np.diag(z.cpu().numpy()) == 0)
    return dm, info, rep


@pytest.mark.parametrize("m,n", [(6, 4), (7, 5), (3, 1), (1, 2)])
def test_edge_fill_parity_sphere(gk, oracle, forced, m, n):
    dm, info, rep = _check(gk, oracle, sphere(gk, 3), m, n, 2 * np.pi, mopts=forced)
    assert info["blocks"] > 1 and info["work_ratio"] < 0.85, info
    # the far threshold is the measured reversed-edge rounding / (32 u)
    assert 0 < info["delta"] < 1e-15
    assert info["r_far"] == info["delta"] * 2.0 ** 48
    # the shared edges did run: fewer evaluations than the reference's calls
    assert rep.evaluations < 0.8 * rep.actual_calls


def test_edge_fill_parity_lossy_plate(gk, oracle, forced):
    """C4's medium (attenuation coupled to the phase reduction) on an open,
    row-major plate: blocks follow the bisection order."""
    mesh = gk.generate_plate_mesh(1.0, 20)
    k = complex(gk.wavenumber(gk.Medium(1.0, 4.0, 1.0, -0.4)))
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, k, mopts=forced)
    assert info["ordered"]
    assert rep.evaluations < 0.85 * rep.actual_calls


def test_edge_fill_exp_kind(gk, oracle, forced):
    mesh = sphere(gk, 3)
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, 2 * np.pi, kind=gk.KernelKind.PlainExp,
                           mopts=forced)
    assert rep.evaluations < 0.8 * rep.actual_calls


def test_edge_fill_close_to_per_triangle_fill(gk, forced):
    """same matrix as the reference-order kernel up to rounding"""
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    ze, re_ = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    zt, rt = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, options=per_tri(gk))
    assert rt.evaluations == rt.actual_calls and re_.evaluations < rt.evaluations
    rel = ((ze - zt).abs() / zt.abs().clamp_min(1e-300)).max().item()
    assert rel < 1e-12


def test_edge_near_tiles_bit_identical_to_per_triangle_fill(gk, ctx_edges):
    """blocks as large as the mesh: every tile is near and takes the
    reference's own points in the reference's order (bitwise the v4 kernel)"""
    import torch
    mesh = sphere(gk, 2)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    z1, r1 = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    z0, r0 = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, options=per_tri(gk))
    assert torch.equal(z1, z0)
    assert r1.evaluations == r0.evaluations == r0.actual_calls


def test_edge_row_blocks_union_bit_exact(gk, forced):
    import torch
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    full, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    N = dm.N
    parts, evals = [], 0
    for b, e in [(0, 417), (417, 418), (418, 1000), (1000, N)]:
        z, r = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, row_begin=b, row_end=e)
        parts.append(z)
        evals += r.evaluations
    assert torch.equal(torch.cat(parts), full)
    assert evals == rep.evaluations


def test_edge_fill_host_pipeline_and_async(gk, forced):
    """the streamed host fill and the asynchronous fill take the same path"""
    import torch
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    zh = np.empty((dm.N, dm.N), np.complex128)
    reph = gk.fill_rows_host(dm, gk.Mode.DIRECT, zh, k=2 * np.pi)
    assert np.array_equal(zh, z.cpu().numpy()) and reph.evaluations == rep.evaluations
    za, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, report=False)
    assert dm.ctx.fill_check() == 0
    assert torch.equal(za, z)


def test_edge_blocks_skip_meshes_without_shared_edges(gk, oracle, ctx_edges):
    """disconnected triangles share no edge: the per-triangle kernel runs"""
    rng = np.random.default_rng(7)
    N = 300
    base = rng.uniform(-1, 1, (N, 1, 3))
    verts = (base + rng.uniform(-0.05, 0.05, (N, 3, 3))).reshape(-1, 3)
    tris = np.arange(3 * N, dtype=np.uint32).reshape(N, 3)
    mesh = gk.TriangleMesh(verts, tris)
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, 2 * np.pi)
    assert info["work_ratio"] >= 0.85 and rep.evaluations == rep.actual_calls


def _table(gk, oracle, dm, k, S, r_min=None):
    lo, hi = dm.distance_range()
    med = gk.Medium(lambda0=2 * np.pi / k)
    t = gk.DeviceTable(gk.SamplingConfig(r_min=r_min or lo, r_max=hi, samples_per_wavelength=S),
                       med)
    d = t.download()
    return t, oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), t.k)


@pytest.mark.parametrize("m,n", [(6, 4), (7, 5)])
def test_table_edge_fill_parity(gk, oracle, forced, m, n):
    """K3e: the paper's table on shared edges (a table too large for shared
    memory, so the edge kernel runs) against the CPU direct fill within the
    interpolation bound, and against the CPU table fill on the same plan
    within rounding"""
    from oracle.pyoracle import TABLE
    mesh = sphere(gk, 3)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n), options=forced)
    t, ev = _table(gk, oracle, dm, k, 10000)
    zt, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    zt = zt.cpu().numpy()
    ref_d, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k, threads=8)
    ref_t, rep_t = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, TABLE, k, ev=ev, threads=8)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, ev, k, ULPS)
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, k, ULPS)
    assert np.all(np.abs(zt - ref_d) <= B_t)
    assert np.all(np.abs(zt - ref_t) <= B_d)
    assert rep.evaluations < 0.8 * rep.actual_calls
    assert rep.fallback_calls == rep_t.fallback_calls == 0


@pytest.mark.parametrize("r_min", [0.03, 0.08])
def test_table_edge_fallback_counts_match_reference(gk, oracle, forced, r_min):
    """a table starting above the nearest pairs: near tiles fall back exactly
    like the reference (evaluator.hpp:199-205); far tiles (>= max(r_far,
    r_min) apart: r_far = 0.044 m here) never do"""
    from oracle.pyoracle import TABLE
    mesh = sphere(gk, 3)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    assert 0.03 < dm.edge_info()["r_far"] < 0.08
    t, ev = _table(gk, oracle, dm, k, 10000, r_min=r_min)
    zt, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    ref_t, rep_t = oracle.fill_rows(mesh.vertices, mesh.triangles, 6, 4, TABLE, k, ev=ev, threads=8)
    assert rep.fallback_calls == rep_t.fallback_calls > 0
    assert rep.evaluations < 0.8 * rep.actual_calls
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, 6, 4, None, k, ULPS)
    assert np.all(np.abs(zt.cpu().numpy() - ref_t) <= B_d)


def test_table_edge_dispatch_by_table_size(gk, forced):
    """a table staged whole in shared memory stays per triangle (S = 300);
    one too large for that but L1-sized (<= 300 KB of records) takes K3e"""
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    lo, hi = dm.distance_range()
    for S, shared in ((300, False), (1000, True)):
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S))
        _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
        assert (rep.evaluations < rep.actual_calls) == shared, (S, t.info.nodes)


@pytest.mark.parametrize("mode", ["direct", "lossy", "table"])
def test_edge_fused_pair_equals_separate_fills(gk, forced, mode):
    """gk_fill_rows_pair on shared edges: Exp and Green from one pass, bitwise
    equal to the two separate shared-edge fills (direct, C4's lossy medium,
    and the table read through L1)"""
    import torch
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=forced)
    med = gk.Medium(1.0, 4.0, 1.0, -0.4) if mode == "lossy" else gk.Medium()
    kw = dict(k=gk.wavenumber(med))
    if mode == "table":
        lo, hi = dm.distance_range()
        kw = dict(table=gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi,
                                                         samples_per_wavelength=10000), med))
    md = gk.Mode.TABLE if mode == "table" else gk.Mode.DIRECT
    ze, zg, rep = gk.fill_rows_pair(dm, md, **kw)
    e, re_ = gk.fill_rows(dm, md, kind=gk.KernelKind.PlainExp, **kw)
    g, rg = gk.fill_rows(dm, md, kind=gk.KernelKind.GreenOverR, **kw)
    assert torch.equal(ze, e) and torch.equal(zg, g)
    assert rep.actual_calls == 2 * rg.actual_calls and rep.fallback_calls == 0
    assert rep.evaluations == re_.evaluations + rg.evaluations < 0.8 * rep.actual_calls


def test_edge_fill_parity_mesh_far_from_origin(gk, oracle, forced):
    """a mesh 3e4 m from the origin: the two orientations of an edge still
    round to the same points up to delta (measured; the ulp of the large
    coordinate cancels between them), so the shared points stay within the
    bound on the far tiles"""
    mesh = sphere(gk, 3)
    mesh = gk.TriangleMesh(mesh.vertices + np.array([3.0e4, 0.0, 0.0]), mesh.triangles)
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, 2 * np.pi, mopts=forced)
    assert rep.evaluations < 0.8 * rep.actual_calls


def test_edge_fill_parity_inconsistent_orientation(gk, oracle, forced):
    """every third triangle flipped: the sides that run the owner's way share
    its points exactly (g with g), the others pair g with n-1-g; the measured
    delta stays at the rounding level and the shared edges stay in use"""
    mesh = sphere(gk, 3)
    tris = mesh.triangles.copy()
    tris[::3] = tris[::3, ::-1]
    mesh = gk.TriangleMesh(mesh.vertices, tris)
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, 2 * np.pi, mopts=forced)
    assert 0 < info["delta"] < 1e-15
    assert rep.evaluations < 0.8 * rep.actual_calls


@pytest.mark.parametrize("chunks", [1, 6, 12])
def test_edge_block_sizes_launch_and_agree(gk, ctx_edges, chunks):
    """every block size launches (6 chunks put the K3e edge sums at exactly
    48 KB of dynamic shared memory beside the static weights) and agrees with
    the per-triangle kernels"""
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), options=gk.MeshOptions(edge_chunks=chunks))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=10000))
    for md, kw in ((gk.Mode.DIRECT, dict(k=2 * np.pi)), (gk.Mode.TABLE, dict(table=t))):
        z, rep = gk.fill_rows(dm, md, **kw)
        z0, _ = gk.fill_rows(dm, md, options=per_tri(gk), **kw)
        rel = ((z - z0).abs() / z0.abs().clamp_min(1e-300)).max().item()
        assert rel < 1e-12, (md, rel)


@pytest.mark.parametrize("m", [1, 3, 4, 6, 7])
def test_edge_kernels_every_rule_agree_with_per_triangle(gk, forced, m):
    """every outer rule x n = 1..5, direct (lossless and C4's lossy medium)
    and table (K3e): the shared-edge fill agrees with the per-triangle one"""
    mesh = sphere(gk, 3)
    for n in range(1, 6):
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n), options=forced)
        lo, hi = dm.distance_range()
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=10000))
        kl = complex(gk.wavenumber(gk.Medium(1.0, 4.0, 1.0, -0.4)))
        for md, kw in ((gk.Mode.DIRECT, dict(k=2 * np.pi)), (gk.Mode.DIRECT, dict(k=kl)),
                       (gk.Mode.TABLE, dict(table=t))):
            z, rep = gk.fill_rows(dm, md, **kw)
            z0, rep0 = gk.fill_rows(dm, md, options=per_tri(gk), **kw)
            rel = ((z - z0).abs() / z0.abs().clamp_min(1e-300)).max().item()
            assert rel < 1e-12, (m, n, md, rel)
            assert rep.evaluations < rep0.evaluations == rep0.actual_calls, (m, n, md, kw.keys())


@pytest.mark.parametrize("radius,lam", [(1e-3, 1e-3), (1e3, 1e3)])
def test_edge_fill_parity_scaled_meshes(gk, oracle, forced, radius, lam):
    """the far threshold scales with the mesh (delta is measured on its own
    points): millimetre and kilometre spheres stay within the bound"""
    mesh = gk.jitter(gk.generate_sphere_mesh(radius, 3), 1901, 1e-3 * radius)
    dm, info, rep = _check(gk, oracle, mesh, 6, 4, 2 * np.pi / lam, mopts=forced)
    assert 0.01 * radius < info["r_far"] < 0.1 * radius
    assert rep.evaluations < 0.8 * rep.actual_calls
