"""Randomised parity: seeded random triangle soups (not meshes: arbitrary
orientations, sizes, near-touching pairs), random quadrature (m in
{1,3,4,6,7}, n in 1..6), random real or complex k, both modes, against the
oracle under the per-entry bound of tests/test_gpu_fill.py."""
import numpy as np
import pytest

from oracle.pyoracle import DIRECT, TABLE

pytestmark = pytest.mark.gpu
ULPS = 64.0


def soup(gk, rng, N):
    """N random triangles in [0, 2]^3 with area > 1e-3 (TriangleMesh rejects <= 1e-12)"""
    verts, tris = [], []
    while len(tris) < N:
        c = rng.uniform(0.0, 2.0, 3)
        e1, e2 = rng.normal(0, 0.15, 3), rng.normal(0, 0.15, 3)
        if 0.5 * np.linalg.norm(np.cross(e1, e2)) < 1e-3:
            continue
        b = len(verts)
        verts += [c, c + e1, c + e2]
        tris.append([b, b + 1, b + 2])
    return gk.TriangleMesh(np.array(verts), np.array(tris))


@pytest.mark.parametrize("seed", range(24))
def test_random_soup_parity(gk, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(20, 160))
    mesh = soup(gk, rng, N)
    m = int(rng.choice([1, 3, 4, 6, 7]))
    n = int(rng.integers(1, 7))
    lam = float(rng.uniform(0.2, 2.0))
    lossy = seed % 3 == 2
    med = gk.Medium(lambda0=lam, eps_r=float(rng.uniform(1.0, 6.0)),
                    eps_r_im=-float(rng.uniform(0.05, 1.0)) if lossy else 0.0)
    k = complex(gk.wavenumber(med))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
    lo, hi = dm.distance_range()
    olo, ohi = oracle.distance_range(mesh.vertices, mesh.triangles, m, n)
    assert lo <= olo <= lo * (1 + 2.0 ** -47) and hi * (1 - 2.0 ** -47) <= ohi <= hi
    zd, rd = gk.fill_rows(dm, gk.Mode.DIRECT, k=k)
    ref_d, rep = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k.real,
                                  k_im=k.imag, threads=8)
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, abs(k), ULPS)
    assert np.all(np.abs(zd.cpu().numpy() - ref_d) <= B_d)
    assert rd.actual_calls == rep.actual_calls == 3 * m * n * N * (N - 1)
    S = int(rng.choice([300, 1000, 4000]))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
    d = t.download()
    ev = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), k.real, k_im=k.imag)
    zt, rt = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    ref_t, rept = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, TABLE, k.real, ev=ev,
                                   k_im=k.imag, threads=8)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, ev, abs(k), ULPS)
    zt = zt.cpu().numpy()
    assert np.all(np.abs(zt - ref_d) <= B_t)
    assert np.all(np.abs(zt - ref_t) <= B_d)
    assert rt.fallback_calls == rept.fallback_calls == 0


@pytest.mark.parametrize("seed", range(12))
def test_random_closed_mesh_shared_edges(gk, oracle, seed):
    """Seeded random closed meshes through the shared-edge kernels (K4e / K3e):
    random sphere radius, jitter, subdivision level, block size (1..6 chunks:
    far, near and padded tiles in every mix), block order, quadrature (n <= 5),
    real or complex k, kind; the bar is the direct fill's per-entry bound."""
    from oracle.pyoracle import EXP, GREEN
    rng = np.random.default_rng(7000 + seed)
    level = int(rng.choice([2, 3]))
    radius = float(10.0 ** rng.uniform(-2.0, 2.0))
    mesh = gk.jitter(gk.generate_sphere_mesh(radius, level), 100 + seed, 1e-3 * radius)
    m = int(rng.choice([1, 3, 4, 6, 7]))
    n = int(rng.integers(1, 6))
    lam = radius * float(rng.uniform(0.3, 3.0))
    lossy = seed % 4 == 3
    med = gk.Medium(lambda0=lam, eps_r=float(rng.uniform(1.0, 4.0)),
                    eps_r_im=-float(rng.uniform(0.05, 0.5)) if lossy else 0.0)
    k = complex(gk.wavenumber(med))
    exp_kind = seed % 3 == 1
    kind = gk.KernelKind.PlainExp if exp_kind else gk.KernelKind.GreenOverR
    mopts = gk.MeshOptions(edge_chunks=int(rng.integers(1, 7)), edge_order=int(rng.integers(0, 2)))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n), options=mopts)
    N = mesh.triangle_count()
    opts = gk.FillOptions(shared_edges=1)
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, kind=kind, options=opts)
    ref, orep = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k.real,
                                 kind=EXP if exp_kind else GREEN, k_im=k.imag, threads=8)
    err = np.abs(z.cpu().numpy() - ref)
    if exp_kind:  # the Exp bar of test_gpu_fill.test_fill_exp_kind
        assert np.max(err) <= 1e-13 * np.abs(ref).max() * 80
    else:
        B = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, abs(k), ULPS)
        assert np.all(err <= B), float(np.max(err / np.maximum(B, 1e-300)))
    assert rep.actual_calls == orep.actual_calls == 3 * m * n * N * (N - 1)
    # the dispatch keeps the per-triangle kernel where the blocks share too few
    # edges (slots / 3N >= 0.85) or the attenuation table is too long
    assert rep.path_name in ("direct_edge", "direct") and rep.evaluations <= rep.actual_calls
    info = dm.edge_info()
    if info["work_ratio"] < 0.85 and not lossy:
        assert rep.path_name == "direct_edge", info
    assert np.all(np.diag(z.cpu().numpy()) == 0)
    # the same matrix up to rounding as the per-triangle kernel, and the row
    # blocks' union is bitwise the whole
    zt, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, kind=kind, options=gk.FillOptions(shared_edges=0))
    scale = zt.abs().max().item()
    assert ((z - zt).abs().max().item()) <= 1e-11 * scale
    cut = int(rng.integers(1, N - 1))
    import torch
    za, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, kind=kind, options=opts, row_end=cut)
    zb, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, kind=kind, options=opts, row_begin=cut)
    assert torch.equal(torch.cat([za, zb]), z)
