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
