"""K0 points, K1 range, K3/K4 fills vs the oracle (parity tests proper).

Tolerance (stated here in code): for each entry
  |Z_gpu - Z_cpu_direct| <= B_pq = sum_{o,i} |w_o w_i| (pw(r_oi) + 64 2^-53 (1 + |k| r) / r)
with pw = pointwise_bound(ev, Green, Lagrange, r) (bounds.hpp:97-111) for the
table mode and 0 for the direct mode; the (1 + |k| r) factor is the rounding
of the phase k r, which the reference itself carries.
"""
import numpy as np
import pytest

from oracle.pyoracle import DIRECT, EXP, TABLE

pytestmark = pytest.mark.gpu

ULPS = 64.0


def sphere(gk, level, radius=1.0, seed=1901, amp=1e-3):
    return gk.jitter(gk.generate_sphere_mesh(radius, level), seed, amp)


def test_points_bit_exact(gk, oracle):
    for mesh, m, n in [(sphere(gk, 2), 6, 4), (sphere(gk, 1, 0.5), 7, 5),
                       (gk.generate_plate_mesh(1.0, 10), 4, 3), (sphere(gk, 0), 1, 1),
                       (sphere(gk, 1), 3, 2), (sphere(gk, 1), 3, 6), (sphere(gk, 1), 6, 32)]:
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
        go, gi = dm.points()
        oo, oi = oracle.points(mesh.vertices, mesh.triangles, m, n)
        assert np.array_equal(go, oo) and np.array_equal(gi, oi)


def test_distance_range_brackets_exact(gk, oracle):
    mesh = sphere(gk, 2)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    for rb, re in [(0, 320), (0, 160), (160, 320), (17, 18)]:
        lo, hi = dm.distance_range(rb, re)
        olo, ohi = oracle.distance_range(mesh.vertices, mesh.triangles, 6, 4, rb, re)
        assert lo <= olo <= lo * (1 + 2.0 ** -47)
        assert hi * (1 - 2.0 ** -47) <= ohi <= hi


def _fill_case(gk, oracle, mesh, m, n, k, S=1000):
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
    lo, hi = dm.distance_range()
    med = gk.Medium(lambda0=2 * np.pi / k)
    cfg = gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S)
    t = gk.DeviceTable(cfg, med)
    plan = oracle.make_plan(t.download()["abscissae"], t.download()["zeros"])
    ev = oracle.evaluator(plan, t.k)
    return dm, t, ev


@pytest.mark.parametrize("level,m,n,S", [(1, 6, 4, 1000), (2, 6, 4, 1000), (2, 4, 3, 10000),
                                         (1, 7, 5, 1000), (1, 1, 1, 1000), (1, 3, 2, 10000)])
def test_fill_parity_sphere(gk, oracle, level, m, n, S):
    mesh = sphere(gk, level)
    k = 2 * np.pi
    dm, t, ev = _fill_case(gk, oracle, mesh, m, n, k, S)
    zd, rd = gk.fill_rows(dm, gk.Mode.DIRECT, k=k)
    zt, rt = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    zd, zt = zd.cpu().numpy(), zt.cpu().numpy()
    ref_d, rep = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k, threads=8)
    ref_t, rep_t = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, TABLE, k, ev=ev,
                                    threads=8)
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, k, ULPS)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, ev, k, ULPS)
    assert np.all(np.abs(zd - ref_d) <= B_d), np.max(np.abs(zd - ref_d) / np.maximum(B_d, 1e-300))
    assert np.all(np.abs(zt - ref_d) <= B_t), np.max(np.abs(zt - ref_d) / np.maximum(B_t, 1e-300))
    # same plan on both sides: only rounding separates GPU-table and CPU-table
    assert np.all(np.abs(zt - ref_t) <= B_d)
    N = mesh.triangle_count()
    assert rd.actual_calls == rt.actual_calls == rep.actual_calls == 3 * m * n * N * (N - 1)
    assert rd.predicted_calls == 3 * m * n * N * N
    assert rt.fallback_calls == 0 == rep_t.fallback_calls
    assert np.all(np.diag(zd) == 0) and np.all(np.diag(zt) == 0)


def test_fill_exp_kind(gk, oracle):
    mesh = sphere(gk, 1, 0.5)
    k = 2 * np.pi
    dm, t, ev = _fill_case(gk, oracle, mesh, 4, 3, k)
    zd, _ = gk.fill_rows(dm, gk.Mode.DIRECT, kind=gk.KernelKind.PlainExp, k=k)
    zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, kind=gk.KernelKind.PlainExp, table=t)
    ref_d, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, DIRECT, k, kind=EXP)
    ref_t, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, TABLE, k, ev=ev, kind=EXP)
    scale = np.abs(ref_d).max()
    assert np.max(np.abs(zd.cpu().numpy() - ref_d)) <= 1e-13 * scale * 80
    assert np.max(np.abs(zt.cpu().numpy() - ref_t)) <= 1e-12 * scale * 80


def test_fallback_routing_below_rmin(gk, oracle):
    """test_matfill.cpp:152-165: r_min = 0.3 forces a fat near-field region."""
    mesh = gk.generate_sphere_mesh(0.5, 1)
    k = 2 * np.pi
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    hi = oracle.max_vertex_distance(mesh.vertices) * 1.01
    t = gk.DeviceTable(gk.SamplingConfig(r_min=0.3, r_max=hi))
    zt, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    d = t.download()
    ev = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), k)
    ref, orep = oracle.fill_rows(mesh.vertices, mesh.triangles, 1, 1, TABLE, k, ev=ev)
    assert 0 < rep.fallback_calls < rep.actual_calls
    assert rep.fallback_calls == orep.fallback_calls
    B = oracle.entry_bounds(mesh.vertices, mesh.triangles, 1, 1, None, k, ULPS)
    assert np.all(np.abs(zt.cpu().numpy() - ref) <= B + np.abs(ref) * 1e-12)


def test_above_rmax_is_out_of_range(gk):
    mesh = gk.generate_sphere_mesh(0.5, 1)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=1e-3, r_max=0.5))
    with pytest.raises(gk.OutOfRange):
        gk.fill_rows(dm, gk.Mode.TABLE, table=t)


def test_row_blocks_union_bit_exact(gk):
    """test_matfill.cpp:98-105 (threads) mirrored as row blocks (GPU shards)."""
    mesh = sphere(gk, 2)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi))
    for mode, kw in ((gk.Mode.DIRECT, dict(k=2 * np.pi)), (gk.Mode.TABLE, dict(table=t))):
        full, _ = gk.fill_rows(dm, mode, **kw)
        N = dm.N
        parts = []
        for w in range(3):
            chunk = (N + 2) // 3
            b, e = w * chunk, min(N, (w + 1) * chunk)
            z, rep = gk.fill_rows(dm, mode, row_begin=b, row_end=e, **kw)
            assert rep.actual_calls == 3 * 6 * 4 * (e - b) * (N - 1)
            parts.append(z)
        import torch
        assert torch.equal(torch.cat(parts), full)


def test_lossy_plate_parity(gk, oracle):
    """C4 shape at small N: complex k, direct and table vs the complex-k oracle."""
    mesh = gk.generate_plate_mesh(1.0, 8)
    med = gk.Medium(lambda0=1.0, eps_r=4.0, eps_r_im=-0.4)
    k = gk.wavenumber(med)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi), med)
    d = t.download()
    ev = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), k.real, k_im=k.imag)
    zd, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k)
    zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
    ref, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 6, 4, DIRECT, k.real, k_im=k.imag,
                              threads=8)
    B_d = oracle.entry_bounds(mesh.vertices, mesh.triangles, 6, 4, None, abs(k), ULPS)
    B_t = oracle.entry_bounds(mesh.vertices, mesh.triangles, 6, 4, ev, abs(k), ULPS)
    assert np.all(np.abs(zd.cpu().numpy() - ref) <= B_d)
    assert np.all(np.abs(zt.cpu().numpy() - ref) <= B_t)


@pytest.mark.parametrize("kval", ["c4", "eps1-20j", "1-6j"])
@pytest.mark.parametrize("m,n", [(6, 4), (3, 7)])
def test_lossy_attenuation_paths(gk, oracle, kval, m, n):
    """Both lossy direct paths vs the complex-k oracle: attenuation coupled to
    the phase reduction (|Im k| <= 2.6 Re k: C4's medium and eps_r = 1 - 20j)
    and the attenuation table (an explicit k = 1 - 6j; no physical medium with
    eps_r > 0 gets there); the fused kernel (n <= 5) and the generic one (n = 7)."""
    mesh = gk.generate_plate_mesh(1.0, 6)
    k = {"c4": lambda: complex(gk.wavenumber(gk.Medium(1.0, 4.0, 1.0, -0.4))),
         "eps1-20j": lambda: complex(gk.wavenumber(gk.Medium(1.0, 1.0, 1.0, -20.0))),
         "1-6j": lambda: complex(1.0, -6.0)}[kval]()
    assert k.imag < 0
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
    zd, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k)
    ref, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, m, n, DIRECT, k.real, k_im=k.imag,
                              threads=8)
    B = oracle.entry_bounds(mesh.vertices, mesh.triangles, m, n, None, abs(k), ULPS)
    err = np.abs(zd.cpu().numpy() - ref)
    assert np.all(err <= B), float(np.max(err / np.maximum(B, 1e-300)))


def test_fill_matrix_host_end_to_end(gk, oracle):
    mesh = sphere(gk, 1)
    k = 2 * np.pi
    z, rep = gk.fill_matrix(mesh, gk.QuadratureSpec(4, 3), gk.Mode.TABLE, gk.Medium())
    ref, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, DIRECT, k)
    assert rep.actual_calls == 3 * 4 * 3 * 80 * 79 and rep.fallback_calls == 0
    re, im = oracle.compare_fills(z, ref)
    assert max(re, im) <= 1e-4   # acceptance criterion 5 gate


def test_hand_summed_static_kernel(gk):
    """test_matfill.cpp:38-59: m = n = 1, k = 0, hand sum of 1/r."""
    mesh = gk.TriangleMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1],
                                     [0, 1, 1]], float), np.array([[0, 1, 2], [3, 4, 5]]))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=0.0)
    z = z.cpu().numpy()
    c = np.array([1 / 3, 1 / 3, 0.0])
    mids = np.array([[0.5, 0, 1], [0.5, 0.5, 1], [0, 0.5, 1]])
    lens = [1.0, np.sqrt(2.0), 1.0]
    expect = sum(0.5 * lens[e] / np.linalg.norm(c - mids[e]) for e in range(3))
    assert abs(z[0, 1].real - expect) <= expect * 1e-14
    assert z[0, 1].imag == 0.0 and z[0, 0] == 0 and z[1, 1] == 0
    assert rep.actual_calls == 6 and rep.predicted_calls == 12


def test_mesh_validation(gk):
    mesh = gk.generate_sphere_mesh(0.5, 0)
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceMesh(mesh, gk.QuadratureSpec(5, 1))
    with pytest.raises(gk.InvalidArgument, match="<= 32"):   # device limit (documented)
        gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 33))
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 0))
    bad = gk.TriangleMesh(mesh.vertices, np.array([[0, 1, 99]]))
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceMesh(bad, gk.QuadratureSpec(4, 3))


def test_fill_rows_host_matches_device(gk):
    mesh = sphere(gk, 2)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    zd, rep_d = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, row_begin=5, row_end=301)
    zh = np.zeros((296, dm.N), np.complex128)
    rep_h = gk.fill_rows_host(dm, gk.Mode.DIRECT, zh, k=2 * np.pi, row_begin=5, row_end=301)
    assert np.array_equal(zh, zd.cpu().numpy())
    assert rep_h.actual_calls == rep_d.actual_calls


@pytest.mark.parametrize("mode", ["direct", "table", "lossy", "lossy_table"])
@pytest.mark.parametrize("m,n", [(6, 4), (7, 5), (3, 7)])
def test_fused_pair_fill_equals_separate_fills(gk, mode, m, n):
    """gk_fill_rows_pair: Exp and Green from one pass, bitwise equal to two
    fills (real k, and the C4 complex k in both modes)."""
    import torch
    mesh = sphere(gk, 2)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
    med = gk.Medium(1.0, 4.0, 1.0, -0.4) if mode.startswith("lossy") else gk.Medium()
    kw = dict(k=gk.wavenumber(med))
    if mode.endswith("table"):
        lo, hi = dm.distance_range()
        kw = dict(table=gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi), med))
    md = gk.Mode.TABLE if mode.endswith("table") else gk.Mode.DIRECT
    ze, zg, rep = gk.fill_rows_pair(dm, md, **kw)
    e, _ = gk.fill_rows(dm, md, kind=gk.KernelKind.PlainExp, **kw)
    g, rg = gk.fill_rows(dm, md, kind=gk.KernelKind.GreenOverR, **kw)
    assert torch.equal(ze, e) and torch.equal(zg, g)
    assert rep.actual_calls == 2 * rg.actual_calls and rep.fallback_calls == 0


def test_zero_distance_pair_is_domain_error(gk, oracle):
    """A source edge through an observation quadrature point: r = 0 exactly.
    The reference throws domain_error (kernel.hpp:51-53); so does the device fill."""
    v = np.array([[0, 0, 0], [3, 0, 0], [0, 3, 0],          # p: centroid (1, 1, 0)
                  [0.5, 1, 0], [1.5, 1, 0], [1, 1, 1]], float)  # q: edge midpoint (1, 1, 0)
    t = np.array([[0, 1, 2], [3, 4, 5]])
    mesh = gk.TriangleMesh(v, t)
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError) as e:
        oracle.fill_rows(mesh.vertices, mesh.triangles, 1, 1, DIRECT, 2 * np.pi)
    assert e.value.status == 2
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    with pytest.raises(gk.DomainError):
        gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    with pytest.raises(gk.DomainError):
        gk.fill_matrix(mesh, gk.QuadratureSpec(1, 1), gk.Mode.DIRECT, gk.Medium())


def test_zero_distance_pair_plain_exp(gk, oracle):
    """The same r = 0 pair with the PlainExp kind is defined: eval_analytic(PlainExp,
    k, 0) = (1, 0) (kernel.hpp:58-60).  Direct mode returns it; table mode takes it
    as a counted fallback below r_min (evaluator.hpp:199-205) -- as the reference."""
    v = np.array([[0, 0, 0], [3, 0, 0], [0, 3, 0],
                  [0.5, 1, 0], [1.5, 1, 0], [1, 1, 1]], float)
    t = np.array([[0, 1, 2], [3, 4, 5]])
    mesh = gk.TriangleMesh(v, t)
    k = 2 * np.pi
    ref, rrep = oracle.fill_rows(mesh.vertices, mesh.triangles, 1, 1, DIRECT, k, kind=EXP)
    assert np.all(np.isfinite(ref))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    for opts in (None, gk.FillOptions(shared_edges=0)):
        z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, kind=gk.KernelKind.PlainExp, k=k, options=opts)
        z = z.cpu().numpy()
        assert np.all(np.isfinite(z))
        assert np.abs(z - ref).max() <= 1e-14
    table = gk.DeviceTable(gk.SamplingConfig(r_min=0.1, r_max=4.0, samples_per_wavelength=1000))
    d = table.download()
    ev = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), k)
    reft, treport = oracle.fill_rows(mesh.vertices, mesh.triangles, 1, 1, TABLE, k, ev=ev, kind=EXP)
    z, rep = gk.fill_rows(dm, gk.Mode.TABLE, kind=gk.KernelKind.PlainExp, table=table)
    z = z.cpu().numpy()
    assert np.all(np.isfinite(z)) and np.abs(z - reft).max() <= 1e-12
    assert rep.fallback_calls == treport.fallback_calls >= 1


@pytest.mark.parametrize("level,S,r_min", [(2, 1000, None), (3, 10000, None), (2, 1000, 0.3)])
def test_table_staging_paths_bit_identical(gk, level, S, r_min):
    """The L1 table kernel, the shared-memory kernel with the whole table staged,
    with per-tile TMA windows, and with windows overflowing a small budget (global
    reads inside the staged kernel) all give the same bits, fallbacks included."""
    import torch
    mesh = sphere(gk, level)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=r_min or lo, r_max=hi, samples_per_wavelength=S))
    G, Sh = gk.GK_TABLE_GLOBAL, gk.GK_TABLE_SHARED
    settings = [(G, 0), (Sh, 0), (Sh, 65536), (Sh, 8192)]
    outs = []
    for place, budget in settings:
        o = gk.FillOptions(table_placement=place, smem_budget=budget)
        ze, zg, rep = gk.fill_rows_pair(dm, gk.Mode.TABLE, table=t, options=o)
        g, rg = gk.fill_rows(dm, gk.Mode.TABLE, table=t, row_begin=7, row_end=dm.N - 3,
                             options=o)
        outs.append((ze, zg, g, rep.fallback_calls, rg.fallback_calls))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])
        assert torch.equal(o[2], outs[0][2]) and o[3:] == outs[0][3:]
    assert (outs[0][3] > 0) == (r_min is not None)


def test_degenerate_sizes_and_strided_output(gk, oracle):
    """N = 1 (only the self pair: Z = 0, no calls), N = 2, empty row ranges,
    and an output block with ldz > N (a window of a larger matrix)."""
    import torch
    one = gk.TriangleMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 2]]))
    for mode, kw in ((gk.Mode.DIRECT, dict(k=2 * np.pi)), (gk.Mode.TABLE, None)):
        dm = gk.DeviceMesh(one, gk.QuadratureSpec(6, 4))
        if kw is None:   # the only pair is the self pair: the range is empty
            kw = dict(table=gk.DeviceTable(gk.SamplingConfig(r_min=0.1, r_max=2.0)))
        z, rep = gk.fill_rows(dm, mode, **kw)
        assert z.shape == (1, 1) and complex(z[0, 0].item()) == 0
        assert rep.actual_calls == 0 and rep.predicted_calls == 3 * 6 * 4
    two = gk.TriangleMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 0.7], [1, 0, 0.7],
                                    [0, 1, 0.7]], float), np.array([[0, 1, 2], [3, 4, 5]]))
    dm = gk.DeviceMesh(two, gk.QuadratureSpec(4, 3))
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    ref, orep = oracle.fill_rows(two.vertices, two.triangles, 4, 3, DIRECT, 2 * np.pi)
    B = oracle.entry_bounds(two.vertices, two.triangles, 4, 3, None, 2 * np.pi, ULPS)
    assert np.all(np.abs(z.cpu().numpy() - ref) <= B) and rep.actual_calls == orep.actual_calls
    # empty row range
    mesh = sphere(gk, 1)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, row_begin=7, row_end=7)
    assert z.shape[0] == 0 and rep.actual_calls == 0
    # strided output: rows 10..30 into columns [5, 5 + N) of a wider buffer
    big = torch.full((20, dm.N + 13), complex(7, 7), dtype=torch.complex128, device="cuda:0")
    win = big[:, 5:5 + dm.N]
    gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi, row_begin=10, row_end=30, out=win)
    full, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    assert torch.equal(win, full[10:30])
    assert torch.all(big[:, :5] == complex(7, 7)) and torch.all(big[:, 5 + dm.N:] == complex(7, 7))


def test_separate_contexts_on_separate_host_threads(gk):
    """SURVEY 8b threading contract: a context is not re-entrant, but separate
    contexts (each with its own stream) may be driven from separate host
    threads concurrently; every thread gets the single-threaded result."""
    import threading

    import torch
    mesh = sphere(gk, 2)
    ref, _ = gk.fill_rows(gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4)), gk.Mode.DIRECT,
                          k=2 * np.pi)
    ref = ref.cpu()
    results, errors = {}, []

    def work(i):
        try:
            ctx = gk.Context(0)   # its own gk_ctx and stream
            dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), ctx)
            lo, hi = dm.distance_range()
            t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi), gk.Medium(), ctx=ctx)
            for _ in range(3):
                z, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
                zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
            results[i] = (z.cpu(), zt.cpu())
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for i in range(4):
        assert torch.equal(results[i][0], ref)
        assert torch.equal(results[i][1], results[0][1])


def test_async_fill_errors_surface_at_fill_check(gk):
    """Asynchronous fills (report=False) accumulate their counts in the
    context; fill_check returns the fallbacks and raises the reference's
    exceptions like the synchronous call."""
    ctx = gk.Context.get(0)
    ctx.fill_check()   # start clean
    mesh = gk.generate_sphere_mesh(0.5, 1)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(1, 1))
    from oracle.pyoracle import Oracle
    hi = Oracle().max_vertex_distance(mesh.vertices) * 1.01
    t = gk.DeviceTable(gk.SamplingConfig(r_min=0.3, r_max=hi))
    _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t)           # synchronous reference
    for _ in range(3):
        gk.fill_rows(dm, gk.Mode.TABLE, table=t, report=False)
    assert ctx.fill_check() == 3 * rep.fallback_calls > 0
    assert ctx.fill_check() == 0                                 # reset
    low = gk.DeviceTable(gk.SamplingConfig(r_min=1e-3, r_max=0.5))
    gk.fill_rows(dm, gk.Mode.TABLE, table=low, report=False)     # radii above r_max
    with pytest.raises(gk.OutOfRange):
        ctx.fill_check()
    v = np.array([[0, 0, 0], [3, 0, 0], [0, 3, 0], [0.5, 1, 0], [1.5, 1, 0], [1, 1, 1]], float)
    zero = gk.DeviceMesh(gk.TriangleMesh(v, np.array([[0, 1, 2], [3, 4, 5]])),
                         gk.QuadratureSpec(1, 1))
    gk.fill_rows(zero, gk.Mode.DIRECT, k=2 * np.pi, report=False)
    with pytest.raises(gk.DomainError):
        ctx.fill_check()
    assert ctx.fill_check() == 0


@pytest.mark.parametrize("lam", [0.01, 1000.0])
def test_extreme_wavelengths(gk, oracle, lam):
    """kr up to ~1250 (lambda = 1 cm on the unit sphere: phase rounding grows
    like the reference's, the (1 + |k| r) factor of the bound) and kr ~ 0.01
    (lambda = 1 km: G ~ 1/r), both modes."""
    mesh = sphere(gk, 2)
    k = 2 * np.pi / lam
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 3))
    zd, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, row_begin=0, row_end=64)
    ref, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, DIRECT, k, threads=8,
                              row_begin=0, row_end=64)
    B = oracle.entry_bounds(mesh.vertices, mesh.triangles, 4, 3, None, k, ULPS,
                            row_begin=0, row_end=64)
    assert np.all(np.abs(zd.cpu().numpy() - ref) <= B)
    lo, hi = dm.distance_range()
    # S such that the base interval is <= 1 mm (lambda = 1 km at S = 1000 would
    # leave fewer than two intervals: build_plan rejects it, like the reference)
    S = max(1000, int(lam / 1e-3))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S),
                       gk.Medium(lambda0=lam))
    d = t.download()
    ev = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), k)
    zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t, row_begin=0, row_end=64)
    ref_t, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, TABLE, k, ev=ev, threads=8,
                                row_begin=0, row_end=64)
    Bt = oracle.entry_bounds(mesh.vertices, mesh.triangles, 4, 3, ev, k, ULPS, row_begin=0,
                             row_end=64)
    assert np.all(np.abs(zt.cpu().numpy() - ref) <= Bt)
    assert np.all(np.abs(zt.cpu().numpy() - ref_t) <= B)


def test_no_device_memory_growth_over_repeated_lifecycles(gk):
    """Create / fill / destroy meshes, tables, bench_compare and streamed host
    fills repeatedly: after a warm-up cycle the device's free memory stays
    flat (every stream-ordered allocation is freed and reused by the pool)."""
    import gc

    import torch

    def cycle():
        mesh = sphere(gk, 2)
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
        lo, hi = dm.distance_range()
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=4000))
        gk.fill_rows(dm, gk.Mode.TABLE, table=t)
        gk.fill_rows_pair(dm, gk.Mode.DIRECT, k=2 * np.pi)
        z = np.zeros((50, dm.N), np.complex128)
        gk.fill_rows_host(dm, gk.Mode.DIRECT, z, k=2 * np.pi, row_begin=0, row_end=50)
        t.error_sweep(gk.KernelKind.GreenOverR, probe_count=10000)
        gk.bench_compare(gk.generate_sphere_mesh(0.5, 1), gk.QuadratureSpec(4, 3))
        del t, dm
        gc.collect()
        torch.cuda.synchronize()

    cycle()
    free0 = torch.cuda.mem_get_info(0)[0]
    for _ in range(5):
        cycle()
    free1 = torch.cuda.mem_get_info(0)[0]
    assert free0 - free1 <= 64 << 20, (free0 - free1) / 2 ** 20


def test_fill_rows_rejects_bad_output(gk):
    """A too-small, strided or wrong-dtype output is rejected before launch."""
    import torch
    dm = gk.DeviceMesh(sphere(gk, 1), gk.QuadratureSpec(4, 3))
    for bad in (torch.empty((10, dm.N), dtype=torch.complex128, device="cuda:0"),       # rows
                torch.empty((dm.N, dm.N - 1), dtype=torch.complex128, device="cuda:0"),  # cols
                torch.empty((dm.N, dm.N), dtype=torch.complex64, device="cuda:0"),
                torch.empty((dm.N, 2 * dm.N), dtype=torch.complex128, device="cuda:0")[:, ::2],
                torch.empty((dm.N, dm.N), dtype=torch.complex128)):
        with pytest.raises(gk.InvalidArgument):
            gk.fill_rows(dm, gk.Mode.DIRECT, k=1.0, out=bad)


@pytest.mark.parametrize("S,refine", [(1000, True), (10000, True), (300, True), (1000, False)])
def test_table_arithmetic_locate_bit_identical(gk, S, refine):
    """The arithmetic interval index on verified runs of the uniform base grid
    (TableDev::coarse) gives exactly the lookup path's bits: fills through the
    staged, L1 and global-fallback paths and eval_batch, with
    FillOptions.arith_locate on and off."""
    import torch
    mesh = sphere(gk, 3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S,
                                         refine=refine), gk.Medium(lambda0=0.3))
    r = torch.linspace(lo, hi, 200001, dtype=torch.float64, device="cuda:0")
    out = {}
    for arith in (1, 0):
        res = []
        for place in (gk.GK_TABLE_GLOBAL, gk.GK_TABLE_SHARED, gk.GK_AUTO):
            o = gk.FillOptions(arith_locate=arith, table_placement=place)
            ze, zg, rep = gk.fill_rows_pair(dm, gk.Mode.TABLE, table=t, row_begin=100,
                                            row_end=300, options=o)
            res += [ze, zg]
        t.ctx.set_fill_options(gk.FillOptions(arith_locate=arith))  # eval_batch: the context's
        try:
            res.append(t.eval_batch(gk.KernelKind.GreenOverR, r))
            res.append(t.eval_batch(gk.KernelKind.PlainExp, r))
        finally:
            t.ctx.set_fill_options(None)
        out[arith] = res
    for a, b in zip(out[1], out[0]):
        assert torch.equal(a, b)
