"""K2 device table build and K5 evaluation vs the oracle (parity tests proper).

Plan and reference-format hash: bit-exact vs the oracle's build_plan /
build_hash (which is pinned bitwise to the reference, test_oracle_vs_ref.py).
Node values: device sincos vs glibc, <= 4 ulp.  Interpolated values: GPU table
vs CPU table on the same plan, rounding-level; vs direct evaluation, within
the reference's own per-probe bound (bounds.hpp:97-111) plus FP64 rounding.
"""
import math

import numpy as np
import pytest

from oracle.pyoracle import EXP, GREEN, SamplingConfig as OCfg, splitmix64_uniform

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -52


def _cfg(g, **kw):
    return g.SamplingConfig(**kw)


def _ocfg(c):
    return OCfg(c.r_min, c.r_max, c.samples_per_wavelength, c.refine_interval_divisor,
                c.refine_halfwidth_in_t, c.dedup_fraction, c.refine)


def _oracle_plan(oracle, c, med):
    if med.eps_r_im == 0.0:
        return oracle.build_plan(_ocfg(c), med.lambda0, med.eps_r, med.mu_r)
    n = np.sqrt(complex(med.eps_r * med.mu_r, med.eps_r_im * med.mu_r))
    k = 2.0 * math.pi * n / med.lambda0
    t = med.lambda0 / (c.samples_per_wavelength * n.real)
    return oracle.build_plan_core(_ocfg(c), k.real, t)


def _random_configs(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        lam = float(rng.uniform(0.3, 3.0))
        out.append((dict(r_min=1e-4 * lam, r_max=lam * 1.3,
                         samples_per_wavelength=int(rng.integers(40, 4001)),
                         refine_interval_divisor=int(rng.integers(2, 5)),
                         refine_halfwidth_in_t=float(rng.uniform(1.0, 3.0)),
                         dedup_fraction=float(rng.uniform(0.25, 1.0))),
                    dict(lambda0=lam)))
    return out


FIXED = [
    (dict(), dict()),                                            # reference default config
    (dict(refine=False), dict()),                                # plain grid, 1001 nodes
    (dict(r_min=1e-3, r_max=2.0), dict(lambda0=0.5)),            # C1, S = 1e3
    (dict(r_min=1e-3, r_max=2.0, samples_per_wavelength=10000), dict(lambda0=0.5)),  # C1 1e4
    (dict(r_min=0.0118, r_max=1.9997), dict()),                  # C2-like range
    (dict(r_min=1.4e-3, r_max=2.0, samples_per_wavelength=10000), dict(lambda0=0.15)),  # C5
    (dict(r_min=0.26, r_max=0.49), dict()),                      # no zero in range
    (dict(r_min=0.25, r_max=1.0), dict()),                       # zeros on both endpoints
    (dict(r_min=1e-4, r_max=1.0, samples_per_wavelength=20, refine_halfwidth_in_t=3.0),
     dict()),                                                    # overlapping windows
    (dict(r_min=1e-3, r_max=1.5, samples_per_wavelength=1000), dict(eps_r=4.0, eps_r_im=-0.4)),
]


@pytest.mark.parametrize("cfg_kw,med_kw", FIXED + _random_configs(24, 991))
def test_plan_and_hash_bit_exact(gk, oracle, cfg_kw, med_kw):
    c = gk.SamplingConfig(**cfg_kw)
    med = gk.Medium(**med_kw)
    t = gk.DeviceTable(c, med)
    d = t.download()
    p = _oracle_plan(oracle, c, med)
    assert d["abscissae"].size == p.abscissae.size
    assert np.array_equal(d["abscissae"], p.abscissae)
    assert np.array_equal(d["zeros"], p.zeros)
    assert d["t"] == p.t and d["dr_min"] == p.dr_min
    b, dr, inv = oracle.build_hash(p.abscissae, p.zeros)
    assert np.array_equal(d["buckets"], b)
    assert t.info.inv_dr_min == inv


def test_refine_off_plan_size(gk):
    t = gk.DeviceTable(gk.SamplingConfig(refine=False))
    assert t.info.nodes == 1001 and t.info.zeros == 0   # test_sampling.cpp:122-129


def test_zero_locations_quarter_period(gk):
    t = gk.DeviceTable(gk.SamplingConfig())
    assert list(t.download()["zeros"]) == [0.25, 0.5, 0.75, 1.0]  # test_sampling.cpp:42-49


@pytest.mark.parametrize("S", [1000, 10000])
def test_node_values_vs_glibc(gk, oracle, S):
    c = gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=S)
    med = gk.Medium(lambda0=0.5)
    t = gk.DeviceTable(c, med)
    d = t.download()
    p = _oracle_plan(oracle, c, med)
    ev = oracle.evaluator(p, oracle.wavenumber(0.5))
    e, g = ev.tables()
    assert np.all(np.abs(d["exp"] - e) <= 4 * ULP * np.abs(e))
    assert np.all(np.abs(d["green"] - g) <= 4 * ULP * np.abs(g))


def _c1(gk, oracle, S, n=1 << 20, lo=1e-3, seed=1901):
    c = gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=S)
    med = gk.Medium(lambda0=0.5)
    t = gk.DeviceTable(c, med)
    p = _oracle_plan(oracle, c, med)
    ev = oracle.evaluator(p, oracle.wavenumber(0.5))
    r = splitmix64_uniform(seed, n, lo, 2.0)
    return t, ev, r


@pytest.mark.parametrize("S", [1000, 10000])
def test_eval_batch_table_vs_cpu_table(gk, oracle, S):
    """C1 (2^20 seeded radii): same plan, GPU vs CPU interpolation."""
    t, ev, r = _c1(gk, oracle, S, lo=1e-4)  # straddles r_min: fallbacks exercised
    for kind in (EXP, GREEN):
        got = t.eval_batch(gk.KernelKind(kind), r).cpu().numpy()
        ref = ev.eval_batch(kind, r)
        scale = np.abs(ref) + (1.0 if kind == EXP else 1.0 / r)
        err = np.abs(got - ref) / scale
        assert err.max() <= 1e-11, (kind, err.max(), r[err.argmax()])
    assert t.fallbacks == ev.fallbacks and ev.fallbacks > 0


@pytest.mark.parametrize("S", [1000, 10000])
def test_eval_batch_green_within_pointwise_bound(gk, oracle, S):
    t, ev, r = _c1(gk, oracle, S, n=1 << 16)
    got = t.eval_batch(gk.KernelKind.GreenOverR, r).cpu().numpy()
    k = oracle.wavenumber(0.5)
    exact = np.array([oracle.eval_analytic(GREEN, k, x) for x in r])
    bound = np.array([ev.pointwise_bound(GREEN, 1, x) for x in r])
    tol = bound + 64 * 2.0 ** -53 * (1 + k * r) / r
    assert np.all(np.abs(got - exact) <= tol)


def test_nodes_reproduced_exactly(gk):
    t = gk.DeviceTable(gk.SamplingConfig())
    d = t.download()
    a = d["abscissae"]
    assert np.array_equal(t.eval_batch(gk.KernelKind.GreenOverR, a).cpu().numpy(), d["green"])
    assert np.array_equal(t.eval_batch(gk.KernelKind.PlainExp, a).cpu().numpy(), d["exp"])


@pytest.fixture
def eval_method(gk, request):
    ctx = gk.Context.get()
    ctx.set_fill_options(gk.FillOptions(eval_libdevice=request.param))
    yield request.param
    ctx.set_fill_options(None)


@pytest.mark.parametrize("eval_method", [0, 1], indirect=True)
def test_eval_batch_direct_vs_glibc(gk, oracle, eval_method):
    """direct eval_batch: the phase-table path (default, real k) and the
    libdevice sincos path (complex k, fallbacks; FillOptions.eval_libdevice
    through the context), both within a few ulp of glibc"""
    r = splitmix64_uniform(7, 1 << 16, 1e-3, 2.0)
    r[:3] = [0.25, 0.5, 1.0]   # quarter-period known answers (test_kernel.cpp:32-81)
    k = 4.0 * math.pi
    for kind in (EXP, GREEN):
        got = gk.eval_batch(gk.KernelKind(kind), r, k=k).cpu().numpy()
        ref = np.array([oracle.eval_analytic(kind, k, x) for x in r])
        assert np.all(np.abs(got - ref) <= 8 * ULP * (1 + k * r) * np.abs(ref))


def test_eval_batch_errors_carry_index(gk):
    t = gk.DeviceTable(gk.SamplingConfig())
    with pytest.raises(gk.InvalidArgument, match=r"\[2\]"):
        t.eval_batch(gk.KernelKind.PlainExp, [0.2, 0.3, -1.0, 0.4])
    with pytest.raises(gk.InvalidArgument, match=r"\[1\]"):
        t.eval_batch(gk.KernelKind.GreenOverR, [0.2, 1.5])          # above r_max
    with pytest.raises(gk.InvalidArgument, match=r"\[0\]"):
        gk.eval_batch(gk.KernelKind.GreenOverR, [0.0], k=1.0)      # singular
    assert gk.eval_batch(gk.KernelKind.PlainExp, [], k=1.0).numel() == 0
    assert complex(gk.eval_batch(gk.KernelKind.PlainExp, [0.0], k=7.3).cpu()[0]) == 1.0


def test_config_validation(gk):
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceTable(gk.SamplingConfig(r_min=-1.0))
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceTable(gk.SamplingConfig(r_min=0.1, r_max=0.1 + 1.5e-3))  # < two intervals
    with pytest.raises(gk.InvalidArgument):
        gk.DeviceTable(gk.SamplingConfig(), gk.Medium(lambda0=0.0))


def test_wire_formats_readable_by_reference(gk, oracle, ref, tmp_path):
    """io.hpp formats written from a DEVICE table: the plan CSV is byte-identical
    to the reference's dump_plan_csv, and the reference's load_table_binary reads
    the GKTB dump (radii bitwise, values within 4 ulp of glibc)."""
    c = gk.SamplingConfig(r_min=1e-3, r_max=2.0)
    t = gk.DeviceTable(c, gk.Medium(lambda0=0.5))
    d = t.download()
    t.dump_plan_csv(str(tmp_path / "gpu.csv"))
    p = oracle.build_plan(_ocfg(c), 0.5)
    ref.dump_plan_csv(p, str(tmp_path / "ref.csv"))
    assert (tmp_path / "gpu.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    for kind in (EXP, GREEN):
        path = str(tmp_path / f"t{kind}.gktb")
        t.dump_table_binary(gk.KernelKind(kind), path)
        k_kind, k, r, v = ref.load_table_binary(path)
        assert k_kind == kind and k == t.k
        assert np.array_equal(r, p.abscissae)
        e, g = oracle.evaluator(p, oracle.wavenumber(0.5)).tables()
        want = e if kind == EXP else g
        assert np.all(np.abs(v - want) <= 4 * ULP * np.abs(want))
        assert np.array_equal(v, d["exp"] if kind == EXP else d["green"])


def test_eval_batch_async_matches_sync_and_reports(gk, oracle):
    """gk_eval_batch_async: same bits as gk_eval_batch; fallbacks and the first
    bad radius accumulate in the device status and raise at read()."""
    import torch
    t, ev, r = _c1(gk, oracle, 1000, n=1 << 16, lo=1e-4)
    rd = torch.as_tensor(r, device="cuda:0")
    st = gk.EvalStatus(t.ctx)
    f0 = t.fallbacks
    for kind in (gk.KernelKind.PlainExp, gk.KernelKind.GreenOverR):
        out = torch.empty(r.size, dtype=torch.complex128, device="cuda:0")
        gk.eval_batch_async(kind, rd, out, st, table=t)
        assert torch.equal(out, t.eval_batch(kind, rd))
    fb_sync = t.fallbacks - f0
    assert fb_sync > 0 and st.read() == fb_sync
    bad = rd.clone()
    bad[9] = 3.0     # above r_max
    bad[5] = -1.0
    st.reset()
    out = torch.empty(r.size, dtype=torch.complex128, device="cuda:0")
    gk.eval_batch_async(gk.KernelKind.GreenOverR, bad, out, st, table=t)
    with pytest.raises(gk.InvalidArgument, match=r"\[5\]"):
        st.read()
    st.reset()
    gk.eval_batch_async(gk.KernelKind.PlainExp, rd, out, st, k=2.0)  # direct: no fallbacks
    assert st.read() == 0
    with pytest.raises(gk.InvalidArgument):   # host tensors are rejected, not dereferenced
        gk.eval_batch_async(gk.KernelKind.PlainExp, rd.cpu(), out, st, k=2.0)
    with pytest.raises(gk.InvalidArgument):
        gk.eval_batch_async(gk.KernelKind.PlainExp, rd, out[:10], st, k=2.0)


@pytest.mark.parametrize("degree", [1, 2, 4, 5, 7])
def test_lagrange_degrees_vs_oracle(gk, oracle, degree):
    """Green interpolation of degree != 3 (the reference's generic
    interp_lagrange, evaluator.hpp:40-95, with its stencil rule): device
    records vs the oracle's evaluator of the same degree on the same plan --
    rounding-level, eval_batch and a table-mode fill; test_evaluator.cpp:167-186
    checks degrees 2 and 4 against the pointwise bound, done here too."""
    c = gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=1000)
    med = gk.Medium(lambda0=0.5)
    t = gk.DeviceTable(c, med, lagrange_degree=degree)
    assert t.info.degree == degree
    p = _oracle_plan(oracle, c, med)
    ev = oracle.evaluator(p, oracle.wavenumber(0.5), degree=degree)
    r = splitmix64_uniform(3, 1 << 16, 1e-3, 2.0)
    got = t.eval_batch(gk.KernelKind.GreenOverR, r).cpu().numpy()
    ref = ev.eval_batch(GREEN, r)
    assert np.max(np.abs(got - ref) / (np.abs(ref) + 1.0 / r)) <= 1e-11
    k = oracle.wavenumber(0.5)
    exact = oracle.eval_analytic_batch(GREEN, k, r[::16])
    bound = oracle.pointwise_bounds(ev, GREEN, 1, r[::16])
    assert np.all(np.abs(got[::16] - exact) <= bound + 64 * 2.0 ** -53 * (1 + k * r[::16]) / r[::16])
    # table-mode fill with this degree
    mesh = gk.jitter(gk.generate_sphere_mesh(0.5, 1), 5, 1e-3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 3))
    lo, hi = dm.distance_range()
    tf = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=2000),
                        gk.Medium(), lagrange_degree=degree)
    d = tf.download()
    evf = oracle.evaluator(oracle.make_plan(d["abscissae"], d["zeros"]), 2 * math.pi,
                           degree=degree)
    zt, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=tf)
    ref_t, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, 4, 3, 1, 2 * math.pi, ev=evf,
                                threads=8)
    B = oracle.entry_bounds(mesh.vertices, mesh.triangles, 4, 3, None, 2 * math.pi, 64.0)
    assert np.all(np.abs(zt.cpu().numpy() - ref_t) <= B)


def test_accumulate_batch_vs_reference(gk, oracle, ref):
    """gk_accumulate_batch: the reference's Kernel::accumulate for many blocks at
    once -- TableKernel (accumulate_green, evaluator.hpp:150-194) and
    AnalyticKernel (matfill.hpp:58-68) -- vs the reference itself per block."""
    c = gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=1000)
    med = gk.Medium(lambda0=0.5)
    t = gk.DeviceTable(c, med)
    d = t.download()
    plan = oracle.make_plan(d["abscissae"], d["zeros"])
    k = oracle.wavenumber(0.5)
    rev = ref.evaluator(plan, k)
    nb, ln = 400, 72
    r = splitmix64_uniform(11, nb * ln, 2e-4, 2.0).reshape(nb, ln)   # some below r_min
    w = np.random.default_rng(5).uniform(-1.0, 1.0, (nb, ln))
    f0 = t.fallbacks
    got, fb = gk.accumulate_batch(gk.KernelKind.GreenOverR, r, w, table=t)
    got = got.cpu().numpy()
    assert fb == t.fallbacks - f0 == int(np.sum(r < d["abscissae"][0])) > 0
    for b in range(0, nb, 7):
        want = rev.accumulate_green(r[b], w[b])
        scale = np.sum(np.abs(w[b]) / r[b])
        assert abs(got[b] - want) <= 1e-11 * scale, b
    # Exp through the table and both kinds direct (AnalyticKernel{k})
    ge, _ = gk.accumulate_batch(gk.KernelKind.PlainExp, r, w, table=t)
    ev_vals = rev.eval_batch(EXP, r.reshape(-1)).reshape(nb, ln)
    assert np.max(np.abs(ge.cpu().numpy() - np.sum(ev_vals * w, axis=1))) <= 1e-12 * ln
    for kind in (EXP, GREEN):
        gd, fbd = gk.accumulate_batch(gk.KernelKind(kind), r, w, k=k)
        vals = oracle.eval_analytic_batch(kind, k, r.reshape(-1)).reshape(nb, ln)
        tol = np.sum(np.abs(w) * 8 * ULP * (1 + k * r) * np.abs(vals), axis=1) * 4
        assert np.all(np.abs(gd.cpu().numpy() - np.sum(vals * w, axis=1)) <= tol) and fbd == 0
    # errors carry the flat index of the first bad radius
    bad = r.copy()
    bad[3, 5] = 3.0
    with pytest.raises(gk.InvalidArgument, match=r"\[221\]"):
        gk.accumulate_batch(gk.KernelKind.GreenOverR, bad, w, table=t)
    bad[3, 5] = 0.0
    with pytest.raises(gk.InvalidArgument, match=r"\[221\]"):
        gk.accumulate_batch(gk.KernelKind.GreenOverR, bad, w, k=k)
    empty, fbe = gk.accumulate_batch(gk.KernelKind.GreenOverR, np.zeros((0, 4)), np.zeros((0, 4)), k=k)
    assert empty.numel() == 0 and fbe == 0


def test_wire_format_write_errors(gk, tmp_path):
    """io.hpp's writers throw runtime_error on an unwritable path; so do ours."""
    t = gk.DeviceTable(gk.SamplingConfig())
    bad = str(tmp_path / "missing_dir" / "x.gktb")
    with pytest.raises(gk.RuntimeErrorGk):
        t.dump_table_binary(gk.KernelKind.GreenOverR, bad)
    with pytest.raises(gk.RuntimeErrorGk):
        t.dump_plan_csv(str(tmp_path / "missing_dir" / "plan.csv"))
