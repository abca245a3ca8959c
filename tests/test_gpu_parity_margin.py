"""The parity MARGIN at BASELINE.json's full sizes, on SURVEY 8d's 64-row
deterministic sample p = floor(s N / 64), s = 0..63, for C2-C5.

For every sampled entry the device fill is compared with the reference's own
fill of the same rows (oracle/_ref: AnalyticKernel / TableKernel through the
reference's staging loop; for C4's complex k, which the reference has no path
for, the oracle restatement pinned bitwise to it).  Recorded per config and
mode (written to gpurun_out/r02_parity_margin.json; committed as
profiles/r02_parity_margin.json):

* ratio = max |dZ| / B_pq, B_pq the stated bar (tests/test_gpu_fill.py):
  sum |w_o w_i| (pw(r) + 64 u (1 + |k| r) / r), pw = the reference's
  pointwise_bound on the same plan in table mode, 0 in direct mode;
* ratio_survey = the same against SURVEY 8c's form without the (1 + |k| r)
  factor (direct mode; asserted where kr is small, C2);
* compare_fills = the reference's componentwise max relative error
  (matfill.hpp:237-254: diagonal and exact-zero components skipped);
* max |dZ| / |Z|.
"""
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import DIRECT, TABLE

pytestmark = pytest.mark.gpu
ULPS = 64.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out", "r02_parity_margin.json")

CONFIGS = {  # BASELINE.json configs[1..4]
    "c2": dict(level=3, m=6, n=4, lambda0=1.0),
    "c3": dict(level=5, m=7, n=5, lambda0=0.3),
    "c4": dict(plate=100, m=6, n=4, lambda0=1.0, eps_r=4.0, eps_r_im=-0.4),
    "c5": dict(level=6, m=6, n=4, lambda0=0.15),
}
RESULTS = {}


def sample_rows(N):
    return np.array([(s * N) // 64 for s in range(64)], np.uint64)


def _mesh(gk, c):
    if "plate" in c:
        return gk.generate_plate_mesh(1.0, c["plate"])
    return gk.jitter(gk.generate_sphere_mesh(1.0, c["level"]), 1901, 1e-3)


def _device_rows(gk, dm, rows, mode, **kw):
    out = np.empty((rows.size, dm.N), np.complex128)
    calls = 0
    for i, p in enumerate(rows):
        z, rep = gk.fill_rows(dm, mode, row_begin=int(p), row_end=int(p) + 1, **kw)
        out[i] = z.cpu().numpy()[0]
        calls += rep.actual_calls
    return out, calls


def _oracle_rows(oracle, mesh, c, rows, mode, k, ev=None):
    kc = complex(k)
    out = np.empty((rows.size, mesh.triangle_count()), np.complex128)
    for i, p in enumerate(rows):
        z, _ = oracle.fill_rows(mesh.vertices, mesh.triangles, c["m"], c["n"], mode, kc.real,
                                ev=ev, k_im=kc.imag, threads=8, row_begin=int(p),
                                row_end=int(p) + 1)
        out[i] = z[0]
    return out


def _compare_fills(test, ref, rows):
    """matfill.hpp:237-254 on sampled rows: skip the self pair (q == p) and
    exactly-zero reference components"""
    mask = np.ones(ref.shape, bool)
    mask[np.arange(rows.size), rows.astype(np.int64)] = False
    out = []
    for part in (np.real, np.imag):
        a, b = part(ref), part(test)
        ok = mask & (a != 0.0)
        out.append(float(np.max(np.abs(b[ok] - a[ok]) / np.abs(a[ok]))) if ok.any() else 0.0)
    return out


def _margin(z, want, B, rows, B_survey=None):
    mask = np.ones(z.shape, bool)
    mask[np.arange(rows.size), rows.astype(np.int64)] = False
    err = np.abs(z - want)
    assert np.all(err[~mask] == 0) and np.all(z[~mask] == 0)   # zero diagonal
    r = {"ratio": float(np.max(err[mask] / B[mask])),
         "max_rel_to_entry": float(np.max(err[mask] / np.abs(want[mask]))),
         "compare_fills_re_im": _compare_fills(z, want, rows)}
    if B_survey is not None:
        r["ratio_survey"] = float(np.max(err[mask] / B_survey[mask]))
    return r


def _record(name, key, val):
    RESULTS.setdefault(name, {})[key] = val
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    old = {}
    if os.path.exists(OUT):
        try:
            old = json.load(open(OUT))
        except ValueError:
            old = {}
    old.setdefault(name, {})[key] = val
    json.dump(old, open(OUT, "w"), indent=1, sort_keys=True)


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def case(request, gk):
    c = CONFIGS[request.param]
    mesh = _mesh(gk, c)
    med = gk.Medium(lambda0=c["lambda0"], eps_r=c.get("eps_r", 1.0),
                    eps_r_im=c.get("eps_r_im", 0.0))
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(c["m"], c["n"]))
    return request.param, c, mesh, med, dm, sample_rows(mesh.triangle_count())


def test_direct_margin_64_rows(gk, oracle, ref, case):
    name, c, mesh, med, dm, rows = case
    k = gk.wavenumber(med)
    kc = complex(k)
    m, n, N = c["m"], c["n"], mesh.triangle_count()
    z, calls = _device_rows(gk, dm, rows, gk.Mode.DIRECT, k=k)
    if kc.imag == 0.0:   # the reference itself
        want, rcalls, _ = ref.fill_sampled_rows(mesh.vertices, mesh.triangles, m, n, DIRECT,
                                                kc.real, rows, threads=8)
        assert rcalls == calls
        against = "reference AnalyticKernel (oracle/_ref)"
    else:
        want = _oracle_rows(oracle, mesh, c, rows, DIRECT, k)
        against = "oracle restatement (complex k: no reference path)"
    B = oracle.entry_bounds_rows(mesh.vertices, mesh.triangles, m, n, None, abs(kc), rows, ULPS)
    Bs = oracle.entry_bounds_rows(mesh.vertices, mesh.triangles, m, n, None, 0.0, rows, ULPS)
    r = _margin(z, want, B, rows, Bs)
    r.update(rows=int(rows.size), N=N, against=against, entries=int(rows.size * (N - 1)))
    _record(name, "direct", r)
    # measured on a B200 (profiles/r02_parity_margin.json): 0.07-0.13 of the
    # stated bar; asserted with room for another GPU's rounding
    assert r["ratio"] <= 0.25, r
    if name != "c5":   # kr <= 25: within SURVEY 8c's form without the (1 + |k| r)
        assert r["ratio_survey"] <= 1.0, r   # factor (C5's far pairs reach kr = 84: 1.06)


@pytest.mark.parametrize("S", [1000, 10000])
def test_table_margin_64_rows(gk, oracle, ref, case, S):
    name, c, mesh, med, dm, rows = case
    m, n, N = c["m"], c["n"], mesh.triangle_count()
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
    d = t.download()
    kc = complex(t.k)
    z, calls = _device_rows(gk, dm, rows, gk.Mode.TABLE, table=t)
    plan = oracle.make_plan(d["abscissae"], d["zeros"])
    ev = oracle.evaluator(plan, kc.real, k_im=kc.imag)
    if kc.imag == 0.0:   # the reference's direct and TableKernel fills of the same rows
        want_d, _, _ = ref.fill_sampled_rows(mesh.vertices, mesh.triangles, m, n, DIRECT,
                                             kc.real, rows, threads=8)
        rev = ref.evaluator(plan, kc.real)
        want_t, rcalls, _ = ref.fill_sampled_rows(mesh.vertices, mesh.triangles, m, n, TABLE,
                                                  kc.real, rows, ev=rev, threads=8)
        assert rcalls == calls
        against = "reference AnalyticKernel / TableKernel on the device table's plan"
    else:
        want_d = _oracle_rows(oracle, mesh, c, rows, DIRECT, kc)
        want_t = _oracle_rows(oracle, mesh, c, rows, TABLE, kc, ev=ev)
        against = "oracle restatement (complex k: no reference path)"
    B_t = oracle.entry_bounds_rows(mesh.vertices, mesh.triangles, m, n, ev, abs(kc), rows, ULPS)
    B_d = oracle.entry_bounds_rows(mesh.vertices, mesh.triangles, m, n, None, abs(kc), rows, ULPS)
    vs_direct = _margin(z, want_d, B_t, rows)
    vs_table = _margin(z, want_t, B_d, rows)
    r = {"vs_direct (bar: interpolation bound + rounding)": vs_direct,
         "vs_table_same_plan (bar: rounding)": vs_table, "S": S, "nodes": int(d["abscissae"].size),
         "rows": int(rows.size), "N": N, "against": against}
    _record(name, f"table_S{S}", r)
    # vs direct: the interpolation bound dominates (0.65-0.94 measured, the
    # reference's own table reaches 0.69 / 0.86 at C2); vs the
    # reference's table on the same plan: rounding only (0.04-0.10 measured)
    assert vs_direct["ratio"] <= 1.0 and vs_table["ratio"] <= 0.25, r
