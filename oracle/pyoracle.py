"""ctypes front end for the parity checkers under oracle/.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package.  Two libraries are wrapped with the same Python surface:

* ``Oracle``  -> oracle/liboracle.so, the C restatement (gk_oracle.c);
* ``Ref``     -> oracle/_ref/libgkref.so, the unmodified reference headers
                 (/root/reference/proj/include) compiled through ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgkref.so")

STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "domain_error", 3: "out_of_range",
                4: "overflow_error", 5: "runtime_error"}
EXP, GREEN = 0, 1
DIRECT, TABLE = 0, 1

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {what}")


def _chk(status: int, what: str = "") -> None:
    if status:
        raise OracleError(status, what)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def build(ref: bool = True) -> None:
    """make -C oracle (liboracle always; _ref only when /root/reference exists)."""
    target = "all" if ref else "oracle"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


class _SamplingCfg(C.Structure):
    _fields_ = [("r_min", C.c_double), ("r_max", C.c_double),
                ("samples_per_wavelength", C.c_int), ("refine_interval_divisor", C.c_int),
                ("refine_halfwidth_in_t", C.c_double), ("dedup_fraction", C.c_double),
                ("refine", C.c_int)]


class _Plan(C.Structure):
    _fields_ = [("absc", _dp), ("n", C.c_size_t), ("zeros", _dp), ("nz", C.c_size_t),
                ("t", C.c_double), ("dr_min", C.c_double)]


class _Hash(C.Structure):
    _fields_ = [("r_min", C.c_double), ("r_max", C.c_double), ("dr_min", C.c_double),
                ("inv_dr_min", C.c_double), ("buckets", _u32p), ("nb", C.c_size_t)]


class FillReport(C.Structure):
    _fields_ = [("N", C.c_uint64), ("m", C.c_int), ("n", C.c_int),
                ("predicted_calls", C.c_uint64), ("actual_calls", C.c_uint64),
                ("fallback_calls", C.c_uint64), ("wall_time_s", C.c_double)]


@dataclass
class SamplingConfig:
    """Mirror of gktab::SamplingConfig (sampling.hpp:18-45) with its defaults."""
    r_min: float = 1e-4
    r_max: float = 1.0
    samples_per_wavelength: int = 1000
    refine_interval_divisor: int = 2
    refine_halfwidth_in_t: float = 2.0
    dedup_fraction: float = 0.5
    refine: bool = True

    def c(self) -> _SamplingCfg:
        return _SamplingCfg(self.r_min, self.r_max, self.samples_per_wavelength,
                            self.refine_interval_divisor, self.refine_halfwidth_in_t,
                            self.dedup_fraction, int(bool(self.refine)))


@dataclass
class Plan:
    abscissae: np.ndarray
    zeros: np.ndarray
    t: float
    dr_min: float


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C {HERE}`")
    return C.CDLL(path)


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path) and path == ORACLE_SO:
            build(ref=False)
        L = self.L = _load(path)
        L.go_evaluator_create.restype = C.c_void_p
        L.go_evaluator_create.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_double,
                                          C.c_double, C.c_int, C.POINTER(C.c_int)]
        L.go_evaluator_free.argtypes = [C.c_void_p]
        L.go_evaluator_fallbacks.restype = C.c_uint64
        L.go_evaluator_fallbacks.argtypes = [C.c_void_p]
        L.go_evaluator_hash.restype = C.POINTER(_Hash)
        L.go_evaluator_hash.argtypes = [C.c_void_p]
        L.go_max_vertex_distance.restype = C.c_double
        L.go_triangle_area.restype = C.c_double
        for name in ("go_eval_batch", "go_accumulate_green", "go_pointwise_bound",
                     "go_eval_exp", "go_eval_green", "go_eval_kernel", "go_interp_linear",
                     "go_interp_lagrange", "go_evaluator_tables"):
            getattr(L, name).argtypes = None
        L.go_jitter.argtypes = [_dp, C.c_size_t, C.c_uint64, C.c_double]
        L.go_jitter.restype = None

    # -- kernel.hpp
    def wavenumber(self, lambda0=1.0, eps_r=1.0, mu_r=1.0) -> float:
        k = C.c_double()
        med = (C.c_double * 3)(lambda0, eps_r, mu_r)
        _chk(self.L.go_wavenumber(med, C.byref(k)), "wavenumber")
        return k.value

    def eval_analytic(self, kind: int, k: float, r: float, k_im: float = 0.0) -> complex:
        out = (C.c_double * 2)()
        _chk(self.L.go_eval_analytic_ck(C.c_int(kind), C.c_double(k), C.c_double(k_im),
                                        C.c_double(r), out), "eval_analytic")
        return complex(out[0], out[1])

    def eval_analytic_batch(self, kind: int, k: float, radii, k_im: float = 0.0) -> np.ndarray:
        r = np.ascontiguousarray(radii, np.float64)
        out = np.zeros(r.size, np.complex128)
        _chk(self.L.go_eval_analytic_batch(C.c_int(kind), C.c_double(k), C.c_double(k_im),
                                           dptr(r), C.c_size_t(r.size),
                                           out.ctypes.data_as(C.c_void_p)), "eval_analytic")
        return out

    def pointwise_bounds(self, ev, kind: int, method: int, radii) -> np.ndarray:
        r = np.ascontiguousarray(radii, np.float64)
        return np.array([ev.pointwise_bound(kind, method, x) for x in r])

    # -- sampling.hpp
    def zero_crossings(self, k: float, r_min: float, r_max: float) -> np.ndarray:
        cnt = C.c_size_t()
        _chk(self.L.go_zero_crossings(C.c_double(k), C.c_double(r_min), C.c_double(r_max),
                                      None, C.c_size_t(0), C.byref(cnt)), "zero_crossings")
        out = np.zeros(cnt.value, np.float64)
        self.L.go_zero_crossings(C.c_double(k), C.c_double(r_min), C.c_double(r_max),
                                 dptr(out), C.c_size_t(out.size), C.byref(cnt))
        return out

    def _plan_out(self, p: _Plan) -> Plan:
        absc = np.ctypeslib.as_array(p.absc, shape=(p.n,)).copy()
        zeros = (np.ctypeslib.as_array(p.zeros, shape=(p.nz,)).copy() if p.nz
                 else np.zeros(0, np.float64))
        res = Plan(absc, zeros, p.t, p.dr_min)
        self.L.go_plan_free(C.byref(p))
        return res

    def build_plan(self, cfg: SamplingConfig, lambda0=1.0, eps_r=1.0, mu_r=1.0) -> Plan:
        p = _Plan()
        med = (C.c_double * 3)(lambda0, eps_r, mu_r)
        _chk(self.L.go_build_plan(C.byref(cfg.c()), med, C.byref(p)), "build_plan")
        return self._plan_out(p)

    def build_plan_core(self, cfg: SamplingConfig, k_zero: float, t_nominal: float) -> Plan:
        p = _Plan()
        _chk(self.L.go_build_plan_core(C.byref(cfg.c()), C.c_double(k_zero),
                                       C.c_double(t_nominal), C.byref(p)), "build_plan_core")
        return self._plan_out(p)

    def make_plan(self, absc, zeros=()) -> Plan:
        a = np.ascontiguousarray(absc, np.float64)
        z = np.ascontiguousarray(zeros, np.float64)
        p = _Plan()
        _chk(self.L.go_make_plan(dptr(a), C.c_size_t(a.size), dptr(z) if z.size else None,
                                 C.c_size_t(z.size), C.byref(p)), "make_plan")
        return self._plan_out(p)

    # -- table.hpp
    def build_hash(self, absc, zeros=()):
        a = np.ascontiguousarray(absc, np.float64)
        z = np.ascontiguousarray(zeros, np.float64)
        p = _Plan()
        _chk(self.L.go_make_plan(dptr(a), C.c_size_t(a.size), dptr(z) if z.size else None,
                                 C.c_size_t(z.size), C.byref(p)), "make_plan")
        h = _Hash()
        st = self.L.go_build_hash(C.byref(p), C.byref(h))
        self.L.go_plan_free(C.byref(p))
        _chk(st, "build_hash")
        b = np.ctypeslib.as_array(h.buckets, shape=(h.nb,)).copy()
        dr, inv = h.dr_min, h.inv_dr_min
        self.L.go_hash_free(C.byref(h))
        return b, dr, inv

    def evaluator(self, plan: Plan, k: float, degree: int = 3, k_im: float = 0.0):
        return OracleEvaluator(self, plan, k, degree, k_im)

    # -- quadrature.hpp
    def triangle_rule(self, m: int) -> np.ndarray:
        out = np.zeros((4, 7), np.float64)
        _chk(self.L.go_triangle_rule(C.c_int(m), dptr(out[0]), dptr(out[1]), dptr(out[2]),
                                     dptr(out[3])), "triangle_rule")
        return out[:, :m].copy()

    def gauss_legendre_unit(self, n: int) -> np.ndarray:
        out = np.zeros((2, n), np.float64)
        _chk(self.L.go_gauss_legendre_unit(C.c_int(n), dptr(out[0]), dptr(out[1])),
             "gauss_legendre_unit")
        return out

    # -- mesh.hpp
    def _mesh_out(self, vp, nv, tp, nt):
        v = np.ctypeslib.as_array(vp, shape=(nv.value * 3,)).copy().reshape(-1, 3)
        t = np.ctypeslib.as_array(tp, shape=(nt.value * 3,)).copy().reshape(-1, 3)
        self.L.go_mesh_free(vp, tp)
        return v, t

    def sphere_mesh(self, radius: float, subdivisions: int):
        vp, tp = _dp(), _u32p()
        nv, nt = C.c_size_t(), C.c_size_t()
        _chk(self.L.go_sphere_mesh(C.c_double(radius), C.c_int(subdivisions), C.byref(vp),
                                   C.byref(nv), C.byref(tp), C.byref(nt)), "sphere_mesh")
        return self._mesh_out(vp, nv, tp, nt)

    def plate_mesh(self, side: float, cells: int):
        vp, tp = _dp(), _u32p()
        nv, nt = C.c_size_t(), C.c_size_t()
        _chk(self.L.go_plate_mesh(C.c_double(side), C.c_int(cells), C.byref(vp), C.byref(nv),
                                  C.byref(tp), C.byref(nt)), "plate_mesh")
        return self._mesh_out(vp, nv, tp, nt)

    def jitter(self, verts: np.ndarray, seed: int, amp: float) -> np.ndarray:
        v = np.ascontiguousarray(verts, np.float64).copy()
        self.L.go_jitter(dptr(v.reshape(-1)), v.shape[0], seed, amp)
        return v

    def max_vertex_distance(self, verts) -> float:
        v = np.ascontiguousarray(verts, np.float64)
        return self.L.go_max_vertex_distance(dptr(v.reshape(-1)), C.c_size_t(v.shape[0]))

    def points(self, verts, tris, m: int, n: int):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nv, nt = v.size // 3, t.size // 3
        outer = np.zeros((4, nt * m), np.float64)
        inner = np.zeros((4, nt * 3 * n), np.float64)
        _chk(self.L.go_outer_points(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt),
                                    C.c_int(m), *[dptr(outer[i]) for i in range(4)]), "outer")
        _chk(self.L.go_inner_points(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt),
                                    C.c_int(n), *[dptr(inner[i]) for i in range(4)]), "inner")
        return outer, inner

    # -- matfill.hpp
    def fill_rows(self, verts, tris, m: int, n: int, mode: int, k: float, ev=None,
                  kind: int = GREEN, threads: int = 1, row_begin: int = 0, row_end=None,
                  k_im: float = 0.0):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nv, nt = v.size // 3, t.size // 3
        row_end = nt if row_end is None else row_end
        z = np.zeros((row_end - row_begin, nt), np.complex128)
        rep = FillReport()
        _chk(self.L.go_fill_rows(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt), C.c_int(m),
                                 C.c_int(n), C.c_int(mode), C.c_double(k), C.c_double(k_im),
                                 C.c_void_p(ev.h if ev is not None else None), C.c_int(kind),
                                 C.c_int(threads), C.c_size_t(row_begin), C.c_size_t(row_end),
                                 z.ctypes.data_as(C.c_void_p), C.c_size_t(nt), C.byref(rep)),
             "fill_rows")
        return z, rep

    def compare_fills(self, test: np.ndarray, ref: np.ndarray):
        a = np.ascontiguousarray(test, np.complex128)
        b = np.ascontiguousarray(ref, np.complex128)
        re, im = C.c_double(), C.c_double()
        _chk(self.L.go_compare_fills(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                     C.c_size_t(a.shape[0]), C.byref(re), C.byref(im)), "cmp")
        return re.value, im.value

    def entry_bounds(self, verts, tris, m, n, ev, k_abs, ulps=64.0, row_begin=0, row_end=None):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nv, nt = v.size // 3, t.size // 3
        row_end = nt if row_end is None else row_end
        b = np.zeros((row_end - row_begin, nt), np.float64)
        _chk(self.L.go_entry_bounds(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt),
                                    C.c_int(m), C.c_int(n),
                                    C.c_void_p(ev.h if ev is not None else None),
                                    C.c_double(k_abs), C.c_double(ulps), C.c_size_t(row_begin),
                                    C.c_size_t(row_end), dptr(b), C.c_size_t(nt)), "bounds")
        return b

    def entry_bounds_rows(self, verts, tris, m, n, ev, k_abs, rows, ulps=64.0, threads=8):
        """entry_bounds for an arbitrary row list (full-size sampled rows)"""
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nv, nt = v.size // 3, t.size // 3
        rws = np.ascontiguousarray(rows, np.uint64)
        b = np.zeros((rws.size, nt), np.float64)
        _chk(self.L.go_entry_bounds_rows(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt),
                                         C.c_int(m), C.c_int(n),
                                         C.c_void_p(ev.h if ev is not None else None),
                                         C.c_double(k_abs), C.c_double(ulps),
                                         rws.ctypes.data_as(_u64p), C.c_size_t(rws.size),
                                         C.c_int(threads), dptr(b), C.c_size_t(nt)), "bounds")
        return b

    def distance_range(self, verts, tris, m, n, row_begin=0, row_end=None):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nv, nt = v.size // 3, t.size // 3
        row_end = nt if row_end is None else row_end
        lo, hi = C.c_double(), C.c_double()
        _chk(self.L.go_distance_range(dptr(v), C.c_size_t(nv), u32ptr(t), C.c_size_t(nt),
                                      C.c_int(m), C.c_int(n), C.c_size_t(row_begin),
                                      C.c_size_t(row_end), C.byref(lo), C.byref(hi)), "range")
        return lo.value, hi.value

    def predicted_calls(self, N, m, n) -> int:
        out = C.c_uint64()
        _chk(self.L.go_predicted_calls(C.c_uint64(N), C.c_uint64(m), C.c_uint64(n),
                                       C.byref(out)), "predicted_calls")
        return out.value


class OracleEvaluator:
    """Mirror of gktab::KernelEvaluator over the C restatement."""

    def __init__(self, o: Oracle, plan: Plan, k: float, degree: int, k_im: float):
        self.o, self.plan, self.k, self.k_im, self.degree = o, plan, k, k_im, degree
        a, z = plan.abscissae, plan.zeros
        st = C.c_int()
        self.h = o.L.go_evaluator_create(dptr(a), C.c_size_t(a.size),
                                         dptr(z) if z.size else None, C.c_size_t(z.size),
                                         C.c_double(k), C.c_double(k_im), C.c_int(degree),
                                         C.byref(st))
        _chk(st.value, "KernelEvaluator")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.go_evaluator_free(C.c_void_p(self.h))
            self.h = None

    @property
    def fallbacks(self) -> int:
        return self.o.L.go_evaluator_fallbacks(C.c_void_p(self.h))

    def tables(self):
        n = self.plan.abscissae.size
        e = np.zeros(n, np.complex128)
        g = np.zeros(n, np.complex128)
        self.o.L.go_evaluator_tables(C.c_void_p(self.h), e.ctypes.data_as(C.c_void_p),
                                     g.ctypes.data_as(C.c_void_p))
        return e, g

    def buckets(self) -> np.ndarray:
        h = self.o.L.go_evaluator_hash(C.c_void_p(self.h)).contents
        return np.ctypeslib.as_array(h.buckets, shape=(h.nb,)).copy()

    def eval_batch(self, kind: int, radii) -> np.ndarray:
        r = np.ascontiguousarray(radii, np.float64)
        out = np.zeros(r.size, np.complex128)
        fail = C.c_size_t()
        st = self.o.L.go_eval_batch(C.c_void_p(self.h), C.c_int(kind), dptr(r),
                                    C.c_size_t(r.size), out.ctypes.data_as(C.c_void_p),
                                    C.byref(fail))
        _chk(st, f"eval_batch: radius [{fail.value}]")
        return out

    def _scalar(self, fn, *args) -> complex:
        out = (C.c_double * 2)()
        _chk(fn(C.c_void_p(self.h), *args, out), fn.__name__)
        return complex(out[0], out[1])

    def eval_exp(self, r):
        return self._scalar(self.o.L.go_eval_exp, C.c_double(r))

    def eval_green(self, r):
        return self._scalar(self.o.L.go_eval_green, C.c_double(r))

    def eval_kernel(self, kind, r):
        return self._scalar(self.o.L.go_eval_kernel, C.c_int(kind), C.c_double(r))

    def interp_lagrange(self, kind, degree, r):
        return self._scalar(self.o.L.go_interp_lagrange, C.c_int(kind), C.c_int(degree),
                            C.c_double(r))

    def accumulate_green(self, radii, weights) -> complex:
        r = np.ascontiguousarray(radii, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        out = (C.c_double * 2)()
        _chk(self.o.L.go_accumulate_green(C.c_void_p(self.h), dptr(r), dptr(w),
                                          C.c_size_t(r.size), out), "accumulate_green")
        return complex(out[0], out[1])

    def pointwise_bound(self, kind, method, r) -> float:
        out = C.c_double()
        _chk(self.o.L.go_pointwise_bound(C.c_void_p(self.h), C.c_int(kind), C.c_int(method),
                                         C.c_double(r), C.byref(out)), "pointwise_bound")
        return out.value


class Ref:
    """The unmodified reference compiled in place (oracle/_ref/libgkref.so)."""

    def __init__(self, path: str = REF_SO):
        L = self.L = _load(path)
        for fn in ("gr_plan_create", "gr_make_plan", "gr_evaluator_create"):
            getattr(L, fn).restype = C.c_void_p
        L.gr_plan_create.argtypes = [C.POINTER(_SamplingCfg), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int)]
        L.gr_plan_free.argtypes = [C.c_void_p]
        L.gr_evaluator_free.argtypes = [C.c_void_p]
        L.gr_fallbacks.restype = C.c_uint64
        L.gr_fallbacks.argtypes = [C.c_void_p]
        L.gr_max_vertex_distance.restype = C.c_double

    def wavenumber(self, lambda0=1.0, eps_r=1.0, mu_r=1.0) -> float:
        k = C.c_double()
        _chk(self.L.gr_wavenumber((C.c_double * 3)(lambda0, eps_r, mu_r), C.byref(k)), "k")
        return k.value

    def eval_analytic(self, kind, k, r) -> complex:
        out = (C.c_double * 2)()
        _chk(self.L.gr_eval_analytic(C.c_int(kind), C.c_double(k), C.c_double(r), out), "ea")
        return complex(out[0], out[1])

    def _plan(self, h) -> Plan:
        n, nz = C.c_size_t(), C.c_size_t()
        t, dr = C.c_double(), C.c_double()
        self.L.gr_plan_info(C.c_void_p(h), C.byref(n), C.byref(nz), C.byref(t), C.byref(dr))
        a = np.zeros(n.value, np.float64)
        z = np.zeros(nz.value, np.float64)
        self.L.gr_plan_copy(C.c_void_p(h), dptr(a), dptr(z) if z.size else dptr(np.zeros(1)))
        self.L.gr_plan_free(C.c_void_p(h))
        return Plan(a, z, t.value, dr.value)

    def build_plan(self, cfg: SamplingConfig, lambda0=1.0, eps_r=1.0, mu_r=1.0) -> Plan:
        st = C.c_int()
        c = cfg.c()
        h = self.L.gr_plan_create(C.byref(c), (C.c_double * 3)(lambda0, eps_r, mu_r),
                                  C.byref(st))
        _chk(st.value, "build_plan")
        return self._plan(h)

    def build_hash(self, absc, zeros=()):
        a = np.ascontiguousarray(absc, np.float64)
        z = np.ascontiguousarray(zeros, np.float64)
        st = C.c_int()
        h = self.L.gr_make_plan(dptr(a), C.c_size_t(a.size), dptr(z) if z.size else None,
                                C.c_size_t(z.size), C.byref(st))
        _chk(st.value, "make_plan")
        nb, dr, inv = C.c_size_t(), C.c_double(), C.c_double()
        _chk(self.L.gr_build_hash(C.c_void_p(h), C.byref(nb), None, C.c_size_t(0),
                                  C.byref(dr), C.byref(inv)), "build_hash")
        b = np.zeros(nb.value, np.uint32)
        self.L.gr_build_hash(C.c_void_p(h), C.byref(nb), u32ptr(b), C.c_size_t(b.size),
                             C.byref(dr), C.byref(inv))
        self.L.gr_plan_free(C.c_void_p(h))
        return b, dr.value, inv.value

    def evaluator(self, plan: Plan, k: float, degree: int = 3):
        return RefEvaluator(self, plan, k, degree)

    def triangle_rule(self, m):
        out = np.zeros((4, 7), np.float64)
        _chk(self.L.gr_triangle_rule(C.c_int(m), dptr(out[0]), dptr(out[1]), dptr(out[2]),
                                     dptr(out[3])), "triangle_rule")
        return out[:, :m].copy()

    def gauss_legendre_unit(self, n):
        out = np.zeros((2, n), np.float64)
        _chk(self.L.gr_gauss_legendre_unit(C.c_int(n), dptr(out[0]), dptr(out[1])), "gl")
        return out

    def sphere_mesh(self, radius, subdivisions):
        nv, nt = C.c_size_t(), C.c_size_t()
        _chk(self.L.gr_sphere_mesh(C.c_double(radius), C.c_int(subdivisions), None,
                                   C.byref(nv), None, C.byref(nt)), "sphere")
        v = np.zeros((nv.value, 3), np.float64)
        t = np.zeros((nt.value, 3), np.uint32)
        self.L.gr_sphere_mesh(C.c_double(radius), C.c_int(subdivisions), dptr(v.reshape(-1)),
                              C.byref(nv), u32ptr(t.reshape(-1)), C.byref(nt))
        return v, t

    def max_vertex_distance(self, verts):
        v = np.ascontiguousarray(verts, np.float64)
        return self.L.gr_max_vertex_distance(dptr(v.reshape(-1)), C.c_size_t(v.shape[0]))

    def points(self, verts, tris, m, n):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nt = t.size // 3
        outer = np.zeros((4, nt * m), np.float64)
        inner = np.zeros((4, nt * 3 * n), np.float64)
        _chk(self.L.gr_points(dptr(v), C.c_size_t(v.size // 3), u32ptr(t), C.c_size_t(nt),
                              C.c_int(m), C.c_int(n), dptr(outer.reshape(-1)),
                              dptr(inner.reshape(-1))), "points")
        return outer, inner

    def fill_matrix(self, verts, tris, m, n, mode, k, ev=None, kind=GREEN, threads=1):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nt = t.size // 3
        z = np.zeros((nt, nt), np.complex128)
        rep = FillReport()
        _chk(self.L.gr_fill_matrix(dptr(v), C.c_size_t(v.size // 3), u32ptr(t), C.c_size_t(nt),
                                   C.c_int(m), C.c_int(n), C.c_int(mode), C.c_double(k),
                                   C.c_void_p(ev.h if ev is not None else None), C.c_int(kind),
                                   C.c_int(threads), z.ctypes.data_as(C.c_void_p),
                                   C.byref(rep)), "fill_matrix")
        return z, rep

    def fill_sampled_rows(self, verts, tris, m, n, mode, k, rows, ev=None, kind=GREEN,
                          threads=1):
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.uint32).reshape(-1)
        nt = t.size // 3
        rws = np.ascontiguousarray(rows, np.uint64)
        z = np.zeros((rws.size, nt), np.complex128)
        calls, wall = C.c_uint64(), C.c_double()
        _chk(self.L.gr_fill_sampled_rows(dptr(v), C.c_size_t(v.size // 3), u32ptr(t),
                                         C.c_size_t(nt), C.c_int(m), C.c_int(n), C.c_int(mode),
                                         C.c_double(k),
                                         C.c_void_p(ev.h if ev is not None else None),
                                         C.c_int(kind), C.c_int(threads),
                                         rws.ctypes.data_as(_u64p), C.c_size_t(rws.size),
                                         z.ctypes.data_as(C.c_void_p), C.byref(calls),
                                         C.byref(wall)), "fill_sampled_rows")
        return z, calls.value, wall.value

    def analytic_batch(self, kind, k, radii, threads=1):
        r = np.ascontiguousarray(radii, np.float64)
        out = np.zeros(r.size, np.complex128)
        _chk(self.L.gr_analytic_batch_threaded(C.c_int(kind), C.c_double(k), dptr(r),
                                               C.c_size_t(r.size),
                                               out.ctypes.data_as(C.c_void_p),
                                               C.c_int(threads)), "analytic_batch")
        return out

    def dump_plan_csv(self, plan: Plan, path: str) -> None:
        a, z = plan.abscissae, plan.zeros
        _chk(self.L.gr_dump_plan_csv(dptr(a), C.c_size_t(a.size), dptr(z) if z.size else None,
                                     C.c_size_t(z.size), path.encode()), "dump_plan_csv")

    def error_sweep(self, ev, kind: int, method: int, probes: int):
        """the reference's error_sweep (bounds.hpp:128-186) on a reference evaluator"""
        d = np.zeros(5, np.float64)
        hist = np.zeros(24, np.uint64)
        _chk(self.L.gr_error_sweep(C.c_void_p(ev.h), C.c_int(kind), C.c_int(method),
                                   C.c_uint64(probes), dptr(d), hist.ctypes.data_as(C.c_void_p)),
             "error_sweep")
        return dict(max_rel_re=d[0], max_rel_im=d[1], max_abs=d[2], worst_r=d[3],
                    max_abs_at_exact_zero=d[4], decade_histogram=hist.tolist())

    def write_bench_csv(self, ints, dbls, path: str) -> None:
        """the reference's write_bench_csv (io.hpp:147-156) of a report"""
        i = np.ascontiguousarray(ints, np.uint64)
        d = np.ascontiguousarray(dbls, np.float64)
        _chk(self.L.gr_write_bench_csv(i.ctypes.data_as(C.c_void_p), dptr(d), path.encode()),
             "write_bench_csv")

    def write_sweep_csv(self, kind, method, degree, probes, dbls, path: str) -> None:
        """the reference's write_sweep_csv_header + _row (io.hpp:134-145)"""
        d = np.ascontiguousarray(dbls, np.float64)
        _chk(self.L.gr_write_sweep_csv(C.c_int(kind), C.c_int(method), C.c_int(degree),
                                       C.c_uint64(probes), dptr(d), path.encode()),
             "write_sweep_csv")

    def load_table_binary(self, path: str):
        kind, k, cnt = C.c_int(), C.c_double(), C.c_size_t()
        _chk(self.L.gr_load_table_binary(path.encode(), C.byref(kind), C.byref(k), C.byref(cnt),
                                         None, None), "load_table_binary")
        r = np.zeros(cnt.value, np.float64)
        v = np.zeros(cnt.value, np.complex128)
        _chk(self.L.gr_load_table_binary(path.encode(), C.byref(kind), C.byref(k), C.byref(cnt),
                                         dptr(r), v.ctypes.data_as(C.c_void_p)),
             "load_table_binary")
        return kind.value, k.value, r, v

    def compare_fills(self, test, ref):
        a = np.ascontiguousarray(test, np.complex128)
        b = np.ascontiguousarray(ref, np.complex128)
        re, im = C.c_double(), C.c_double()
        _chk(self.L.gr_compare_fills(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                     C.c_size_t(a.shape[0]), C.byref(re), C.byref(im)), "cmp")
        return re.value, im.value


class RefEvaluator:
    def __init__(self, ref: Ref, plan: Plan, k: float, degree: int):
        self.ref, self.plan, self.k, self.degree = ref, plan, k, degree
        a, z = plan.abscissae, plan.zeros
        st = C.c_int()
        self.h = ref.L.gr_evaluator_create(dptr(a), C.c_size_t(a.size),
                                           dptr(z) if z.size else None, C.c_size_t(z.size),
                                           C.c_double(k), C.c_int(degree), C.byref(st))
        _chk(st.value, "KernelEvaluator")

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.gr_evaluator_free(C.c_void_p(self.h))
            self.h = None

    @property
    def fallbacks(self) -> int:
        return self.ref.L.gr_fallbacks(C.c_void_p(self.h))

    def tables(self):
        n = self.plan.abscissae.size
        e = np.zeros(n, np.complex128)
        g = np.zeros(n, np.complex128)
        self.ref.L.gr_tables(C.c_void_p(self.h), e.ctypes.data_as(C.c_void_p),
                             g.ctypes.data_as(C.c_void_p))
        return e, g

    def eval_batch(self, kind, radii, threads: int = 1):
        r = np.ascontiguousarray(radii, np.float64)
        out = np.zeros(r.size, np.complex128)
        _chk(self.ref.L.gr_eval_batch_threaded(C.c_void_p(self.h), C.c_int(kind), dptr(r),
                                               C.c_size_t(r.size),
                                               out.ctypes.data_as(C.c_void_p),
                                               C.c_int(threads)), "eval_batch")
        return out

    def eval_kernel(self, kind, r) -> complex:
        out = (C.c_double * 2)()
        _chk(self.ref.L.gr_eval_kernel(C.c_void_p(self.h), C.c_int(kind), C.c_double(r), out),
             "eval_kernel")
        return complex(out[0], out[1])

    def accumulate_green(self, radii, weights) -> complex:
        r = np.ascontiguousarray(radii, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        out = (C.c_double * 2)()
        _chk(self.ref.L.gr_accumulate_green(C.c_void_p(self.h), dptr(r), dptr(w),
                                            C.c_size_t(r.size), out), "accumulate_green")
        return complex(out[0], out[1])

    def pointwise_bound(self, kind, method, r) -> float:
        out = C.c_double()
        _chk(self.ref.L.gr_pointwise_bound(C.c_void_p(self.h), C.c_int(kind), C.c_int(method),
                                           C.c_double(r), C.byref(out)), "pointwise_bound")
        return out.value


def splitmix64_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """Seeded U[lo, hi) radii: splitmix64, top 53 bits."""
    out = np.empty(n, np.float64)
    M = (1 << 64) - 1
    s = seed & M
    # vectorised splitmix64 over a counter sequence
    ctr = (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
           + np.uint64(s))
    z = ctr
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    out[:] = lo + (hi - lo) * u
    return out
