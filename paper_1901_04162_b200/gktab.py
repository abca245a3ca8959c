"""Python mirror of the reference's operator surface for the fill hot path.

The names, argument meaning and error behaviour follow ``gktab``
(/root/reference/proj/include/gktab/): ``Medium``, ``SamplingConfig``,
``QuadratureSpec``, ``KernelKind``, ``wavenumber``, ``generate_sphere_mesh``,
``KernelEvaluator`` (here ``DeviceTable``: built on the GPU), ``eval_batch``,
``fill_matrix`` and ``FillReport``.  All compute runs in libgk.so (sm_100a
CUDA); torch supplies device memory and the current CUDA stream only.
"""
from __future__ import annotations

import ctypes as C
import enum
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import FillReportC, Medium as _MediumC, SamplingConfigC, TableInfoC, check, lib


class KernelKind(enum.IntEnum):
    """gktab::KernelKind (kernel.hpp:14-17)"""

    PlainExp = 0
    GreenOverR = 1


class InterpMethod(enum.IntEnum):
    """gktab::InterpMethod (bounds.hpp:15)"""

    Linear = 0
    Lagrange = 1


class Mode(enum.IntEnum):
    """AnalyticKernel (DIRECT) vs TableKernel (TABLE), matfill.hpp:59-87"""

    DIRECT = 0
    TABLE = 1


@dataclass
class Medium:
    """gktab::Medium (kernel.hpp:25-38); eps_r_im < 0 = lossy extension."""

    lambda0: float = 1.0
    eps_r: float = 1.0
    mu_r: float = 1.0
    eps_r_im: float = 0.0

    def c(self) -> _MediumC:
        return _MediumC(self.lambda0, self.eps_r, self.mu_r, self.eps_r_im)


@dataclass
class SamplingConfig:
    """gktab::SamplingConfig (sampling.hpp:18-45), same defaults."""

    r_min: float = 1e-4
    r_max: float = 1.0
    samples_per_wavelength: int = 1000
    refine_interval_divisor: int = 2
    refine_halfwidth_in_t: float = 2.0
    dedup_fraction: float = 0.5
    refine: bool = True

    def c(self) -> SamplingConfigC:
        return SamplingConfigC(self.r_min, self.r_max, int(self.samples_per_wavelength),
                               int(self.refine_interval_divisor), self.refine_halfwidth_in_t,
                               self.dedup_fraction, int(bool(self.refine)))


@dataclass
class QuadratureSpec:
    """gktab::QuadratureSpec (quadrature.hpp:15-26)"""

    outer_points: int = 4
    inner_points_per_edge: int = 3


@dataclass
class TriangleMesh:
    """gktab::TriangleMesh (mesh.hpp:33-58): vertices (nv,3) f64, triangles (nt,3) u32"""

    vertices: np.ndarray
    triangles: np.ndarray

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, np.float64).reshape(-1, 3)
        self.triangles = np.ascontiguousarray(self.triangles, np.uint32).reshape(-1, 3)

    def triangle_count(self) -> int:
        return self.triangles.shape[0]


@dataclass
class FillReport:
    """gktab::FillReport (matfill.hpp:33-47), the fields fill_matrix sets."""

    N: int = 0
    m: int = 0
    n: int = 0
    predicted_calls: int = 0
    actual_calls: int = 0
    fallback_calls: int = 0
    wall_time_s: float = 0.0
    # set by bench_compare (matfill.hpp:41-46)
    max_rel_re: float = 0.0
    max_rel_im: float = 0.0
    speedup: float = 0.0
    analytic_time_s: float = 0.0
    interp_time_s: float = 0.0
    table_build_s: float = 0.0
    # kernel evaluations the device performed (<= actual_calls: shared edges)
    evaluations: int = 0
    # the fill kernel that ran (gk_fill_path: PATH_NAMES)
    path: int = 0

    @classmethod
    def from_c(cls, r: FillReportC) -> "FillReport":
        return cls(r.N, r.m, r.n, r.predicted_calls, r.actual_calls, r.fallback_calls,
                   r.wall_time_s, evaluations=r.evaluations, path=r.path)

    @property
    def path_name(self) -> str:
        return PATH_NAMES.get(self.path, "none")


@dataclass
class ErrorSweepReport:
    """gktab::ErrorSweepReport (bounds.hpp:113-124)"""

    probe_count: int = 0
    max_rel_re: float = 0.0
    max_rel_im: float = 0.0
    max_abs: float = 0.0
    worst_r: float = 0.0
    max_abs_at_exact_zero: float = 0.0
    decade_histogram: list = field(default_factory=lambda: [0] * 24)


def wavenumber(medium: Medium) -> complex:
    """k = 2 pi sqrt(eps_r mu_r) / lambda0 (kernel.hpp:41-44); complex if lossy"""
    kr, ki = C.c_double(), C.c_double()
    check(lib().gk_wavenumber(C.byref(medium.c()), C.byref(kr), C.byref(ki)), "wavenumber")
    return complex(kr.value, ki.value) if ki.value else kr.value


def predicted_calls(N: int, m: int, n: int) -> int:
    out = C.c_uint64()
    check(lib().gk_predicted_calls(N, m, n, C.byref(out)), "predicted_calls")
    return out.value


def _mesh_from(fn, *args) -> TriangleMesh:
    nv, nt = C.c_size_t(), C.c_size_t()
    check(fn(*args, None, C.byref(nv), None, C.byref(nt)), fn.__name__)
    v = np.zeros((nv.value, 3), np.float64)
    t = np.zeros((nt.value, 3), np.uint32)
    check(fn(*args, v.ctypes.data, C.byref(nv), t.ctypes.data, C.byref(nt)), fn.__name__)
    return TriangleMesh(v, t)


def generate_sphere_mesh(radius: float, subdivisions: int) -> TriangleMesh:
    """generate_sphere_mesh (mesh.hpp:154-202), bit-identical"""
    return _mesh_from(lib().gk_sphere_mesh, C.c_double(radius), C.c_int(subdivisions))


def generate_plate_mesh(side: float, cells: int) -> TriangleMesh:
    """flat side x side plate, cells x cells grid, two right triangles per cell"""
    return _mesh_from(lib().gk_plate_mesh, C.c_double(side), C.c_int(cells))


def jitter(mesh: TriangleMesh, seed: int, amp: float) -> TriangleMesh:
    """splitmix64(seed) per coordinate, U(-amp, amp)"""
    v = mesh.vertices.copy()
    check(lib().gk_jitter(v.ctypes.data, v.shape[0], seed, amp), "jitter")
    return TriangleMesh(v, mesh.triangles.copy())


def _torch():
    import torch  # plumbing only: device memory + streams

    return torch


@dataclass
class FillOptions:
    """gk_fill_options: the choice between equivalent kernels, per call
    (AUTO = -1 everywhere = the measured best; see include/gk/gk.h)."""

    shared_edges: int = _lib.GK_AUTO      # 0: per-triangle (reference order), 1: forced
    table_placement: int = _lib.GK_AUTO   # 0: GLOBAL (L1/L2), 1: SHARED (staged)
    arith_locate: int = _lib.GK_AUTO
    lossy_phase: int = _lib.GK_AUTO
    unrolled: int = _lib.GK_AUTO
    eval_libdevice: int = _lib.GK_AUTO
    smem_budget: int = 0

    def c(self) -> _lib.FillOptionsC:
        return _lib.FillOptionsC(self.shared_edges, self.table_placement, self.arith_locate,
                                 self.lossy_phase, self.unrolled, self.eval_libdevice,
                                 self.smem_budget)


# gk_fill_path (include/gk/gk.h): the fill kernels of DESIGN.md §5
PATH_NAMES = {1: "direct", 2: "direct_edge", 3: "table_l1", 4: "table_staged",
              5: "table_edge", 6: "table_sweep"}


@dataclass
class MeshOptions:
    """gk_mesh_options: shared-edge block construction at mesh creation."""

    shared_edges: int = _lib.GK_AUTO
    edge_chunks: int = 0                  # 0: 11
    edge_order: int = _lib.GK_AUTO        # 0: mesh order, 1: bisection order
    leaf_pct: int = 0                     # 0: 61
    sweep_chunks: int = 0                 # 0: 2 (the table sweep's block set)

    def c(self) -> _lib.MeshOptionsC:
        return _lib.MeshOptionsC(self.shared_edges, self.edge_chunks, self.edge_order,
                                 self.leaf_pct, self.sweep_chunks)


def _opts(options: FillOptions | None):
    return C.byref(options.c()) if options is not None else None


class Context:
    """One gk_ctx per CUDA device, running on torch's current stream (bound
    again by every launching call, so ``with torch.cuda.stream(s):`` is
    honoured)."""

    _cache: dict[int, "Context"] = {}

    def __init__(self, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.RuntimeErrorGk("no CUDA device: libgk has no CPU fallback")
        self.device = device
        h = C.c_void_p()
        check(lib().gk_ctx_create(device, C.byref(h)), "gk_ctx_create")
        self.h = h

    def __del__(self):
        # tables and meshes hold a reference to their context, so this runs
        # only after they are gone (gk_ctx_destroy's ordering rule)
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            try:
                _lib._lib.gk_ctx_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        """The cached context of `device` (default: torch's current CUDA
        device, i.e. the one torch.cuda.set_device(local_rank) selected),
        bound to torch's current stream."""
        if device is None:
            device = _torch().cuda.current_device()
        if device not in cls._cache:
            cls._cache[device] = cls(device)
        ctx = cls._cache[device]
        ctx.bind_stream()
        return ctx

    def bind_stream(self, stream=None) -> None:
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().gk_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream)), "set_stream")

    def synchronize(self) -> None:
        check(lib().gk_ctx_synchronize(self.h), "synchronize")

    def set_fill_options(self, options: FillOptions | None) -> None:
        """The context's default kernel selection (gk_ctx_set_fill_options):
        used by calls that take no options (fill_matrix, bench_compare,
        eval_batch).  None restores the library defaults."""
        check(lib().gk_ctx_set_fill_options(self.h, _opts(options)), "set_fill_options")

    def fill_check(self) -> int:
        """Synchronise; raise like a synchronous fill if any asynchronous fill
        (report=False) since the last check met r > r_max or r = 0; return and
        reset their accumulated fallback count."""
        fb = C.c_uint64()
        check(lib().gk_fill_check(self.h, C.byref(fb)), "fill_matrix")
        return fb.value

    def fp64_peak_tflops(self) -> float:
        out = C.c_double()
        check(lib().gk_bench_fp64_peak(self.h, C.byref(out)), "fp64_peak")
        return out.value

    def device_info(self) -> dict:
        sm, clk, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().gk_device_info(self.h, C.byref(sm), C.byref(clk), C.byref(ma),
                                   C.byref(mi)), "device_info")
        return {"sm_count": sm.value, "clock_khz": clk.value, "cc": f"{ma.value}.{mi.value}"}


@dataclass
class TableInfo:
    nodes: int
    zeros: int
    hash_buckets: int
    lookup_buckets: int
    r_min: float
    r_max: float
    t: float
    dr_min: float
    inv_dr_min: float
    k: complex
    degree: int
    device_bytes: int
    build_ms: float


class DeviceTable:
    """gktab::KernelEvaluator built on the device (evaluator.hpp:102-309).

    Plan and reference-format hash are bit-identical to build_plan /
    build_hash; Exp uses linear and Green degree-d Lagrange interpolation on
    the reference's stencils; r < r_min falls back to direct evaluation and
    is counted.
    """

    def __init__(self, cfg: SamplingConfig, medium: Medium = Medium(), lagrange_degree: int = 3,
                 ctx: Context | None = None):
        self.ctx = ctx or Context.get()
        self.cfg, self.medium = cfg, medium
        h = C.c_void_p()
        self.ctx.bind_stream()
        check(lib().gk_table_build(self.ctx.h, C.byref(cfg.c()), C.byref(medium.c()),
                                   lagrange_degree, C.byref(h)), "KernelEvaluator")
        self.h = h
        ic = TableInfoC()
        check(lib().gk_table_info_get(self.h, C.byref(ic)), "table_info")
        self.info = TableInfo(ic.nodes, ic.zeros, ic.hash_buckets, ic.lookup_buckets, ic.r_min,
                              ic.r_max, ic.t, ic.dr_min, ic.inv_dr_min,
                              complex(ic.k_re, ic.k_im) if ic.k_im else ic.k_re, ic.degree,
                              ic.device_bytes, ic.build_ms)
        self.fallbacks = 0

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            try:
                _lib._lib.gk_table_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    @property
    def k(self):
        return self.info.k

    def download(self) -> dict:
        """Host copies: abscissae, zero_locations, exp/green node values, buckets."""
        n, nz, nb = self.info.nodes, self.info.zeros, self.info.hash_buckets
        a = np.zeros(n, np.float64)
        z = np.zeros(max(nz, 1), np.float64)
        e = np.zeros(n, np.complex128)
        g = np.zeros(n, np.complex128)
        b = np.zeros(nb, np.uint32)
        check(lib().gk_table_download(self.h, a.ctypes.data, z.ctypes.data, e.ctypes.data,
                                      g.ctypes.data, b.ctypes.data), "download")
        return {"abscissae": a, "zeros": z[:nz], "exp": e, "green": g, "buckets": b,
                "t": self.info.t, "dr_min": self.info.dr_min}

    def dump_table_binary(self, kind: KernelKind, path: str) -> None:
        """The reference's GKTB table dump (io.hpp:77-96) of this device table."""
        check(lib().gk_table_dump_binary(self.h, int(kind), path.encode()), "dump_table_binary")

    def dump_plan_csv(self, path: str) -> None:
        """The reference's plan CSV (io.hpp:60-74) of this device table's plan."""
        check(lib().gk_plan_dump_csv(self.h, path.encode()), "dump_plan_csv")

    def eval_batch(self, kind: KernelKind, radii):
        """KernelEvaluator::eval_batch (evaluator.hpp:209-221) on the device.

        ``radii``: torch CUDA float64 tensor (stays on device) or array-like
        (copied).  Returns a complex128 tensor on the device.
        """
        return eval_batch(kind, radii, table=self, ctx=self.ctx)

    def locate(self, radii):
        """locate (table.hpp:87-102): bracketing interval index per radius (device)."""
        torch = _torch()
        r = _as_device_f64(radii, self.ctx.device)
        out = torch.empty(r.numel(), dtype=torch.int32, device=r.device)
        self.ctx.bind_stream()
        check(lib().gk_locate(self.ctx.h, self.h, r.data_ptr() if r.numel() else None, r.numel(),
                              out.data_ptr() if r.numel() else None), "locate")
        return out

    def error_sweep(self, kind: KernelKind, method: InterpMethod | None = None,
                    probe_count: int = 10000) -> ErrorSweepReport:
        """error_sweep (bounds.hpp:128-186) on the device: the device's methods
        (Exp linear, Green Lagrange) against the device analytic evaluation."""
        if method is None:
            method = InterpMethod.Linear if kind == KernelKind.PlainExp else InterpMethod.Lagrange
        r = _lib.SweepReportC()
        self.ctx.bind_stream()
        check(lib().gk_error_sweep(self.ctx.h, self.h, int(kind), int(method), probe_count,
                                   C.byref(r)), "error_sweep")
        return ErrorSweepReport(r.probe_count, r.max_rel_re, r.max_rel_im, r.max_abs, r.worst_r,
                                r.max_abs_at_exact_zero, list(r.decade_histogram))

    def eval_exp(self, r: float) -> complex:
        return complex(self.eval_batch(KernelKind.PlainExp, [r]).cpu()[0])

    def eval_green(self, r: float) -> complex:
        return complex(self.eval_batch(KernelKind.GreenOverR, [r]).cpu()[0])


def _as_device_f64(x, device: int):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device=f"cuda:{device}", dtype=torch.float64)
    else:
        t = torch.as_tensor(np.ascontiguousarray(x, np.float64), device=f"cuda:{device}")
    return t.contiguous()


def eval_batch(kind: KernelKind, radii, table: DeviceTable | None = None, k: complex = 0.0,
               ctx: Context | None = None):
    """eval_batch with a table, or eval_analytic elementwise (table=None)."""
    torch = _torch()
    ctx = ctx or (table.ctx if table else Context.get())
    r = _as_device_f64(radii, ctx.device)
    out = torch.empty(r.numel(), dtype=torch.complex128, device=r.device)
    fb = C.c_uint64()
    kc = complex(k)
    ctx.bind_stream()
    check(lib().gk_eval_batch(ctx.h, table.h if table else None, int(kind), kc.real, kc.imag,
                              r.data_ptr() if r.numel() else None, r.numel(),
                              out.data_ptr() if r.numel() else None, C.byref(fb)), "eval_batch")
    if table is not None:
        table.fallbacks += fb.value
    return out


def accumulate_batch(kind: KernelKind, radii, weights, table: "DeviceTable | None" = None,
                     k: complex = 0.0, ctx: "Context | None" = None):
    """Kernel::accumulate (matfill.hpp:59-87) for a batch of blocks:
    out[b] = sum_i K(radii[b, i]) weights[b, i], with TableKernel semantics
    (KernelEvaluator::accumulate_green, evaluator.hpp:150-194) when a table is
    given and AnalyticKernel{k} otherwise.  radii/weights: (nblocks, block_len)
    arrays or tensors.  Returns (complex128 CUDA tensor [nblocks], fallbacks)."""
    torch = _torch()
    ctx = ctx or (table.ctx if table else Context.get())
    r = _as_device_f64(radii, ctx.device)
    w = _as_device_f64(weights, ctx.device)
    if r.dim() == 1:
        r, w = r.reshape(1, -1), w.reshape(1, -1)
    if r.shape != w.shape or r.dim() != 2:
        raise _lib.InvalidArgument("accumulate_batch: radii and weights must be (nblocks, len)")
    nb, ln = r.shape
    out = torch.empty(nb, dtype=torch.complex128, device=r.device)
    fb = C.c_uint64()
    kc = complex(k)
    ctx.bind_stream()
    check(lib().gk_accumulate_batch(ctx.h, table.h if table else None, int(kind), kc.real,
                                    kc.imag, r.data_ptr() if r.numel() else None,
                                    w.data_ptr() if w.numel() else None, ln, nb,
                                    out.data_ptr() if nb else None, C.byref(fb)), "accumulate")
    if table is not None:
        table.fallbacks += fb.value
    return out, fb.value


class EvalStatus:
    """Device-resident status of stream-ordered eval_batch calls
    (gk_eval_batch_async): fallback count and the first failing radius."""

    def __init__(self, ctx: Context | None = None):
        torch = _torch()
        self.ctx = ctx or Context.get()
        self.words = torch.empty(2, dtype=torch.int64, device=f"cuda:{self.ctx.device}")
        self.reset()

    def reset(self) -> None:
        self.ctx.bind_stream()
        check(lib().gk_eval_status_reset(self.ctx.h, self.words.data_ptr()), "eval_status")

    def read(self) -> int:
        """Synchronises; raises like eval_batch if any radius was invalid; returns fallbacks."""
        fb = C.c_uint64()
        self.ctx.bind_stream()
        check(lib().gk_eval_status_read(self.ctx.h, self.words.data_ptr(), C.byref(fb)),
              "eval_batch")
        return fb.value


def eval_batch_async(kind: KernelKind, radii, out, status: EvalStatus,
                     table: DeviceTable | None = None, k: complex = 0.0) -> None:
    """Stream-ordered eval_batch into a preallocated complex128 ``out``; errors
    and fallbacks accumulate in ``status`` (no host synchronisation)."""
    ctx = status.ctx
    kc = complex(k)
    n = radii.numel()
    if (out.numel() < n or out.dtype != _torch().complex128 or radii.dtype != _torch().float64
            or not (radii.is_cuda and out.is_cuda) or not (radii.is_contiguous()
                                                           and out.is_contiguous())):
        raise _lib.InvalidArgument("eval_batch_async: contiguous CUDA float64 radii and "
                                   "complex128 out[n]")
    ctx.bind_stream()
    check(lib().gk_eval_batch_async(ctx.h, table.h if table else None, int(kind), kc.real, kc.imag,
                                    radii.data_ptr() if n else None, n,
                                    out.data_ptr() if n else None, status.words.data_ptr()),
          "eval_batch")


def edge_blocks_plan(mesh: TriangleMesh, chunks: int = 11, order_mode: int = -1,
                     leaf_pct: int = 0, rho_cap: float = 0.0) -> dict:
    """The host part of the shared-edge blocks (gk_edge_blocks_plan; no
    device needed): block positions, triangle order and block-local edge
    indices."""
    nt = mesh.triangle_count()
    order = np.zeros(nt, np.uint32)
    eidx = np.zeros((nt, 3), np.uint32)
    start = np.zeros(nt + 1, np.uint32)
    nedge = np.zeros(nt, np.uint32)
    nb = C.c_uint64()
    ordered = C.c_int()
    check(lib().gk_edge_blocks_plan(mesh.vertices.ctypes.data, mesh.vertices.shape[0],
                                    mesh.triangles.ctypes.data, nt, chunks, order_mode,
                                    leaf_pct, rho_cap, order.ctypes.data, eidx.ctypes.data,
                                    start.ctypes.data,
                                    nedge.ctypes.data, C.byref(nb), C.byref(ordered)),
          "edge_blocks_plan")
    n = nb.value
    return dict(order=order, edge_index=eidx, block_start=np.append(start[:n], nt),
                block_edges=nedge[:n], ordered=bool(ordered.value))


class DeviceMesh:
    """A mesh resident on the device with its quadrature points (K0)."""

    def __init__(self, mesh: TriangleMesh, spec: QuadratureSpec, ctx: Context | None = None,
                 options: MeshOptions | None = None):
        self.ctx = ctx or Context.get()
        self.ctx.bind_stream()
        self.mesh, self.spec = mesh, spec
        h = C.c_void_p()
        check(lib().gk_mesh_create_ex(self.ctx.h, mesh.vertices.ctypes.data,
                                      mesh.vertices.shape[0], mesh.triangles.ctypes.data,
                                      mesh.triangles.shape[0], spec.outer_points,
                                      spec.inner_points_per_edge,
                                      C.byref(options.c()) if options is not None else None,
                                      C.byref(h)),
              "fill_matrix")
        self.h = h
        self.N = mesh.triangle_count()

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            try:
                _lib._lib.gk_mesh_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def points(self):
        """(outer[4][N m], inner[4][N 3n]) in the reference's SoA order"""
        m, n = self.spec.outer_points, self.spec.inner_points_per_edge
        o = np.zeros((4, self.N * m), np.float64)
        i = np.zeros((4, self.N * 3 * n), np.float64)
        check(lib().gk_mesh_points_download(self.h, o.ctypes.data, i.ctypes.data), "points")
        return o, i

    def edge_info(self) -> dict:
        """Shared-edge blocks of the direct fill (gk_mesh_edge_info_get)."""
        out = (C.c_double * 13)()
        check(lib().gk_mesh_edge_info_get(self.h, C.cast(out, C.c_void_p)), "edge_info")
        raw = bytes(out)
        rho_max = np.frombuffer(raw[64:72], np.float64)[0]
        s_blocks, s_slots = np.frombuffer(raw[72:88], np.uint64)
        s_ratio, s_rho = np.frombuffer(raw[88:104], np.float64)
        blocks, slots = np.frombuffer(raw[:16], np.uint64)
        ratio, delta, r_far = np.frombuffer(raw[16:40], np.float64)
        edges = np.frombuffer(raw[40:48], np.uint64)[0]
        rho = np.frombuffer(raw[48:56], np.float64)[0]
        ordered = np.frombuffer(raw[56:60], np.int32)[0]
        return dict(blocks=int(blocks), edge_slots=int(slots), work_ratio=float(ratio),
                    delta=float(delta), r_far=float(r_far), edges=int(edges),
                    rho_mean=float(rho), ordered=bool(ordered), rho_max=float(rho_max),
                    sweep=dict(blocks=int(s_blocks), edge_slots=int(s_slots),
                               work_ratio=float(s_ratio), rho_max=float(s_rho)))

    def max_vertex_distance(self) -> float:
        """max_vertex_distance (mesh.hpp:62-68), exact, on the device."""
        out = C.c_double()
        self.ctx.bind_stream()
        check(lib().gk_max_vertex_distance(self.ctx.h, self.h, C.byref(out)),
              "max_vertex_distance")
        return out.value

    def distance_range(self, row_begin: int = 0, row_end: int | None = None):
        """K1: min/max quadrature pair distance over rows x all q != p"""
        row_end = self.N if row_end is None else row_end
        lo, hi = C.c_double(), C.c_double()
        self.ctx.bind_stream()
        check(lib().gk_distance_range(self.ctx.h, self.h, row_begin, row_end, C.byref(lo),
                                      C.byref(hi)), "distance_range")
        return lo.value, hi.value


def fill_rows(dmesh: DeviceMesh, mode: Mode, kind: KernelKind = KernelKind.GreenOverR,
              table: DeviceTable | None = None, k: complex = 0.0, row_begin: int = 0,
              row_end: int | None = None, out=None, report: bool = True,
              options: FillOptions | None = None):
    """fill_rows (matfill.hpp:169-203) for rows [row_begin,row_end) on the device.

    Returns (Z, FillReport | None); Z is a (rows, N) complex128 CUDA tensor.
    ``report=False`` launches asynchronously on the current stream.
    ``options`` chooses between equivalent kernels (None: the context's).
    """
    torch = _torch()
    ctx = dmesh.ctx
    ctx.bind_stream()
    N = dmesh.N
    row_end = N if row_end is None else row_end
    rows = row_end - row_begin
    if out is None:
        out = torch.empty((rows, N), dtype=torch.complex128, device=f"cuda:{ctx.device}")
    if not (out.dtype == torch.complex128 and out.is_cuda and out.dim() == 2
            and out.stride(1) == 1 and out.shape[0] >= rows and out.shape[1] >= N
            and (rows <= 1 or out.stride(0) >= N)):
        raise _lib.InvalidArgument(
            f"fill_rows: out must be a CUDA complex128 ({rows}, >= {N}) view with unit "
            f"column stride (got {tuple(out.shape)}, {out.dtype})")
    kc = complex(k)
    rep = FillReportC()
    check(lib().gk_fill_rows(ctx.h, dmesh.h, int(mode), table.h if table else None, int(kind),
                             kc.real, kc.imag, row_begin, row_end,
                             out.data_ptr() if rows else None, out.stride(0) if rows else N,
                             _opts(options), C.byref(rep) if report else None), "fill_matrix")
    return out, (FillReport.from_c(rep) if report else None)


def compare_fills(test, ref, row_begin: int = 0, ctx: Context | None = None):
    """compare_fills (matfill.hpp:237-254) on device matrices: (max_rel_re,
    max_rel_im) over the rows given, skipping the diagonal (row index
    row_begin + r == column) and exactly-zero reference components."""
    torch = _torch()
    if test.shape != ref.shape:
        raise _lib.InvalidArgument("compare_fills: size mismatch")
    ctx = ctx or Context.get(test.device.index or 0)
    t = test.contiguous()
    r = ref.contiguous()
    rows, N = (t.shape[0], t.shape[1]) if t.dim() == 2 else (0, 0)
    assert t.dtype == r.dtype == torch.complex128 and t.is_cuda and r.is_cuda
    re, im = C.c_double(), C.c_double()
    ctx.bind_stream()
    check(lib().gk_compare_fills(ctx.h, t.data_ptr() if t.numel() else None,
                                 r.data_ptr() if r.numel() else None, rows, N, row_begin,
                                 max(N, 1), C.byref(re), C.byref(im)), "compare_fills")
    return re.value, im.value


def bench_compare(mesh: TriangleMesh, spec: QuadratureSpec, medium: Medium = Medium(),
                  cfg: SamplingConfig | None = None, lagrange_degree: int = 3,
                  kind: KernelKind = KernelKind.GreenOverR, repeats: int = 1,
                  ctx: Context | None = None) -> FillReport:
    """bench_compare (matfill.hpp:262-294) on the device (gk_bench_compare):
    direct fill, then the table fill over a plan with r_max = 1.01 x
    max_vertex_distance (cfg.r_min kept), the table build charged to the
    table side; with repeats > 1 the fills interleave and the fastest device
    time per side counts."""
    ctx = ctx or Context.get()
    cfg = cfg or SamplingConfig()
    r = _lib.BenchReportC()
    ctx.bind_stream()
    check(lib().gk_bench_compare(ctx.h, mesh.vertices.ctypes.data, mesh.vertices.shape[0],
                                 mesh.triangles.ctypes.data, mesh.triangles.shape[0],
                                 spec.outer_points, spec.inner_points_per_edge,
                                 C.byref(medium.c()), C.byref(cfg.c()), lagrange_degree,
                                 int(kind), repeats, C.byref(r)), "bench_compare")
    rep = FillReport.from_c(r.fill)
    rep.max_rel_re, rep.max_rel_im = r.max_rel_re, r.max_rel_im
    rep.speedup, rep.analytic_time_s = r.speedup, r.analytic_time_s
    rep.interp_time_s, rep.table_build_s = r.interp_time_s, r.table_build_s
    return rep


def fill_rows_pair(dmesh: DeviceMesh, mode: Mode, table: DeviceTable | None = None,
                   k: complex = 0.0, row_begin: int = 0, row_end: int | None = None,
                   report: bool = True, options: FillOptions | None = None):
    """Fused Exp + Green fill sharing r (and the table lookup): returns
    (Z_exp, Z_green, FillReport) with each matrix identical to its separate fill."""
    torch = _torch()
    ctx = dmesh.ctx
    ctx.bind_stream()
    N = dmesh.N
    row_end = N if row_end is None else row_end
    rows = row_end - row_begin
    ze = torch.empty((rows, N), dtype=torch.complex128, device=f"cuda:{ctx.device}")
    zg = torch.empty_like(ze)
    kc = complex(k)
    rep = FillReportC()
    check(lib().gk_fill_rows_pair(ctx.h, dmesh.h, int(mode), table.h if table else None, kc.real,
                                  kc.imag, row_begin, row_end, ze.data_ptr() if rows else None,
                                  zg.data_ptr() if rows else None, N, _opts(options),
                                  C.byref(rep) if report else None), "fill_matrix")
    return ze, zg, (FillReport.from_c(rep) if report else None)


def fill_rows_host(dmesh: DeviceMesh, mode: Mode, out: np.ndarray,
                   kind: KernelKind = KernelKind.GreenOverR, table: DeviceTable | None = None,
                   k: complex = 0.0, row_begin: int = 0, row_end: int | None = None,
                   options: FillOptions | None = None) -> FillReport:
    """fill_rows straight into host memory (``out``: (rows, N) complex128, C order;
    pinned memory gets full PCIe bandwidth).  Chunked + double-buffered."""
    ctx = dmesh.ctx
    ctx.bind_stream()
    N = dmesh.N
    row_end = N if row_end is None else row_end
    assert out.dtype == np.complex128 and out.flags.c_contiguous and out.shape[1] == N
    assert out.shape[0] >= row_end - row_begin
    kc = complex(k)
    rep = FillReportC()
    check(lib().gk_fill_rows_host(ctx.h, dmesh.h, int(mode), table.h if table else None,
                                  int(kind), kc.real, kc.imag, row_begin, row_end,
                                  out.ctypes.data, N, _opts(options), C.byref(rep)),
          "fill_matrix")
    return FillReport.from_c(rep)


def fill_matrix(mesh: TriangleMesh, spec: QuadratureSpec, mode: Mode, medium: Medium = Medium(),
                cfg: SamplingConfig | None = None, kind: KernelKind = KernelKind.GreenOverR,
                ctx: Context | None = None, out: np.ndarray | None = None):
    """fill_matrix<Kernel> (matfill.hpp:144-228) end to end from host buffers.

    TABLE mode: ``cfg.r_min/r_max <= 0`` selects the device-computed pair
    distance range (K1).  Returns (Z as a host complex128 (N,N) array, report).
    """
    ctx = ctx or Context.get()
    N = mesh.triangle_count()
    z = out if out is not None else np.empty((N, N), np.complex128)
    assert z.dtype == np.complex128 and z.flags.c_contiguous and z.shape == (N, N)
    rep = FillReportC()
    cfg_c = (cfg or SamplingConfig(r_min=0.0, r_max=0.0)).c()
    ctx.bind_stream()
    check(lib().gk_fill_matrix_host(ctx.h, mesh.vertices.ctypes.data, mesh.vertices.shape[0],
                                    mesh.triangles.ctypes.data, N, spec.outer_points,
                                    spec.inner_points_per_edge, int(mode), C.byref(cfg_c),
                                    C.byref(medium.c()), int(kind), z.ctypes.data,
                                    C.byref(rep)), "fill_matrix")
    return z, FillReport.from_c(rep)
