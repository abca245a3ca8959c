"""ctypes binding of libgk.so (the C ABI declared in include/gk/gk.h).

The library is built in-tree (``python -m paper_1901_04162_b200.build``) and
loaded from this package directory only; a missing library is an error, never
a silent fallback.
"""
from __future__ import annotations

import ctypes as C
import os

# GK_LIB: an alternative in-tree build of the same library (kernel A/B
# experiments, scripts/build_variant.sh); default: the package's libgk.so
LIB_PATH = os.environ.get("GK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "libgk.so")

GK_OK = 0


class GkError(RuntimeError):
    """Base of the status-code exceptions (gk_status != GK_OK)."""

    status = 5


class InvalidArgument(GkError, ValueError):
    """std::invalid_argument"""

    status = 1


class DomainError(GkError, ArithmeticError):
    """std::domain_error"""

    status = 2


class OutOfRange(GkError, IndexError):
    """std::out_of_range"""

    status = 3


class OverflowErrorGk(GkError, OverflowError):
    """std::overflow_error"""

    status = 4


class RuntimeErrorGk(GkError):
    """std::runtime_error / CUDA failure"""

    status = 5


_BY_STATUS = {1: InvalidArgument, 2: DomainError, 3: OutOfRange, 4: OverflowErrorGk,
              5: RuntimeErrorGk}


class Medium(C.Structure):
    _fields_ = [("lambda0", C.c_double), ("eps_r", C.c_double), ("mu_r", C.c_double),
                ("eps_r_im", C.c_double)]


class SamplingConfigC(C.Structure):
    _fields_ = [("r_min", C.c_double), ("r_max", C.c_double),
                ("samples_per_wavelength", C.c_int), ("refine_interval_divisor", C.c_int),
                ("refine_halfwidth_in_t", C.c_double), ("dedup_fraction", C.c_double),
                ("refine", C.c_int)]


class FillReportC(C.Structure):
    _fields_ = [("N", C.c_uint64), ("m", C.c_int), ("n", C.c_int),
                ("predicted_calls", C.c_uint64), ("actual_calls", C.c_uint64),
                ("fallback_calls", C.c_uint64), ("wall_time_s", C.c_double),
                ("evaluations", C.c_uint64), ("path", C.c_int)]


GK_AUTO = -1
GK_TABLE_GLOBAL, GK_TABLE_SHARED, GK_TABLE_SWEEP = 0, 1, 2


class FillOptionsC(C.Structure):
    """gk_fill_options (include/gk/gk.h): kernel selection per call."""
    _fields_ = [("shared_edges", C.c_int), ("table_placement", C.c_int),
                ("arith_locate", C.c_int), ("lossy_phase", C.c_int), ("unrolled", C.c_int),
                ("eval_libdevice", C.c_int), ("smem_budget", C.c_uint64)]


class MeshOptionsC(C.Structure):
    """gk_mesh_options (include/gk/gk.h): shared-edge block construction."""
    _fields_ = [("shared_edges", C.c_int), ("edge_chunks", C.c_int), ("edge_order", C.c_int),
                ("leaf_pct", C.c_int), ("sweep_chunks", C.c_int)]


class SweepReportC(C.Structure):
    _fields_ = [("probe_count", C.c_uint64), ("max_rel_re", C.c_double),
                ("max_rel_im", C.c_double), ("max_abs", C.c_double), ("worst_r", C.c_double),
                ("max_abs_at_exact_zero", C.c_double), ("decade_histogram", C.c_uint64 * 24)]


class BenchReportC(C.Structure):
    _fields_ = [("fill", FillReportC), ("max_rel_re", C.c_double), ("max_rel_im", C.c_double),
                ("speedup", C.c_double), ("analytic_time_s", C.c_double),
                ("interp_time_s", C.c_double), ("table_build_s", C.c_double)]


class TableInfoC(C.Structure):
    _fields_ = [("nodes", C.c_uint64), ("zeros", C.c_uint64), ("hash_buckets", C.c_uint64),
                ("lookup_buckets", C.c_uint64), ("r_min", C.c_double), ("r_max", C.c_double),
                ("t", C.c_double), ("dr_min", C.c_double), ("inv_dr_min", C.c_double),
                ("k_re", C.c_double), ("k_im", C.c_double), ("degree", C.c_int),
                ("device_bytes", C.c_uint64), ("build_ms", C.c_double)]


_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)

# name -> argtypes (restype gk_status = int unless noted)
PROTOTYPES = {
    "gk_ctx_create": [C.c_int, C.POINTER(_vp)],
    "gk_ctx_destroy": [_vp],
    "gk_ctx_set_stream": [_vp, _vp],
    "gk_ctx_use_own_stream": [_vp],
    "gk_ctx_synchronize": [_vp],
    "gk_ctx_set_fill_options": [_vp, C.POINTER(FillOptionsC)],
    "gk_wavenumber": [C.POINTER(Medium), _dp, _dp],
    "gk_table_build": [_vp, C.POINTER(SamplingConfigC), C.POINTER(Medium), C.c_int,
                       C.POINTER(_vp)],
    "gk_table_info_get": [_vp, C.POINTER(TableInfoC)],
    "gk_table_download": [_vp, _vp, _vp, _vp, _vp, _vp],
    "gk_table_destroy": [_vp],
    "gk_table_dump_binary": [_vp, C.c_int, C.c_char_p],
    "gk_plan_dump_csv": [_vp, C.c_char_p],
    "gk_eval_batch": [_vp, _vp, C.c_int, C.c_double, C.c_double, _vp, C.c_size_t, _vp, _u64p],
    "gk_eval_batch_async": [_vp, _vp, C.c_int, C.c_double, C.c_double, _vp, C.c_size_t, _vp, _vp],
    "gk_eval_status_reset": [_vp, _vp],
    "gk_eval_status_read": [_vp, _vp, _u64p],
    "gk_locate": [_vp, _vp, _vp, C.c_size_t, _vp],
    "gk_eval_batch_host": [_vp, _vp, C.c_int, C.c_double, C.c_double, _vp, C.c_size_t, _vp,
                           _u64p],
    "gk_mesh_create": [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_int, C.c_int, C.POINTER(_vp)],
    "gk_mesh_create_ex": [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_int, C.c_int,
                          C.POINTER(MeshOptionsC), C.POINTER(_vp)],
    "gk_mesh_points_download": [_vp, _vp, _vp],
    "gk_mesh_destroy": [_vp],
    "gk_mesh_edge_info_get": [_vp, _vp],
    "gk_edge_blocks_plan": [_vp, C.c_size_t, _vp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                            C.c_double, _vp, _vp, _vp,
                            _vp, _u64p, C.POINTER(C.c_int)],
    "gk_distance_range": [_vp, _vp, C.c_size_t, C.c_size_t, _dp, _dp],
    "gk_fill_rows": [_vp, _vp, C.c_int, _vp, C.c_int, C.c_double, C.c_double, C.c_size_t,
                     C.c_size_t, _vp, C.c_size_t, C.POINTER(FillOptionsC),
                     C.POINTER(FillReportC)],
    "gk_fill_rows_pair": [_vp, _vp, C.c_int, _vp, C.c_double, C.c_double, C.c_size_t,
                          C.c_size_t, _vp, _vp, C.c_size_t, C.POINTER(FillOptionsC),
                          C.POINTER(FillReportC)],
    "gk_fill_matrix_host": [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                            C.POINTER(SamplingConfigC), C.POINTER(Medium), C.c_int, _vp,
                            C.POINTER(FillReportC)],
    "gk_fill_rows_host": [_vp, _vp, C.c_int, _vp, C.c_int, C.c_double, C.c_double, C.c_size_t,
                          C.c_size_t, _vp, C.c_size_t, C.POINTER(FillOptionsC),
                          C.POINTER(FillReportC)],
    "gk_predicted_calls": [C.c_uint64, C.c_uint64, C.c_uint64, _u64p],
    "gk_rows_of": [C.c_uint64, C.c_int, C.c_int, _u64p, _u64p],
    "gk_comm_unique_id": [_vp],
    "gk_comm_init": [_vp, _vp, C.c_int, C.c_int, C.POINTER(_vp)],
    "gk_comm_init_all": [_vp, C.c_int, _vp],
    "gk_comm_destroy": [_vp],
    "gk_comm_info": [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "gk_distance_range_global": [_vp, _vp, _vp, _dp, _dp],
    "gk_fill_sharded": [_vp, _vp, _vp, C.c_int, C.POINTER(SamplingConfigC), C.POINTER(Medium),
                        C.c_int, _vp, C.c_size_t, C.POINTER(FillOptionsC),
                        C.POINTER(FillReportC), _dp],
    "gk_gather_rows": [_vp, _vp, _vp, C.c_uint64, C.c_int, _vp],
    "gk_compare_fills": [_vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp],
    "gk_max_vertex_distance": [_vp, _vp, _dp],
    "gk_error_sweep": [_vp, _vp, C.c_int, C.c_int, C.c_uint64, _vp],
    "gk_fill_check": [_vp, _u64p],
    "gk_accumulate_batch": [_vp, _vp, C.c_int, C.c_double, C.c_double, _vp, _vp, C.c_size_t,
                            C.c_size_t, _vp, _u64p],
    "gk_accumulate_batch_host": [_vp, _vp, C.c_int, C.c_double, C.c_double, _vp, _vp,
                                 C.c_size_t, C.c_size_t, _vp, _u64p],
    "gk_shared_alloc": [_vp, C.c_size_t, C.POINTER(C.c_void_p), _vp],
    "gk_shared_free": [_vp, _vp],
    "gk_ipc_open": [_vp, _vp, C.POINTER(C.c_void_p)],
    "gk_ipc_close": [_vp, _vp],
    "gk_bench_compare": [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_int, C.c_int, _vp, _vp,
                         C.c_int, C.c_int, C.c_int, _vp],
    "gk_sphere_mesh": [C.c_double, C.c_int, _vp, _szp, _vp, _szp],
    "gk_plate_mesh": [C.c_double, C.c_int, _vp, _szp, _vp, _szp],
    "gk_jitter": [_vp, C.c_size_t, C.c_uint64, C.c_double],
    "gk_bench_fp64_peak": [_vp, _dp],
    "gk_device_info": [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                       C.POINTER(C.c_int)],
}
VOID_PROTOTYPES = {
    "gk_fill_options_init": [C.POINTER(FillOptionsC)],
    "gk_mesh_options_init": [C.POINTER(MeshOptionsC)],
}
EXPORTS = sorted(PROTOTYPES) + sorted(VOID_PROTOTYPES) + [
    "gk_abi_version", "gk_last_error", "gk_launch_count"]

_lib = None


def lib() -> C.CDLL:
    """Load libgk.so from the package directory (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1901_04162_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, args in PROTOTYPES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, args in VOID_PROTOTYPES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = None
    L.gk_launch_count.restype = C.c_uint64
    L.gk_launch_count.argtypes = []
    L.gk_abi_version.restype = C.c_int
    L.gk_abi_version.argtypes = []
    L.gk_last_error.restype = C.c_char_p
    L.gk_last_error.argtypes = []
    _lib = L
    return L


def check(status: int, where: str = "") -> None:
    if status == GK_OK:
        return
    msg = lib().gk_last_error().decode(errors="replace")
    cls = _BY_STATUS.get(status, RuntimeErrorGk)
    raise cls(f"{where}: {msg}" if where else msg)
