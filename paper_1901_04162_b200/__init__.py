"""B200-native (sm_100a) MoM triangle-pair Green-function fill, arXiv 1901.04162.

Drop-in for the reference ``gktab`` fill hot path: device table build,
table lookup/evaluation, direct evaluation and the triangle-pair fill driver,
all in hand-written CUDA (libgk.so, C ABI in include/gk/gk.h).
"""
from .gktab import (Context, DeviceMesh, DeviceTable, ErrorSweepReport, EvalStatus, FillOptions,
                    FillReport, MeshOptions,
                    InterpMethod, KernelKind, Medium, Mode, QuadratureSpec, SamplingConfig,
                    TriangleMesh, accumulate_batch, bench_compare, compare_fills, edge_blocks_plan,
                    eval_batch,
                    eval_batch_async, fill_matrix, fill_rows, fill_rows_host, fill_rows_pair,
                    generate_plate_mesh, generate_sphere_mesh, jitter, predicted_calls,
                    wavenumber)
from ._lib import (GK_AUTO, GK_TABLE_GLOBAL, GK_TABLE_SHARED, GK_TABLE_SWEEP, DomainError, GkError,
                   InvalidArgument, OutOfRange, OverflowErrorGk, RuntimeErrorGk, LIB_PATH)

__all__ = [
    "Context", "DeviceMesh", "DeviceTable", "ErrorSweepReport", "EvalStatus", "FillOptions",
    "FillReport", "MeshOptions", "GK_AUTO", "GK_TABLE_GLOBAL", "GK_TABLE_SHARED", "GK_TABLE_SWEEP",
    "InterpMethod", "KernelKind", "Medium", "Mode", "QuadratureSpec", "SamplingConfig",
    "TriangleMesh", "accumulate_batch", "bench_compare", "compare_fills", "edge_blocks_plan",
    "eval_batch",
    "eval_batch_async", "fill_matrix", "fill_rows", "fill_rows_host", "fill_rows_pair",
    "generate_plate_mesh", "generate_sphere_mesh", "jitter", "predicted_calls", "wavenumber",
    "DomainError", "GkError", "InvalidArgument", "OutOfRange", "OverflowErrorGk",
    "RuntimeErrorGk", "LIB_PATH",
]
