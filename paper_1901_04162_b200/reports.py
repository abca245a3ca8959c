"""Report writers of the reference (io.hpp:134-156), byte for byte.

``write_bench_csv`` renders a FillReport from ``bench_compare`` and
``write_sweep_csv_header`` / ``write_sweep_csv_row`` an ErrorSweepReport,
with the reference's %.17g number format (io.hpp:23-27), so reports from
the device path diff cleanly against the reference's own.
"""
from __future__ import annotations

from .gktab import ErrorSweepReport, FillReport, InterpMethod, KernelKind


def format_g17(v: float) -> str:
    """detail::format_g17 (io.hpp:23-27): snprintf("%.17g")"""
    return "%.17g" % v


def kernel_name(kind: KernelKind) -> str:
    """kernel_name (kernel.hpp:19-21)"""
    return "exp" if kind == KernelKind.PlainExp else "green"


def method_name(method: InterpMethod) -> str:
    """method_name (bounds.hpp:17-19)"""
    return "linear" if method == InterpMethod.Linear else "lagrange"


def write_bench_csv(out, rep: FillReport) -> None:
    """write_bench_csv (io.hpp:147-156): header + one row"""
    out.write("N,m,n,predicted_calls,actual_calls,fallback_calls,analytic_s,interp_s,speedup,"
              "max_rel_re,max_rel_im\n")
    out.write(f"{rep.N},{rep.m},{rep.n},{rep.predicted_calls},{rep.actual_calls},"
              f"{rep.fallback_calls},{format_g17(rep.analytic_time_s)},"
              f"{format_g17(rep.interp_time_s)},{format_g17(rep.speedup)},"
              f"{format_g17(rep.max_rel_re)},{format_g17(rep.max_rel_im)}\n")


def write_sweep_csv_header(out) -> None:
    """write_sweep_csv_header (io.hpp:134-136)"""
    out.write("kernel,method,probes,max_rel_re,max_rel_im,max_abs,worst_r\n")


def write_sweep_csv_row(out, kind: KernelKind, method: InterpMethod, lagrange_degree: int,
                        rep: ErrorSweepReport) -> None:
    """write_sweep_csv_row (io.hpp:138-145)"""
    m = method_name(method) + (str(lagrange_degree) if method == InterpMethod.Lagrange else "")
    out.write(f"{kernel_name(kind)},{m},{rep.probe_count},{format_g17(rep.max_rel_re)},"
              f"{format_g17(rep.max_rel_im)},{format_g17(rep.max_abs)},"
              f"{format_g17(rep.worst_r)}\n")
