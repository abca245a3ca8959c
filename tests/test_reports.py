"""Report writers (paper_1901_04162_b200.reports) byte-identical to the
reference's io.hpp:134-156 (write_bench_csv, write_sweep_csv_header/_row),
checked against the reference compiled in place (oracle/_ref)."""
import io

import numpy as np
import pytest

CASES = [
    ((80, 4, 3, 76800, 75840, 0), (0.0123, 0.0045, 2.7333333333333334, 1.39e-11, 2.1e-11)),
    ((20, 4, 3, 14400, 13680, 0), (0.1, 1 / 3, 3.0000000000000004, 0.0, 5e-324)),
    ((81920, 6, 4, 483183820800, 483177922560, 17), (123456789.123, 1e-17, 1e300, float("inf"),
                                                    -0.0)),
]


@pytest.mark.parametrize("ints,dbls", CASES)
def test_write_bench_csv_matches_reference(ref, tmp_path, ints, dbls):
    from paper_1901_04162_b200.gktab import FillReport
    from paper_1901_04162_b200.reports import write_bench_csv
    rep = FillReport(N=ints[0], m=ints[1], n=ints[2], predicted_calls=ints[3],
                     actual_calls=ints[4], fallback_calls=ints[5], analytic_time_s=dbls[0],
                     interp_time_s=dbls[1], speedup=dbls[2], max_rel_re=dbls[3],
                     max_rel_im=dbls[4])
    buf = io.StringIO()
    write_bench_csv(buf, rep)
    path = str(tmp_path / "bench.csv")
    ref.write_bench_csv(ints, dbls, path)
    assert buf.getvalue().encode() == open(path, "rb").read()


@pytest.mark.parametrize("kind,method,degree", [(0, 0, 3), (1, 1, 3), (1, 1, 5), (0, 1, 2),
                                                (1, 0, 3)])
def test_write_sweep_csv_matches_reference(ref, tmp_path, kind, method, degree):
    from paper_1901_04162_b200.gktab import ErrorSweepReport, InterpMethod, KernelKind
    from paper_1901_04162_b200.reports import write_sweep_csv_header, write_sweep_csv_row
    rng = np.random.default_rng(kind * 10 + method + degree)
    d = [float(x) for x in rng.uniform(0, 1, 4) * np.array([1e-6, 1e-9, 1e-3, 2.0])]
    rep = ErrorSweepReport(probe_count=10000, max_rel_re=d[0], max_rel_im=d[1], max_abs=d[2],
                           worst_r=d[3])
    buf = io.StringIO()
    write_sweep_csv_header(buf)
    write_sweep_csv_row(buf, KernelKind(kind), InterpMethod(method), degree, rep)
    path = str(tmp_path / "sweep.csv")
    ref.write_sweep_csv(kind, method, degree, 10000, d, path)
    assert buf.getvalue().encode() == open(path, "rb").read()
