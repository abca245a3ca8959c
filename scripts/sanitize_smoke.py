#!/usr/bin/env python3
"""Small end-to-end exercise of every device entry point, for compute-sanitizer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_04162_b200 as gk  # noqa: E402

mesh = gk.jitter(gk.generate_sphere_mesh(1.0, 2), 1901, 1e-3)
for m, n in ((6, 4), (7, 5), (3, 7)):
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(m, n))
    lo, hi = dm.distance_range()
    for S in (1000, 10000):
        t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S))
        for kind in (gk.KernelKind.GreenOverR, gk.KernelKind.PlainExp):
            gk.fill_rows(dm, gk.Mode.TABLE, kind=kind, table=t, row_begin=3, row_end=250)
        gk.fill_rows_pair(dm, gk.Mode.TABLE, table=t)
        r = np.linspace(lo * 0.5, hi, 5000)
        t.eval_batch(gk.KernelKind.GreenOverR, r)
        t.locate(np.linspace(lo, hi, 777))
    for kind in (gk.KernelKind.GreenOverR, gk.KernelKind.PlainExp):
        gk.fill_rows(dm, gk.Mode.DIRECT, kind=kind, k=2 * np.pi)
    gk.fill_rows_pair(dm, gk.Mode.DIRECT, k=2 * np.pi, row_begin=10, row_end=17)
    z = np.zeros((40, dm.N), np.complex128)
    gk.fill_rows_host(dm, gk.Mode.DIRECT, z, k=2 * np.pi, row_begin=100, row_end=140)
plate = gk.generate_plate_mesh(1.0, 6)
med = gk.Medium(1.0, 4.0, 1.0, -0.4)
gk.fill_matrix(plate, gk.QuadratureSpec(6, 4), gk.Mode.DIRECT, med)
gk.fill_matrix(plate, gk.QuadratureSpec(6, 4), gk.Mode.TABLE, med)
gk.DeviceTable(gk.SamplingConfig(samples_per_wavelength=20, refine_halfwidth_in_t=3.0))  # sequential plan
gk.DeviceTable(gk.SamplingConfig(refine=False))
gk.eval_batch(gk.KernelKind.GreenOverR, np.linspace(0.01, 2, 1000), k=3.0)
print("sanitize_smoke: done")
