#!/usr/bin/env python3
"""Run one fill launch of a configuration (for ncu): warm-up launch + one
profiled launch.  Usage: profile_fill.py CONFIG MODE [ROWS] [S]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
mode = sys.argv[2]
rows = int(sys.argv[3]) if len(sys.argv) > 3 else 0
S = int(sys.argv[4]) if len(sys.argv) > 4 else 10000
mesh = bench.make_mesh(gk, cfg)
N = mesh.triangle_count()
rows = rows or N
dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]))
med = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0), eps_r_im=cfg.get("eps_r_im", 0.0))
k = gk.wavenumber(med)
t = None
opts = None
if mode in ("sweep", "tedge"):  # the table through the sweep (K3s) / K3e
    opts = gk.FillOptions(table_placement=gk.GK_TABLE_SWEEP if mode == "sweep" else gk.GK_TABLE_GLOBAL)
    mode = "table"
if mode == "table":
    lo, hi = dm.distance_range()
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
Z = torch.empty((rows, N), dtype=torch.complex128, device="cuda")
for _ in range(2):
    if mode == "pair":
        del Z
        _, _, rep = gk.fill_rows_pair(dm, gk.Mode.DIRECT, k=k, row_end=rows)
        Z = None
    else:
        z, rep = gk.fill_rows(dm, gk.Mode.TABLE if t else gk.Mode.DIRECT, table=t, k=k,
                              row_end=rows, out=Z, options=opts)
print(f"{sys.argv[1]} {mode} {rep.path_name} rows={rows} N={N} fill {rep.wall_time_s*1e3:.3f} ms "
      f"{rep.actual_calls / rep.wall_time_s:.3e} evals/s fallbacks={rep.fallback_calls}")
