#!/usr/bin/env python3
"""A/B of the shared-edge table fill (K3e) against the per-triangle table
kernels (FillOptions(shared_edges=0)) on the bench configurations, at S = 10^3 and 10^4.
Usage: table_edge_ab.py [c3 c4 c5] [--rows R]"""
import os  # noqa: F401
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402


def fill(dm, t, rows, Z, opts, reps=2):
    best = None
    for _ in range(reps):
        _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, row_end=rows, out=Z, options=opts)
        best = rep if best is None or rep.wall_time_s < best.wall_time_s else best
    return best


def main():
    names = [a for a in sys.argv[1:] if a.startswith("c")] or ["c3", "c4", "c5"]
    rows_arg = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 0
    for name in names:
        cfg = bench.CONFIGS[name]
        mesh = bench.make_mesh(gk, cfg)
        N = mesh.triangle_count()
        rows = rows_arg or (N if N <= 20480 else 4096)
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]))
        med = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0),
                        eps_r_im=cfg.get("eps_r_im", 0.0))
        lo, hi = dm.distance_range()
        Za = torch.empty((rows, N), dtype=torch.complex128, device="cuda")
        Zb = torch.empty_like(Za)
        for S in (1000, 10000):
            t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
            ra = fill(dm, t, rows, Za, gk.FillOptions(shared_edges=0))
            rb = fill(dm, t, rows, Zb, gk.FillOptions())
            rf = None
            if "--forced" in sys.argv:  # K3e also where the table is staged in shared memory
                rf = fill(dm, t, rows, Zb, gk.FillOptions(table_placement=gk.GK_TABLE_GLOBAL))
            rel = ((Zb - Za).abs() / Za.abs().clamp_min(1e-300)).max().item()
            print(f"{name} S={S} rows={rows} per-triangle {ra.wall_time_s * 1e3:.2f} ms, "
                  f"edge {rb.wall_time_s * 1e3:.2f} ms (x{ra.wall_time_s / rb.wall_time_s:.3f}); "
                  f"evaluations {rb.evaluations / rb.actual_calls:.4f}; fallbacks "
                  f"{ra.fallback_calls}/{rb.fallback_calls}; max |dZ|/|Z| = {rel:.3e}"
                  + (f"; forced K3e {rf.wall_time_s * 1e3:.2f} ms" if rf else ""), flush=True)
        del Za, Zb


if __name__ == "__main__":
    main()
