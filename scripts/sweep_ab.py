#!/usr/bin/env python3
"""A/B of the table sweep (K3s, csrc/fill_sweep.cuh) against the other table
paths -- K3e (shared edges, table through L1) and the staged per-triangle
kernel -- on the bench configurations at S = 10^3 and 10^4.
Usage: sweep_ab.py [c3 c4 c5] [--rows R] [--chunks C] [--full]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402


def arg(name, default):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def fill(dm, t, rows, Z, opts, reps=2):
    best = None
    for _ in range(reps):
        _, rep = gk.fill_rows(dm, gk.Mode.TABLE, table=t, row_end=rows, out=Z, options=opts)
        best = rep if best is None or rep.wall_time_s < best.wall_time_s else best
    return best


def main():
    names = [a for a in sys.argv[1:] if a in bench.CONFIGS] or ["c3", "c4", "c5"]
    rows_arg = arg("--rows", 0)
    chunks = arg("--chunks", 0)
    for name in names:
        cfg = bench.CONFIGS[name]
        mesh = bench.make_mesh(gk, cfg)
        N = mesh.triangle_count()
        rows = N if "--full" in sys.argv else (rows_arg or (N if N <= 20480 else 4096))
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]),
                           options=gk.MeshOptions(sweep_chunks=chunks))
        info = dm.edge_info()
        print(f"{name}: N={N} sweep blocks {info['sweep']}, K3e blocks {info['blocks']} "
              f"rho_max {info['rho_max']:.4f}", flush=True)
        med = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0),
                        eps_r_im=cfg.get("eps_r_im", 0.0))
        lo, hi = dm.distance_range()
        Zb = torch.empty((rows, N), dtype=torch.complex128, device="cuda")
        Za = Zb if "--only" in sys.argv else torch.empty_like(Zb)
        for S in (10000, 1000):
            t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
            rs = fill(dm, t, rows, Zb, gk.FillOptions(table_placement=gk.GK_TABLE_SWEEP))
            if "--only" in sys.argv:
                print(f"{name} S={S} rows={rows}: {rs.path_name} {rs.wall_time_s * 1e3:.2f} ms "
                      f"({rs.evaluations / rs.wall_time_s:.3e}/s performed)", flush=True)
                continue
            re_ = fill(dm, t, rows, Za, gk.FillOptions(table_placement=gk.GK_TABLE_GLOBAL))
            rel = ((Zb - Za).abs() / Za.abs().clamp_min(1e-300)).max().item()
            rst = fill(dm, t, rows, Za, gk.FillOptions(table_placement=gk.GK_TABLE_SHARED,
                                                       shared_edges=0), reps=1)
            print(f"{name} S={S} rows={rows}: {rs.path_name} {rs.wall_time_s * 1e3:.2f} ms "
                  f"(evals {rs.evaluations / rs.actual_calls:.4f}, "
                  f"{rs.evaluations / rs.wall_time_s:.3e}/s performed); "
                  f"{re_.path_name} {re_.wall_time_s * 1e3:.2f} ms "
                  f"(evals {re_.evaluations / re_.actual_calls:.4f}); "
                  f"{rst.path_name} {rst.wall_time_s * 1e3:.2f} ms; "
                  f"speed-up vs K3e x{re_.wall_time_s / rs.wall_time_s:.3f}; "
                  f"fallbacks {rs.fallback_calls}/{re_.fallback_calls}; "
                  f"max |dZ|/|Z| {rel:.3e}", flush=True)
        del Za, Zb


if __name__ == "__main__":
    main()
