#!/usr/bin/env python3
"""A/B of the shared-edge direct fill (K4e) against the per-triangle kernel
(FillOptions(shared_edges=0)) on the bench configurations: fill time, evaluations performed and
the largest entrywise difference relative to the entry's modulus.
Usage: edge_ab.py [c2 c3 c4 c5] [--rows R]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402


def fill(dm, k, rows, Z, opts, reps=3):
    best = None
    for _ in range(reps):
        _, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, row_end=rows, out=Z, options=opts)
        best = rep if best is None or rep.wall_time_s < best.wall_time_s else best
    return best


def main():
    names = [a for a in sys.argv[1:] if a.startswith("c")] or ["c2", "c3", "c4", "c5"]
    rows_arg = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 0
    chunks = sys.argv[sys.argv.index("--chunks") + 1].split(",") if "--chunks" in sys.argv else [None]
    for name, ch in [(n, c) for n in names for c in chunks]:
        mopts = gk.MeshOptions()
        if ch:
            mopts.edge_chunks = int(ch)
            print(f"edge_chunks={ch}", end=" ")
        cfg = bench.CONFIGS[name]
        mesh = bench.make_mesh(gk, cfg)
        N = mesh.triangle_count()
        rows = rows_arg or (N if N <= 20480 else 8192)
        if "--order" in sys.argv:
            mopts.edge_order = int(sys.argv[sys.argv.index("--order") + 1])
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]), options=mopts)
        med = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0),
                        eps_r_im=cfg.get("eps_r_im", 0.0))
        k = gk.wavenumber(med)
        info = dm.edge_info()
        Za = torch.empty((rows, N), dtype=torch.complex128, device="cuda")
        Zb = torch.empty_like(Za)
        ra = fill(dm, k, rows, Za, gk.FillOptions(shared_edges=0))
        rb = fill(dm, k, rows, Zb, gk.FillOptions(shared_edges=1))  # forced: small meshes too
        d = (Zb - Za).abs()
        rel = (d / Za.abs().clamp_min(1e-300)).max().item()
        R = info["edges"] / (3.0 * N)
        ev = rb.evaluations / rb.actual_calls
        near = (ev - R) / (1.0 - R)
        print(f"{name} N={N} rows={rows} blocks={info['blocks']} ordered={info['ordered']} "
              f"edges/3N={R:.3f} slots/3N={info['work_ratio']:.3f} rho_mean={info['rho_mean']:.3f} "
              f"delta={info['delta']:.3e} r_far={info['r_far']:.4f} near~{near:.3f} | per-triangle "
              f"{ra.wall_time_s * 1e3:.2f} ms, edge {rb.wall_time_s * 1e3:.2f} ms "
              f"(x{ra.wall_time_s / rb.wall_time_s:.3f}); evaluations {rb.evaluations / rb.actual_calls:.4f} "
              f"of the reference's; max |dZ|/|Z| = {rel:.3e}", flush=True)
        del Za, Zb


if __name__ == "__main__":
    main()
