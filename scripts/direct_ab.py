#!/usr/bin/env python3
"""Direct-fill timings (K4e shared edges and K4 per triangle) on the bench
configurations, full matrices; for A/B of libgk builds (GK_LIB=...).
Usage: direct_ab.py [c3 c4 c5] [--reps R] [--edge-only] [--leaf P1,P2,...] [--chunks C1,C2,...]
(--leaf / --chunks: K4e only, one line per bisection leaf size / block size)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if a in bench.CONFIGS] or ["c3", "c4", "c5"]
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    for name in names:
        cfg = bench.CONFIGS[name]
        mesh = bench.make_mesh(gk, cfg)
        N = mesh.triangle_count()
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]))
        med = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0),
                        eps_r_im=cfg.get("eps_r_im", 0.0))
        k = gk.wavenumber(med)
        Z = torch.empty((N, N), dtype=torch.complex128, device="cuda")
        leaf = sys.argv[sys.argv.index("--leaf") + 1].split(",") if "--leaf" in sys.argv else []
        chunks = sys.argv[sys.argv.index("--chunks") + 1].split(",") if "--chunks" in sys.argv else [0]
        for lp in leaf:
            for ch in chunks:
                dmv = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]),
                                    options=gk.MeshOptions(leaf_pct=int(lp), edge_chunks=int(ch)))
                best = None
                for _ in range(reps):
                    _, rep = gk.fill_rows(dmv, gk.Mode.DIRECT, k=k, out=Z)
                    best = rep if best is None or rep.wall_time_s < best.wall_time_s else best
                info = dmv.edge_info()
                print(f"{name} leaf_pct={lp} chunks={ch or 'default'} blocks={info['blocks']} "
                      f"slots/3N={info['work_ratio']:.4f}: {best.wall_time_s * 1e3:.2f} ms "
                      f"(evaluations {best.evaluations / best.actual_calls:.4f})", flush=True)
                del dmv
        if leaf:
            continue
        variants = (("edge", None), ("pertri", gk.FillOptions(shared_edges=0)))
        if "--edge-only" in sys.argv:
            variants = variants[:1]
        for label, opts in variants:
            best = None
            for _ in range(reps):
                _, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=k, out=Z, options=opts)
                best = rep if best is None or rep.wall_time_s < best.wall_time_s else best
            print(f"{name} {label} {best.path_name}: {best.wall_time_s * 1e3:.2f} ms "
                  f"({best.evaluations / best.wall_time_s:.3e} performed/s)", flush=True)
        del Z


if __name__ == "__main__":
    main()
