#!/usr/bin/env python3
"""K1 distance range and device table build (K2) times per config and S."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402
for key in ("c2", "c3", "c5"):
    cfg = bench.CONFIGS[key]
    mesh = bench.make_mesh(gk, cfg)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]))
    med = gk.Medium(lambda0=cfg["lambda0"])
    for S in (1000, 10000):
        for rep in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            lo, hi = dm.distance_range()
            torch.cuda.synchronize(); t1 = time.perf_counter()
            t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S), med)
            torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"{key} S={S}: K1 {1e3*(t1-t0):.3f} ms, build {1e3*(t2-t1):.3f} ms (device {t.info.build_ms:.3f} ms), nodes {t.info.nodes}")
