#!/usr/bin/env python3
"""eval_batch against its HBM roofline (24 B per radius) as the batch grows:
C1's 2^20 radii are 24 MB per launch, where launch ramp and drain matter (a
plain device copy of 24 MB is no faster, scripts/copy_ceiling.py); larger
batches show what the kernel itself sustains.  Buffers rotate over > 126 MB
(L2) so every launch reads and writes HBM."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04162_b200 as gk  # noqa: E402

peak = 6532.2
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
ctx = gk.Context.get(0)
rng = np.random.default_rng(1901)
med = gk.Medium(lambda0=0.5)
k = gk.wavenumber(med)
tables = {"direct": None}
for S in (1000, 10000):
    tables[f"table_S{S}"] = gk.DeviceTable(
        gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=S), med)
print(f"HBM peak (copy) {peak:.0f} GB/s")
for logn in (20, 22, 24, 26):
    n = 1 << logn
    sets = max(2, (192 << 20) // (24 * n) + 1)
    rs = [torch.as_tensor(rng.uniform(1e-3, 2.0, n), device="cuda") for _ in range(sets)]
    outs = [torch.empty(n, dtype=torch.complex128, device="cuda") for _ in range(sets)]
    iters = max(8, (1 << 30) // n // 4)
    for name, t in tables.items():
        for kind in (gk.KernelKind.PlainExp, gk.KernelKind.GreenOverR):
            st = gk.EvalStatus(ctx)
            for i in range(min(iters, 2 * sets)):
                gk.eval_batch_async(kind, rs[i % sets], outs[i % sets], st, table=t, k=k)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(iters):
                gk.eval_batch_async(kind, rs[i % sets], outs[i % sets], st, table=t, k=k)
            e1.record()
            torch.cuda.synchronize()
            st.read()
            us = e0.elapsed_time(e1) * 1e3 / iters
            gbs = n * 24 / us / 1e3
            print(f"n=2^{logn} {name:12s} {kind.name:10s} {us:9.2f} us/batch  {gbs:7.0f} GB/s  "
                  f"{gbs / peak:.3f} of HBM", flush=True)
    del rs, outs
