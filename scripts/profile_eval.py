#!/usr/bin/env python3
"""A few eval_batch launches (C1: 2^20 radii, k = 4 pi) for ncu: warm-up,
then the profiled launches.  Usage: profile_eval.py [direct|table] [exp|green]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04162_b200 as gk  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "direct"
kind = gk.KernelKind.PlainExp if (len(sys.argv) > 2 and sys.argv[2] == "exp") else \
    gk.KernelKind.GreenOverR
ctx = gk.Context.get(0)
n = 1 << 20
rng = np.random.default_rng(1901)
rs = [torch.as_tensor(rng.uniform(1e-3, 2.0, n), device="cuda") for _ in range(8)]
outs = [torch.empty(n, dtype=torch.complex128, device="cuda") for _ in range(8)]
med = gk.Medium(lambda0=0.5)
t = gk.DeviceTable(gk.SamplingConfig(r_min=1e-3, r_max=2.0), med) if mode == "table" else None
st = gk.EvalStatus(ctx)
for i in range(24):
    gk.eval_batch_async(kind, rs[i % 8], outs[i % 8], st, table=t, k=gk.wavenumber(med))
torch.cuda.synchronize()
st.read()
print("profile_eval: done")
