#!/usr/bin/env python3
"""C1 eval_batch: back-to-back launches vs one CUDA graph of the same launches."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_04162_b200 as gk  # noqa: E402

n, sets, iters = 1 << 20, 8, 512
ctx = gk.Context.get(0)
rng = np.random.default_rng(1901)
rs = [torch.as_tensor(rng.uniform(1e-3, 2.0, n), device="cuda") for _ in range(sets)]
outs = [torch.empty(n, dtype=torch.complex128, device="cuda") for _ in range(sets)]
med = gk.Medium(lambda0=0.5)
k = gk.wavenumber(med)
for name, S in (("direct", None), ("table_S1000", 1000)):
    t = gk.DeviceTable(gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=S), med) \
        if S else None
    for kind in (gk.KernelKind.PlainExp, gk.KernelKind.GreenOverR):
        st = gk.EvalStatus(ctx)

        def run():
            for i in range(iters):
                gk.eval_batch_async(kind, rs[i % sets], outs[i % sets], st, table=t, k=k)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        plain = e0.elapsed_time(e1) * 1e3 / iters
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ctx.bind_stream()
            with torch.cuda.graph(g, stream=s):
                ctx.bind_stream()
                run()
        ctx.bind_stream()
        torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) * 1e3 / iters
        st.read()
        print(f"{name} {kind.name}: plain {plain:.2f} us/batch ({n*24/plain/1e3:.0f} GB/s), "
              f"graph {graph:.2f} us/batch ({n*24/graph/1e3:.0f} GB/s)")
