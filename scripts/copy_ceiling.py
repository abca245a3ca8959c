#!/usr/bin/env python3
"""The practical ceiling for a 24 MB streaming kernel on this GPU: torch's own
device copy of 12 MB (12 MB read + 12 MB written, C1 eval_batch moves 8 + 16)
as 1024 launches over 8 rotating buffer pairs, back to back and as one CUDA
graph -- the same timing harness as bench.run_c1."""
import json

import torch

n_bytes, sets, iters = 12 << 20, 8, 1024
src = [torch.empty(n_bytes, dtype=torch.uint8, device="cuda") for _ in range(sets)]
dst = [torch.empty_like(s) for s in src]


def run():
    for i in range(iters):
        dst[i % sets].copy_(src[i % sets])


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / iters
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    with torch.cuda.graph(g, stream=side):
        run()
g.replay()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ug = e0.elapsed_time(e1) * 1e3 / iters
print(json.dumps({"bytes_moved": 2 * n_bytes, "us_per_copy": us, "graph_us_per_copy": ug,
                  "graph_gbs": 2 * n_bytes / (ug * 1e-6) / 1e9}))
