#!/usr/bin/env python3
"""The e2e ceiling on this box: a pure device->host copy with the e2e's pattern
(26 windows of 3276 C5 rows, 1 GiB chunks into one pinned window) next to the
same 26 gk_fill_rows_host calls (fill + copy pipelined)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_04162_b200 as gk  # noqa: E402
N = 81920; rows_win = 3276; row_bytes = N * 16
dev = torch.empty((1 << 30) // 8, dtype=torch.float64, device="cuda")
host = torch.empty(rows_win * N * 2, dtype=torch.float64, pin_memory=True)
s = torch.cuda.Stream()
def pure():
    total = 0
    with torch.cuda.stream(s):
        for w in range(26):
            off = 0
            while off < rows_win * row_bytes:
                n = min(1 << 30, rows_win * row_bytes - off)
                host.view(torch.uint8)[off:off + n].copy_(dev.view(torch.uint8)[:n], non_blocking=True)
                off += n; total += n
    s.synchronize(); return total
pure()
t = time.perf_counter(); tot = pure(); dt = time.perf_counter() - t
print(f"pure D2H: {tot/1e9:.1f} GB in {dt:.3f} s = {tot/dt/1e9:.1f} GB/s")
cfg = bench.CONFIGS["c5"]; mesh = bench.make_mesh(gk, cfg)
ctx = gk.Context.get(0); dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4), ctx)
z = host.numpy().view(np.complex128).reshape(-1, N)[:rows_win]
gk.fill_rows_host(dm, gk.Mode.DIRECT, z, k=2*np.pi/0.15, row_begin=0, row_end=rows_win)
t = time.perf_counter()
for b in range(0, N, rows_win):
    gk.fill_rows_host(dm, gk.Mode.DIRECT, z, k=2*np.pi/0.15, row_begin=b, row_end=min(N, b + rows_win))
dt = time.perf_counter() - t
print(f"fill_rows_host x26: {dt:.3f} s = {N*N*16/dt/1e9:.1f} GB/s")

# the pure copy again, with a C5 direct fill running concurrently on another stream
zdev = torch.empty((8192, N), dtype=torch.complex128, device="cuda")
fs = torch.cuda.Stream()
with torch.cuda.stream(fs):
    ctx.bind_stream(fs)
    for b in range(0, 6):
        gk.fill_rows(dm, gk.Mode.DIRECT, k=2*np.pi/0.15, row_begin=0, row_end=8192, out=zdev,
                     report=False)
t = time.perf_counter(); tot = pure(); dt = time.perf_counter() - t
torch.cuda.synchronize()
ctx.bind_stream()
print(f"pure D2H beside a running fill: {tot/1e9:.1f} GB in {dt:.3f} s = {tot/dt/1e9:.1f} GB/s")
