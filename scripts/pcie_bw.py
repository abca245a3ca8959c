#!/usr/bin/env python3
"""Pinned host <-> device copy bandwidth on this box (the e2e ceiling: every byte of Z
crosses PCIe).  Measured on the pool B200: D2H 57.3 GB/s, H2D 55.6 GB/s (Gen5 x16)."""
import torch, time
n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d.fill_(1)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for chunk in (64 << 20, 256 << 20, 1 << 30, 4 << 30):
    torch.cuda.synchronize(); t = time.perf_counter()
    for rep in range(3):
        for o in range(0, n, chunk):
            h[o:o+chunk].copy_(d[o:o+chunk], non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    print(f"D2H chunk {chunk>>20} MiB: {n/dt/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for rep in range(3):
    half = n // 2
    h[:half].copy_(d[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"D2H two streams: {n/dt/1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
for rep in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"H2D: {n/dt/1e9:.1f} GB/s")
