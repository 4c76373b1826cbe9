#!/usr/bin/env python3
"""PCIe probe: pinned H2D / D2H bandwidth for one big copy, chunked copies on
one stream, and concurrent H2D + D2H (full duplex)."""
import time
import torch

N = 1 << 30  # 1 GiB
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
torch.cuda.synchronize()


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best


print("h2d GB/s", N / t(lambda: d.copy_(h, non_blocking=True)) / 1e9)
print("d2h GB/s", N / t(lambda: h.copy_(d, non_blocking=True)) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s1.synchronize(); s2.synchronize()


print("duplex (each direction) GB/s", N / t(duplex) / 1e9)
