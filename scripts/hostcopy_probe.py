#!/usr/bin/env python3
"""Host-side copy rates: pinned -> fresh pageable (page faults) vs pre-touched."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_1711_03888_b200 import hostio

N = 1 << 30
print("torch threads", torch.get_num_threads(), "cpus", os.cpu_count())
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
src = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
for label, fresh in (("fresh", True), ("touched", False)):
    b, v = hostio.new_bytes(N)
    if not fresh:
        v.fill_(1)
    t0 = time.perf_counter()
    for off in range(0, N, 64 << 20):
        v[off:off + (64 << 20)].copy_(src)
    dt = time.perf_counter() - t0
    print(label, f"{N / dt / 1e9:.1f} GB/s")
