#!/usr/bin/env python3
"""Cost of making a fresh multi-GB host output DMA-able: cudaHostAlloc vs
THP pages + parallel first touch + cudaHostRegister, per call."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

from paper_1711_03888_b200 import hostio

n = 6 * 262144000
src = torch.empty(n, dtype=torch.float32, device="cuda").fill_(1.0)
cudart = torch.cuda.cudart()
print("pageable access attr:", torch.cuda.get_device_properties(0))


def reg_path(touch):
    t0 = time.perf_counter()
    h = hostio.empty_host(n)
    if touch:
        h.zero_()
    t1 = time.perf_counter()
    rc = cudart.cudaHostRegister(h.data_ptr(), 4 * n, 0)
    t2 = time.perf_counter()
    h.copy_(src)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    cudart.cudaHostUnregister(h.data_ptr())
    t4 = time.perf_counter()
    print(f"touch={touch} rc={int(rc)} alloc+touch {1e3*(t1-t0):.0f} register {1e3*(t2-t1):.0f} "
          f"d2h {1e3*(t3-t2):.0f} unregister {1e3*(t4-t3):.0f} total {1e3*(t4-t0):.0f} ms", flush=True)


for touch in (True, False):
    for _ in range(2):
        reg_path(touch)
for _ in range(2):
    t0 = time.perf_counter()
    h = hostio.empty_host(n)
    hostio.to_host(src.view(torch.uint8), h.view(torch.uint8))
    print(f"staged {1e3*(time.perf_counter()-t0):.0f} ms", flush=True)
