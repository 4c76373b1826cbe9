#!/usr/bin/env python3
"""Does MADV_POPULATE_WRITE work here, and how fast (1..8 threads)?"""
import ctypes, os, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_1711_03888_b200 import hostio

libc = ctypes.CDLL(None, use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
N = 1 << 30
print(os.uname().release)
for nt in (1, 4, 8):
    b, v = hostio.new_bytes(N)
    addr = v.data_ptr()
    a0 = (addr + 4095) & ~4095
    ln = (addr + N - a0) & ~4095
    CH = 64 << 20
    t0 = time.perf_counter()
    def pf(off):
        r = libc.madvise(ctypes.c_void_p(a0 + off), ctypes.c_size_t(min(CH, ln - off)), 23)
        return r, ctypes.get_errno()
    with ThreadPoolExecutor(nt) as ex:
        res = list(ex.map(pf, range(0, ln, CH)))
    dt = time.perf_counter() - t0
    print(nt, "threads populate", f"{N / dt / 1e9:.1f} GB/s", "rc", res[0])
    src = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
    t0 = time.perf_counter()
    for off in range(0, N, 64 << 20):
        v[off:off + (64 << 20)].copy_(src)
    print("  copy after populate", f"{N / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
