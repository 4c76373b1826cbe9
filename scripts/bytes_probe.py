#!/usr/bin/env python3
"""Fresh-bytes fill strategies (page faults vs THP vs populate)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

for p in ("/sys/kernel/mm/transparent_hugepage/enabled", "/sys/kernel/mm/transparent_hugepage/defrag"):
    try:
        print(p, open(p).read().strip())
    except OSError as e:
        print(p, e)
n = 1_342_495_820
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(3)
api = ctypes.pythonapi
api.PyBytes_FromStringAndSize.restype = ctypes.py_object
api.PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
api.PyBytes_AsString.restype = ctypes.c_void_p
api.PyBytes_AsString.argtypes = [ctypes.py_object]
libc = ctypes.CDLL(None, use_errno=True)


def fresh(advice):
    b = api.PyBytes_FromStringAndSize(None, n)
    addr = api.PyBytes_AsString(b)
    if advice is not None:
        a0 = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
        ln = (addr + n - a0) & ~((2 << 20) - 1)
        rc = libc.madvise(ctypes.c_void_p(a0), ctypes.c_size_t(ln), advice)
        if rc != 0:
            print("madvise", advice, "errno", ctypes.get_errno())
    return b, addr


def fill(advice, threads=None):
    if threads:
        torch.set_num_threads(threads)
    t = time.perf_counter()
    b, addr = fresh(advice)
    t1 = time.perf_counter()
    dst = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(addr)))
    dst.copy_(pin)
    t2 = time.perf_counter()
    del b
    return 1e3 * (t1 - t), 1e3 * (t2 - t1)


for label, adv in (("plain", None), ("hugepage", 14), ("populate_write", 23)):
    for rep in range(3):
        a, c = fill(adv)
        print(f"{label:15s} alloc+advise {a:.1f} ms  copy {c:.1f} ms", flush=True)
for th in (8, 32, 64):
    a, c = fill(14, th)
    print(f"hugepage threads {th}: {a:.1f} + {c:.1f} ms", flush=True)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
