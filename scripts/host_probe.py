#!/usr/bin/env python3
"""Host-transfer strategies for the e2e leg (pinned pool vs staged vs
registered), measured on the GPU box."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

from paper_1711_03888_b200 import hostio


def t_(f, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append(1e3 * (time.perf_counter() - t))
    return " ".join(f"{x:.0f}" for x in out) + " ms"


n_out = 6 * 262144000 * 4
n_arc = 1_340_000_000
src = torch.empty(n_out, dtype=torch.uint8, device="cuda").fill_(1)


def d2h_pool():
    h = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
    h.copy_(src)
    del h


def d2h_staged():
    h = hostio.empty_host(n_out // 4)
    hostio.to_host(src, h.view(torch.uint8))


print("d2h 6.29GB pinned pool :", t_(d2h_pool), flush=True)
print("d2h 6.29GB staged      :", t_(d2h_staged), flush=True)

wire = hostio.bytes_from(src[:n_arc].cpu(), n_arc)
dst = torch.empty(n_arc + 64, dtype=torch.uint8, device="cuda")
print("h2d 1.34GB staged      :", t_(lambda: hostio.to_device(wire, dst[:n_arc])), flush=True)

cudart = torch.cuda.cudart()


def h2d_register():
    mv = memoryview(wire)
    addr = ctypes.c_char_p.from_buffer  # noqa (documentation only)
    a = np.frombuffer(wire, np.uint8).ctypes.data
    rc = cudart.cudaHostRegister(a, n_arc, 0)
    assert int(rc) == 0, rc
    h = torch.from_numpy(np.frombuffer(wire, np.uint8))
    dst[:n_arc].copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    cudart.cudaHostUnregister(a)


try:
    print("h2d 1.34GB register    :", t_(h2d_register), flush=True)
except Exception as e:  # noqa
    print("register failed", e)


def h2d_pageable():
    h = torch.from_numpy(np.frombuffer(wire, np.uint8).copy()) if False else None
    t = torch.frombuffer(bytearray(0), dtype=torch.uint8) if False else None
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = torch.frombuffer(wire, dtype=torch.uint8)
    dst[:n_arc].copy_(h)


print("h2d 1.34GB pageable    :", t_(h2d_pageable), flush=True)

pin = hostio.pinned("serialize", n_arc)
pin[:n_arc].copy_(src[:n_arc])
print("bytes_from 1.34GB      :", t_(lambda: hostio.bytes_from(pin, n_arc)), flush=True)
print("d2h 1.34GB to pinned   :", t_(lambda: pin[:n_arc].copy_(src[:n_arc])), flush=True)
for c in (8 << 20, 32 << 20, 128 << 20):
    hostio.CHUNK = c
    print(f"h2d 1.34GB staged {c>>20}MB :", t_(lambda: hostio.to_device(wire, dst[:n_arc])), flush=True)
