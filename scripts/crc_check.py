#!/usr/bin/env python3
"""CRC-64 kernel check and timing on cuda:0: random buffers at every
alignment / length class against the oracle's CRC, then the time of one
nbzg_crc64_many over config-2-sized payloads (6 buffers, 1.34 GB)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1711_03888_b200 import io as nio  # noqa: E402

rng = np.random.default_rng(7)
big = rng.integers(0, 256, (3 << 20) + 77, dtype=np.uint8)
d = torch.from_numpy(big).cuda()
bad = 0
cases = [(0, 0), (0, 1), (3, 5), (1, 15), (0, 16), (5, 16), (15, 17), (7, 511), (0, 512), (9, 513),
         (0, 65536), (3, 65536), (13, 65537), (1, (1 << 19) - 1), (0, 1 << 19), (2, (1 << 19) + 1),
         (11, (1 << 20) + 12345), (0, big.size), (5, big.size - 5), (16, big.size - 16)]
for off in range(0, 17):
    for ln in (1, 2, 15, 16, 17, 31, 32, 33, 100, 1000, 2049, 70001):
        cases.append((off, ln))
parts = [(d[o:], n) for o, n in cases]
for i in range(0, len(parts), 7):
    got = nio.crc64_device_many(parts[i:i + 7])
    for (o, n), g in zip(cases[i:i + 7], got):
        w = oracle.crc64(big[o:o + n].tobytes())
        if g != w:
            bad += 1
            if bad < 10:
                print("MISMATCH off", o, "len", n, hex(g), hex(w))
print("crc cases", len(cases), "bad", bad)
assert nio.crc64(b"123456789") == 0x995DC9BBDF1939FA

# timing: config-2 payload sizes
sizes = [105_000_000, 125_000_000, 143_000_000, 322_000_000, 322_000_000, 322_000_000]
buf = torch.randint(0, 256, (sum(sizes) + 64,), dtype=torch.uint8, device="cuda")
parts, o = [], 3
for s in sizes:
    parts.append((buf[o:], s))
    o += s
for _ in range(3):
    nio.crc64_device_async(parts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    nio.crc64_device_async(parts)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("crc64_many %.3f ms for %.3f GB -> %.1f GB/s" % (ms, sum(sizes) * 1e-9, sum(sizes) / ms * 1e-6))
sys.exit(1 if bad else 0)
