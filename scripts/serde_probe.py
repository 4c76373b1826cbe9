#!/usr/bin/env python3
"""Where serialized() / deserialize_archive() spend their time at C2."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen, hostio
from paper_1711_03888_b200 import io as nio

n = int(sys.argv[1]) if len(sys.argv) > 1 else 640 ** 3
host_t = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(6)]
host = [t.numpy() for t in host_t]
datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, n, out=host)
snap = nbz.ParticleSnapshot(*host)
res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
ar = res.archive
d = ar._dev


def tm(label, f, reps=3):
    ts = []
    r = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"{label:28s}", " ".join(f"{x:.1f}" for x in ts), "ms", flush=True)
    return r


tm("payload crcs (6 fields)", lambda: nio._payload_crcs(ar))
o, ln = d.offsets[0], d.lengths[0]
tm("crc64_device one field", lambda: nio.crc64_device(d.arena[o:o + ln], ln))
wire = tm("serialized total", lambda: nio.serialize_archive(ar))
print("wire bytes", len(wire))
tm("deserialize total", lambda: nio.deserialize_archive(wire))
dst = torch.empty(len(wire) + 64, dtype=torch.uint8, device="cuda")
tm("to_device(wire)", lambda: hostio.to_device(wire, dst[:len(wire)]))
ar2 = nio.deserialize_archive(wire)
tm("decompress(device=True)", lambda: nbz.decompress(ar2, device=True))
tm("decompress(device=False)", lambda: nbz.decompress(ar2, device=False))
