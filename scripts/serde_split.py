#!/usr/bin/env python3
"""Split serialized() / deserialize_archive() into their parts (C2 archive)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen, hostio, io as nio

n = 640 ** 3
dev = [torch.from_numpy(f).cuda() for f in datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, n)]
snap = nbz.ParticleSnapshot(*dev)
res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
ar = res.archive
d = ar._dev
tot = sum(ar.payload_lengths())
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    crcs = nio._payload_crcs(ar); t1 = time.perf_counter()
    out, view = hostio.new_bytes(tot); t2 = time.perf_counter()
    hostio.to_host(d.arena[:tot], view[:tot]); t3 = time.perf_counter()
    ar._wire = None
    w = ar.serialized(); t4 = time.perf_counter()
    a2 = nio.deserialize_archive(w); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"crc {1e3*(t1-t0):.1f} ms  new_bytes {1e3*(t2-t1):.1f} ms  to_host {1e3*(t3-t2):.1f} ms "
          f"serialized {1e3*(t4-t3):.1f} ms  deserialize {1e3*(t5-t4):.1f} ms  ({tot/1e9:.2f} GB)", flush=True)
