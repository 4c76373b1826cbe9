#!/usr/bin/env python3
"""Wall-clock split of the e2e leg (host in -> bytes -> host out)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen, io as nio

n = int(sys.argv[1]) if len(sys.argv) > 1 else 640 ** 3
host_t = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(6)]
host = [t.numpy() for t in host_t]
datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, n, out=host)
snap = nbz.ParticleSnapshot(*host)
for rep in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4)); torch.cuda.synchronize(); t.append(time.perf_counter())
    wire = res.archive.serialized(); t.append(time.perf_counter())
    ar = nio.deserialize_archive(wire); torch.cuda.synchronize(); t.append(time.perf_counter())
    out = nbz.decompress(ar, device=False); t.append(time.perf_counter())
    names = ["compress(h2d)", "serialized", "deserialize", "decompress(d2h)"]
    print(" ".join(f"{nm} {1e3*(b-a):.0f}ms" for nm, a, b in zip(names, t, t[1:])),
          f"total {1e3*(t[-1]-t[0]):.0f}ms  -> {24*n/(t[-1]-t[0])/1e9:.2f} GB/s", flush=True)
