#!/usr/bin/env python3
"""Per-field decode time (the other fields masked as constants) -- used to
balance SMs across fields.  python scripts/field_times.py [--n N]"""
import argparse, copy, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
args = ap.parse_args()
fields = datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, args.n)
snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
ar = res.archive
for _ in range(2):
    nbz.decompress(ar, device=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); nbz.decompress(ar, device=True); e1.record(); torch.cuda.synchronize()
print(f"all fields: {e0.elapsed_time(e1):.3f} ms")
for fi in range(6):
    a2 = copy.copy(ar)
    a2.constant_mask = 0x3F & ~(1 << fi)
    nbz.decompress(a2, device=True)
    e0.record(); nbz.decompress(a2, device=True); e1.record(); torch.cuda.synchronize()
    print(f"field {fi}: {e0.elapsed_time(e1):.3f} ms  payload {ar._dev.lengths[fi]} B")
