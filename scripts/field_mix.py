#!/usr/bin/env python3
"""Decode time of field subsets (the others masked as constants): do the
fields' CTAs slow each other down?  python scripts/field_mix.py [--n N]"""
import argparse, copy, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen
from paper_1711_03888_b200 import _native as N

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=262144000)
args = ap.parse_args()
fields = datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, args.n)
snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
del fields
res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
ar = res.archive
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for sub in [(3,), (3, 4, 5), (0, 1, 2), (0, 3), (0, 1, 2, 3, 4, 5), (3,), (0,)]:
    a2 = copy.copy(ar)
    a2.constant_mask = 0x3F & ~sum(1 << f for f in sub)
    def dec():
        try:
            nbz.decompress(a2, device=True)
        except Exception:  # timing experiments may decode garbage
            pass
    dec()
    ts = []
    N.trace_enable(True)
    for _ in range(5):
        e0.record(); dec(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    tr = N.trace_read()
    N.trace_enable(False)
    dq = sorted(ms for name, ms in tr if name == "dq_decode")
    print(f"fields {sub}: {min(ts):.3f} ms  dq_decode {dq[0]:.3f} .. {dq[-1]:.3f} ms", flush=True)
