#!/usr/bin/env python3
"""BASELINE config 4 scale check on one GPU: 1024^3 = 1,073,741,824 HACC-like
particles (25.8 GB), sz-lv-prx eb_rel 1e-4.  Generated on the host in
slabs straight into device memory; compress, decompress, then the error
bound is checked at every point on the device (no oracle at this size:
the per-stage bit-exactness is covered by the C0-C3 tests).
    python scripts/c4_check.py [side] [mode]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
mode = sys.argv[2] if len(sys.argv) > 2 else "sz-lv-prx"
spec = datagen.HaccSpec((side, side, side), 2.5)
n = spec.n
dev = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(6)]
t0 = time.time()
step = 1 << 26
buf = [np.empty(step, np.float32) for _ in range(6)]
for p0 in range(0, n, step):
    p1 = min(n, p0 + step)
    out = [b[:p1 - p0] for b in buf]
    datagen.generate(spec, p0, p1, out=out)
    for f, o in zip(dev, out):
        f[p0:p1].copy_(torch.from_numpy(o))
torch.cuda.synchronize()
print(f"generated n={n} in {time.time() - t0:.0f}s", flush=True)
snap = nbz.ParticleSnapshot(*dev)
for rep in range(2):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
    e1.record()
    rec = nbz.decompress(res.archive, device=True)
    e2.record()
    torch.cuda.synchronize()
    tc, td = e0.elapsed_time(e1), e1.elapsed_time(e2)
    print(f"compress {tc:.1f} ms ({24 * n / tc / 1e6:.0f} GB/s)  decompress {td:.1f} ms "
          f"({24 * n / td / 1e6:.0f} GB/s)  ratio {nbz.ratio(res.archive):.4f}", flush=True)
order = res.order_device()
worst = 0.0
for fi in range(6):
    x = dev[fi][order].double()
    err = (x - rec.field(fi).double()).abs().max().item()
    b = res.archive.bounds[fi]
    worst = max(worst, err / b)
    assert err <= b, (fi, err, b)
print(f"{mode}: bound holds at every point (max err/bound {worst:.4f})")
if mode in ("sz-cpc2000", "cpc2000"):
    # the serialized archive decodes to the same values (v2 index path)
    from paper_1711_03888_b200 import io as nio
    rec2 = nbz.decompress(nio.deserialize_archive(res.archive.serialized()), device=True)
    for fi in range(6):
        assert torch.equal(rec2.field(fi), rec.field(fi)), fi
    print(f"{mode}: wire round trip identical")
