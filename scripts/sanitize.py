#!/usr/bin/env python3
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): compress + decompress of one snapshot in every mode, both
archive versions, through the public API and the wire.
    compute-sanitizer --tool memcheck python scripts/sanitize.py [--n N]"""
import argparse, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import datagen, io as nio

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--profile", default="hacc")
args = ap.parse_args()
if args.profile == "hacc":
    L = round(args.n ** (1 / 3))
    fields = datagen.small_hacc(L)
else:
    fields = datagen.small_amdf(args.n)
snap = nbz.ParticleSnapshot(*fields)
spec = nbz.ErrorBoundSpec.relative(1e-4)
runs = [(m, 2) for m in ("sz-lv", "sz-lv-prx", "sz-lcf", "sz-cpc2000", "cpc2000")]
runs += [("sz-lv", 1), ("sz-lv-prx", 1)]
for mode, ver in runs:
    res = nbz.compress(snap, mode, spec, version=ver)
    wire = res.archive.serialized()
    out = nbz.decompress(nio.deserialize_archive(wire))
    order = res.order
    worst = 0.0
    for fi in range(6):
        x = fields[fi] if order is None else fields[fi][order]
        err = float(np.abs(x.astype(np.float64) - np.asarray(out.field(fi), np.float64)).max())
        assert err <= res.archive.bounds[fi], (mode, ver, fi)
        worst = max(worst, err / res.archive.bounds[fi])
    print(f"{mode} v{ver}: n={snap.n} ratio {nbz.ratio(res.archive):.3f} max err/bound {worst:.3f}",
          flush=True)
torch.cuda.synchronize()
print("sanitize workload ok")
