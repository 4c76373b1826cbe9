#!/usr/bin/env python3
"""One CPC-mode compress + decompress of a HACC-like slab on cuda:0 (ncu target)."""
import argparse, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--mode", default="cpc2000")
args = ap.parse_args()
fields = datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, args.n)
snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
res = nbz.compress(snap, args.mode, nbz.ErrorBoundSpec.relative(1e-4))
out = nbz.decompress(res.archive, device=True)
torch.cuda.synchronize()
print("ratio", nbz.ratio(res.archive))
