#!/usr/bin/env python3
"""Encode / decode path crossover: per-stage trace of a C2-generator slab of n
particles with the block/thread-per-chunk paths forced on and off
(NBZG_ENCODE / NBZG_DECODE), to place the chunk-count thresholds.
    python scripts/path_crossover.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import _native as N, datagen  # noqa: E402

spec = datagen.HaccSpec((640, 640, 640), 2.5)
sizes = [int(a) for a in sys.argv[1:]] or [1 << lg for lg in (21, 22, 23, 24, 25, 26)]
for n in sizes:
    lg = n.bit_length() - 1
    fields = datagen.generate(spec, 0, n)
    snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    for enc, dec in (("t", "thread"), ("w", "warp")):
        os.environ["NBZG_ENCODE"] = enc
        os.environ["NBZG_DECODE"] = dec
        best = {}
        for r in range(4):
            N.trace_enable(True)
            res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
            nbz.decompress(res.archive, device=True)
            torch.cuda.synchronize()
            for k, v in N.trace_read():
                best[k] = min(best.get(k, 1e9), v)
            N.trace_enable(False)
        comp = sum(v for k, v in best.items() if not k.startswith("dq_"))
        sz = sum(best.get(k, 0) for k in ("quantize", "codebook", "layout", "encode"))
        print(f"n={n} (~2^{lg}) chunks/field={n // 16384} enc={enc} dec={dec} "
              f"compress={comp:.3f} sz_stages={sz:.3f} dq_decode={best.get('dq_decode', 0):.3f}", flush=True)
