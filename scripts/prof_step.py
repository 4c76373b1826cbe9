#!/usr/bin/env python3
"""One compress + decompress of a HACC-like slab on cuda:0 -- the short
command profiled with ncu (profiles/*).  Usage:
    python scripts/prof_step.py [--n N] [--mode sz-lv-prx] [--reps R]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--mode", default="sz-lv-prx")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--compress-only", action="store_true")
    ap.add_argument("--trace", action="store_true", help="print per-stage ms of the last rep")
    ap.add_argument("--crc", action="store_true", help="also serialise (payload CRC-64s)")
    ap.add_argument("--eb", type=float, default=1e-4)
    ap.add_argument("--workload", default=None, help="a datagen.CONFIGS name instead of the C2 slab")
    args = ap.parse_args()
    from paper_1711_03888_b200 import _native as N
    if args.workload:
        fields = datagen.generate(args.workload)
    else:
        fields = datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, args.n)
    snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    for r in range(args.reps):
        if args.trace and r == args.reps - 1:
            N.trace_enable(True)
        res = nbz.compress(snap, args.mode, nbz.ErrorBoundSpec.relative(args.eb))
        if args.crc:
            from paper_1711_03888_b200 import io as nio
            nio._payload_crcs(res.archive)
        if not args.compress_only:
            out = nbz.decompress(res.archive, device=True)
    torch.cuda.synchronize()
    if args.trace:
        print(" ".join(f"{k}={v:.3f}" for k, v in N.trace_read()))
        N.trace_enable(False)
    print("ratio", nbz.ratio(res.archive), "n", snap.n)


if __name__ == "__main__":
    main()
