#!/usr/bin/env python3
"""Throughput / ratio sweep over the BASELINE configurations that are not
the bench line (config 1: AMDF 2^22; config 3: 2^26 HACC-like and AMDF-like,
eb_rel 1e-2 .. 1e-6; both SZ modes): device-resident compress (incl. the
payload CRC-64s) and decompress, CUDA-event timed, best of --reps.
    python scripts/sweep.py [--out profiles/r02_sweep.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402


def timed(fn, reps):
    best = 1e30
    out = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workloads", default="C1,C3-hacc,C3-amdf")
    args = ap.parse_args()
    rows = []
    for wl in args.workloads.split(","):
        fields = datagen.generate(wl)
        n = fields[0].size
        snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
        ebs = [1e-4] if wl == "C1" else [1e-2, 1e-3, 1e-4, 1e-5, 1e-6]
        for eb in ebs:
            for mode in ("sz-lv", "sz-lv-prx"):
                spec = nbz.ErrorBoundSpec.relative(eb)
                nbz.decompress(nbz.compress(snap, mode, spec).archive, device=True)  # warm-up
                tc, res = timed(lambda: nbz.compress(snap, mode, spec), args.reps)
                td, out = timed(lambda: nbz.decompress(res.archive, device=True), args.reps)
                # bound check on the device (sorted order for prx)
                worst = 0.0
                od = res.order_device()
                for fi, name in enumerate(nbz.FIELD_NAMES):
                    x = getattr(snap, name)
                    if od is not None:
                        x = x[od]
                    err = (x.double() - getattr(out, name).double()).abs().max().item()
                    worst = max(worst, err / res.archive.bounds[fi] if res.archive.bounds[fi] else 0.0)
                row = dict(workload=wl, n=int(n), eb_rel=eb, mode=mode, ratio=nbz.ratio(res.archive),
                           compress_ms=round(tc, 3), decompress_ms=round(td, 3),
                           compress_gbps=round(24.0 * n / tc * 1e-6, 1),
                           decompress_gbps=round(24.0 * n / td * 1e-6, 1),
                           max_err_over_bound=round(worst, 6))
                rows.append(row)
                print(json.dumps(row), flush=True)
        del snap, fields
        torch.cuda.empty_cache()
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
