#!/usr/bin/env python3
"""Decoder experiments at config 2: `prep` compresses the 640^3 snapshot
once (default library) and keeps the wire + a digest of the decoded fields
in /tmp; `time` decodes that wire with the library NBZG_LIB points at
(an in-tree variant build, csrc/Makefile `variant`) and prints the
dq_decode launch times and whether the output is bit-identical.
    python scripts/dec_variants.py prep|time [--n N] [--reps R]"""
import argparse, hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_1711_03888_b200 as nbz
from paper_1711_03888_b200 import _native as N, datagen, io as nio

ap = argparse.ArgumentParser()
ap.add_argument("what")
ap.add_argument("--n", type=int, default=262144000)
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--mode", default="sz-lv-prx")
ap.add_argument("--wire", default="/tmp/c2.nbz")
args = ap.parse_args()


def digest(out):
    h = hashlib.sha256()
    for f in nbz.FIELD_NAMES:
        t = getattr(out, f)
        h.update(t.view(torch.int32).sum(dtype=torch.int64).cpu().numpy().tobytes())
        h.update((t.view(torch.int32).to(torch.int64) * torch.arange(1, t.numel() + 1,
                 device=t.device) % 1000003).sum().cpu().numpy().tobytes())
    return h.hexdigest()[:16]


if args.what == "prep":
    fields = datagen.generate(datagen.HaccSpec((640, 640, 640), 2.5), 0, args.n)
    snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    del fields
    res = nbz.compress(snap, args.mode, nbz.ErrorBoundSpec.relative(1e-4))
    wire = res.archive.serialized()
    out = nbz.decompress(res.archive, device=True)
    open(args.wire, "wb").write(wire)
    open(args.wire + ".sha", "w").write(digest(out))
    print(json.dumps({"prep": len(wire), "ratio": nbz.ratio(res.archive)}))
else:
    wire = open(args.wire, "rb").read()
    ar = nio.deserialize_archive(wire)
    del wire
    ok = None
    ts, dq = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(args.reps + 2):
        N.trace_enable(True)
        e0.record()
        out = nbz.decompress(ar, device=True)
        e1.record()
        torch.cuda.synchronize()
        tr = N.trace_read()
        N.trace_enable(False)
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
            dq += [ms for name, ms in tr if name == "dq_decode"]
        if r == 0:
            ok = digest(out) == open(args.wire + ".sha").read().strip()
        del out
    print(json.dumps({"lib": os.path.basename(N.LIB_PATH), "ok": ok,
                      "dq_min": round(min(dq), 4), "dq_med": round(float(np.median(dq)), 4),
                      "decomp_min": round(min(ts), 4)}), flush=True)
