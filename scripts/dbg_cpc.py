#!/usr/bin/env python3
"""Debug: GPU vs oracle CPC archives, stream by stream (golden case)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
import oracle as O
import paper_1711_03888_b200 as nbz
from conftest import golden_inputs, load_golden

case = sys.argv[1] if len(sys.argv) > 1 else "cpc_hacc24"
g = load_golden(case)
fields = golden_inputs(g)
ss = int(g["segment_size"])
snap = nbz.ParticleSnapshot(*fields)
for tag in g["tags"]:
    t = str(tag)
    mode, eb = t.split("|")
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(float(eb)), nbz.Settings(segment_size=ss))
    ref = O.compress_cpc(fields, mode, "rel", float(eb), segment_size=ss, fmt=2)
    print(t, "wire equal", res.archive.serialized() == ref["wire"])
    rs = {f: p for k, f, p in ref["streams"]}
    for st in res.archive.streams:
        p = rs.get(st.field)
        if p is None:
            print("  extra stream", st.field); continue
        if st.payload != p:
            a, b = np.frombuffer(st.payload, np.uint8), np.frombuffer(p, np.uint8)
            m = min(a.size, b.size)
            d = np.nonzero(a[:m] != b[:m])[0]
            print("  field", st.field, "len gpu", a.size, "ora", b.size, "first diff", d[:8])
            nseg = (snap.n + ss - 1) // ss
            print("   gpu total_bits", int(np.frombuffer(st.payload[nseg:nseg+8], np.uint64)[0]),
                  "ora", int(np.frombuffer(p[nseg:nseg+8], np.uint64)[0]), "ids", list(a[:nseg][:8]), list(b[:nseg][:8]))
