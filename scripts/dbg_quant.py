#!/usr/bin/env python3
"""Debug: locate positions where the GPU payload of one field decodes
differently from the oracle's (hacc34 golden case)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
import oracle as O
import paper_1711_03888_b200 as nbz
from conftest import golden_inputs, load_golden

case = sys.argv[1] if len(sys.argv) > 1 else "hacc34"
g = load_golden(case)
fields = golden_inputs(g)
snap = nbz.ParticleSnapshot(*fields)
for mode in ("sz-lv", "sz-lv-prx"):
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
    ref = O.compress(fields, mode, "rel", 1e-4, fmt=2)
    for st in res.archive.streams:
        f = st.field
        if st.payload == ref["payloads"][f]:
            continue
        b = res.archive.bounds[f]
        a = O.sz_decode(st.payload, snap.n, b, 65536, 2)
        r = O.sz_decode(ref["payloads"][f], snap.n, b, 65536, 2)
        d = np.nonzero(a.view(np.uint32) != r.view(np.uint32))[0]
        work = fields[f] if res.order is None else fields[f][res.order]
        print(mode, "field", f, "ndiff", d.size, "first", d[:10])
        inv = 1.0 / (2.0 * b)
        for p in d[:5]:
            x = work[p]
            t = np.float32(x) * np.float32(inv)
            print(f"  p={p} (tile pos {p % 16384}) x={x!r} t32={t!r} t64={float(x) * inv!r} gpu={a[p]!r} ref={r[p]!r}")
