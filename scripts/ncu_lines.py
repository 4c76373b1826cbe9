#!/usr/bin/env python3
"""Per-CUDA-source-line hot spots of one kernel in an ncu report: the SASS
page (stall samples, executed instructions) joined with nvdisasm line info
from the in-tree libnbzg.so (must be the build that was profiled).
    python scripts/ncu_lines.py REP KERNEL_SUBSTR [TOP]"""
import collections, csv, glob, io, os, re, subprocess, sys, tempfile

rep, kern = sys.argv[1], sys.argv[2]
# "NCU_REGEX@MANGLED_SUBSTR" when the demangled and mangled names differ
ncu_k, kern = (kern.split("@", 1) if "@" in kern else (kern, kern))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
lib = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1711_03888_b200",
                   "libnbzg.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
sass = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    txt = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True,
                         text=True).stdout
    fn, cur = None, None
    for l in txt.split("\n"):
        m = re.match(r"\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
            sass[fn] = []
            continue
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m and fn:
            sass[fn].append((cur, m.group(2)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base",
                      "mangled", "-k", "regex:" + ncu_k, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # next profiled kernel
    if len(r) == len(hdr):
        data.append(r)
cands = [f for f in sass if kern in f and len(sass[f]) == len(data)]
if not cands:
    sys.exit(f"no SASS function matching {kern} with {len(data)} instructions: " +
             str([(f, len(v)) for f, v in sass.items() if kern in f]))
ins = sass[cands[0]]
agg = collections.defaultdict(lambda: [0, 0, 0])
for (loc, txt), r in zip(ins, data):
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ie = int(r[ix["Instructions Executed"]] or 0)
    ti = int(r[ix["Thread Instructions Executed"]] or 0)
    a = agg[loc]
    a[0] += st
    a[1] += ie
    a[2] += ti
S = sum(v[0] for v in agg.values()) or 1
I = sum(v[1] for v in agg.values()) or 1
print(f"{cands[0]}: {S} stall samples, {I} warp instructions")
for loc, (st, ie, ti) in sorted(agg.items(), key=lambda kv: -kv[1][1 if os.environ.get("BY_INST") else 0])[:top]:
    print(f"{100*st/S:5.1f}% stall {100*ie/I:5.1f}% inst  {ti/max(ie,1):4.1f} thr  {loc}")
