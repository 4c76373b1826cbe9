#!/usr/bin/env python3
"""Group an ncu SASS source page into runs of equal execution count (basic
blocks, roughly) and print the heaviest:  python scripts/ncu_runs.py REP [launch] [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
launch = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None and len(r) == len(cur[1]):
        cur[2].append(r)
name, h, data = blocks[launch]
ix = {k: i for i, k in enumerate(h)}
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print(name, "warp instructions", tot)
runs = []
for n, r in enumerate(data):
    ie = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if runs and abs(runs[-1][2] - ie) <= max(1, 0.02 * ie):
        runs[-1][1] = n; runs[-1][3] += ie; runs[-1][4] += st
    else:
        runs.append([n, n, ie, ie, st])
S = sum(x[4] for x in runs) or 1
for a, b, ie, sm, st in sorted(runs, key=lambda x: -x[3])[:top]:
    print(f"{a:5d}-{b:5d} n={b - a + 1:4d} each={ie / 1e6:7.3f}M inst={100 * sm / tot:5.1f}% "
          f"stall={100 * st / S:5.1f}% {data[a][ix['Source']].strip()[:60]}")
