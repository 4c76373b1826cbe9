#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches, mean and total time and share of our kernels' time.
    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.md"""
import collections, csv, re, sys

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name).replace("void ", "")
    short = re.sub(r"^nbzg::", "", short)
    ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else
                                     1e6 if r["Metric Unit"] == "ms" else 1.0)
    rows.append((short, ns, r["Grid Size"], r["Block Size"]))
agg = collections.OrderedDict()
for short, ns, g, b in rows:
    a = agg.setdefault(short, [0, 0.0, g, b])
    a[0] += 1
    a[1] += ns
ours = {k: v for k, v in agg.items() if "at::" not in k and "cub" not in k.lower()}
tot = sum(v[1] for v in ours.values()) or 1.0
print(f"# ncu launch list summary ({sys.argv[1]})\n")
print("cold-cache, serialised per-launch times (ncu); shares are of this library's kernels\n")
print("| kernel | launches | mean ms | total ms | share | grid | block |")
print("|---|---|---|---|---|---|---|")
for k, (c, ns, g, b) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {c} | {ns / c / 1e6:.3f} | {ns / 1e6:.2f} | {ns / tot:.1%} | {g} | {b} |")
others = {k: v for k, v in agg.items() if k not in ours}
if others:
    print(f"\nother (torch) kernels: {sum(v[0] for v in others.values())} launches, "
          f"{sum(v[1] for v in others.values()) / 1e6:.2f} ms")
