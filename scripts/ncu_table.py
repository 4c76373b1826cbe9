#!/usr/bin/env python3
"""Per-launch table of an `ncu --set full` report: time, DRAM bytes, issue /
warp activity, the busiest pipes and the top stall reasons.
    python scripts/ncu_table.py REPORT.ncu-rep [--json traffic.json]"""
import csv, json, re, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]


def g(r, k, f=float):
    try:
        return f(r[h.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return None


out, traffic = [], {}
print("| kernel | ms | DRAM GB (r+w) | issue % | warps % | L1TEX % | ALU % | top stalls |")
print("|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "")
    ms = g(r, "gpu__time_duration.sum")
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    unit = r[h.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h else ""
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    stalls = ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:3])
    print(f"| {name} | {ms:.3f} | {rd:.3f} + {wr:.3f} | "
          f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{g(r, 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.0f} | {stalls} |")
    short = {"minmax_seg_kernel": "minmax6", "rindex_csort_kernel": "rindex_sort",
             "quantize_kernel<1>": "quantize", "encode_tpc_kernel": "encode",
             "decode_lv_kernel": "dq_decode"}.get(name)
    if short:  # GB (ncu's unit) -> bytes, summed over the launches of the stage
        traffic[short] = traffic.get(short, 0) + int(round((rd + wr) * 1e9))
if len(sys.argv) > 3 and sys.argv[2] == "--json":
    json.dump(traffic, open(sys.argv[3], "w"), indent=1)
