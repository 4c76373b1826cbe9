#!/usr/bin/env python3
"""Print the headline metrics and top stall reasons of an ncu report:
    python scripts/ncu_metrics.py gpurun_out/x.ncu-rep [launch-index]"""
import csv, subprocess, sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
v = rows[2 + idx]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in want:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]}")
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:8]))
