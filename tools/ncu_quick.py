#!/usr/bin/env python
"""Quick look at an ncu report: key throughput counters, stall reasons, instruction mix, top stalled SASS.
Usage: python tools/ncu_quick.py <report.ncu-rep> [kernel_regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kf = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in d:
        print(f"{k:75s} {d[k]}")
st = [(k, float(val)) for k, val in d.items() if k.startswith("smsp__average_warp_latency_issue_stalled") or
      (k.startswith("smsp__warp_issue_stalled") and k.endswith("_per_warp_active.pct"))]
for k, val in sorted(st, key=lambda x: -x[1])[:12]:
    print(f"  stall {k:80s} {val:.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
ie = lambda x: float(x["Instructions Executed"] or 0)
ss = lambda x: float(x["Warp Stall Sampling (All Samples)"] or 0)
tot, tots = sum(map(ie, data)), sum(map(ss, data))
op, ops = Counter(), Counter()
for x in data:
    t = x["Source"].split()
    o = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")).split(".")[0]
    op[o] += ie(x)
    ops[o] += ss(x)
print(f"instructions executed {tot:.4g}, stall samples {tots:.0f}")
for k, val in op.most_common(16):
    print(f"  {k:10s} {val / tot * 100:6.2f}% inst {ops[k] / tots * 100:6.2f}% samples")
print("top stalled instructions:")
for x in sorted(data, key=ss, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    print(f"  {x['Address'][-5:]} {x['Source'][:64]:64s} exec {ie(x):10.0f} samples {ss(x):6.0f}")
