#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (our kernels vs input generation) and the key counters of a
--set full capture.  Usage:
  python tools/ncu_summary.py launches <launches.csv> <out.txt>
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [traffic_key pairs_per_launch]
"""
import csv
import json
import os
import re
import subprocess
import sys

OURS = re.compile(r"ttc::|inner_|contract_kernel|splice_kernel|reconstruct_kernel|ttsvd_")


def short(name):
    m = re.search(r"(inner_r16_kernel|inner_r64_kernel|inner_r64tc_kernel|inner_ffma_kernel|inner_tc_kernel<[^>]*>|inner_generic_kernel|contract_kernel|splice_kernel|reconstruct_kernel|ttsvd_kernel)", name)
    return m.group(1) if m else name.split("(")[0][-60:]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    data = [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    ours = [d for d in data if OURS.search(d["Kernel Name"])]
    other = [d for d in data if not OURS.search(d["Kernel Name"])]
    tot_ours = sum(float(d["Metric Value"]) for d in ours)
    lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised launches)",
             f"launches: {len(data)} total, {len(ours)} of ours, {len(other)} others (input generation / torch)",
             f"{'ID':>5} {'kernel':40s} {'grid':>12} {'block':>12} {'ns':>10}"]
    for d in ours:
        lines.append(f"{d['ID']:>5} {short(d['Kernel Name']):40s} {d['Grid Size']:>12} {d['Block Size']:>12} "
                     f"{float(d['Metric Value']):>10.0f}")
    lines.append(f"sum of our launches: {tot_ours:.0f} ns; mean {tot_ours / max(1, len(ours)):.0f} ns per launch")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:3] + lines[-1:]))


def full(rep, out, key=None, pairs=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
            "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__cycles_active.avg",
            "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct"]
    lines = [f"ncu --set full --clock-control none capture of {os.path.basename(rep)}"]
    for k in want:
        if k in d:
            lines.append(f"{k:60s} {d[k]} {u.get(k, '')}")
    stalls = []
    for k, v in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if m:
            try:
                stalls.append((float(v), m.group(1)))
            except ValueError:
                pass
    lines.append("warp stall reasons (cycles per issued instruction):")
    for v, k in sorted(stalls, reverse=True)[:10]:
        lines.append(f"  {k:30s} {v:.3f}")
    def num(k):
        try:
            x = float(d[k].replace(",", ""))
        except Exception:
            return None
        unit = u.get(k, "")
        return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    if rd is not None and wr is not None:
        lines.append(f"DRAM traffic per launch: {rd + wr:.6g} bytes (read {rd:.6g}, write {wr:.6g})")
        if key:
            tp = os.path.join(os.path.dirname(out), "traffic.json")
            tj = json.load(open(tp)) if os.path.exists(tp) else {}
            tj[key] = {"bytes": rd + wr, "pairs": int(pairs) if pairs else None,
                       "source": os.path.basename(out)}
            json.dump(tj, open(tp, "w"), indent=1)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None,
             sys.argv[5] if len(sys.argv) > 5 else None)
