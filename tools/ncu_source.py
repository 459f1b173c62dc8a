#!/usr/bin/env python
"""Per-instruction warp-stall samples from an ncu report's SASS source page.
Usage: python tools/ncu_source.py <report.ncu-rep> [top_n] [kernel_regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 3:
        cmd += ["-k", "regex:" + sys.argv[3]]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    print(f"instructions {len(data)}, samples {tot}")
    ops = Counter()
    stalls = Counter()
    for d in data:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        op = d["Source"].split()[0] if d["Source"].strip() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        ops[op.split(".")[0]] += s
        for c in stall_cols:
            stalls[c] += int(d[c] or 0)
    print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(14)))
    print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in stalls.most_common(10)))
    print(f"top {top} instructions:")
    idx = sorted(range(len(data)), key=lambda i: -int(data[i]["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for i in sorted(idx):
        d = data[i]
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        reasons = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{n}:{v}" for v, n in reasons if v)
        print(f"{i:5d} {s / tot:6.2%} {d['Source'].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
