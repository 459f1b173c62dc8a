#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (mixed sass,cuda source view).
Usage: python tools/ncu_lines.py <report.ncu-rep> [units_for_normalisation] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = {}
fn = ""
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
    if len(r) < 8 or r[0] in ("Line No", "File Path", "Function Name") or not r[0]:
        continue
    try:
        e, smp = float(r[7]), float(r[4])
    except ValueError:
        continue
    key = (int(r[0]), r[1].strip()[:80])
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += e
    a[1] += smp
tot = sum(v[0] for v in agg.values())
print(f"total instructions {tot:.4g}  per unit {tot / units:.1f}")
for (ln, src), (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {e / units:9.1f} {100 * e / tot:5.1f}% samples {s:7.0f}  {src}")
