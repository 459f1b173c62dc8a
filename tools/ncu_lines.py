#!/usr/bin/env python
"""Per-source-line instructions executed and warp-stall samples from an ncu report (CUDA source view; needs
-lineinfo and --import-source on).  Usage: python tools/ncu_lines.py <report.ncu-rep> [top_n] [kernel_regex]"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(sys.argv) > 3:
        cmd += ["-k", "regex:" + sys.argv[3]]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    lines, cur = [], None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r[0].isdigit():
            lines.append((cur, int(r[0]), r[1].strip()[:90], num(r[4]), num(r[7])))
    ts = sum(x[3] for x in lines) or 1
    ti = sum(x[4] for x in lines) or 1
    print(f"samples {ts}, warp instructions {ti}")
    for f, ln, src, smp, ins in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"{f}:{ln:<5} samples {100 * smp / ts:5.1f}%  inst {100 * ins / ti:5.1f}%  {src}")


if __name__ == "__main__":
    main()
