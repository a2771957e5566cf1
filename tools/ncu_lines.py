#!/usr/bin/env python
"""Per-source-line instruction counts of one kernel in an ncu report (needs -lineinfo):
usage: tools/ncu_lines.py REPORT.ncu-rep [WORK_UNITS] [MIN_PER_UNIT]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, res = None, []
for x in csv.reader(io.StringIO(out)):
    if len(x) == 2 and x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if len(x) < 8 or x[0] in ("Line No", ""):
        continue
    try:
        res.append((cur, int(x[0]), x[1][:90], int(x[7]), int(x[4])))
    except ValueError:
        pass
tot = sum(r[3] for r in res)
print(f"total {tot} instr = {tot / units:.1f} per unit; samples {sum(r[4] for r in res)}")
for r in sorted(res, key=lambda r: (r[0], r[1])):
    if r[3] / units >= thr:
        print(f"{r[0][:16]:16s} {r[1]:5d} {r[3] / units:7.1f} {r[4]:5d}  {r[2]}")
