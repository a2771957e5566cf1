#!/usr/bin/env python
"""Summarise an `ncu --set full` report into a short text file for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--units N --bytes-per-unit B] > profiles/rNN_x.txt

Prints the speed-of-light block, pipe utilisation, DRAM bytes per launch,
warp-stall samples and the SASS opcode mix (per launch and per work unit).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import re
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", type=float, default=0.0, help="work units per launch (e.g. token-heads)")
    ap.add_argument("--unit-name", default="unit")
    ap.add_argument("--bytes-per-unit", type=float, default=0.0)
    a = ap.parse_args()

    raw = ncu_csv(a.report, "--page", "raw")
    h, v = raw[0], raw[2]
    m = dict(zip(h, v))
    name = m.get("Kernel Name", "?")
    print(f"kernel: {name}")
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
            "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sass__inst_executed_local_loads"]
    for k in keys:
        if k in m:
            print(f"  {k:60s} {m[k]} {raw[1][h.index(k)]}")
    print("pipes (% of peak, active cycles):")
    for k in h:
        if re.match(r"sm__inst_executed_pipe_\w+\.avg\.pct_of_peak_sustained_active$", k) or \
           re.match(r"sm__pipe_\w+_cycles_active\.avg\.pct_of_peak_sustained_active$", k):
            try:
                if float(m[k]) >= 0.5:
                    print(f"  {k:70s} {m[k]}")
            except ValueError:
                pass
    print("warp stall samples:")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(m[k] or 0)) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    for k, x in sorted(st.items(), key=lambda t: -t[1])[:12]:
        print(f"  {k:28s} {x:7d} {100.0 * x / tot:5.1f}%")

    src = ncu_csv(a.report, "--page", "source", "--print-source", "sass")
    hh = src[1]
    iS, iE = hh.index("Source"), hh.index("Instructions Executed")
    ops = collections.Counter()
    for r in src[2:]:
        mm = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS])
        if mm:
            ops[mm.group(2)] += int(r[iE] or 0)
    total = sum(ops.values())
    per = f" per {a.unit_name}" if a.units else ""
    print(f"SASS warp-instructions executed: {total}" + (f" ({total / a.units:.2f}{per})" if a.units else ""))
    for k, x in ops.most_common(28):
        extra = f" {x / a.units:7.3f}{per}" if a.units else ""
        print(f"  {k:10s} {x:10d}{extra}")
    if a.units and a.bytes_per_unit:
        t = float(m["gpu__time_duration.sum"])
        tu = raw[1][h.index("gpu__time_duration.sum")]
        scale = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(tu, 1e-9)
        alg = a.units * a.bytes_per_unit
        print(f"algorithmic bytes per launch {alg / 1e6:.1f} MB -> {alg / (t * scale) / 1e9:.0f} GB/s "
              f"(cold-cache, serialised launch under ncu)")


if __name__ == "__main__":
    main()
