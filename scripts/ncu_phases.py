#!/usr/bin/env python3
"""Stall-reason breakdown per source-line range (kernel phase) of one kernel
in an .ncu-rep.  usage: python scripts/ncu_phases.py REP name=file:lo-hi,..."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, spec = sys.argv[1], sys.argv[2]
groups = []
for g in spec.split(","):
    name, rng = g.split("=")
    f, lohi = rng.split(":")
    lo, hi = map(int, lohi.split("-"))
    groups.append((name, f, lo, hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
REASONS = ["stall_long_sb", "stall_short_sb", "stall_mio", "stall_lg", "stall_wait", "stall_math",
           "stall_branch_resolving", "stall_barrier", "stall_no_inst", "stall_not_selected",
           "stall_selected", "stall_dispatch", "stall_drain", "stall_membar", "stall_tex",
           "stall_misc"]
agg = defaultdict(lambda: defaultdict(float))
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    ln = int(r[0])
    key = "other"
    for name, f, lo, hi in groups:
        if fname == f and lo <= ln <= hi:
            key = name
            break
    for k in REASONS + ["Warp Stall Sampling (All Samples)", "Instructions Executed"]:
        try:
            agg[key][k] += float(d.get(k, 0) or 0)
        except ValueError:
            pass
tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values()) or 1
toti = sum(a["Instructions Executed"] for a in agg.values()) or 1
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"]):
    s = a["Warp Stall Sampling (All Samples)"]
    top = sorted(((a[k], k) for k in REASONS), reverse=True)[:4]
    print(f"{key:10s} stall {100 * s / tot:5.1f}%  inst {100 * a['Instructions Executed'] / toti:5.1f}%  " +
          "  ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for v, k in top))
