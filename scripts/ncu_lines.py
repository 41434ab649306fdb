#!/usr/bin/env python3
"""Per-CUDA-source-line hot spots of one kernel in an .ncu-rep (needs -lineinfo):
warp-stall samples and executed warp instructions aggregated by ncu per line.

usage: python scripts/ncu_lines.py <rep> [top_n] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        st = int(d["Warp Stall Sampling (All Samples)"])
        ins = int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    rows.append((st, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for st, ins, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*st/tot_s:5.1f}% stall {100*ins/tot_i:5.1f}% inst  {loc:22s} {src}")

if len(sys.argv) > 3:   # optional grouping: name=file:lo-hi,...
    groups = []
    for spec in sys.argv[3].split(","):
        name, rng = spec.split("=")
        f, lohi = rng.split(":")
        lo, hi = map(int, lohi.split("-"))
        groups.append((name, f, lo, hi))
    agg = {g[0]: [0, 0] for g in groups}
    agg["other"] = [0, 0]
    for st, ins, loc, _ in rows:
        f, ln = loc.rsplit(":", 1)
        for name, gf, lo, hi in groups:
            if f == gf and lo <= int(ln) <= hi:
                agg[name][0] += st
                agg[name][1] += ins
                break
        else:
            agg["other"][0] += st
            agg["other"][1] += ins
    for k, (st, ins) in agg.items():
        print(f"{k:14s} stall {100*st/tot_s:5.1f}%  inst {100*ins/tot_i:5.1f}%")
