#!/usr/bin/env python3
"""Summarise ncu captures (.ncu-rep) and launch lists (.csv) into profiles/.

usage: python scripts/ncu_summary.py <tag> <rep> [<rep> ...] [--launches csv] [--no-traffic]
Writes profiles/<tag>_ncu.md and merges per-kernel DRAM bytes into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""

import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 red requests"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / instr"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (u, v) for h, u, v in zip(hdr, units, r)})
    return recs


def stalls(rec):
    out = []
    for h, (u, v) in rec.items():
        if h.startswith("smsp__average_warp_latency_issue_stalled") or (
                "warp_issue_stalled" in h and h.endswith("per_warp_active.pct")):
            try:
                out.append((float(v), h))
            except ValueError:
                pass
    return sorted(out, reverse=True)[:6]


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    launches = None
    if "--launches" in sys.argv:
        launches = sys.argv[sys.argv.index("--launches") + 1]
    os.makedirs("profiles", exist_ok=True)
    traffic_path = "profiles/ncu_traffic.json"
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lines = [f"# ncu summary `{tag}`", ""]
    sums = {}
    for rep in reps:
        for rec in raw(rep):
            name = rec.get("Kernel Name", ("", "?"))[1]
            lines += [f"## {name}", f"source: `{os.path.basename(rep)}` (ncu --set full, "
                      "--clock-control none; cold-cache single replayed launch)", "",
                      "| metric | value |", "|---|---|"]
            for k, label in KEYS:
                if k in rec:
                    u, v = rec[k]
                    lines.append(f"| {label} (`{k}`) | {v} {u} |")
            st = stalls(rec)
            if st:
                lines += ["", "top stall reasons (per-warp-active %):", ""]
                lines += [f"- {h}: {v:.1f}" for v, h in st]
            lines.append("")
            try:
                rd = float(rec["dram__bytes_read.sum"][1]) * UNIT[rec["dram__bytes_read.sum"][0]]
                wr = float(rec["dram__bytes_write.sum"][1]) * UNIT[rec["dram__bytes_write.sum"][0]]
                # the bench's per-step legs: the backward is three kernels, the
                # update two (their DRAM bytes add up per launch of the leg)
                key = ("render_fused_bwd" if any(k in name for k in
                                                 ("march_bwd_kernel", "colour_kernel",
                                                  "scatter_kernel"))
                       else "opt_step" if any(k in name for k in
                                              ("opt_rows_kernel", "touched_compact"))
                       else "tv" if ("tv_dense_kernel" in name or "tv_sparse_kernel" in name or "plx::tv_kernel" in name) else None)
                if key:
                    sums[key] = sums.get(key, 0.0) + rd + wr
            except (KeyError, ValueError):
                pass
    if "--no-traffic" not in sys.argv:
        traffic.update(sums)
    if launches:
        text = open(launches).read().splitlines()
        start = [i for i, l in enumerate(text) if l.startswith('"ID"')][0]
        rows = list(csv.reader(text[start:]))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            try:
                agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
            except (ValueError, IndexError):
                pass
        lines += ["## launch list (gpu__time_duration.sum, serialised, cold cache)", "",
                  "| kernel | launches | mean us | total ms |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e6:.3f} |")
    with open(f"profiles/{tag}_ncu.md", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print(f"wrote profiles/{tag}_ncu.md")


if __name__ == "__main__":
    main()
