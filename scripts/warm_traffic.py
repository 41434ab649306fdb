#!/usr/bin/env python3
"""Per-leg warm-cache DRAM traffic of the bench's timed window from an ncu
capture (`ncu --cache-control none --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum --csv` of `bench.py --steps 20
--warmup 5 --no-cpu-baseline --steady-step 0`, scripts/gpu_final_r2.sh).

Launches are grouped into steps at each march_bwd_kernel (one per step at
C2); steps W..W+K-1 are averaged (the window `value` is measured over).
usage: python scripts/warm_traffic.py <csv> [W] [K] -> profiles/ncu_traffic.json"""
import csv
import io
import json
import sys
from collections import defaultdict

path = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
text = open(path).read()
body = text[text.index('"ID"'):]
launches = defaultdict(dict)
names = {}
for r in csv.DictReader(io.StringIO(body)):
    i = int(r["ID"])
    names[i] = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
             "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
    launches[i][r["Metric Name"]] = v * scale
LEG = {"march_bwd": "render_fused_bwd", "colour_kernel": "render_fused_bwd",
       "scatter_kernel": "render_fused_bwd", "seg_": "render_fused_bwd", "tv_dense_kernel": "tv", "tv_sparse_kernel": "tv", "::tv_kernel": "tv",
       "touched_compact": "opt_step", "opt_rows": "opt_step"}
steps, cur = [], None
for i in sorted(launches):
    n = names[i]
    if "march_bwd" in n:
        cur = defaultdict(float)
        steps.append(cur)
    if cur is None:
        continue
    leg = next((v for k, v in LEG.items() if k in n), None)
    if leg:
        m = launches[i]
        cur[leg] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
win = steps[W:W + K]
assert len(win) == K, (len(steps), W, K)
out = {leg: sum(s[leg] for s in win) / K for leg in ("tv", "render_fused_bwd", "opt_step")}
out["_source"] = ("ncu --cache-control none (warm caches, as in the pipeline), --metrics "
                  "dram__bytes_read/write, the %d timed steps (%d..%d, graph replays) of `bench.py "
                  "--steps %d --warmup %d --no-cpu-baseline --steady-step 0`, mean per step -- the "
                  "window bench.py's algorithmic bytes are averaged over; kernels serialised by ncu; "
                  "scripts/warm_traffic.py on %s" % (K, W, W + K - 1, K, W, path.split("/")[-1]))
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
