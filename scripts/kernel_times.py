#!/usr/bin/env python3
"""Per-kernel device times of the C2 training step in steady operation (warm
caches, normal overlap) via torch.profiler/CUPTI -- complements the ncu
launch list, whose per-launch times are serialised and cold-cache.

usage: python scripts/kernel_times.py [steps] [warm_to_step]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


tr = trainer.Trainer(ds, bench.bench_config(A), device=dev)
for s in range(warm):
    tr.step(s)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(warm, warm + steps):
        tr.step(s)
    torch.cuda.synchronize()
agg = defaultdict(list)
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg[e.name[:70]].append(e.device_time)
# idle gaps between consecutive device operations (launch latency etc.)
evs = sorted(((e.time_range.start, e.time_range.end, e.name[:40]) for e in prof.events()
              if e.device_type.name == "CUDA"))
spans = [(a, b) for a, b, _ in evs]
gaps, end = [], None     # idle = time covered by no operation (streams overlap)
for a, b in spans:
    if end is not None:
        gaps.append(max(0.0, a - end))
    end = b if end is None else max(end, b)
big = [g for g in gaps if g > 50.0]
if os.environ.get("KT_TIMELINE"):   # the ops of the last two steps, in start order
    n_last = 2 * max(1, len(evs) // steps)
    t0, end = evs[-n_last][0], None
    for a, b, name in evs[-n_last:]:
        idle = 0.0 if end is None else max(0.0, a - end)
        end = b if end is None else max(end, b)
        print(f"  +{a - t0:8.1f} us  {b - a:7.1f} us  idle before {idle:5.1f}  {name}")
print(f"device idle between ops: {sum(g for g in gaps if g <= 50.0) / steps:7.1f} us/step "
      f"(+ {len(big)} gaps > 50 us totalling {sum(big):.0f} us)")
tot = 0.0
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    tot += sum(v)
    print(f"{sum(v) / steps:9.1f} us/step  n/step={len(v) / steps:4.1f}  {k}")
print(f"{tot / steps:9.1f} us/step total device time")

# host cost of a step call vs the device step time (no profiler)
import time  # noqa: E402

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
host = 0.0
e0.record()
for s in range(warm + steps, warm + 2 * steps):
    h0 = time.perf_counter()
    tr.step(s)
    host += time.perf_counter() - h0
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1) * 1000 / steps:9.1f} us device-timed, "
      f"{host * 1e6 / steps:9.1f} us host per tr.step() call")

# pure host cost of enqueueing a step (no divergence checks, GPU runs behind)
torch.cuda.synchronize()
h0 = time.perf_counter()
for s in range(warm + 2 * steps, warm + 3 * steps):
    tr.step(s, check_finite=False)
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue only: {(h1 - h0) * 1e6 / steps:9.1f} us per tr.step(check_finite=False)")
