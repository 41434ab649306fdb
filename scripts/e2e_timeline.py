#!/usr/bin/env python3
"""Device timeline of the e2e leg (Trainer.step_rays with packed pinned host
batches) on the C2 bench state: per-op start offsets, durations and the idle
time before each, for the last two profiled steps (CUPTI via torch.profiler)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402
from paper_2112_05131_b200.camera import all_rays  # noqa: E402

dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


tr = trainer.Trainer(ds, bench.bench_config(A), device=dev)
for s in range(5):
    tr.step(s)
o, m, v, gt = all_rays(ds.images, ds.cameras)
rng = np.random.default_rng(0)
host = []
for _ in range(16):
    sel = rng.integers(0, o.shape[0], 5000)
    host.append(torch.from_numpy(np.stack([a[sel] for a in (o, m, v, gt)])).pin_memory())
for i in range(4):
    tr.step_rays(5 + i, host[i])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(8):
        tr.step_rays(9 + i, host[4 + i])
    tr.check_pending()
    torch.cuda.synchronize()
evs = sorted((e.time_range.start, e.time_range.end, e.name[:50]) for e in prof.events()
             if e.device_type.name == "CUDA")
n = len(evs) // 8 * 2
t0, end = evs[-n][0], None
for a, b, name in evs[-n:]:
    idle = 0.0 if end is None else max(0.0, a - end)
    end = b if end is None else max(end, b)
    print(f"  +{a - t0:8.1f} us  {b - a:7.1f} us  idle before {idle:5.1f}  {name}")
