#!/usr/bin/env python3
"""Bench-state diagnostics (C2 workload): density sign statistics of the
grid after N training steps, the share of trilinear cells whose 8 corners
are all negative ("dead"), and the march counters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402

steps = [int(x) for x in (sys.argv[1:] or ["12"])]
dev = torch.device("cuda", 0)
args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


cfg = bench.bench_config(A)
tr = trainer.Trainer(ds, cfg, device=dev)
done = 0
for target in steps:
    while done < target:
        tr.step(done)
        done += 1
    g = tr.grid
    d = g.density.view(*g.dims)
    neg = d < 0
    dead = (neg[:-1, :-1, :-1] & neg[1:, :-1, :-1] & neg[:-1, 1:, :-1] & neg[:-1, :-1, 1:] &
            neg[1:, 1:, :-1] & neg[1:, :-1, 1:] & neg[:-1, 1:, 1:] & neg[1:, 1:, 1:])
    st0 = tr.march_stats.clone()
    tr.step(done)
    done += 1
    st = (tr.march_stats - st0).tolist()
    print(f"step {target}: rows sigma<0 {neg.float().mean().item():.3f}  sigma>0 "
          f"{(d > 0).float().mean().item():.3f}  dead cells {dead.float().mean().item():.3f}  "
          f"positions {st[0]}  samples {st[1]}  chunks {st[2]}  "
          f"U {tr.count.item()}", flush=True)
