#!/usr/bin/env python3
"""Dump the composited-sample records (ray, position, cell) of one C2 training
step at the headline state (step 5) and at step 2000 -> gpurun_out/records_<step>.npz
(for offline analysis of sample sort orders / row sharing)."""
import os
os.environ.setdefault("PLX_PACK", "0")   # reads the unpacked cell array
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import trainer, _lib  # noqa: E402

dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


tr = trainer.Trainer(ds, bench.bench_config(A), device=dev)
g = tr.grid
step = tr._kopts.step
lo, hi = np.array(g.aabb_min, float), np.array(g.aabb_max, float)
cap = int(math.ceil(math.sqrt(((hi - lo) ** 2).sum()) / step)) + 4
B = 5000
nseg_max = (cap + 31) // 32
off = 256
offs = {}
def take(name, nbytes):
    global off
    offs[name] = off
    off = (off + nbytes + 255) & ~255
n = B * cap
for name, nb in [("ns", B * 4), ("segfirst", B * 4), ("segray", B * nseg_max * 4), ("rayd", B * 24),
                 ("basis", B * 48), ("att", n * 8), ("T", n * 8), ("w", n * 8), ("c", n * 16),
                 ("cell", n * 16), ("f", n * 16), ("rows", n * 32), ("sig", n * 8), ("segsum", B * nseg_max * 48)]:
    take(name, nb)
buf = tr._scratch_keep
out = os.path.join("gpurun_out")
os.makedirs(out, exist_ok=True)
s = 0
for target in (5, 2000):
    while s <= target:
        tr.step(s)
        s += 1
    torch.cuda.synchronize()
    ns = buf[offs["ns"]:offs["ns"] + B * 4].view(torch.int32).cpu().numpy()
    cell = buf[offs["cell"]:offs["cell"] + n * 16].view(torch.int32).view(B, cap, 4).cpu().numpy()
    rays, js = [], []
    sel = [cell[r, :ns[r]] for r in range(B)]
    ray = np.concatenate([np.full(ns[r], r, np.int32) for r in range(B)])
    np.savez_compressed(os.path.join(out, f"records_{target}.npz"), ns=ns, ray=ray,
                        cell=np.concatenate(sel), dims=np.array(g.dims))
    print(target, "samples", int(ns.sum()), "cap", cap)
