#!/usr/bin/env python3
"""Empty-space statistics of the C2 bench state at given steps: the share of
8^3-cell bricks whose 9^3 lattice sigma are all < 0 ("dead": no march
position inside can be composited), and the share of the march positions of
one batch that fall in dead bricks (from the positions' cells)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402
from paper_2112_05131_b200.camera import all_rays  # noqa: E402

steps = [int(x) for x in (sys.argv[1:] or ["5", "25", "2000"])]
dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


cfg = bench.bench_config(A)
tr = trainer.Trainer(ds, cfg, device=dev)
o, m, v, gt = all_rays(ds.images, ds.cameras)
rng = np.random.default_rng(0)
sel = rng.integers(0, o.shape[0], 2000)
ot = torch.from_numpy(o[sel]).to(dev)
dt = torch.from_numpy(np.ascontiguousarray(m[sel])).to(dev)
done = 0
for target in steps:
    while done < target:
        tr.step(done)
        done += 1
    torch.cuda.synchronize()
    g = tr.grid
    D = g.dims
    s = g.density.view(1, 1, *D).float()
    pad = F.pad(s, (0, 8 * 33 + 1 - D[2], 0, 8 * 33 + 1 - D[1], 0, 8 * 33 + 1 - D[0]),
                value=-1e30)
    bmax = F.max_pool3d(pad, kernel_size=9, stride=8)[0, 0]
    nb = [(d - 2) // 8 + 1 for d in D]
    bmax = bmax[:nb[0], :nb[1], :nb[2]]
    dead = bmax < 0
    # march positions of the rays (reference step rule), their cells, bricks
    lo = torch.tensor(cfg.aabb[:3], device=dev, dtype=torch.float64)
    hi = torch.tensor(cfg.aabb[3:], device=dev, dtype=torch.float64)
    scale = (torch.tensor(D, device=dev, dtype=torch.float64) - 1) / (hi - lo)
    inv = 1.0 / torch.where(dt.abs() < 1e-15, torch.full_like(dt, 1e-15), dt)
    ta, tb = (lo - ot) * inv, (hi - ot) * inv
    t0 = torch.minimum(ta, tb).amax(1).clamp_min(0)
    t1 = torch.maximum(ta, tb).amin(1)
    step = cfg.step_frac / scale.max()
    tot = 0
    in_dead = 0
    for r in range(ot.shape[0]):
        if t1[r] <= t0[r]:
            continue
        t = torch.arange(t0[r].item(), t1[r].item(), step.item(), device=dev, dtype=torch.float64)
        gp = ((ot[r] + t[:, None] * dt[r]) - lo) * scale
        c = gp.long().clamp(min=0)
        c = torch.minimum(c, torch.tensor(D, device=dev) - 2)
        b = c // 8
        tot += t.numel()
        in_dead += int(dead[b[:, 0], b[:, 1], b[:, 2]].sum())
    print(f"step {target}: dead bricks {dead.float().mean().item():.3f}  "
          f"positions in dead bricks {in_dead / max(tot, 1):.3f} of {tot}", flush=True)
