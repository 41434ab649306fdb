#!/usr/bin/env python3
"""Empty-space statistics at the C5 state (sweep_c5.py's 512^3 toy-sparse grid
after a few training steps): the share of k^3-cell bricks whose (k+1)^3
lattice sigma are all <= 0 or empty ("dead": no march position inside can be
composited, K:211), and the share of one batch's march positions inside
dead bricks, for k = 4, 8, 16."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2112_05131_b200 import grid as gmod, optim, render, scenes, trainer  # noqa: E402

dev = torch.device("cuda", 0)
gt64 = scenes.build_toy_grid(64, device=dev)
g512 = gt64.upsample((512, 512, 512))
cams, _ = scenes.hemisphere_cameras(64, 512, phase=1.0)
opts = render.RenderOptions(background=(1.0, 1.0, 1.0))
imgs = [(np.rint(np.clip(render.render_image(gt64, c, opts), 0, 1) * 255) / 255).astype(np.float32)
        for c in cams]
ds = scenes.Dataset(np.stack(imgs), cams)
cfg = trainer.default_config("bounded")
cfg.aabb = (-1.1, -1.1, -1.1, 1.1, 1.1, 1.1)
cfg.ladder = [trainer.LadderRung(0, (8, 8, 8))]
cfg.lambda_tv_sigma = cfg.lambda_tv_sh = 0.0
cfg.batch_size = 1 << 16
tr = trainer.Trainer(ds, cfg, device=dev)
tr.grid = g512.copy()
tr.state = optim.OptimState(tr.grid.n_rows, device=dev)
tr.grads = gmod.GradientBuffer(tr.grid.n_rows, device=dev)
tr._refresh_cache()
for s in range(int(os.environ.get("STEPS", 5))):
    tr.step(s)
torch.cuda.synchronize()
g = tr.grid
D = g.dims
lat, _ = g.lattice_sigma()
s = lat.view(*D).float().clone()
s[torch.isnan(s)] = -1e30
s = s.view(1, 1, *D)
from paper_2112_05131_b200.camera import all_rays  # noqa: E402
rng = np.random.default_rng(0)
views = rng.integers(0, len(cams), 8)
o, m, v, gt = all_rays(ds.images[views], [cams[i] for i in views])
sel = rng.integers(0, o.shape[0], 1500)
ot = torch.from_numpy(o[sel]).to(dev)
dt = torch.from_numpy(np.ascontiguousarray(m[sel])).to(dev)
lo = torch.tensor(cfg.aabb[:3], device=dev, dtype=torch.float64)
hi = torch.tensor(cfg.aabb[3:], device=dev, dtype=torch.float64)
scale = (torch.tensor(D, device=dev, dtype=torch.float64) - 1) / (hi - lo)
inv = 1.0 / torch.where(dt.abs() < 1e-15, torch.full_like(dt, 1e-15), dt)
ta, tb = (lo - ot) * inv, (hi - ot) * inv
t0 = torch.minimum(ta, tb).amax(1).clamp_min(0)
t1 = torch.maximum(ta, tb).amin(1)
step = cfg.step_frac / scale.max()
cells = []
for r in range(ot.shape[0]):
    if t1[r] <= t0[r]:
        continue
    t = torch.arange(t0[r].item(), t1[r].item(), step.item(), device=dev, dtype=torch.float64)
    gp = ((ot[r] + t[:, None] * dt[r]) - lo) * scale
    c = gp.long().clamp(min=0)
    cells.append(torch.minimum(c, torch.tensor(D, device=dev) - 2))
cells = torch.cat(cells)
for k in (4, 8, 16):
    nb = [(d - 2) // k + 1 for d in D]
    pad = F.pad(s, (0, k * nb[2] + 1 - D[2], 0, k * nb[1] + 1 - D[1], 0, k * nb[0] + 1 - D[0]),
                value=-1e30)
    bmax = F.max_pool3d(pad, kernel_size=k + 1, stride=k)[0, 0][:nb[0], :nb[1], :nb[2]]
    dead = bmax <= 0
    b = cells // k
    pin = dead[b[:, 0], b[:, 1], b[:, 2]].float().mean().item()
    print(f"k={k}: dead bricks {dead.float().mean().item():.3f}, march positions in dead bricks "
          f"{pin:.3f} of {cells.shape[0]}", flush=True)
