#!/usr/bin/env python3
"""Gradient error statistics of the device fused backward vs the f64 oracle
on a trained toy-scene grid (mid-training state): per column class, the
relative L2 error and the signed bias sum(ours - oracle) / sum|oracle|."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import load  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2112_05131_b200 import losses, trainer  # noqa: E402
from paper_2112_05131_b200.camera import all_rays  # noqa: E402
from paper_2112_05131_b200.scenes import dataset_from_arrays  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
z = load("toy128.npz")
ds = dataset_from_arrays(z["imgs"], z["c2w"], z["focal"], tag="train")
cfg = trainer.toy_config(grid_dim=64, total_steps=5000, batch_size=3000)
cfg.eval_every = cfg.log_every = 0
tr = trainer.Trainer(ds, cfg)
for s in range(steps):
    tr.step(s)
torch.cuda.synchronize()
g = tr.grid
links, table = g.to_numpy()
og = orc.Grid(links, table.astype(np.float64), g.aabb_min, g.aabb_max)
o, m, v, gt = all_rays(ds.images, ds.cameras)
rng = np.random.default_rng(5)
idx = rng.permutation(o.shape[0])[:3000]
bo = orc.GradBuf(og.n_rows)
_, mse_o, _ = orc.fused_mse_backward(og, o[idx], m[idx], v[idx], gt[idx], bo, len(idx),
                                     step_frac=cfg.step_frac, stop_thresh=cfg.stop_thresh,
                                     background=cfg.background)
import paper_2112_05131_b200 as px  # noqa: E402
bd = px.GradientBuffer(g.n_rows)
_, mse_d, _ = px.fused_mse_backward(g, o[idx], m[idx], v[idx], gt[idx], bd, tr.opts,
                                    n_total=len(idx))
gd, go = bd.dense(), bo.data
print(f"after {steps} steps: mse dev {mse_d:.9e} oracle {mse_o:.9e}  touched {bd.n_touched} / "
      f"{bo.n_touched}")
for name, cols in (("sigma", [0]), ("DC", [1, 10, 19]), ("SH>0", [c for c in range(1, 28)
                                                                if c not in (1, 10, 19)])):
    a, b = gd[:, cols].ravel(), go[:, cols].ravel()
    l2 = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    bias = (a - b).sum() / max(np.abs(b).sum(), 1e-300)
    sign = np.mean(np.sign(a[b != 0]) != np.sign(b[b != 0]))
    print(f"  {name:6s} rel L2 {l2:.3e}  bias {bias:+.3e}  sign flips {sign:.2e}  "
          f"zero-mismatch {np.mean((a == 0) != (b == 0)):.2e}")
