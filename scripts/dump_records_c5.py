#!/usr/bin/env python3
"""Dump one C5 step's composited-sample cells (512^3 toy-sparse grid, single
wave: B = 2^15 and 40000 rays) -> gpurun_out/records_c5_<B>.npz."""
import os
os.environ.setdefault("PLX_PACK", "0")   # reads the unpacked cell array
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2112_05131_b200 import grid as gmod, optim, render, scenes, trainer
    dev = torch.device("cuda", 0)
    gt64 = scenes.build_toy_grid(64, device=dev)
    g512 = gt64.upsample((512, 512, 512))
    cams, _ = scenes.hemisphere_cameras(64, 512, phase=1.0)
    opts = render.RenderOptions(background=(1.0, 1.0, 1.0))
    imgs = []
    for cam in cams:
        img = render.render_image(gt64, cam, opts)
        imgs.append((np.rint(np.clip(img, 0, 1) * 255) / 255).astype(np.float32))
    ds = scenes.Dataset(np.stack(imgs), cams)
    cfg = trainer.default_config("bounded")
    cfg.aabb = (-1.1, -1.1, -1.1, 1.1, 1.1, 1.1)
    cfg.ladder = [trainer.LadderRung(0, (8, 8, 8))]
    cfg.lambda_tv_sigma = cfg.lambda_tv_sh = 0.0
    for B in (1 << 15, 40000):
        cfg.batch_size = B
        tr = trainer.Trainer(ds, cfg, device=dev)
        tr.grid = g512.copy()
        tr.state = optim.OptimState(tr.grid.n_rows, device=dev)
        tr.grads = gmod.GradientBuffer(tr.grid.n_rows, device=dev)
        tr._refresh_cache()
        for s in range(4):
            tr.step(s)
        torch.cuda.synchronize()
        g = tr.grid
        step = tr._kopts.step
        lo, hi = np.array(g.aabb_min, float), np.array(g.aabb_max, float)
        cap = int(math.ceil(math.sqrt(((hi - lo) ** 2).sum()) / step)) + 4
        nseg_max = (cap + 31) // 32
        off = 256
        offs = {}
        n = B * cap
        for name, nb in [("ns", B * 4), ("segfirst", B * 4), ("segray", B * nseg_max * 4),
                         ("rayd", B * 24), ("basis", B * 48), ("att", n * 8), ("T", n * 8),
                         ("w", n * 8), ("c", n * 16), ("cell", n * 16)]:
            offs[name] = off
            off = (off + nb + 255) & ~255
        buf = tr._scratch_keep
        ns = buf[offs["ns"]:offs["ns"] + B * 4].view(torch.int32).cpu().numpy()
        cell = buf[offs["cell"]:offs["cell"] + n * 16].view(torch.int32).view(B, cap, 4)
        sel = [cell[r, :ns[r]].cpu().numpy() for r in range(B) if ns[r] > 0]
        ray = np.concatenate([np.full(ns[r], r, np.int32) for r in range(B)])

        np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"records_c5_{B}.npz"), ns=ns, ray=ray,
                            cell=np.concatenate(sel), dims=np.array(g.dims), cap=cap)
        print(B, "samples", int(ns.sum()), "cap", cap, "rows", g.n_rows)



main()
