#!/usr/bin/env python3
"""Row sharing of one large C5 wave (512^3 toy-sparse grid): distinct rows vs
the (segment, row) loads of the ray-order segments vs Morton-sorted sample
chunks.  Computed on the device from the render scratch after a step.
usage: python scripts/share_stats_c5.py [B]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def morton(c, bits=10):
    m = torch.zeros(c.shape[0], dtype=torch.int64, device=c.device)
    for b in range(bits):
        for a in range(3):
            m |= ((c[:, a] >> b) & 1) << (3 * b + (2 - a))
    return m


def main():
    from paper_2112_05131_b200 import grid as gmod, optim, render, scenes, trainer
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 150000
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
    lo, hi = np.array(g.aabb_min, float), np.array(g.aabb_max, float)
    cap = int(math.ceil(math.sqrt(((hi - lo) ** 2).sum()) / tr._kopts.step)) + 4
    nseg_max = (cap + 31) // 32
    off, offs = 256, {}
    n = B * cap
    for name, nb in [("ns", B * 4), ("segfirst", B * 4), ("segray", B * nseg_max * 4),
                     ("rayd", B * 24), ("basis", B * 48), ("att", n * 8), ("T", n * 8),
                     ("w", n * 8), ("c", n * 16), ("cell", n * 16)]:
        offs[name] = off
        off = (off + nb + 255) & ~255
    buf = tr._scratch_keep
    ns = buf[offs["ns"]:offs["ns"] + B * 4].view(torch.int32).long()
    cell = buf[offs["cell"]:offs["cell"] + n * 16].view(torch.int32).view(B, cap, 4)[..., :3]
    j = torch.arange(cap, device=dev)
    keep = j[None, :] < ns[:, None]
    c = cell[keep].long()                     # samples in ray order
    ray = torch.arange(B, device=dev)[:, None].expand(B, cap)[keep]
    jj = j[None, :].expand(B, cap)[keep]
    Dx, Dy, Dz = g.dims
    offs8 = torch.tensor([[a, b, e] for a in (0, 1) for b in (0, 1) for e in (0, 1)], device=dev)
    R = ((c[:, None, :] + offs8[None]) * torch.tensor([Dy * Dz, Dz, 1], device=dev)).sum(-1)
    S = c.shape[0]
    distinct = torch.unique(R).numel()
    seg = ray * nseg_max + jj // 32
    segload = torch.unique(seg[:, None] * (Dx * Dy * Dz) + R).numel()
    out = {"B": B, "samples": S, "distinct_rows": distinct, "segment_row_loads": segload}
    o = torch.argsort(morton(c))
    for csz in (32, 128, 512):
        ch = torch.arange(S, device=dev) // csz
        out[f"morton_{csz}"] = torch.unique(ch[:, None] * (Dx * Dy * Dz) + R[o]).numel()
    for bsh in (1, 2, 3):
        ob = torch.argsort(morton(c >> bsh), stable=True)
        for csz in (128, 512):
            ch = torch.arange(S, device=dev) // csz
            out[f"brick{1 << bsh}_{csz}"] = torch.unique(ch[:, None] * (Dx * Dy * Dz) + R[ob]).numel()
    print(out)


main()
