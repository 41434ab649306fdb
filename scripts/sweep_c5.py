#!/usr/bin/env python3
"""BASELINE C5: large-batch throughput sweep on a 512^3 sparse grid (1 GPU).

Grid: the reference's toy ground truth (toy.py:65-99 via scenes.build_toy_grid)
upsampled on the device to 512^3 (SparseGrid.upsample, G:260-285).  Ray pool:
hemisphere views of that scene rendered on the device.  Step = fused
forward/backward + RMSProp update with fused clear (TV off, as SURVEY §8(d)
C5).  For each B in 2^14..2^20: rays/s over K timed steps (CUDA events), the
touched rows U and the compulsory-HBM roofline of the step
(bytes = 60 B + U (4 + 112 + 224 + 672))."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2112_05131_b200 import grid as gmod, optim, render, scenes, trainer
    from paper_2112_05131_b200.camera import all_rays
    import bench

    dev = torch.device("cuda", 0)
    views, res = int(os.environ.get("VIEWS", 64)), int(os.environ.get("RES", 512))
    steps, warm = int(os.environ.get("STEPS", 10)), int(os.environ.get("WARM", 3))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    gt64 = scenes.build_toy_grid(64, device=dev)
    t0.record()
    g512 = gt64.upsample((512, 512, 512))
    t1.record()
    torch.cuda.synchronize()
    up_ms = t0.elapsed_time(t1)
    cams, _ = scenes.hemisphere_cameras(views, res, phase=1.0)
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
    peak, _ = bench.load_peaks()
    out = {"grid": "toy GT upsampled to 512^3", "rows": g512.n_rows, "upsample_64_to_512_ms": up_ms,
           "rays_in_pool": views * res * res, "sweep": []}
    for logb in range(int(os.environ.get("LOGB0", 14)), int(os.environ.get("LOGB1", 21))):
        B = 1 << logb
        cfg.batch_size = B
        tr = trainer.Trainer(ds, cfg, device=dev)
        tr.grid = g512.copy()
        tr.state = optim.OptimState(tr.grid.n_rows, device=dev)
        tr.grads = gmod.GradientBuffer(tr.grid.n_rows, device=dev)
        tr._refresh_cache()
        for s in range(warm):
            tr.step(s)
        torch.cuda.synchronize()
        counts = []
        st0 = tr.march_stats.clone()
        t0.record()
        for s in range(steps):
            tr.step(warm + s)
            counts.append(tr.count.clone())
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        U = float(torch.stack(counts).double().mean())
        step_bytes = 60 * B + U * (4 + 112 + 224 + 672)
        mst = ((tr.march_stats - st0).double() / steps).cpu().numpy()
        rec = {"B": B, "ms_per_step": ms, "rays_per_s": B / (ms / 1e3), "U": U,
               "march_positions": float(mst[0]), "samples": float(mst[1]), "chunks": float(mst[2]),
               "U_frac": U / tr.grid.n_rows, "step_bytes": step_bytes,
               "hbm_roofline_rays_per_s": B * peak * 1e9 / step_bytes,
               "frac_of_roofline": (B / (ms / 1e3)) / (B * peak * 1e9 / step_bytes)}
        out["sweep"].append(rec)
        print(json.dumps(rec), flush=True)
        del tr
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sweep_c5.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "sweep"}))


if __name__ == "__main__":
    main()
