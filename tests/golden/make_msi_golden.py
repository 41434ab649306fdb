#!/usr/bin/env python3
"""Golden vectors for the multi-sphere-image background path (360 scenes),
produced by the REFERENCE (pkg/src/plenoxel/msi.py and _kernels.py K:603-977)
in the build container.  Pins oracle.render_360 / bg_sample / tv_bg /
step_table and, through them, the CUDA path.

  msi.npz  per case: a random f32-quantised grid inside the unit sphere, a
           random background (sigma of both signs, colours of both signs),
           rays from inside the sphere and from outside it, the reference's
           render_rays_with_background forward and backward outputs (grid and
           background gradients, touched sets), sample_background at random
           exterior points, bg_tv_loss values and gradients, and one
           step_table RMSProp update of the background.

Usage:  NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_msi_golden.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from make_golden import grid_dict, random_grid  # noqa: E402  (imports the reference)

import plenoxel as px  # noqa: E402
from plenoxel import msi, optim  # noqa: E402
from plenoxel.grid import GradientBuffer  # noqa: E402
from plenoxel.sh import normalize_dirs  # noqa: E402

OUT = Path(__file__).resolve().parent


def rays_360(rng, n):
    """Half the rays start inside the unit sphere (camera ring at r 0.8),
    half outside it; a few are aimed away from the grid."""
    o = np.empty((n, 3))
    d = np.empty((n, 3))
    for i in range(n):
        if i % 2 == 0:
            th = rng.uniform(0, 2 * np.pi)
            o[i] = [0.8 * np.cos(th), 0.8 * np.sin(th), rng.uniform(-0.2, 0.2)]
        else:
            v = normalize_dirs(rng.normal(size=3))
            o[i] = 1.6 * v
        tgt = rng.uniform(-0.3, 0.3, 3)
        dd = tgt - o[i] if i % 5 else rng.normal(size=3)
        d[i] = normalize_dirs(dd)
    return o, d


def main():
    rng = np.random.default_rng(360)
    out = {}
    cases = [("trilinear", 0.0, 0.0, 1e-4), ("nearest", 0.0, 0.0, 1e-4),
             ("trilinear", 0.01, 0.05, 1e-4), ("trilinear", 0.0, 0.0, 0.0)]
    for ci, (interp, lam_c, lam_b, stop) in enumerate(cases):
        dims = tuple(int(x) for x in rng.integers(4, 9, 3))
        g = random_grid(rng, dims=dims, aabb=0.5, holes=0.3, sigma_range=(-1.0, 3.0))
        L, H, W = int(rng.integers(3, 7)), int(rng.integers(3, 8)), int(rng.integers(4, 10))
        bg = msi.MsiBackground.create(L, H, W)
        bg.data[..., 0] = rng.uniform(-0.5, 2.0, (L, H, W))
        bg.data[..., 1:] = rng.uniform(-0.2, 1.0, (L, H, W, 3))
        bg.data[:] = bg.data.astype(np.float32)
        o, d = rays_360(rng, 48)
        gt = rng.uniform(0, 1, (48, 3))
        opts = px.RenderOptions(background=(0.0, 0.0, 0.0), interp=interp, stop_thresh=stop)
        rgb, tfg, trans, _, _, _ = msi.render_rays_with_background(g, bg, o, d, opts)
        grads = GradientBuffer(g.n_rows)
        bgg = msi.BgGradientBuffer(bg)
        rgb2, tfg2, trans2, mse, craw, braw = msi.render_rays_with_background(
            g, bg, o, d, opts, gt_rgb=gt, grads=grads, bg_grads=bgg, n_total=48,
            lam_cauchy=lam_c, lam_beta=lam_b)
        assert np.array_equal(rgb, rgb2)
        pts = normalize_dirs(rng.normal(size=(32, 3))) * rng.uniform(1.0, 6.0, (32, 1))
        pts[0] = [0.0, 0.0, 1.5]          # the pole
        pts[1] = [-2.0, -1e-12, 0.3]      # the phi seam
        s_sig, s_rgb = msi.sample_background(bg, pts)
        cells = msi.sample_bg_tv_cells(bg, 0.5, rng)
        tvb = msi.BgGradientBuffer(bg)
        tv = msi.bg_tv_loss(bg, cells, 0.9, 1.1, tvb)
        # one background update from the render + TV gradients
        merged = bgg.data + tvb.data
        ids = np.nonzero(np.any(merged != 0.0, axis=1) | (bgg.touched_mask > 0)
                         | (tvb.touched_mask > 0))[0]
        state = optim.OptimState(L * H * W, 4)
        state.v[:] = rng.uniform(0, 0.01, state.v.shape)
        v0 = state.v.copy()
        table = bg.data.reshape(-1, 4).copy()
        optim.step_table(table, merged, ids, len(ids), state, 0.5, 0.1)
        p = f"c{ci}_"
        out.update(grid_dict(p, g))
        out.update({p + "bg": bg.data, p + "radii": bg.radii, p + "o": o, p + "d": d,
                    p + "gt": gt,
                    p + "opts": np.array([interp == "nearest", lam_c, lam_b, stop]),
                    p + "rgb": rgb, p + "tfg": tfg, p + "trans": trans,
                    p + "sums": np.array([mse, craw, braw]),
                    p + "grad": grads.data, p + "touched": np.sort(grads.touched_ids[:grads.n_touched]),
                    p + "bg_grad": bgg.data,
                    p + "bg_touched": np.sort(bgg.touched_ids[:bgg.n_touched]),
                    p + "pts": pts, p + "s_sig": s_sig, p + "s_rgb": s_rgb,
                    p + "tv_cells": cells, p + "tv": np.array(tv), p + "tv_grad": tvb.data,
                    p + "tv_touched": np.sort(tvb.touched_ids[:tvb.n_touched]),
                    p + "opt_ids": ids, p + "opt_grad": merged, p + "opt_v0": v0,
                    p + "opt_v": state.v, p + "opt_table": table})
    np.savez_compressed(OUT / "msi.npz", n=len(cases), **out)
    print("wrote", OUT / "msi.npz")
    # a grid + background container and its state sidecar written by the
    # reference's artifact_io (artifact_io.py:42-62, 138-156)
    from plenoxel import artifact_io
    g = random_grid(rng, dims=(3, 4, 5), aabb=0.5, holes=0.3)
    bg = msi.MsiBackground.create(3, 4, 6)
    bg.data[:] = rng.uniform(-1, 2, bg.data.shape).astype(np.float32)
    st = optim.OptimState(g.n_rows)
    st.v[:] = rng.uniform(0, 1, st.v.shape).astype(np.float32)
    bst = optim.OptimState(bg.n_layers * bg.height * bg.width, 4)
    bst.v[:] = rng.uniform(0, 1, bst.v.shape).astype(np.float32)
    artifact_io.save_checkpoint(OUT / "msi_grid.plnx", g, st, 1234, bg, bst)
    print("wrote", OUT / "msi_grid.plnx")


def make_trainer_360():
    """A 20-step 360 run of the reference's trainer.train (T:350-518 with
    the MSI background) on the tiny toy set loaded as unbounded_360."""
    import dataclasses
    import tempfile

    from make_golden import _dataset_arrays

    with tempfile.TemporaryDirectory() as td:
        px.make_toy_dataset(Path(td) / "t", n_views=4, res=32, n_test=2, grid_dim=16)
        train = px.load_nerf_dataset(Path(td) / "t", "unbounded_360", "train",
                                     background=(0.0, 0.0, 0.0))
        test = px.load_nerf_dataset(Path(td) / "t", "unbounded_360", "test",
                                    background=(0.0, 0.0, 0.0))
    cfg = dataclasses.replace(
        px.toy_config(grid_dim=8, total_steps=20, batch_size=64), scene_type="unbounded_360",
        aabb=(-1.0, -1.0, -1.0, 1.0, 1.0, 1.0), bg_layers=4, bg_height=8, bg_width=16,
        lambda_beta=1e-3, lambda_sparsity=1e-6, background=(0.0, 0.0, 0.0))
    cfg.eval_every = 0
    cfg.log_every = 1
    cfg.seed = 7
    res = px.train(train, cfg, test_ds=test)
    loss = np.array([m["loss"] for m in res.metrics if "loss" in m])
    mse = np.array([m["mse"] for m in res.metrics if "mse" in m])
    nnz = np.array([m["nnz_fraction"] for m in res.metrics if "nnz_fraction" in m])
    psnr = [m["psnr"] for m in res.metrics if "psnr" in m][-1]
    imgs, c2w, focal = _dataset_arrays(train)
    timgs, tc2w, tfocal = _dataset_arrays(test)
    np.savez_compressed(OUT / "trainer_360.npz", imgs=imgs, c2w=c2w, focal=focal,
                        test_imgs=timgs, test_c2w=tc2w, test_focal=tfocal, loss=loss, mse=mse,
                        nnz=nnz, psnr=np.array([psnr]), table=res.grid.table,
                        links=res.grid.links, bg=res.background.data,
                        scene_scale=np.array([res.scene_scale]))
    print("wrote", OUT / "trainer_360.npz", "psnr", psnr, "loss", loss[:3], loss[-1])


if __name__ == "__main__":
    main()
    make_trainer_360()
