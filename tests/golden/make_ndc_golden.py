#!/usr/bin/env python3
"""Golden vectors for the forward-facing NDC path (BASELINE configs[3], C4 at
reduced dims): the reference's camera.to_ndc on random rays,
and a short reference training run of a synthetic forward-facing scene.

Runs only in the build container, where the reference package is importable
(/root/reference/pkg/src); writes tests/golden/ndc.npz.

Scene: a ground-truth grid defined in the NDC cube [-1, 1]^3 (two density
blobs with distinct DC colours), rendered by the reference through its own
to_ndc from 4 LLFF-like cameras (identity rotation, small x/y offsets,
looking down -z) at 40 x 32 px, 8-bit quantised like its PNG round trip.
Training: default_config('forward_facing_ndc') with the ladder cut to one
44 x 36 x 16 rung (the 1408 x 1156 x 128 rung reduced), TV (5e-4, 5e-3),
Cauchy lambda_s = 1e-12, 25 steps of 256 rays, loss / nnz logged every step.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import plenoxel as px  # noqa: E402
from plenoxel import camera as pcam  # noqa: E402
from plenoxel import render as prender  # noqa: E402

OUT = Path(__file__).resolve().parent


def gt_grid(dims=(44, 36, 16)):
    g = px.SparseGrid.dense(dims, (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), sigma=0.0, rgb=0.1)
    ijk = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), -1).reshape(-1, 3)
    p = g.aabb_min + ijk * g.voxel_size
    for centre, rad, rgb in (((-0.3, 0.1, 0.2), 0.35, (0.9, 0.2, 0.2)),
                             ((0.35, -0.2, 0.6), 0.3, (0.1, 0.4, 0.9))):
        inside = np.linalg.norm((p - np.array(centre)) / np.array([1, 1, 0.6]), axis=1) < rad
        rows = g.links.reshape(-1)[inside]
        g.table[rows, 0] = 12.0
        for ch in range(3):
            g.table[rows, 1 + 9 * ch] = rgb[ch] / px.sh.SH_C0
    return g


def cameras(n, w=40, h=32, focal=36.0):
    cams = []
    for i in range(n):
        c2w = np.eye(4)
        c2w[0, 3] = 0.15 * np.cos(2 * np.pi * i / n)
        c2w[1, 3] = 0.1 * np.sin(2 * np.pi * i / n)
        cams.append(pcam.Camera(c2w=c2w, focal=focal, width=w, height=h))
    return cams


def render_views(g, cams):
    opts = prender.RenderOptions(step_frac=0.5, background=(0.0, 0.0, 0.0))
    imgs = []
    for cam in cams:
        o, d = pcam.generate_rays(cam)
        on, dn, valid = pcam.to_ndc(o, d, cam)
        rgb, _, _ = prender.render_rays(g, on, dn, opts, viewdirs=d)
        imgs.append((np.rint(np.clip(rgb, 0, 1) * 255) / 255.0).astype(np.float32)
                    .reshape(cam.height, cam.width, 3))
    return np.stack(imgs)


def main():
    rng = np.random.default_rng(2112)
    # to_ndc on random rays of random forward-facing cameras
    cam = pcam.Camera(c2w=np.eye(4), focal=50.0, width=64, height=48)
    o = rng.normal(scale=0.2, size=(200, 3))
    d = rng.normal(size=(200, 3))
    d[:, 2] = -np.abs(d[:, 2]) - 0.2
    d[:5, 2] = 0.0                       # parallel to the image plane: invalid
    on, dn, valid = pcam.to_ndc(o, d, cam, near=1.0)

    g = gt_grid()
    train_cams, test_cams = cameras(4), cameras(2)
    for c in test_cams:                   # offset the test poses
        c.c2w[0, 3] += 0.05
    train = pcam.Dataset(render_views(g, train_cams), train_cams, "forward_facing_ndc",
                         np.zeros(3))
    test = pcam.Dataset(render_views(g, test_cams), test_cams, "forward_facing_ndc",
                        np.zeros(3))
    cfg = px.default_config("forward_facing_ndc")
    cfg.ladder = [px.trainer.LadderRung(0, (44, 36, 16))]
    cfg.total_steps = 25
    cfg.batch_size = 256
    cfg.eval_every = 0
    cfg.log_every = 1
    cfg.seed = 5
    res = px.train(train, cfg, test_ds=test)
    loss = np.array([m["loss"] for m in res.metrics if "loss" in m])
    nnz = np.array([m["nnz_fraction"] for m in res.metrics if "nnz_fraction" in m])
    psnr = [m["psnr"] for m in res.metrics if "psnr" in m][-1]
    u8 = lambda ims: np.rint(np.asarray(ims) * 255.0).astype(np.uint8)  # noqa: E731
    np.savez_compressed(
        OUT / "ndc.npz", o=o, d=d, on=on, dn=dn, valid=valid, cam_focal=np.array([50.0]),
        cam_wh=np.array([64, 48]),
        imgs=u8(train.images), c2w=np.stack([c.c2w for c in train_cams]),
        focal=np.array([c.focal for c in train_cams]),
        test_imgs=u8(test.images), test_c2w=np.stack([c.c2w for c in test_cams]),
        test_focal=np.array([c.focal for c in test_cams]),
        loss=loss, nnz=nnz, psnr=np.array([psnr]), links=res.grid.links)
    print("wrote", OUT / "ndc.npz", "loss", loss[[0, -1]], "psnr", psnr)


if __name__ == "__main__":
    main()
