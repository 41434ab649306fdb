#!/usr/bin/env python3
"""Coarse-to-fine golden (T:412-439, pkg/tests/test_trainer.py:182-193): the
REFERENCE trainer (imported from /root/reference/pkg/src; build container
only) on the tiny toy set of trainer_tiny.npz with a 2-rung ladder, once per
prune criterion:

  weight :  8^3 -> 12^3 at step 20, prune_threshold 1e-5 (test_trainer.py:185-188)
  density:  8^3 -> 16^3 at step 10, prune_threshold 0.05

Per run: loss / nnz every step, the links of the final grid (the
rung's prune + upsample fixes the links, no later event changes them) and
the final test PSNR -> ladder.npz.

Usage: NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_ladder_golden.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import plenoxel as px  # noqa: E402
from plenoxel.camera import Camera, Dataset  # noqa: E402
from plenoxel.trainer import LadderRung  # noqa: E402

OUT = Path(__file__).resolve().parent

CASES = {"weight": dict(total=40, batch=128, rung=20, dims=12, thr=1e-5),
         "density": dict(total=30, batch=128, rung=10, dims=16, thr=0.05)}


def dataset(z, prefix, tag):
    imgs = (np.asarray(z[f"{prefix}imgs"], dtype=np.float64) / 255.0).astype(np.float32)
    h, w = imgs.shape[1:3]
    cams = [Camera(c2w=c, focal=float(f), width=w, height=h)
            for c, f in zip(z[f"{prefix}c2w"], z[f"{prefix}focal"])]
    return Dataset(images=imgs, cameras=cams, scene_type="bounded",
                   background=np.ones(3), paths=[f"{tag}{i}" for i in range(len(cams))])


def main():
    z = np.load(OUT / "trainer_tiny.npz")
    train, test = dataset(z, "", "train"), dataset(z, "test_", "test")
    out = {}
    for name, c in CASES.items():
        cfg = px.toy_config(grid_dim=8, total_steps=c["total"], batch_size=c["batch"])
        cfg.ladder = [LadderRung(0, (8, 8, 8)), LadderRung(c["rung"], (c["dims"],) * 3)]
        cfg.prune_criterion = name
        cfg.prune_threshold = c["thr"]
        cfg.eval_every = 0
        cfg.log_every = 1
        cfg.seed = 11
        res = px.train(train, cfg, test_ds=test)
        res.grid.validate()
        out[f"{name}_loss"] = np.array([m["loss"] for m in res.metrics if "loss" in m])
        out[f"{name}_nnz"] = np.array([m["nnz_fraction"] for m in res.metrics
                                       if "nnz_fraction" in m])
        out[f"{name}_psnr"] = np.array([[m["psnr"] for m in res.metrics if "psnr" in m][-1]])
        out[f"{name}_links"] = res.grid.links
        print(name, res.grid.dims, res.grid.n_rows, out[f"{name}_psnr"])
    np.savez_compressed(OUT / "ladder.npz", **out)


if __name__ == "__main__":
    main()
