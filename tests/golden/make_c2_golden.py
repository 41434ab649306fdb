#!/usr/bin/env python3
"""C2 PSNR golden (BASELINE configs[1]): the REFERENCE trainer
(imported from /root/reference/pkg/src; build container only) on
make_toy_dataset(100 views, 200^2, 10 test views, 64^3 gt) with
default_config("bounded") at a 256^3 dense rung, 5000-ray batches, TV +
RMSProp, for STEPS steps; then evaluate() on the test views.

Runs the stock reference and K runs with float32 state and +-1 ulp init
perturbations (ref_psnr_spread.py's f32 model of our storage) in parallel.
-> c2_psnr.json: per-run final PSNR, the loss every 10 steps, and sha256 of
every 8-bit train / test image so the device-rendered dataset can be checked
identical.

Usage: python tests/golden/make_c2_golden.py [STEPS] [K]   (~15 min, 3 x 11 GB RAM)
"""
import hashlib
import json
import os
import sys
import tempfile
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
OUT = Path(__file__).resolve().parent


def run(args):
    seed, steps = args
    import numpy as np
    import plenoxel as px
    from plenoxel.trainer import LadderRung

    if seed > 0:
        import ref_psnr_spread as rs
        rs.NOISE = rs.GRAD32 = False
        # reuse the f32-state + perturbed-init patches of ref_psnr_spread.run
        from plenoxel import optim as popt, trainer as ptr
        orig_step = popt.step

        def step_f32(grid, grads, state, *a, **k):
            out = orig_step(grid, grads, state, *a, **k)
            grid.table[:] = grid.table.astype(np.float32)
            state.v[:] = state.v.astype(np.float32)
            return out

        ptr.optim.step = step_f32
        orig_dense = px.SparseGrid.dense.__func__

        def dense_pert(cls, *a, **k):
            g = orig_dense(cls, *a, **k)
            rng = np.random.default_rng(seed)
            t32 = g.table.astype(np.float32)
            up = np.nextafter(t32, np.float32(np.inf))
            dn = np.nextafter(t32, np.float32(-np.inf))
            pick = rng.integers(0, 3, t32.shape)
            g.table[:] = np.where(pick == 0, dn, np.where(pick == 1, t32, up))
            return g

        ptr.SparseGrid.dense = classmethod(dense_pert)
    with tempfile.TemporaryDirectory() as td:
        root = Path(td) / "c2"
        px.make_toy_dataset(root, n_views=100, res=200, n_test=10, grid_dim=64)
        train = px.load_nerf_dataset(root, "bounded", "train")
        test = px.load_nerf_dataset(root, "bounded", "test")
        sha = {"train": [hashlib.sha256(np.rint(im * 255).astype(np.uint8).tobytes()).hexdigest()
                         for im in train.images],
               "test": [hashlib.sha256(np.rint(im * 255).astype(np.uint8).tobytes()).hexdigest()
                        for im in test.images]}
    cfg = px.default_config("bounded")
    cfg.ladder = [LadderRung(0, (256, 256, 256))]
    cfg.total_steps = steps
    cfg.eval_every = 0
    cfg.log_every = 10
    res = px.train(train, cfg, test_ds=test)
    losses = [m["loss"] for m in res.metrics if "loss" in m]
    psnr = [m["psnr"] for m in res.metrics if "psnr" in m][-1]
    ssim = [m["ssim"] for m in res.metrics if "ssim" in m][-1]
    return seed, {"psnr": psnr, "ssim": ssim, "loss_every_10": losses, "sha256": sha}


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    seeds = [0] + list(range(1, k + 1))
    with ProcessPoolExecutor(max_workers=len(seeds)) as ex:
        res = dict(ex.map(run, [(s, steps) for s in seeds]))
    out = {"steps": steps, "batch": 5000, "grid": 256, "views": 100, "res": 200, "n_test": 10,
           "stock": res[0], "f32_perturbed": {str(s): res[s]["psnr"] for s in seeds if s},
           "sha256": res[0]["sha256"]}
    for s in seeds:
        del res[s]["sha256"]
    vals = list(out["f32_perturbed"].values())
    out["f32_perturbed_mean"] = sum(vals) / len(vals) if vals else None
    (OUT / "c2_psnr.json").write_text(json.dumps(out, indent=1))
    print({k: v for k, v in out.items() if k != "sha256"})


if __name__ == "__main__":
    main()
