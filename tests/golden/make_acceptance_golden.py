#!/usr/bin/env python3
"""The reference's acceptance-suite training arms (pkg/tests/test_acceptance.py
criteria 3, 5, 6, 7 and the TV trend), run with the UNMODIFIED reference
(imported from /root/reference/pkg/src; build container only), in parallel
processes -> acceptance_arms.json: the final test PSNR of every arm (and the
coarse-to-fine drift / final PSNR), for tests/test_gpu_acceptance.py to
print and compare against.

Usage: NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_acceptance_golden.py
"""
import json
import os
import sys
import tempfile
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

ARMS = {
    "tri32": {},
    "nn64": {"grid": 64, "interp": "nearest"},
    "nn32": {"grid": 32, "interp": "nearest"},
    "abs32": {"formula": "absolute"},
    "sgd": {"optimizer": "sgd", "lr_sigma": ("delayed_exponential", 3e6, 5e3, 6000, 300, 0.01),
            "lr_sh": ("exponential", 100.0, 1.0, 6000, 0, 0.01)},
    "exp": {"lr_sigma": ("exponential", 2.0, 0.1, 6000, 0, 0.01)},
    "const": {"lr_sigma": ("constant", 1.0, 1.0, 6000, 0, 0.01)},
    "tv10_low": {"_views": 10},
    "tv10_high": {"_views": 10, "lambda_tv_sigma": 1e-5, "lambda_tv_sh": 1e-3},
    "c2f": {"_c2f": True},
}


def run(name):
    import numpy as np
    import plenoxel as px
    from plenoxel.camera import all_rays
    from plenoxel.grid import GradientBuffer
    from plenoxel.optim import LrSchedule
    from plenoxel.render import fused_mse_backward
    from plenoxel.trainer import EpochBatcher, evaluate
    from plenoxel import optim as O

    kw = dict(ARMS[name])
    views = kw.pop("_views", 25)
    c2f = kw.pop("_c2f", False)
    grid = kw.pop("grid", 32)
    with tempfile.TemporaryDirectory() as td:
        d = Path(td) / "toy"
        px.make_toy_dataset(d, n_views=views, res=64, n_test=10, grid_dim=64)
        train = px.load_nerf_dataset(d, "bounded", "train")
        test = px.load_nerf_dataset(d, "bounded", "test")
    cfg = px.toy_config(grid_dim=grid, total_steps=3000, batch_size=2000)
    for k, v in kw.items():
        if k in ("lr_sigma", "lr_sh"):
            v = LrSchedule(kind=v[0], lr_init=v[1], lr_final=v[2], total_steps=v[3],
                           delay_steps=v[4], delay_mult=v[5])
        setattr(cfg, k, v)
    cfg.eval_every = 0
    res = px.train(train, cfg, test_ds=test)
    out = {"psnr": [m for m in res.metrics if "psnr" in m][-1]["psnr"]}
    if c2f:   # test_acceptance.py:231-267
        g = res.grid
        o, m, v, gt = all_rays(train)
        opts = px.RenderOptions(background=(1, 1, 1))
        w = g.max_weight_accumulate(o, m)
        pruned, _ = g.prune("weight", float(w[w > 0].min()), w)
        up = pruned.upsample((64, 64, 64))
        out["p_before"] = evaluate(g, test, opts)[0]
        out["p_after"] = evaluate(up, test, opts)[0]
        rng = np.random.default_rng(0)
        state, grads = O.OptimState(up.n_rows), GradientBuffer(up.n_rows)
        batcher = EpochBatcher(o.shape[0], 2000, rng)
        c64 = px.toy_config(grid_dim=64, total_steps=500, batch_size=2000)
        for s in range(500):
            idx = batcher.next()
            fused_mse_backward(up, np.ascontiguousarray(o[idx]), np.ascontiguousarray(m[idx]),
                               np.ascontiguousarray(v[idx]), np.ascontiguousarray(gt[idx]),
                               grads, opts, n_total=len(idx))
            O.step(up, grads, state, O.lr_at(c64.lr_sigma, s), O.lr_at(c64.lr_sh, s))
            grads.clear()
        out["p_final"] = evaluate(up, test, opts)[0]
    return name, out


def main():
    with ProcessPoolExecutor(max_workers=min(len(ARMS), os.cpu_count() or 1)) as ex:
        res = dict(ex.map(run, list(ARMS)))
    (OUT / "acceptance_arms.json").write_text(json.dumps(res, indent=1))
    print(res)


if __name__ == "__main__":
    main()
