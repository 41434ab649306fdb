#!/usr/bin/env python3
"""Kernel micro-benchmarks at the bench.py training state (diagnostics only).

Times, with CUDA events over R repetitions on the same batch:
  fwd      plx_render_fwd (pass 1 only)
  bwd      plx_render_fused_bwd (pass 1 + records + pass 2 scatter)
  tv, opt  the other two step kernels
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    import bench
    from paper_2112_05131_b200 import grid as gmod, losses, optim, render, trainer

    class A:
        batch, gpus, dims, views, res = 5000, 1, int(os.environ.get("DIMS", 256)), 100, 200

    dev = torch.device("cuda", 0)
    ds = bench.toy_scene(A.views, A.res, dev)
    cfg = bench.bench_config(A)
    tr = trainer.Trainer(ds, cfg, device=dev)
    for s in range(int(os.environ.get("WARM", 5))):
        tr.step(s)
    idx = tr.batcher.next_device()
    o, d, v = tr.pool.origins[idx].contiguous(), tr.pool.dirs[idx].contiguous(), tr.pool.viewdirs[idx].contiguous()
    res = {}
    res["fwd"] = timeit(lambda: render.render_rays(tr.grid, o, d, tr.opts, viewdirs=v))
    sums = torch.zeros(2, dtype=torch.float64, device=dev)

    def bwd():
        render.fused_mse_backward_pool(tr.grid, tr.pool, idx, tr.grads, tr.opts, len(idx), 0.0, sums)
    res["bwd"] = timeit(bwd)
    res["U_render"] = tr.grads.n_touched
    tr.grads.clear()
    gmod.USE_CELL_OCC = False
    tr._refresh_cache()
    res["bwd_no_cellocc"] = timeit(lambda: render.fused_mse_backward_pool(
        tr.grid, tr.pool, idx, tr.grads, tr.opts, len(idx), 0.0, sums))
    gmod.USE_CELL_OCC = True
    tr._refresh_cache()
    tr.grads.clear()
    run = losses.sample_tv_cells(tr.grid, cfg.tv_sample_frac, np.random.default_rng(0))
    res["tv"] = timeit(lambda: losses.tv_loss(tr.grid, run, 1e-5, 1e-3, tr.grads, sums=sums))
    bwd()
    st = tr.state

    def opt():
        optim.step(tr.grid, tr.grads, st, 0.0, 0.0, clear=False)
    res["opt_noclear"] = timeit(opt)
    res["U_total"] = tr.grads.n_touched
    print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()})


if __name__ == "__main__":
    main()
