"""Helper of test_gpu_waves.py (run as a subprocess: the record budget is read
once per process).  Renders the same batches through every wave-sliced entry
point and saves the results to argv[1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import random_grid, ray_batch  # noqa: E402


def main(out):
    import paper_2112_05131_b200 as px
    from paper_2112_05131_b200 import msi, render, scenes, trainer
    res = {}
    rng = np.random.default_rng(0)
    g = random_grid(rng, dims=(9, 8, 10), holes=0.2, sigma_range=(-0.5, 3.0))
    dg = px.SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)
    o, d = ray_batch(rng, 3000)
    gt = rng.uniform(0, 1, (3000, 3))
    for name, opts in (("rel", px.RenderOptions()),
                       ("abs_nearest", px.RenderOptions(formula="absolute", interp="nearest"))):
        buf = px.GradientBuffer(dg.n_rows)
        rgb, mse, _ = px.fused_mse_backward(dg, o, d, d / np.linalg.norm(d, axis=1, keepdims=True),
                                            gt, buf, opts, n_total=3000, lam_cauchy=1e-3)
        res[f"{name}_rgb"], res[f"{name}_mse"] = rgb, np.array([mse])
        res[f"{name}_grad"], res[f"{name}_touched"] = buf.dense(), buf.touched_rows()
    buf = px.GradientBuffer(dg.n_rows)   # upstream mode with jitter
    rgb, _ = px.render_rays_backward(dg, o, d, rng.normal(size=(3000, 3)), buf,
                                     px.RenderOptions(jitter=1.0), rng=np.random.default_rng(3))
    res["jit_rgb"], res["jit_grad"] = rgb, buf.dense()
    bg = msi.MsiBackground.create(6, 8, 12)      # 360: background stage per wave
    bg.data[:] = torch.as_tensor(np.random.default_rng(4).uniform(0, 1, tuple(bg.data.shape)))
    oi = rng.uniform(-0.3, 0.3, (3000, 3))
    di = rng.normal(size=(3000, 3))
    di /= np.linalg.norm(di, axis=1, keepdims=True)
    buf, bgb = px.GradientBuffer(dg.n_rows), msi.BgGradientBuffer(bg)
    rgb, tfg, trans, mse, craw, braw = msi.render_rays_with_background(
        dg, bg, oi, di, px.RenderOptions(background=(0, 0, 0)), gt_rgb=gt, grads=buf,
        bg_grads=bgb, n_total=3000, lam_cauchy=1e-3, lam_beta=1e-2)
    res.update(msi_rgb=rgb, msi_tfg=tfg, msi_trans=trans, msi_sums=np.array([mse, craw, braw]),
               msi_grad=buf.dense(), msi_bggrad=bgb.data.cpu().numpy())
    train, _, _ = scenes.make_toy_dataset(n_views=4, res=48, n_test=1, grid_dim=16)
    cfg = trainer.toy_config(grid_dim=16, total_steps=6, batch_size=2500)   # camera pool, graphs
    cfg.log_every = 1
    r = trainer.train(train, cfg)
    res["train_loss"] = np.array([m["loss"] for m in r.metrics if "loss" in m])
    res["train_table"] = r.grid.table.cpu().numpy()
    np.savez(out, **res)


main(sys.argv[1])
