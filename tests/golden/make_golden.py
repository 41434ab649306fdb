#!/usr/bin/env python3
"""Generate the golden vectors that pin the oracle (and, transitively, the
CUDA path) to the REFERENCE implementation.

Runs only in the build container, where the reference package is importable
from /root/reference/pkg/src (it does not exist on the GPU box; the outputs
committed next to this script are what travels).  Every case calls the
reference's own public API / kernels:

  render.npz     render_rays (R:114-140) on random grids, 4 formula x interp
  backward.npz   fused_mse_backward (R:253-279) / render_rays_backward (R:205)
  tv.npz         tv_loss (L:50-77)
  optim.npz      optim.step (O:81-97) RMSProp + SGD
  maxw.npz       SparseGrid.max_weight_accumulate (G:287-302)
  structure.npz  SparseGrid.prune (G:228-258) / upsample (G:260-285)
  toy.plnx, toy_render.bin, toy_ref.json
                 the reference viewer golden (scripts/make_viewer_fixtures.py:88-120)
  plnx/          g000..g009.plnx regenerated with the fixture script's RNG; their
                 CRC32s must equal pkg/frontend/test/fixtures/golden.json
  trainer_tiny.npz  a 30-step training run (trainer.py:350-518) on a tiny toy
                 dataset: per-step loss / nnz and the final table
  toy128.npz     the acceptance toy dataset (make_toy_dataset 25x128^2 + 10 test)
                 as uint8 images + poses, for the PSNR-parity test

Grid tables are quantised to float32 before the reference runs, so the f32
device tables see exactly the reference's inputs.

Usage:  NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import zlib
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import plenoxel as px  # noqa: E402
from plenoxel.grid import GradientBuffer  # noqa: E402
from plenoxel.losses import tv_loss  # noqa: E402
from plenoxel.render import fused_mse_backward  # noqa: E402
from plenoxel.sh import normalize_dirs  # noqa: E402
from plenoxel import optim  # noqa: E402

OUT = Path(__file__).resolve().parent


def random_grid(rng, dims=(5, 5, 5), aabb=1.0, sigma_range=(0.2, 3.0),
                dc_range=(0.5, 1.5), band_scale=0.05, holes=0.0):
    """pkg/tests/conftest.py:10-31, then f32-quantised."""
    g = px.SparseGrid.dense(dims, (-aabb,) * 3, (aabb,) * 3)
    g.table[:, 0] = rng.uniform(*sigma_range, g.n_rows)
    for ch in range(3):
        g.table[:, 1 + 9 * ch] = rng.uniform(*dc_range, g.n_rows)
        for b in range(1, 9):
            g.table[:, 1 + 9 * ch + b] = rng.uniform(-band_scale, band_scale, g.n_rows)
    if holes > 0:
        links = g.links.copy()
        mask = rng.random(links.shape) < holes
        links[mask] = -1
        keep = np.sort(g.links[links >= 0])
        remap = np.full(g.n_rows, -1, dtype=np.int64)
        remap[keep] = np.arange(len(keep))
        links = np.where(links >= 0, remap[np.maximum(links, 0)], -1)
        g = px.SparseGrid(links.astype(np.int32), g.table[keep], g.aabb_min, g.aabb_max)
    g.table[:] = g.table.astype(np.float32)
    return g


def random_hitting_ray(rng, aabb=1.0):
    """pkg/tests/conftest.py:34-42."""
    target = rng.uniform(-0.6 * aabb, 0.6 * aabb, 3)
    theta = rng.uniform(0, 2 * np.pi)
    z = rng.uniform(-0.9, 0.9)
    r = np.sqrt(1 - z * z)
    origin = 3.0 * aabb * np.array([r * np.cos(theta), r * np.sin(theta), z])
    d = target - origin
    return origin, d / np.linalg.norm(d)


def ray_batch(rng, n, aabb=1.0, n_miss=4):
    o, d = zip(*[random_hitting_ray(rng, aabb) for _ in range(n)])
    o, d = np.array(o), np.array(d)
    # a few rays that miss the box, one axis-parallel ray, one from inside
    for i in range(min(n_miss, n)):
        o[i] = [3.0 * aabb, 3.0 * aabb, 0.0]
        d[i] = normalize_dirs(np.array([1.0, 0.2 * i, 0.1]))
    if n > n_miss + 2:
        o[n_miss] = [-3.0 * aabb, 0.1, 0.05]
        d[n_miss] = [1.0, 0.0, 0.0]
        o[n_miss + 1] = [0.05, -0.1, 0.2]
        d[n_miss + 1] = normalize_dirs(np.array([0.3, -0.5, 0.8]))
    return o, d


def grid_dict(prefix, g):
    return {f"{prefix}links": g.links, f"{prefix}table": g.table,
            f"{prefix}aabb_min": g.aabb_min, f"{prefix}aabb_max": g.aabb_max}


COMBOS = [("relative", "trilinear"), ("relative", "nearest"),
          ("absolute", "trilinear"), ("absolute", "nearest")]


def make_render(rng):
    out = {}
    for ci, (formula, interp) in enumerate(COMBOS):
        dims = tuple(int(x) for x in rng.integers(3, 9, 3))
        g = random_grid(rng, dims=dims, holes=0.25, sigma_range=(-0.5, 4.0))
        o, d = ray_batch(rng, 64)
        bg = rng.uniform(0, 1, 3)
        stop = [1e-4, 0.0, 1e-2, 1e-4][ci]
        step_frac = [0.5, 0.37, 0.5, 0.8][ci]
        opts = px.RenderOptions(formula=formula, interp=interp, background=tuple(bg),
                                stop_thresh=stop, step_frac=step_frac)
        rgb, trans, wsum = px.render_rays(g, o, d, opts)
        out.update(grid_dict(f"c{ci}_", g))
        out.update({f"c{ci}_o": o, f"c{ci}_d": d, f"c{ci}_bg": bg,
                    f"c{ci}_opts": np.array([stop, step_frac, interp == "nearest",
                                             formula == "absolute"], dtype=np.float64),
                    f"c{ci}_rgb": rgb, f"c{ci}_trans": trans, f"c{ci}_wsum": wsum})
    np.savez_compressed(OUT / "render.npz", n=len(COMBOS), **out)


def make_backward(rng):
    out = {}
    cases = COMBOS + [("relative", "trilinear")]     # + a Cauchy / upstream case
    for ci, (formula, interp) in enumerate(cases):
        dims = tuple(int(x) for x in rng.integers(3, 9, 3))
        sig_range = (0.2, 3.0) if formula == "relative" else (0.05, 0.6)
        if ci == 0:
            sig_range = (-0.5, 3.0)        # exercises the sigma<0 skip / sigma=0 record
        g = random_grid(rng, dims=dims, holes=0.2, sigma_range=sig_range)
        o, d = ray_batch(rng, 48)
        vd = normalize_dirs(d)
        gt = rng.uniform(0, 1, (len(o), 3))
        bg = rng.uniform(0, 1, 3)
        stop = [1e-4, 0.0, 1e-3, 0.0, 1e-4][ci]
        opts = px.RenderOptions(formula=formula, interp=interp, background=tuple(bg),
                                stop_thresh=stop)
        lam = 1e-3 if ci == 4 else 0.0
        buf = GradientBuffer(g.n_rows)
        rgb, mse_sum, cauchy = fused_mse_backward(g, o, d, vd, gt, buf, opts,
                                                  n_total=len(o), lam_cauchy=lam)
        out.update(grid_dict(f"c{ci}_", g))
        out.update({f"c{ci}_o": o, f"c{ci}_d": d, f"c{ci}_gt": gt, f"c{ci}_bg": bg,
                    f"c{ci}_opts": np.array([stop, 0.5, interp == "nearest",
                                             formula == "absolute", lam]),
                    f"c{ci}_rgb": rgb, f"c{ci}_sums": np.array([mse_sum, cauchy]),
                    f"c{ci}_grad": buf.dense(), f"c{ci}_touched": buf.touched_rows()})
        if ci == 4:
            # upstream mode (render_rays_backward, R:205-239)
            up = rng.normal(size=(len(o), 3))
            buf2 = GradientBuffer(g.n_rows)
            rgb2, cauchy2 = px.render_rays_backward(g, o, d, up, buf2, opts,
                                                    lam_cauchy=lam)
            out.update({"up_up": up, "up_rgb": rgb2, "up_cauchy": np.array([cauchy2]),
                        "up_grad": buf2.dense(), "up_touched": buf2.touched_rows()})
    np.savez_compressed(OUT / "backward.npz", n=len(cases), **out)


def make_tv(rng):
    out = {}
    for ci in range(3):
        dims = tuple(int(x) for x in rng.integers(3, 9, 3))
        g = random_grid(rng, dims=dims, holes=0.3, sigma_range=(-1.0, 1.0),
                        dc_range=(-1.0, 1.0), band_scale=0.8)
        ncell = int(np.prod(dims))
        if ci == 0:
            cells = np.arange(ncell, dtype=np.int64)
        elif ci == 1:
            cells = rng.permutation(ncell)[:30].astype(np.int64)
        else:
            cells = px.losses.sample_tv_cells(g, 0.3, rng)
        eps = [1e-6, 1e-6, 0.0][ci]
        buf = GradientBuffer(g.n_rows)
        a, b = tv_loss(g, cells, 0.7, 1.3, buf, eps=eps)
        out.update(grid_dict(f"c{ci}_", g))
        out.update({f"c{ci}_cells": cells, f"c{ci}_eps": np.array([eps]),
                    f"c{ci}_loss": np.array([a, b]), f"c{ci}_grad": buf.dense(),
                    f"c{ci}_touched": buf.touched_rows()})
    np.savez_compressed(OUT / "tv.npz", n=3, **out)


def make_optim(rng):
    out = {}
    for ci, method in enumerate(("rmsprop", "sgd")):
        g = random_grid(rng, dims=(4, 4, 4))
        state = optim.OptimState(g.n_rows)
        state.v[:] = rng.uniform(0, 0.5, state.v.shape).astype(np.float32)
        buf = GradientBuffer(g.n_rows)
        for r in rng.permutation(g.n_rows)[:30]:
            vals = rng.normal(size=28).astype(np.float32).astype(np.float64)
            vals[rng.random(28) < 0.3] = 0.0
            buf.add(int(r), vals)
        t0, v0, gd = g.table.copy(), state.v.copy(), buf.dense()
        touched = buf.touched_rows()
        optim.step(g, buf, state, 0.3, 0.01, method)
        out.update({f"c{ci}_table": t0, f"c{ci}_v": v0, f"c{ci}_grad": gd,
                    f"c{ci}_touched": touched, f"c{ci}_table_out": g.table,
                    f"c{ci}_v_out": state.v})
    np.savez_compressed(OUT / "optim.npz", n=2, lr=np.array([0.3, 0.01]), **out)


def make_maxw(rng):
    out = {}
    for ci, interp in enumerate(("trilinear", "nearest")):
        g = random_grid(rng, dims=(7, 6, 8), holes=0.2, sigma_range=(-0.5, 6.0))
        o, d = ray_batch(rng, 64)
        w = g.max_weight_accumulate(o, d, step_frac=0.5, stop_thresh=1e-4, interp=interp)
        out.update(grid_dict(f"c{ci}_", g))
        out.update({f"c{ci}_o": o, f"c{ci}_d": d, f"c{ci}_w": w})
    np.savez_compressed(OUT / "maxw.npz", n=2, **out)


def make_structure(rng):
    out = {}
    # prune: density / weight / lone-voxel dilation (test_grid.py:185-193)
    g = random_grid(rng, dims=(9, 7, 8), holes=0.2, sigma_range=(0.0, 4.0))
    p, kept = g.prune("density", 2.5)
    out.update(grid_dict("pd_", g))
    out.update({"pd_thr": np.array([2.5]), "pd_links_out": p.links, "pd_kept": kept})
    g = random_grid(rng, dims=(10, 6, 7), holes=0.3)
    w = rng.uniform(0, 1, g.n_rows)
    p, kept = g.prune("weight", 0.8, w)
    out.update(grid_dict("pw_", g))
    out.update({"pw_thr": np.array([0.8]), "pw_w": w, "pw_links_out": p.links,
                "pw_kept": kept})
    # upsample cases: identity, 2x, nested 8->15, anisotropic, shrink
    g = random_grid(rng, dims=(8, 8, 8), holes=0.3)
    g = px.SparseGrid(g.links, g.table, (-1.1, -0.9, -1.3), (1.0, 1.2, 0.7))
    out.update(grid_dict("up_", g))
    targets = [(8, 8, 8), (16, 16, 16), (15, 15, 15), (7, 5, 9), (13, 17, 11), (5, 4, 6)]
    for ti, nd in enumerate(targets):
        u = g.upsample(nd)
        out.update({f"up{ti}_dims": np.array(nd), f"up{ti}_links": u.links,
                    f"up{ti}_table": u.table})
    np.savez_compressed(OUT / "structure.npz", n_up=len(targets), **out)


def make_viewer_goldens():
    """Re-run scripts/make_viewer_fixtures.py's logic into tests/golden/."""
    from plenoxel.msi import MsiBackground

    plnx = OUT / "plnx"
    plnx.mkdir(exist_ok=True)
    rng = np.random.default_rng(20240)
    golden = []
    for i in range(10):                          # make_viewer_fixtures.py:29-86
        dims = tuple(int(rng.integers(2, 7)) for _ in range(3))
        aabb = rng.uniform(0.5, 2.0)
        g = px.SparseGrid.dense(dims, (-aabb,) * 3, (aabb,) * 3)
        g.table[:] = rng.normal(size=g.table.shape)
        if rng.random() < 0.5:
            links = g.links.copy()
            links[rng.random(links.shape) < 0.4] = -1
            keep = np.sort(g.links[links >= 0])
            if len(keep) == 0:
                links[0, 0, 0] = 0
                keep = np.array([g.links[0, 0, 0]])
            remap = np.full(g.n_rows, -1, dtype=np.int64)
            remap[keep] = np.arange(len(keep))
            g = px.SparseGrid(np.where(links >= 0, remap[np.maximum(links, 0)], -1)
                              .astype(np.int32), g.table[keep], g.aabb_min, g.aabb_max)
        g.table[:] = g.table.astype(np.float32)
        bg = None
        if i % 4 == 3:
            bg = MsiBackground.create(3, 4, 6)
            bg.data[:] = rng.uniform(0, 1, bg.data.shape).astype(np.float32)
        name = f"g{i:03d}.plnx"
        px.save_grid(g, plnx / name, bg)
        raw = (plnx / name).read_bytes()
        if g.n_rows:
            for _ in range(5):
                rng.integers(0, g.n_rows)
                rng.integers(0, 28)
        for _ in range(5):
            [int(rng.integers(0, d)) for d in g.dims]
        golden.append({"file": name, "crc32": zlib.crc32(raw[:-4]) & 0xFFFFFFFF,
                       "size": len(raw), "has_background": bg is not None})
    committed = json.loads(Path("/root/reference/pkg/frontend/test/fixtures/golden.json")
                           .read_text())
    for a, b in zip(golden, committed):
        assert (a["crc32"], a["size"]) == (b["crc32"], b["size"]), (a, b)
    (OUT / "plnx_golden.json").write_text(json.dumps(golden, indent=1))

    grid = px.build_toy_grid(24)                 # make_viewer_fixtures.py:88-120
    px.save_grid(grid, OUT / "toy.plnx")
    radius, azim, elev = 3.0, 0.8, 0.5
    pos = radius * np.array([np.cos(azim) * np.cos(elev),
                             np.sin(azim) * np.cos(elev), np.sin(elev)])
    zc = pos / np.linalg.norm(pos)
    xc = np.cross([0.0, 0.0, 1.0], zc)
    xc /= np.linalg.norm(xc)
    yc = np.cross(zc, xc)
    c2w = np.eye(4)
    c2w[:3, 0], c2w[:3, 1], c2w[:3, 2], c2w[:3, 3] = xc, yc, zc, pos
    w = h = 40
    focal = 0.5 * w / np.tan(0.5 * 0.6911112)
    cam = px.Camera(c2w=c2w, focal=focal, width=w, height=h)
    opts = px.RenderOptions(step_frac=0.5, stop_thresh=1e-4, background=(1.0, 1.0, 1.0))
    loaded, _ = px.load_grid(OUT / "toy.plnx")
    img = px.render_image(loaded, cam, opts)
    img.astype("<f4").tofile(OUT / "toy_render.bin")
    ref = json.loads(Path("/root/reference/pkg/frontend/test/fixtures/toy_ref.json")
                     .read_text())
    assert np.allclose(ref["c2w"], c2w.tolist(), atol=0) and ref["focal"] == focal
    (OUT / "toy_ref.json").write_text(json.dumps(ref, indent=1))


def _dataset_arrays(ds):
    imgs = np.stack([np.rint(np.asarray(im) * 255.0) for im in ds.images]).astype(np.uint8)
    c2w = np.stack([c.c2w for c in ds.cameras])
    focal = np.array([c.focal for c in ds.cameras])
    return imgs, c2w, focal


def make_trainer_tiny():
    """A 30-step run of trainer.train on the tiny toy set (test_trainer.py:146)."""
    with tempfile.TemporaryDirectory() as td:
        px.make_toy_dataset(Path(td) / "t", n_views=4, res=32, n_test=2, grid_dim=16)
        train = px.load_nerf_dataset(Path(td) / "t", "bounded", "train")
        test = px.load_nerf_dataset(Path(td) / "t", "bounded", "test")
    cfg = px.toy_config(grid_dim=8, total_steps=30, batch_size=64)
    cfg.eval_every = 0
    cfg.log_every = 1
    cfg.seed = 11
    res = px.train(train, cfg, test_ds=test)
    loss = np.array([m["loss"] for m in res.metrics if "loss" in m])
    mse = np.array([m["mse"] for m in res.metrics if "mse" in m])
    nnz = np.array([m["nnz_fraction"] for m in res.metrics if "nnz_fraction" in m])
    psnr = [m["psnr"] for m in res.metrics if "psnr" in m][-1]
    imgs, c2w, focal = _dataset_arrays(train)
    timgs, tc2w, tfocal = _dataset_arrays(test)
    np.savez_compressed(OUT / "trainer_tiny.npz", imgs=imgs, c2w=c2w, focal=focal,
                        test_imgs=timgs, test_c2w=tc2w, test_focal=tfocal,
                        loss=loss, mse=mse, nnz=nnz, psnr=np.array([psnr]),
                        table=res.grid.table, links=res.grid.links)


def make_toy128():
    """The acceptance dataset (conftest.py:74-79 / test_acceptance.py:192-205)."""
    with tempfile.TemporaryDirectory() as td:
        px.make_toy_dataset(Path(td) / "toy128", n_views=25, res=128, n_test=10,
                            grid_dim=64)
        train = px.load_nerf_dataset(Path(td) / "toy128", "bounded", "train")
        test = px.load_nerf_dataset(Path(td) / "toy128", "bounded", "test")
    imgs, c2w, focal = _dataset_arrays(train)
    timgs, tc2w, tfocal = _dataset_arrays(test)
    np.savez_compressed(OUT / "toy128.npz", imgs=imgs, c2w=c2w, focal=focal,
                        test_imgs=timgs, test_c2w=tc2w, test_focal=tfocal,
                        published_psnr=np.array([34.64]))


def main():
    rng = np.random.default_rng(2112_05131)
    make_render(rng)
    make_backward(rng)
    make_tv(rng)
    make_optim(rng)
    make_maxw(rng)
    make_structure(rng)
    make_viewer_goldens()
    make_trainer_tiny()
    make_toy128()
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
