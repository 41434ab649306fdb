#!/usr/bin/env python3
"""Throughput of the 360 path: the fused grid + MSI
background render with the MSE / Cauchy / beta backward (plx_msi_render), the
background TV and the background update, at the reference's 360 defaults
(T:133-154: 128^3 dense first rung, 64 x 1024 x 2048 layers, 5000 rays per
step), device-timed with CUDA events; beside it the CPU oracle
(oracle/plx_oracle.c: oracle_render_360, the reference's K:661-881 restated,
1 core) on a bounded sample of the same rays.  Prints one JSON line.

usage: python scripts/bench_msi.py [--steps K] [--warmup W] [--oracle-rays N]"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--rays", type=int, default=5000)
    ap.add_argument("--dims", type=int, default=128)
    ap.add_argument("--layers", type=int, default=64)
    ap.add_argument("--height", type=int, default=1024)
    ap.add_argument("--width", type=int, default=2048)
    ap.add_argument("--oracle-rays", type=int, default=100)
    args = ap.parse_args()

    from paper_2112_05131_b200 import _lib, msi
    from paper_2112_05131_b200.grid import GradientBuffer, SparseGrid
    from paper_2112_05131_b200.render import RenderOptions, kernel_opts

    dev = torch.device("cuda", 0)
    D = args.dims
    grid = SparseGrid.dense((D,) * 3, (-1.0,) * 3, (1.0,) * 3, sigma=0.1, rgb=0.1, device=dev)
    bg = msi.MsiBackground.create(args.layers, args.height, args.width, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    bg.data[..., 0] = 0.1 + 0.05 * torch.rand(bg.data.shape[:3], generator=g, device=dev,
                                              dtype=torch.float64)
    bg.data[..., 1:] = 0.1
    rng = np.random.default_rng(0)
    n = args.rays
    th = rng.uniform(0, 2 * np.pi, n)
    o = np.stack([0.9 * np.cos(th), 0.9 * np.sin(th), rng.uniform(-0.2, 0.2, n)], 1)
    tgt = rng.uniform(-0.3, 0.3, (n, 3))
    d = tgt - o
    d[::3] = rng.normal(size=d[::3].shape)       # a third look outwards / sideways
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    gt = rng.uniform(0, 1, (n, 3))
    ot, dt, gtt = (torch.from_numpy(a).to(dev) for a in (o, d, gt))
    opts = RenderOptions(background=(0.0, 0.0, 0.0))
    grads, bgg = GradientBuffer(grid.n_rows, device=dev), msi.BgGradientBuffer(bg)
    st = msi.BgOptimState(bg)
    cg, ko, cb = grid._c(with_occ=True), kernel_opts(grid, opts), bg._c()
    L = _lib.lib()
    need = int(L.plx_msi_scratch_bytes(ctypes.byref(cg), ctypes.byref(cb), ctypes.byref(ko), n))
    scratch = torch.empty(need, dtype=torch.uint8, device=dev)
    r = _lib.PlxRays()
    r.origins, r.dirs, r.viewdirs, r.target = ot.data_ptr(), dt.data_ptr(), None, gtt.data_ptr()
    r.jitter, r.idx, r.n = None, None, n
    rgb = torch.empty((n, 3), dtype=torch.float64, device=dev)
    tfg = torch.empty(n, dtype=torch.float64, device=dev)
    trans = torch.empty(n, dtype=torch.float64, device=dev)
    sums = torch.zeros(3, dtype=torch.float64, device=dev)
    cgrad, cbgg = grads._c(with_ids=False), bgg._c()
    cells_rng = np.random.default_rng(1)
    stream = _lib.stream_ptr()

    def render():
        _lib.check(L.plx_msi_render(ctypes.byref(cg), ctypes.byref(cb), ctypes.byref(r),
                                    ctypes.byref(ko), 1, 2.0 / n, 1e-11, 1e-5, 1e-6,
                                    ctypes.byref(cgrad), ctypes.byref(cbgg), rgb.data_ptr(),
                                    tfg.data_ptr(), trans.data_ptr(), sums.data_ptr(),
                                    scratch.data_ptr(), need, stream), "msi_render")

    def render_fwd():
        _lib.check(L.plx_msi_render(ctypes.byref(cg), ctypes.byref(cb), ctypes.byref(r),
                                    ctypes.byref(ko), 1, 2.0 / n, 1e-11, 1e-5, 1e-6,
                                    None, None, rgb.data_ptr(), tfg.data_ptr(),
                                    trans.data_ptr(), sums.data_ptr(), scratch.data_ptr(),
                                    need, stream), "msi_render_fwd")

    legs = {"render_bwd": 0.0, "bg_tv": 0.0, "bg_update": 0.0, "grid_clear": 0.0}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def step(timed=False):
        ev[0].record()
        render()
        ev[1].record()
        run = msi.sample_bg_tv_cells(bg, 0.01, cells_rng)
        _lib.check(L.plx_msi_tv(ctypes.byref(cb), None, run.start, run.count, 1e-6,
                                1e-3 / run.count, 1e-3 / run.count, ctypes.byref(cbgg),
                                sums.data_ptr(), stream), "msi_tv")
        ev[2].record()
        msi.step_table(bg, bgg, st, 1.0, 0.01)
        ev[3].record()
        grads.clear()
        ev[4].record()
        if timed:
            torch.cuda.synchronize()
            for i, k in enumerate(legs):
                legs[k] += ev[i].elapsed_time(ev[i + 1]) / args.steps

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if os.environ.get("MSI_PROFILE"):   # per-kernel device times of the render (CUPTI)
        from collections import defaultdict
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(10):
                render()
                grads.clear()
                bgg.clear()
            torch.cuda.synchronize()
        agg = defaultdict(float)
        for ev_ in prof.events():
            if ev_.device_type.name == "CUDA":
                agg[ev_.name[:60]] += ev_.device_time / 10
        for k_, v_ in sorted(agg.items(), key=lambda kv: -kv[1]):
            print(f"{v_:9.1f} us/render  {k_}", file=sys.stderr)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t_render = t_step = 0.0
    for _ in range(args.steps):
        e[0].record()
        render()
        e[1].record()
        torch.cuda.synchronize()
        t_render += e[0].elapsed_time(e[1])
        grads.clear()
        bgg.clear()
    for _ in range(args.steps):
        e[2].record()
        step(timed=True)
        e[3].record()
        torch.cuda.synchronize()
        t_step += e[2].elapsed_time(e[3])
    ms_render, ms_step = t_render / args.steps, t_step / args.steps
    t_fwd = 0.0
    for _ in range(args.steps):
        e[0].record()
        render_fwd()
        e[1].record()
        torch.cuda.synchronize()
        t_fwd += e[0].elapsed_time(e[1])
    ms_fwd = t_fwd / args.steps

    # Roofline of the fused render/backward on its compulsory bytes: every
    # distinct grid row it touches read once (112 B of the 128-B row) and its
    # gradient row read + written once (the red.add lines), every distinct
    # background texel the same at 32 B, plus the ray inputs / outputs; the
    # per-sample record scratch is this design's, not compulsory.
    grads.clear()
    bgg.clear()
    render()
    torch.cuda.synchronize()
    rows, texels = grads.n_touched, bgg.n_touched
    grads.clear()
    bgg.clear()
    alg = rows * 3 * 112 + texels * 3 * 32 + n * (9 + 3 + 3 + 2) * 8
    peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "MEASURED_PEAKS.json")
    peak = json.load(open(peaks))["hbm_gbs"] if os.path.exists(peaks) else 7700.0
    achieved = alg / (ms_render * 1e-3) / 1e9

    # CPU oracle on a bounded sample of the same rays (1 core)
    from oracle import oracle as orc
    og = orc.Grid.dense((D,) * 3, (-1.0,) * 3, (1.0,) * 3, sigma=0.1, rgb=0.1)
    og.table[:] = og.table.astype(np.float32)
    # per-ray work does not depend on the texel count: a 64 x 128 layer
    # lattice keeps the host copy small
    bgd = np.full((args.layers, 64, 128, 4), 0.1)
    k = args.oracle_rays
    buf, bgb = orc.GradBuf(og.n_rows), orc.BgGradBuf(bgd.shape[0] * 64 * 128)
    t0 = time.perf_counter()
    orc.render_360(og, bgd, bg.radii, o[:k], d[:k], gt_rgb=gt[:k], buf=buf, bg_buf=bgb,
                   n_total=n, lam_cauchy=1e-11, lam_beta=1e-5)
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": "360 train rays/sec (grid + MSI background fused render/backward)",
        "config": {"grid": f"{D}^3 dense", "background": f"{args.layers}x{args.height}x"
                   f"{args.width} f64 texels", "rays": n, "steps": args.steps},
        "render_bwd_ms": ms_render, "render_fwd_only_ms": ms_fwd, "render_bwd_rays_per_s": n / (ms_render / 1e3),
        "step_ms": ms_step, "step_rays_per_s": n / (ms_step / 1e3), "step_legs_ms": legs,
        "roofline": {"kernel": "msi_render (fused render/backward)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "algorithmic_bytes": alg,
                     "touched_rows": rows, "touched_texels": texels,
                     "model": "rows*3*112 + texels*3*32 + rays*17*8"},
        "step_note": "render+backward, background TV (1% texels), background update + clear, "
                     "grid gradient clear",
        "cpu_oracle": {"rays_per_s": k / cpu_s, "rays": k, "cores": 1,
                       "kind": "port (oracle_render_360, K:661-881)"},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
