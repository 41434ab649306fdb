#!/usr/bin/env python3
"""BASELINE C4 throughput on 1 GPU: forward-facing NDC scene at the final
rung's 1408 x 1156 x 128 sparse grid (tests/test_gpu_configs.py::_c4_grid:
two density blobs, ~2 % of 208 M lattice points occupied), the reference's
forward-facing defaults (T:130-140: TV 5e-4 / 5e-3 on 1 % of the cells,
Cauchy 1e-12, RMSProp), 5000-ray batches from a forward-facing camera pool
(rays generated and NDC-warped on the device).  Device-timed steps of
Trainer.step (CUDA-graph replay)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2112_05131_b200 import grid as gmod, optim, scenes, trainer
    from paper_2112_05131_b200.camera import Camera
    from test_gpu_configs import _c4_grid

    dev = torch.device("cuda", 0)
    n_views = int(os.environ.get("VIEWS", 20))
    cams = []
    for i in range(n_views):
        c2w = np.eye(4)
        a = 2 * np.pi * i / n_views
        c2w[0, 3], c2w[1, 3] = 0.15 * np.cos(a), 0.1 * np.sin(a)
        cams.append(Camera(c2w=c2w, focal=1100.0, width=1008, height=756))
    rng = np.random.default_rng(0)
    imgs = rng.uniform(0, 1, (n_views, 756, 1008, 3)).astype(np.float32)
    ds = scenes.Dataset(imgs, cams, "forward_facing_ndc", np.zeros(3))
    cfg = trainer.default_config("forward_facing_ndc")
    cfg.batch_size = int(os.environ.get("B", 5000))
    cfg.ladder = [trainer.LadderRung(0, (64, 64, 16))]   # replaced by the C4 grid below
    tr = trainer.Trainer(ds, cfg, device=dev)
    tr.grid = _c4_grid()
    tr.state = optim.OptimState(tr.grid.n_rows, device=dev)
    tr.grads = gmod.GradientBuffer(tr.grid.n_rows, device=dev)
    tr._refresh_cache()
    warm, steps = int(os.environ.get("WARM", 5)), int(os.environ.get("STEPS", 20))
    for s in range(warm):
        tr.step(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = tr.march_stats.clone()
    e0.record()
    for s in range(warm, warm + steps):
        tr.step(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    mst = ((tr.march_stats - st0).double() / steps / cfg.batch_size).cpu().numpy()
    out = {"config": "C4 forward-facing NDC, 1408x1156x128 sparse (%d rows), %d views of "
                     "1008x756, batch %d, TV 1%%, RMSProp" % (tr.grid.n_rows, n_views, cfg.batch_size),
           "ms_per_step": ms, "rays_per_s": cfg.batch_size / ms * 1e3,
           "march_per_ray": {"positions": float(mst[0]), "samples": float(mst[1]),
                             "chunks": float(mst[2])},
           "bricks": tr.grid._bricks is not None}
    if os.environ.get("C4_PROFILE"):
        from collections import defaultdict
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for s in range(warm + steps, warm + steps + 10):
                tr.step(s)
            torch.cuda.synchronize()
        agg = defaultdict(float)
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                agg[ev.name[:50]] += ev.device_time / 10
        out["kernel_us_per_step"] = {k: round(v, 1) for k, v in
                                     sorted(agg.items(), key=lambda kv: -kv[1])[:8]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
