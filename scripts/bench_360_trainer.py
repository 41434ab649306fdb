#!/usr/bin/env python3
"""Wall-clock throughput of Trainer.step on an unbounded_360 scene at the
reference's 360 defaults (T:133-154: 128^3 first rung, 64 x 1024 x 2048
background layers, 5000-ray batches, grid + background TV, beta and Cauchy
terms, both updates), 20 views of 200 x 200 on a camera ring (synthetic
images).  The 360 step reads its loss every step (the reference's order), so
this is host + device time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2112_05131_b200 import scenes, trainer
    from paper_2112_05131_b200.camera import Camera

    n_views, res = 20, 200
    cams = []
    for i in range(n_views):
        a = 2 * np.pi * i / n_views
        eye = np.array([2.5 * np.cos(a), 2.5 * np.sin(a), 0.3])
        f = -eye / np.linalg.norm(eye)
        r = np.cross(f, [0.0, 0.0, 1.0])
        r /= np.linalg.norm(r)
        u = np.cross(r, f)
        c2w = np.eye(4)
        c2w[:3, 0], c2w[:3, 1], c2w[:3, 2], c2w[:3, 3] = r, u, -f, eye
        cams.append(Camera(c2w=c2w, focal=200.0, width=res, height=res))
    rng = np.random.default_rng(0)
    ds = scenes.Dataset(rng.uniform(0, 1, (n_views, res, res, 3)).astype(np.float32), cams,
                        "unbounded_360", np.zeros(3))
    cfg = trainer.default_config("unbounded_360")
    cfg.batch_size = 5000
    tr = trainer.Trainer(ds, cfg, device=torch.device("cuda", 0))
    warm, steps = 5, int(os.environ.get("STEPS", 50))
    for s in range(warm):
        tr.step(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(warm, warm + steps):
        tr.step(s)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / steps * 1e3
    print(json.dumps({"config": "360 trainer step, 128^3 + 64x1024x2048 background, 5000 rays",
                      "ms_per_step_wall": ms, "rays_per_s": 5000 / ms * 1e3}))


if __name__ == "__main__":
    main()
