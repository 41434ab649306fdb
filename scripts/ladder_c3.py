#!/usr/bin/env python3
"""BASELINE C3: coarse-to-fine 256^3 -> 512^3 with density pruning, 1 GPU.

Trains the bounded default config on the device for S1 steps at 256^3, fires
the rung event (max-weight-free density prune at 5.0 ... here the bounded
config's criterion switched to 'density' per C3, G:228-258), upsamples to 512^3
(G:260-285), and trains S2 more steps.  Reports step rates before/after and
the rung event cost (prune + upsample + state reset), all device-timed."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2112_05131_b200 import trainer

    class A:
        batch, gpus, dims, views, res = 5000, 1, 256, 100, 200

    dev = torch.device("cuda", 0)
    S1, S2 = int(os.environ.get("S1", 200)), int(os.environ.get("S2", 100))
    ds = bench.toy_scene(A.views, A.res, dev)
    cfg = bench.bench_config(A)
    cfg.ladder = [trainer.LadderRung(0, (256, 256, 256)), trainer.LadderRung(S1, (512, 512, 512))]
    cfg.prune_criterion = "density"
    cfg.prune_threshold = float(os.environ.get("THR", 1.0))
    cfg.total_steps = S1 + S2
    tr = trainer.Trainer(ds, cfg, device=dev)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for s in range(5):
        tr.step(s)
    torch.cuda.synchronize()
    e[0].record()
    for s in range(5, S1):
        tr.step(s)
    e[1].record()
    torch.cuda.synchronize()
    rows_before = tr.grid.n_rows
    w0 = time.perf_counter()
    e[2].record()
    tr.rung_event((512, 512, 512), None, S1)
    e[3].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    for s in range(S1, S1 + 5):
        tr.step(s)
    torch.cuda.synchronize()
    e[4].record()
    for s in range(S1 + 5, S1 + S2):
        tr.step(s)
    e[5].record()
    torch.cuda.synchronize()
    ms1 = e[0].elapsed_time(e[1]) / (S1 - 5)
    ms2 = e[4].elapsed_time(e[5]) / (S2 - 5)
    st0 = tr.march_stats.clone()
    for s in range(S1 + S2, S1 + S2 + 10):
        tr.step(s)
    torch.cuda.synchronize()
    mst = ((tr.march_stats - st0).double() / 10 / A.batch).cpu().numpy()
    e[0].record()
    for _ in range(10):
        tr.grid.rebuild_bricks()
    e[1].record()
    torch.cuda.synchronize()
    brick_ms = e[0].elapsed_time(e[1]) / 10
    kt = None
    if os.environ.get("C3_PROFILE"):   # per-kernel device times at 512^3 (CUPTI)
        from collections import defaultdict
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for s in range(S1 + S2 + 10, S1 + S2 + 20):
                tr.step(s)
            torch.cuda.synchronize()
        agg = defaultdict(float)
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                agg[ev.name[:50]] += ev.device_time / 10
        kt = {k: round(v, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]}
    out = {"config": "C3 256^3 -> 512^3, density prune thr %.2f" % cfg.prune_threshold,
           "kernel_us_per_step_512": kt,
           "march_per_ray_512": {"positions": float(mst[0]), "samples": float(mst[1]),
                                 "chunks": float(mst[2])},
           "brick_rebuild_ms": brick_ms if tr.grid._bricks is not None else None,
           "rows_256": rows_before, "rows_512": tr.grid.n_rows,
           "ms_per_step_256": ms1, "rays_per_s_256": A.batch / ms1 * 1e3,
           "ms_per_step_512": ms2, "rays_per_s_512": A.batch / ms2 * 1e3,
           "rung_event_ms_device": e[2].elapsed_time(e[3]), "rung_event_s_wall": wall,
           "nnz_fraction_512": tr.nnz_fraction()}
    print(json.dumps(out))
    with open("gpurun_out/ladder_c3.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
