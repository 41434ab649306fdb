#!/usr/bin/env python3
"""The reference's own PSNR spread on the toy acceptance run
(pkg/tests/test_acceptance.py:192-205: 25 views x 128^2, 64^3, 5000 x 3000).

The reference is deterministic (one thread, float64), so its published
34.64 dB is ONE draw of a trajectory that is chaotic at the voxel level:
RMSProp normalises gradient magnitude, so rounding-level differences in a
gradient flip whole updates.  To know what "within 0.05 dB" can mean for a
float32 / atomic-accumulation implementation, this script runs the UNMODIFIED
reference trainer (imported from /root/reference/pkg/src in this container
only) several times:
  stock    : as published (expect 34.64);
  f32      : table and RMSProp state rounded to float32 after every
             optimiser step (our storage precision), init perturbed by a
             random +-1 f32 ulp per value with seeds 1..K.
Writes tests/golden/psnr_spread.json.  Usage: python ref_psnr_spread.py K
(runs K+1 trainings in parallel processes, ~4 min each on one core)."""
import json
import os
import sys
import tempfile
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def run(seed):
    import numpy as np
    import plenoxel as px
    from plenoxel import optim as popt, trainer as ptr

    if seed > 0:
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
        px.make_toy_dataset(Path(td) / "toy", n_views=25, res=128, n_test=10, grid_dim=64)
        train = px.load_nerf_dataset(Path(td) / "toy", "bounded", "train")
        test = px.load_nerf_dataset(Path(td) / "toy", "bounded", "test")
        cfg = px.load_config(Path(td) / "toy" / "toy_config.yaml")
    cfg.eval_every = 0
    res = px.train(train, cfg, test_ds=test)
    return seed, [m for m in res.metrics if "psnr" in m][-1]["psnr"]


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    with ProcessPoolExecutor(max_workers=min(k + 1, os.cpu_count() or 1)) as ex:
        res = dict(ex.map(run, range(k + 1)))
    out = {"stock": res[0], "f32_perturbed": [res[s] for s in range(1, k + 1)]}
    (OUT / "psnr_spread.json").write_text(json.dumps(out, indent=1))
    print(out)


if __name__ == "__main__":
    main()
