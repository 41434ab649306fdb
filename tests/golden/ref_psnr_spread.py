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
             random +-1 f32 ulp per value with seeds 1..K;
  REF_GRAD_F32=1: additionally the gradients rounded to float32 before each
             update (-> psnr_spread_grad32.json).
Writes tests/golden/psnr_spread.json.  Usage: python ref_psnr_spread.py K
[FIRST] (runs the stock run plus seeds FIRST..FIRST+K-1 in parallel
processes, ~4 min each on one core; seeds already in the file are kept)."""
import json
import os
import sys
import tempfile
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


GRAD32 = os.environ.get("REF_GRAD_F32") == "1"
# per-step noise of the order of f32 atomic-accumulation reordering
NOISE = os.environ.get("REF_GRAD_NOISE") == "1"


def run(seed):
    import numpy as np
    import plenoxel as px
    from plenoxel import optim as popt, trainer as ptr

    if seed > 0:
        orig_step = popt.step

        def step_f32(grid, grads, state, *a, **k):
            if NOISE:    # f32 accumulation in a nondeterministic order
                rs = np.random.default_rng(seed * 1000003 + int(state.step_count))
                g32 = grads.data.astype(np.float32).astype(np.float64)
                ulp = np.spacing(np.abs(g32).astype(np.float32)).astype(np.float64)
                grads.data[:] = np.where(g32 != 0.0, g32 + ulp * rs.integers(-2, 3, g32.shape),
                                         0.0)
            elif GRAD32:   # gradients as an f32 accumulator would hold them
                grads.data[:] = grads.data.astype(np.float32)
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
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    path = OUT / ("psnr_spread_noise.json" if NOISE else
                  "psnr_spread_grad32.json" if GRAD32 else "psnr_spread.json")
    old = json.loads(path.read_text()) if path.exists() else {}
    seeds = list(range(first, first + k)) + ([] if "stock" in old else [0])
    with ProcessPoolExecutor(max_workers=min(len(seeds), os.cpu_count() or 1)) as ex:
        res = dict(ex.map(run, seeds))
    per_seed = {int(s): v for s, v in old.get("f32_perturbed_by_seed", {}).items()}
    if not per_seed and "f32_perturbed" in old:   # first format: seeds 1..n
        per_seed = {i + 1: v for i, v in enumerate(old["f32_perturbed"])}
    per_seed.update({s: v for s, v in res.items() if s > 0})
    vals = [per_seed[s] for s in sorted(per_seed)]
    out = {"stock": res.get(0, old.get("stock")),
           "f32_perturbed_by_seed": {str(s): per_seed[s] for s in sorted(per_seed)},
           "f32_perturbed_mean": sum(vals) / len(vals),
           "f32_perturbed_min": min(vals), "f32_perturbed_max": max(vals)}
    path.write_text(json.dumps(out, indent=1))
    print(out)


if __name__ == "__main__":
    main()
