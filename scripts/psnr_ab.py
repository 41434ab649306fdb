#!/usr/bin/env python3
"""Toy acceptance run (pkg/tests/test_acceptance.py:192-205 setup: 25 views x
128^2, 64^3, 5000 steps x 3000 rays) repeated N times; prints the final PSNR
of each run and, with --out, appends a per-run record to a JSON log (kernel
A/B via PLX_LIB; a tag names the variant).

  python scripts/psnr_ab.py N [--out gpurun_out/psnr_runs.json] [--tag name]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import load  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402
from paper_2112_05131_b200.scenes import dataset_from_arrays  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="?", default=3)
ap.add_argument("--out", default=None)
ap.add_argument("--tag", default=os.environ.get("PLX_LIB", "default"))
ap.add_argument("--seed", type=int, default=0, help="trainer seed (batch order / TV cells)")
args = ap.parse_args()

z = load("toy128.npz")
tr_ds = dataset_from_arrays(z["imgs"], z["c2w"], z["focal"], tag="train")
te_ds = dataset_from_arrays(z["test_imgs"], z["test_c2w"], z["test_focal"], tag="test")
out = []
for i in range(args.n):
    cfg = trainer.toy_config(grid_dim=64, total_steps=5000, batch_size=3000)
    cfg.eval_every = 0
    cfg.log_every = 0
    cfg.seed = args.seed
    t0 = time.perf_counter()
    res = trainer.train(tr_ds, cfg, test_ds=te_ds)
    out.append([m["psnr"] for m in res.metrics if "psnr" in m][-1])
    print(f"run {i}: {out[-1]:.4f} dB ({time.perf_counter() - t0:.1f} s)", flush=True)
print(args.tag, " ".join(f"{p:.4f}" for p in out), "mean %.4f std %.4f" % (np.mean(out), np.std(out)))
if args.out:
    log = json.load(open(args.out)) if os.path.exists(args.out) else {}
    rec = log.setdefault(args.tag, {"runs": []})
    rec["runs"] += out
    rec["mean"] = float(np.mean(rec["runs"]))
    rec["std"] = float(np.std(rec["runs"]))
    rec["n"] = len(rec["runs"])
    json.dump(log, open(args.out, "w"), indent=1)
