#!/usr/bin/env python3
"""Train the toy acceptance run (pkg/tests/test_acceptance.py:192-205 setup)
and save the final grid as .plnx (for cross-evaluation with the reference's
own evaluate on the host).  usage: python scripts/psnr_export.py OUT.plnx"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import load  # noqa: E402
from paper_2112_05131_b200 import artifact_io, trainer  # noqa: E402
from paper_2112_05131_b200.scenes import dataset_from_arrays  # noqa: E402

z = load("toy128.npz")
tr_ds = dataset_from_arrays(z["imgs"], z["c2w"], z["focal"], tag="train")
te_ds = dataset_from_arrays(z["test_imgs"], z["test_c2w"], z["test_focal"], tag="test")
cfg = trainer.toy_config(grid_dim=64, total_steps=5000, batch_size=3000)
cfg.eval_every = 0
cfg.log_every = 0
res = trainer.train(tr_ds, cfg, test_ds=te_ds)
print("ours psnr", [m["psnr"] for m in res.metrics if "psnr" in m][-1])
artifact_io.save_grid(res.grid, sys.argv[1])
