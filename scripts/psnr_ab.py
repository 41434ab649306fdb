#!/usr/bin/env python3
"""Toy acceptance run (pkg/tests/test_acceptance.py:192-205 setup) repeated
N times; prints the final PSNR of each run (kernel A/B via PLX_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from helpers import load  # noqa: E402
from paper_2112_05131_b200 import trainer  # noqa: E402
from paper_2112_05131_b200.scenes import dataset_from_arrays  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
z = load("toy128.npz")
tr_ds = dataset_from_arrays(z["imgs"], z["c2w"], z["focal"], tag="train")
te_ds = dataset_from_arrays(z["test_imgs"], z["test_c2w"], z["test_focal"], tag="test")
out = []
for i in range(n):
    cfg = trainer.toy_config(grid_dim=64, total_steps=5000, batch_size=3000)
    cfg.eval_every = 0
    cfg.log_every = 0
    res = trainer.train(tr_ds, cfg, test_ds=te_ds)
    out.append([m["psnr"] for m in res.metrics if "psnr" in m][-1])
print(os.environ.get("PLX_LIB", "default"), " ".join(f"{p:.4f}" for p in out),
      "mean %.4f" % np.mean(out))
