"""Mean final PSNR of N toy acceptance runs (test_gpu_trainer.py's protocol) for
the package found first on sys.path (bisecting a PSNR shift across builds):
python scripts/psnr_mean.py [pkg_root] [N]"""
import os
import sys

root = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-" else os.getcwd()
sys.path.insert(0, root)
sys.path.insert(1, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402

from helpers import load  # noqa: E402
sys.path.insert(0, os.getcwd())
from paper_2112_05131_b200 import trainer  # noqa: E402
import paper_2112_05131_b200 as px  # noqa: E402


n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_trainer as T  # noqa: E402
z = load("toy128.npz")
tr_ds, te_ds = T._ds(z), T._ds(z, "test_")
runs = []
for _ in range(n):
    cfg = trainer.toy_config(grid_dim=64, total_steps=5000, batch_size=3000)
    cfg.eval_every = 0
    cfg.log_every = 0
    res = trainer.train(tr_ds, cfg, test_ds=te_ds)
    runs.append([m["psnr"] for m in res.metrics if "psnr" in m][-1])
print(f"{px.__file__}: mean of {n} runs {np.mean(runs):.4f} std {np.std(runs):.4f}", flush=True)
