import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from collections import defaultdict
from torch.profiler import ProfilerActivity, profile
from paper_2112_05131_b200 import msi
dev = torch.device("cuda", 0)
bg = msi.MsiBackground.create(64, 1024, 2048, device=dev)
bg.data[..., 0] = 0.1
g = msi.BgGradientBuffer(bg)
st = msi.BgOptimState(bg)
n = bg.n_texels
idx = torch.randint(0, n, (3_000_000,), device=dev)
def fill():
    g.touched_mask[idx] = 1
    g.data[idx] = 0.01
for _ in range(2):
    fill(); msi.step_table(bg, g, st, 1.0, 0.01)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        fill(); msi.step_table(bg, g, st, 1.0, 0.01)
    torch.cuda.synchronize()
agg = defaultdict(float)
for e in prof.events():
    if e.device_type.name == "CUDA": agg[e.name[:70]] += e.device_time / 3
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]: print(f"{v:9.1f} us  {k}")
