import os, sys, json
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from collections import defaultdict
from torch.profiler import ProfilerActivity, profile
from paper_2112_05131_b200 import grid as gmod, optim, render, scenes, trainer
dev = torch.device("cuda", 0)
gt64 = scenes.build_toy_grid(64, device=dev)
g512 = gt64.upsample((512, 512, 512))
cams, _ = scenes.hemisphere_cameras(64, 512, phase=1.0)
opts = render.RenderOptions(background=(1.0, 1.0, 1.0))
imgs = [(np.rint(np.clip(render.render_image(gt64, c, opts), 0, 1) * 255) / 255).astype(np.float32) for c in cams]
ds = scenes.Dataset(np.stack(imgs), cams)
cfg = trainer.default_config("bounded"); cfg.aabb = (-1.1,)*3 + (1.1,)*3
cfg.ladder = [trainer.LadderRung(0, (8, 8, 8))]; cfg.lambda_tv_sigma = cfg.lambda_tv_sh = 0.0
cfg.batch_size = int(os.environ.get("B", 1 << 18))
tr = trainer.Trainer(ds, cfg, device=dev)
tr.grid = g512.copy(); tr.state = optim.OptimState(tr.grid.n_rows, device=dev)
tr.grads = gmod.GradientBuffer(tr.grid.n_rows, device=dev); tr._refresh_cache()
for s in range(3): tr.step(s)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(5): tr.step(3 + s)
    torch.cuda.synchronize()
agg = defaultdict(float)
for e in prof.events():
    if e.device_type.name == "CUDA": agg[e.name[:60]] += e.device_time / 5
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]: print(f"{v:9.1f} us  {k}")
print("n events", sum(1 for e in prof.events() if e.device_type.name == "CUDA"))
