#!/usr/bin/env python3
"""How much of the update and the next step's march can overlap (C2 state,
step 5): the update (compaction + opt_rows) and a forward render of the next
batch (march_kernel<FWD>, the march's proxy) timed alone and on two streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import optim, render, trainer, _lib  # noqa: E402

dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


tr = trainer.Trainer(ds, bench.bench_config(A), device=dev)
for s in range(6):
    tr.step(s)
torch.cuda.synchronize()
# gradients of one step without its update: render + TV through the public API
idx = tr.batcher.next_device()
o, d, vd, gt = tr.pool.materialize(idx)
tr.grads.clear()
render.fused_mse_backward(tr.grid, o, d, vd, gt, tr.grads, tr.opts, n_total=5000)
torch.cuda.synchronize()
g_keep, m_keep = tr.grads.data.clone(), tr.grads.touched_mask.clone()
idx2 = tr.batcher.next_device()
o2, d2, vd2, _ = tr.pool.materialize(idx2)
st_keep = tr.state.v.clone()
sh_keep, den_keep = tr.grid.sh.clone(), tr.grid.density.clone()
s_up, s_m = torch.cuda.Stream(), torch.cuda.Stream()


def restore():
    tr.grads.data.copy_(g_keep)
    tr.grads.touched_mask.copy_(m_keep)
    tr.state.v.copy_(st_keep)
    tr.grid.sh.copy_(sh_keep)
    tr.grid.density.copy_(den_keep)
    torch.cuda.synchronize()


def upd():
    optim.step(tr.grid, tr.grads, tr.state, 0.1, 0.01, clear=True)


def mar():
    render.render_rays(tr.grid, o2, d2, tr.opts, viewdirs=vd2)


def timed(fn, reps=10):
    tot = 0.0
    for _ in range(reps):
        restore()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1000


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s_up.wait_event(ev)
    s_m.wait_event(ev)
    with torch.cuda.stream(s_up):
        upd()
    with torch.cuda.stream(s_m):
        mar()
    cur.wait_stream(s_up)
    cur.wait_stream(s_m)


print(f"update alone  {timed(upd):7.1f} us")
print(f"fwd render    {timed(mar):7.1f} us")
print(f"serial        {timed(lambda: (upd(), mar())):7.1f} us")
print(f"two streams   {timed(both):7.1f} us")
