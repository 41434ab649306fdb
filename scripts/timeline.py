#!/usr/bin/env python3
"""Warp timeline of one bwd_kernel launch at the C2 bench state (needs a
-DPLX_TIMELINE build via PLX_LIB): per-warp start/end -> the tail (time the
kernel runs with fewer than half / a quarter of its warps still active)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_05131_b200 import _lib, trainer  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 12
dev = torch.device("cuda", 0)
ds = bench.toy_scene(100, 200, dev)


class A:
    batch, gpus, dims = 5000, 1, 256


tr = trainer.Trainer(ds, bench.bench_config(A), device=dev)
for s in range(warm):
    tr.step(s)
torch.cuda.synchronize()
L = _lib.lib()
n = 8192
buf = (ctypes.c_ulonglong * (2 * n))()
L.plx_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.plx_debug_timeline(buf, n)
a = np.array(buf, dtype=np.float64).reshape(n, 2)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
start, end = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
T = end.max()
ends = np.sort(end)
print(f"warps {len(a)}  kernel {T:.1f} us  starts within {start.max():.1f} us")
for q in (0.5, 0.75, 0.9, 0.99):
    print(f"  {int(q * 100)}% of warps done at {ends[int(q * len(ends)) - 1]:.1f} us")

# per-ray march times (start, end, positions)
L.plx_debug_raylog.argtypes = [ctypes.c_void_p, ctypes.c_int]
rb = (ctypes.c_ulonglong * (3 * 5000))()
L.plx_debug_raylog(rb, 5000)
r = np.array(rb, dtype=np.float64).reshape(5000, 3)
rs, re, rp = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3, r[:, 2]
dur = re - rs
print(f"rays: duration mean {dur.mean():.1f} us, p50 {np.median(dur):.1f}, max {dur.max():.1f}; "
      f"positions mean {rp.mean():.0f}, max {rp.max():.0f}; ns/position {1e3 * dur.sum() / rp.sum():.2f}")
late = rs > np.percentile(rs, 60)
print(f"rays started after the first wave: {int((rs > 1.0).sum())}, their mean duration {dur[rs > 1.0].mean():.1f} us, "
      f"first-wave rays {dur[rs <= 1.0].mean():.1f} us")
for t in range(0, int(T) + 5, 5):
    act = int(((start <= t) & (end > t)).sum())
    print(f"  t={t:4d} us  active warps {act}")
