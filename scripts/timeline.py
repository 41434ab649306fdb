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

# per-ray phase times vs march positions / samples
L.plx_debug_raylog.argtypes = [ctypes.c_void_p, ctypes.c_int]
rb = (ctypes.c_ulonglong * (4 * 5000))()
L.plx_debug_raylog(rb, 5000)
r = np.array(rb, dtype=np.uint64).reshape(5000, 4)
tA, tB, tC = r[:, 0] / 1e3, r[:, 1] / 1e3, r[:, 2] / 1e3
pos, ns = (r[:, 3] >> np.uint64(32)).astype(np.int64), (r[:, 3] & np.uint64(0xffffffff)).astype(np.int64)
tot = tA + tB + tC
print(f"per ray (us): A {tA.mean():.1f}  B {tB.mean():.1f}  C {tC.mean():.1f}  total mean "
      f"{tot.mean():.1f} p90 {np.percentile(tot, 90):.1f} max {tot.max():.1f}")
print(f"  positions mean {pos.mean():.0f} max {pos.max()}  samples mean {ns.mean():.0f} max {ns.max()}")
top = np.argsort(-tot)[:8]
for i in top:
    print(f"  ray {i:5d}: {tot[i]:6.1f} us  A {tA[i]:5.1f} B {tB[i]:5.1f} C {tC[i]:5.1f}  "
          f"pos {pos[i]} samples {ns[i]}")
print(f"  A us per 32 positions {np.sum(tA) / (np.sum(pos) / 32):.2f}; B+C us per 32 samples "
      f"{np.sum(tB + tC) / max(np.sum(ns) / 32, 1):.2f}")
