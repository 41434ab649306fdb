"""Training losses and image metrics (drop-in for pkg/src/plenoxel/losses.py).

tv_loss (L:50-77) runs the sm_100a TV kernel; sample_tv_cells (L:41-47)
draws the same contiguous wrapped run from the same numpy RNG call but hands
the kernel (start, count) instead of materialising the id array.  MSE /
Cauchy / PSNR / SSIM are host-side helpers with the reference's semantics.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .grid import GradientBuffer, SparseGrid

TV_EPS = 1e-6


def mse_loss(pred, target):
    """L:24-38 -> (loss, dL/dpred)."""
    pred = np.asarray(pred, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    if pred.shape != target.shape:
        raise ValueError("prediction / target shape mismatch")
    if pred.size == 0:
        raise ValueError("empty batch")
    n = pred.shape[0]
    diff = pred - target
    return float(np.sum(diff * diff) / n), 2.0 * diff / n


class CellRun:
    """A contiguous wrapped run of lattice cells (start + arange(count)) % n.
    Behaves like the reference's int64 id array (np.asarray works)."""

    def __init__(self, start: int, count: int, n_cells: int):
        self.start, self.count, self.n_cells = int(start), int(count), int(n_cells)

    @property
    def size(self) -> int:
        return self.count

    def __len__(self) -> int:
        return self.count

    def split(self, rank: int, size: int) -> "CellRun":
        """Contiguous sub-run for one rank (dist.shard_range)."""
        from .dist import shard_range
        s, c = shard_range(self.count, rank, size)
        return CellRun((self.start + s) % self.n_cells, c, self.n_cells)

    def __array__(self, dtype=None, copy=None):
        a = ((self.start + np.arange(self.count)) % self.n_cells).astype(np.int64)
        return a if dtype is None else a.astype(dtype)


def sample_tv_cells(grid: SparseGrid, fraction: float, rng) -> CellRun:
    """L:41-47 (same RNG draw: one rng.integers(0, n_cells))."""
    n_cells = int(np.prod(grid.dims))
    count = max(1, int(round(fraction * n_cells)))
    start = int(rng.integers(0, n_cells))
    return CellRun(start, count, n_cells)


def tv_loss(grid: SparseGrid, cells, lam_sigma: float, lam_sh: float,
            grads: GradientBuffer | None = None, eps: float = TV_EPS,
            wrap=(False, False, False), sums: torch.Tensor | None = None,
            n_norm: int | None = None, _cgrid=None, _cgrad=None):
    """L:50-77 -> (lam_sigma * tv_sigma, lam_sh * tv_sh).

    With a device float64[2] `sums`, the raw (sigma_sum, sh_sum) are
    accumulated there and (sums, n) is returned without a host sync.
    `n_norm` overrides the averaging count (a rank's sub-run of a larger run
    normalises by the global count, dist.py)."""
    if isinstance(cells, CellRun):
        n, start, cptr, keep = cells.count, cells.start, None, None
    else:
        c = torch.as_tensor(np.asarray(cells, dtype=np.int64)) if not isinstance(
            cells, torch.Tensor) else cells
        keep = c.to(grid.device, torch.int64).contiguous()
        n, start, cptr = keep.numel(), 0, keep.data_ptr()
    if n == 0:
        return 0.0, 0.0
    dims = grid.dims
    nn = int(n_norm) if n_norm is not None else n
    dev_sums = sums if sums is not None else torch.zeros(2, dtype=torch.float64,
                                                         device=grid.device)
    gb = (_cgrad if _cgrad is not None else grads._c()) if grads is not None else None
    c_ = _cgrid if _cgrid is not None else grid._c(with_occ=False)
    _lib.check(_lib.lib().plx_tv(
        ctypes.byref(c_), cptr, start, n, dims[0] / 256.0, dims[1] / 256.0, dims[2] / 256.0,
        float(eps), lam_sigma / nn, lam_sh / nn, int(wrap[0]), int(wrap[1]), int(wrap[2]),
        int(grads is not None), ctypes.byref(gb) if gb is not None else None,
        dev_sums.data_ptr(), _lib.stream_ptr()), "tv")
    del keep
    if sums is not None:
        return dev_sums, n
    s = dev_sums.cpu().numpy()
    return lam_sigma * float(s[0]) / nn, lam_sh * float(s[1]) / nn


def cauchy_sparsity_loss(sigmas, lam: float):
    """L:80-88."""
    s = np.asarray(sigmas, dtype=np.float64)
    return lam * float(np.sum(np.log1p(2.0 * s * s))), lam * 4.0 * s / (1.0 + 2.0 * s * s)


def psnr(a, b) -> float:
    """L:110-119."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("image dimension mismatch")
    mse = float(np.mean((a - b) ** 2))
    if mse == 0.0:
        return math.inf
    return -10.0 * math.log10(mse)


def _gaussian_window(radius: int = 5, sigma: float = 1.5) -> np.ndarray:
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return w / w.sum()


def ssim(a, b, k1: float = 0.01, k2: float = 0.03) -> float:
    """L:128-165 (11x11 Gaussian, sigma 1.5, valid interior)."""
    from scipy.ndimage import correlate1d

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("image dimension mismatch")
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    radius = 5
    win = _gaussian_window(radius)
    if a.shape[0] <= 2 * radius or a.shape[1] <= 2 * radius:
        raise ValueError("image smaller than the SSIM window")
    c1, c2 = k1 * k1, k2 * k2

    def filt(img):
        out = correlate1d(img, win, axis=0, mode="constant")
        out = correlate1d(out, win, axis=1, mode="constant")
        return out[radius:-radius, radius:-radius]

    vals = []
    for ch in range(a.shape[2]):
        x, y = a[..., ch], b[..., ch]
        mx, my = filt(x), filt(y)
        vx = filt(x * x) - mx * mx
        vy = filt(y * y) - my * my
        cov = filt(x * y) - mx * my
        num = (2 * mx * my + c1) * (2 * cov + c2)
        den = (mx * mx + my * my + c1) * (vx + vy + c2)
        vals.append(np.mean(num / den))
    return float(np.mean(vals))
