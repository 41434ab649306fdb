"""Training losses and image metrics (drop-in for pkg/src/plenoxel/losses.py).

tv_loss (L:50-77) runs the sm_100a TV kernel; sample_tv_cells (L:41-47)
draws the same contiguous wrapped run from the same numpy RNG call but hands
the kernel (start, count) instead of materialising the id array.  PSNR /
SSIM (L:110-165) run on the device (plx_image_metrics); MSE / Cauchy are
host-side helpers with the reference's semantics.
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


BETA_EPS = 1e-6


def beta_loss(trans_fg, lam: float, eps: float = BETA_EPS):
    """L:91-102: lam * sum(log T + log(1 - T)) over the foreground
    transmittances, T clamped to [eps, 1 - eps] -> (loss, dL/dT), the gradient
    zero where the clamp is active.  A CUDA tensor stays on the device (the
    360 training step computes the same terms inside msi_bg_kernel)."""
    if isinstance(trans_fg, torch.Tensor):
        t = trans_fg.to(torch.float64)
        tc = t.clamp(eps, 1.0 - eps)
        loss = lam * float(torch.sum(torch.log(tc) + torch.log1p(-tc)))
        grad = lam * (1.0 / tc - 1.0 / (1.0 - tc))
        grad = torch.where((t < eps) | (t > 1.0 - eps), torch.zeros_like(grad), grad)
        return loss, grad
    t = np.asarray(trans_fg, dtype=np.float64)
    tc = np.clip(t, eps, 1.0 - eps)
    loss = lam * float(np.sum(np.log(tc) + np.log1p(-tc)))
    grad = lam * (1.0 / tc - 1.0 / (1.0 - tc))
    grad = np.where((t < eps) | (t > 1.0 - eps), 0.0, grad)
    return loss, grad


def _gaussian_window(radius: int = 5, sigma: float = 1.5) -> np.ndarray:
    """L:124-128."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return w / w.sum()


_WINDOW = _gaussian_window(5)


def _image_tensor(x, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)


def image_metrics(a, b, with_ssim: bool = True, k1: float = 0.01, k2: float = 0.03,
                  device=None):
    """(psnr, ssim) of two images in [0, 1] (L:110-165) computed on the device
    (plx_image_metrics): one (H, W[, C]) pair -> two scalars, no image leaves
    the device.  ssim is None when with_ssim is False."""
    dev = torch.device(device) if device is not None else (
        a.device if isinstance(a, torch.Tensor) and a.is_cuda else torch.device("cuda"))
    ta, tb = _image_tensor(a, dev), _image_tensor(b, dev)
    if ta.shape != tb.shape:
        raise ValueError("image dimension mismatch")
    if ta.dim() == 2:
        ta, tb = ta[..., None], tb[..., None]
    if ta.dim() != 3:
        raise ValueError("images must be (H, W) or (H, W, C)")
    h, w, c = (int(x) for x in ta.shape)
    radius = 5
    if with_ssim and (h <= 2 * radius or w <= 2 * radius):
        raise ValueError("image smaller than the SSIM window")
    L = _lib.lib()
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    scratch, nb = None, 0
    if with_ssim:
        nb = int(L.plx_image_metrics_scratch_bytes(h, w, c))
        scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    _lib.check(L.plx_image_metrics(
        ta.data_ptr(), tb.data_ptr(), h, w, c,
        _WINDOW.ctypes.data_as(ctypes.c_void_p) if with_ssim else None, k1, k2,
        sums.data_ptr(), _lib.ptr(scratch), nb, _lib.stream_ptr()), "image_metrics")
    sq, ss = (float(x) for x in sums.cpu())
    mse = sq / (h * w * c)
    p = math.inf if mse == 0.0 else -10.0 * math.log10(mse)
    s = ss / ((h - 2 * radius) * (w - 2 * radius) * c) if with_ssim else None
    return p, s


def psnr(a, b) -> float:
    """L:110-119 on the device: inf if the images are equal."""
    return image_metrics(a, b, with_ssim=False)[0]


def ssim(a, b, k1: float = 0.01, k2: float = 0.03) -> float:
    """L:128-165 on the device: 11x11 Gaussian window (sigma 1.5), statistics
    over the valid interior, averaged over colour channels."""
    return image_metrics(a, b, True, k1, k2)[1]
