"""Multi-sphere-image background for unbounded 360 scenes, on the device.

Mirrors the reference's msi.py (MsiBackground, layer_radii,
sample_background, BgGradientBuffer, render_rays_with_background,
sample_bg_tv_cells, bg_tv_loss) and optim.step_table for the background
(O:100-107), over the C ABI of include/plx.h (plx_msi_render, plx_msi_tv,
plx_msi_opt_step; kernels in csrc/plx_msi.cu, reference K:603-977).

Concentric equirectangular layers carry f64 (sigma, r, g, b) texels; layer
radii run linearly in inverse radius from 1 to infinity (the scene is
pre-scaled into the unit sphere).  A ray samples the foreground grid as the
bounded render does, then the layers once per sphere crossing beyond the
grid's exit, and composites the residual over black.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .grid import GradientBuffer, SparseGrid, _dev


def layer_radii(n_layers: int) -> np.ndarray:
    """msi.py:63-67: radii whose inverses run linearly from 1 down to 0."""
    inv = np.linspace(1.0, 0.0, n_layers)
    with np.errstate(divide="ignore"):
        return 1.0 / inv


class MsiBackground:
    """msi.py:24-60: `data` (layers, H, W, 4) float64 in HBM; `radii`
    (layers,) increasing, the last one infinite."""

    def __init__(self, data, radii=None, device=None):
        dev = _dev(device if device is not None else
                   (data.device if isinstance(data, torch.Tensor) and data.is_cuda else None))
        t = torch.as_tensor(np.asarray(data) if not isinstance(data, torch.Tensor) else data,
                            dtype=torch.float64)
        if t.dim() != 4 or t.shape[3] != 4:
            raise ValueError("background data must be (layers, H, W, 4)")
        self.data = t.to(dev).contiguous()
        if radii is None:
            radii = layer_radii(self.n_layers)
        self.radii = np.asarray(radii, dtype=np.float64)
        if self.radii.shape != (self.n_layers,):
            raise ValueError("one radius per layer required")
        if np.any(np.diff(self.radii) <= 0):
            raise ValueError("layer radii must be strictly increasing")
        self._radii_dev = torch.from_numpy(self.radii.copy()).to(dev)

    @classmethod
    def create(cls, n_layers: int = 64, height: int = 1024, width: int = 2048,
               device=None) -> "MsiBackground":
        dev = _dev(device)
        return cls(torch.zeros((n_layers, height, width, 4), dtype=torch.float64, device=dev),
                   device=dev)

    @property
    def n_layers(self) -> int:
        return int(self.data.shape[0])

    @property
    def height(self) -> int:
        return int(self.data.shape[1])

    @property
    def width(self) -> int:
        return int(self.data.shape[2])

    @property
    def n_texels(self) -> int:
        return self.n_layers * self.height * self.width

    @property
    def device(self):
        return self.data.device

    def copy(self) -> "MsiBackground":
        return MsiBackground(self.data.clone(), self.radii.copy())

    def _c(self) -> _lib.PlxMsi:
        c = _lib.PlxMsi()
        c.data, c.radii = self.data.data_ptr(), self._radii_dev.data_ptr()
        c.L, c.H, c.W = self.n_layers, self.height, self.width
        return c


def sample_background(bg: MsiBackground, pts):
    """msi.py:75-108: trilinear (sigma, rgb) at exterior points |p| >= 1 over
    (inverse-radius layer coordinate, theta, phi), phi wrapping; clamped at 0.
    Host numpy (a utility of the reference's tests and viewer, not on the
    training path)."""
    data = bg.data.cpu().numpy()
    L, H, W = bg.n_layers, bg.height, bg.width
    pts = np.asarray(pts, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.atleast_2d(pts)
    r = np.linalg.norm(pts, axis=-1)
    if np.any(r < 1.0 - 1e-9):
        raise ValueError("background sample inside the unit sphere")
    phi = np.arctan2(pts[:, 1], pts[:, 0])
    theta = np.arccos(np.clip(pts[:, 2] / r, -1.0, 1.0))
    u = (phi + np.pi) / (2.0 * np.pi) * W - 0.5
    u = u - np.floor(u / W) * W
    v = np.clip(theta / np.pi * H - 0.5, 0.0, H - 1.0)
    lc = np.clip((1.0 - 1.0 / r) * (L - 1), 0.0, L - 1)
    l0 = np.minimum(np.floor(lc).astype(np.int64), L - 2)
    fl = lc - l0
    i0 = np.minimum(np.floor(u).astype(np.int64), W - 1)
    fu = u - i0
    i1 = (i0 + 1) % W
    j0 = np.minimum(np.floor(v).astype(np.int64), H - 2)
    fv = v - j0
    out = np.zeros((len(pts), 4))
    for dl, wl in ((0, 1.0 - fl), (1, fl)):
        for jj, wv in ((j0, 1.0 - fv), (j0 + 1, fv)):
            for ii, wu in ((i0, 1.0 - fu), (i1, fu)):
                out += (wl * wv * wu)[:, None] * data[l0 + dl, jj, ii]
    out = np.maximum(out, 0.0)
    if single:
        return float(out[0, 0]), out[0, 1:]
    return out[:, 0], out[:, 1:]


class BgGradientBuffer:
    """msi.py:111-127: touched-texel accumulator over the flattened layer
    lattice, (L*H*W, 4) float64 + byte mask (+ the compacted list the update
    fills)."""

    def __init__(self, bg: MsiBackground):
        n = bg.n_texels
        dev = bg.device
        self.data = torch.zeros((n, 4), dtype=torch.float64, device=dev)
        self.touched_mask = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.touched_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self._count = torch.zeros(1, dtype=torch.int64, device=dev)

    @property
    def n_touched(self) -> int:
        return int(self.touched_mask.count_nonzero().item())

    def touched_rows(self) -> np.ndarray:
        return torch.nonzero(self.touched_mask).flatten().cpu().numpy().astype(np.int64)

    def clear(self) -> None:
        """clear_grad (K:593-600) of the touched texels."""
        idx = torch.nonzero(self.touched_mask).flatten()
        self.data[idx] = 0.0
        self.touched_mask.zero_()

    def _c(self) -> _lib.PlxMsiGrad:
        c = _lib.PlxMsiGrad()
        c.grad, c.tmask = self.data.data_ptr(), self.touched_mask.data_ptr()
        c.tids, c.tcnt = self.touched_ids.data_ptr(), self._count.data_ptr()
        return c


def render_rays_with_background(grid: SparseGrid, bg: MsiBackground, origins, dirs, opts=None,
                                gt_rgb=None, grads: GradientBuffer | None = None,
                                bg_grads: BgGradientBuffer | None = None, n_total: int = 1,
                                lam_cauchy: float = 0.0, lam_beta: float = 0.0,
                                beta_eps: float = 1e-6):
    """msi.py:130-183: composite foreground grid and sphere layers along world
    rays.  Forward-only when `grads` is None; with ground truth and both
    gradient buffers, the fused MSE backward (upstream 2 (C - gt) / n_total)
    with the Cauchy and beta regulariser gradients.

    Returns (rgb, trans_fg, trans_final, mse_sum, cauchy_raw, beta_raw);
    numpy in -> numpy out, tensors in -> device tensors out."""
    from .render import RenderOptions, _step_size, kernel_opts

    opts = opts or RenderOptions(background=(0.0, 0.0, 0.0))
    as_np = not isinstance(origins, torch.Tensor)
    dev = grid.device
    o = torch.as_tensor(np.atleast_2d(origins) if as_np else origins,
                        dtype=torch.float64).reshape(-1, 3).to(dev).contiguous()
    d = torch.as_tensor(np.atleast_2d(dirs) if as_np else dirs,
                        dtype=torch.float64).reshape(-1, 3).to(dev).contiguous()
    n = int(o.shape[0])
    with_grad = grads is not None
    if with_grad and (gt_rgb is None or bg_grads is None):
        raise ValueError("backward pass needs ground truth and both buffers")
    gt = (torch.zeros((n, 3), dtype=torch.float64, device=dev) if gt_rgb is None else
          torch.as_tensor(np.atleast_2d(gt_rgb) if not isinstance(gt_rgb, torch.Tensor)
                          else gt_rgb, dtype=torch.float64).reshape(-1, 3).to(dev).contiguous())
    rgb = torch.empty((n, 3), dtype=torch.float64, device=dev)
    tfg = torch.empty(n, dtype=torch.float64, device=dev)
    trans = torch.empty(n, dtype=torch.float64, device=dev)
    sums = torch.zeros(3, dtype=torch.float64, device=dev)
    if n:
        cg = grid._c(with_occ=opts.interp == "trilinear")
        ko = kernel_opts(grid, opts)
        cb = bg._c()
        need = int(_lib.lib().plx_msi_scratch_bytes(ctypes.byref(cg), ctypes.byref(cb),
                                                    ctypes.byref(ko), n))
        if need < 0:
            raise ValueError("bad render arguments")
        scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        r = _lib.PlxRays()
        r.origins, r.dirs, r.viewdirs, r.target = o.data_ptr(), d.data_ptr(), None, gt.data_ptr()
        r.jitter, r.idx, r.n = None, None, n
        cgrad = grads._c(with_ids=False) if with_grad else None
        cbg = bg_grads._c() if with_grad else None
        _lib.check(_lib.lib().plx_msi_render(
            ctypes.byref(cg), ctypes.byref(cb), ctypes.byref(r), ctypes.byref(ko), 1,
            2.0 / max(n_total, 1), float(lam_cauchy), float(lam_beta), float(beta_eps),
            ctypes.byref(cgrad) if with_grad else None,
            ctypes.byref(cbg) if with_grad else None, rgb.data_ptr(), tfg.data_ptr(),
            trans.data_ptr(), sums.data_ptr(), scratch.data_ptr(), need,
            _lib.stream_ptr()), "msi_render")
        del scratch
    s = sums.cpu().numpy()
    if as_np:
        return rgb.cpu().numpy(), tfg.cpu().numpy(), trans.cpu().numpy(), \
            float(s[0]), float(s[1]), float(s[2])
    return rgb, tfg, trans, float(s[0]), float(s[1]), float(s[2])


class BgCellRun:
    """The texel run of sample_bg_tv_cells as (start, count) -- the kernel
    walks it on the device; np.asarray(run) gives the reference's int64
    array (msi.py:190)."""

    def __init__(self, start: int, count: int, n_cells: int):
        self.start, self.count, self.n_cells = int(start), int(count), int(n_cells)

    def __array__(self, dtype=None, copy=None):
        a = ((self.start + np.arange(self.count)) % self.n_cells).astype(np.int64)
        return a if dtype is None else a.astype(dtype)

    def __len__(self) -> int:
        return self.count

    @property
    def size(self) -> int:
        return self.count


def sample_bg_tv_cells(bg: MsiBackground, fraction: float, rng) -> BgCellRun:
    """msi.py:186-190 (same RNG draws): a contiguous run of texels."""
    n_cells = bg.n_texels
    count = max(1, int(round(fraction * n_cells)))
    start = int(rng.integers(0, n_cells))
    return BgCellRun(start, count, n_cells)


def bg_tv_loss(bg: MsiBackground, cells, lam_sigma: float, lam_rgb: float,
               bg_grads: BgGradientBuffer | None = None, eps: float = 1e-6):
    """msi.py:193-208 -> tv_bg (K:884-977): TV over (layer, theta, phi), phi
    wrapping.  Returns the lambda-scaled (tv_sigma, tv_rgb) means."""
    dev = bg.device
    if isinstance(cells, BgCellRun):   # a run: walked on the device, no upload
        n, start, ct = cells.count, cells.start, None
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        n, start = int(cells.size), 0
        ct = torch.from_numpy(cells).to(dev)
    if n == 0:
        return 0.0, 0.0
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    cbg = bg_grads._c() if bg_grads is not None else None
    _lib.check(_lib.lib().plx_msi_tv(ctypes.byref(bg._c()), _lib.ptr(ct), start, n, float(eps),
                                     lam_sigma / n, lam_rgb / n,
                                     ctypes.byref(cbg) if cbg is not None else None,
                                     sums.data_ptr(), _lib.stream_ptr()), "msi_tv")
    s = sums.cpu().numpy()
    return lam_sigma * float(s[0]) / n, lam_rgb * float(s[1]) / n


class BgOptimState:
    """The background's RMSProp state (O:58-78 on a (L*H*W, 4) f64 table)."""

    def __init__(self, bg: MsiBackground, beta: float = 0.95, eps: float = 1e-8):
        self.v = torch.zeros((bg.n_texels, 4), dtype=torch.float64, device=bg.device)
        self.beta, self.eps = beta, eps
        self.step_count = 0


def step_table(bg: MsiBackground, bg_grads: BgGradientBuffer, state: BgOptimState,
               lr_first: float, lr_rest: float, method: str = "rmsprop",
               clear: bool = True) -> int:
    """optim.step_table (O:100-107) on the background over its touched
    texels (column 0 = opacity uses lr_first), then bg_grads.clear()
    (T:487-492).  Returns nothing the caller must sync on; the touched count
    stays on the device in bg_grads._count."""
    _lib.check(_lib.lib().plx_msi_opt_step(
        bg.data.data_ptr(), state.v.data_ptr(), ctypes.byref(bg_grads._c()), bg.n_texels,
        float(lr_first), float(lr_rest), state.beta, state.eps, int(method == "rmsprop"),
        int(bool(clear)), None, _lib.stream_ptr()), "msi_opt_step")
    state.step_count += 1
