"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the B200 path.

ctypes front-end over liboracle.so (plx_oracle.c), a sequential float64 C
restatement of the reference kernels (pkg/src/plenoxel/_kernels.py:27-600)
plus prune/upsample (pkg/src/plenoxel/grid.py:228-285).  The wrappers below
mirror the reference's L1 call sites so tests read like the reference's own:

  render_rays            <- render.py:114-140  (render_forward,  K:173-238)
  render_rays_backward   <- render.py:205-239  (render_backward, K:241-411)
  fused_mse_backward     <- render.py:253-279  (render_backward, mse_mode)
  max_weight_accumulate  <- grid.py:287-302    (max_weight_accum, K:414-453)
  tv_loss                <- losses.py:50-77    (tv_grid, K:456-569)
  opt_step / clear_grad  <- optim.py:81-97, grid.py:62-64 (K:572-600)
  prune / upsample       <- grid.py:228-285

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ROW = 28
SH_C0 = 0.28209479177387814


def build() -> str:
    """Compile liboracle.so in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "plx_oracle.c")
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_prune.restype = ctypes.c_int64
        _lib.oracle_upsample.restype = ctypes.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


_d = ctypes.c_double
_i = ctypes.c_int64


@dataclass
class Grid:
    """Minimal float64 twin of the reference SparseGrid (grid.py:71-139)."""

    links: np.ndarray
    table: np.ndarray
    aabb_min: np.ndarray
    aabb_max: np.ndarray

    def __post_init__(self):
        self.links = np.ascontiguousarray(self.links, dtype=np.int32)
        self.table = np.ascontiguousarray(self.table, dtype=np.float64)
        self.aabb_min = np.asarray(self.aabb_min, dtype=np.float64).reshape(3)
        self.aabb_max = np.asarray(self.aabb_max, dtype=np.float64).reshape(3)

    @classmethod
    def dense(cls, dims, aabb_min, aabb_max, sigma=0.0, rgb=None):
        dims = tuple(int(d) for d in dims)
        n = dims[0] * dims[1] * dims[2]
        table = np.zeros((n, ROW))
        table[:, 0] = sigma
        if rgb is not None:
            for ch in range(3):
                table[:, 1 + 9 * ch] = rgb / SH_C0
        return cls(np.arange(n, dtype=np.int32).reshape(dims), table,
                   aabb_min, aabb_max)

    @property
    def dims(self):
        return self.links.shape

    @property
    def n_rows(self):
        return self.table.shape[0]

    @property
    def extent(self):
        return self.aabb_max - self.aabb_min

    @property
    def voxel_size(self):
        return self.extent / (np.array(self.dims, dtype=np.float64) - 1.0)

    @property
    def lattice_scale(self):
        return (np.array(self.dims, dtype=np.float64) - 1.0) / self.extent

    def copy(self):
        return Grid(self.links.copy(), self.table.copy(), self.aabb_min.copy(),
                    self.aabb_max.copy())


class GradBuf:
    """Twin of GradientBuffer (grid.py:25-68)."""

    def __init__(self, n_rows):
        self.data = np.zeros((n_rows, ROW))
        self.touched_mask = np.zeros(n_rows, dtype=np.uint8)
        self.touched_ids = np.zeros(max(n_rows, 1), dtype=np.int64)
        self._count = np.zeros(1, dtype=np.int64)

    @property
    def n_touched(self):
        return int(self._count[0])

    def touched_rows(self):
        return np.sort(self.touched_ids[: self.n_touched])

    def clear(self):
        lib().oracle_clear_grad(_p(self.data), _p(self.touched_mask),
                                _p(self.touched_ids), _p(self._count), _i(ROW))


def _geom(grid, step_frac):
    step = step_frac * float(np.min(grid.voxel_size))           # R:63-64
    dmax = np.array(grid.dims, dtype=np.float64) - 1.0          # R:132
    return step, dmax, _f64(grid.lattice_scale)


def _max_samples(grid, step):                                   # R:67-69
    return int(math.ceil(float(np.linalg.norm(grid.extent)) / step)) + 4


def normalize_dirs(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def render_rays(grid, origins, dirs, step_frac=0.5, stop_thresh=1e-4,
                background=(1.0, 1.0, 1.0), interp="trilinear",
                formula="relative", viewdirs=None, jitter_t=None):
    o = _f64(np.atleast_2d(origins))
    d = _f64(np.atleast_2d(dirs))
    v = normalize_dirs(d) if viewdirs is None else _f64(np.atleast_2d(viewdirs))
    n = o.shape[0]
    step, dmax, scale = _geom(grid, step_frac)
    jt = np.zeros(n) if jitter_t is None else _f64(jitter_t)
    rgb, trans, wsum = np.empty((n, 3)), np.empty(n), np.empty(n)
    Dx, Dy, Dz = grid.dims
    lib().oracle_render_forward(
        _p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table), _p(grid.aabb_min),
        _p(grid.aabb_max), _p(scale), _p(dmax), _d(step), _p(o), _p(d), _p(v),
        _i(n), _p(_f64(background)), _d(stop_thresh), ctypes.c_int(interp == "nearest"),
        ctypes.c_int(formula == "absolute"), _p(jt), _p(rgb), _p(trans), _p(wsum))
    return rgb, trans, wsum


def render_backward(grid, origins, dirs, viewdirs, target, buf, mse_mode,
                    up_scale, lam_cauchy=0.0, step_frac=0.5, stop_thresh=1e-4,
                    background=(1.0, 1.0, 1.0), interp="trilinear",
                    formula="relative", jitter_t=None):
    """render_backward (K:241-411); returns (rgb, mse_sum, cauchy_sum)."""
    o = _f64(np.atleast_2d(origins))
    d = _f64(np.atleast_2d(dirs))
    v = normalize_dirs(d) if viewdirs is None else _f64(np.atleast_2d(viewdirs))
    tg = _f64(np.atleast_2d(target))
    n = o.shape[0]
    step, dmax, scale = _geom(grid, step_frac)
    jt = np.zeros(n) if jitter_t is None else _f64(jitter_t)
    rgb = np.empty((n, 3))
    sums = np.zeros(2)
    Dx, Dy, Dz = grid.dims
    lib().oracle_render_backward(
        _p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table), _p(grid.aabb_min),
        _p(grid.aabb_max), _p(scale), _p(dmax), _d(step), _p(o), _p(d), _p(v), _i(n),
        _p(_f64(background)), _d(stop_thresh), ctypes.c_int(interp == "nearest"),
        ctypes.c_int(formula == "absolute"), _p(jt), _p(tg), ctypes.c_int(bool(mse_mode)),
        _d(up_scale), _d(lam_cauchy), _p(buf.data), _p(buf.touched_mask),
        _p(buf.touched_ids), _p(buf._count), _p(rgb), _i(_max_samples(grid, step)),
        _p(sums))
    return rgb, float(sums[0]), float(sums[1])


def fused_mse_backward(grid, origins, dirs, viewdirs, gt, buf, n_total,
                       lam_cauchy=0.0, **opts):
    """render.fused_mse_backward (R:253-279)."""
    return render_backward(grid, origins, dirs, viewdirs, gt, buf, True,
                           2.0 / n_total, lam_cauchy, **opts)


def render_rays_backward(grid, origins, dirs, upstream, buf, viewdirs=None,
                         lam_cauchy=0.0, **opts):
    """render.render_rays_backward (R:205-239); returns (rgb, cauchy_sum)."""
    rgb, _, cs = render_backward(grid, origins, dirs, viewdirs, upstream, buf,
                                 False, 0.0, lam_cauchy, **opts)
    return rgb, cs


def max_weight_accumulate(grid, origins, dirs, step_frac=0.5, stop_thresh=1e-4,
                          interp="trilinear"):
    o = _f64(np.atleast_2d(origins))
    d = _f64(np.atleast_2d(dirs))
    out = np.zeros(grid.n_rows)
    step, dmax, scale = _geom(grid, step_frac)
    Dx, Dy, Dz = grid.dims
    lib().oracle_max_weight_accum(
        _p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table), _p(grid.aabb_min),
        _p(grid.aabb_max), _p(scale), _p(dmax), _d(step), _p(o), _p(d), _i(o.shape[0]),
        _d(stop_thresh), ctypes.c_int(interp == "nearest"), _p(out))
    return out


def sample_tv_cells(dims, fraction, rng):
    """losses.sample_tv_cells (L:41-47)."""
    n_cells = int(np.prod(dims))
    count = max(1, int(round(fraction * n_cells)))
    start = int(rng.integers(0, n_cells))
    return ((start + np.arange(count)) % n_cells).astype(np.int64)


def tv_loss(grid, cells, lam_sigma, lam_sh, buf=None, eps=1e-6,
            wrap=(False, False, False)):
    """losses.tv_loss (L:50-77)."""
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    if cells.size == 0:
        return 0.0, 0.0
    n = cells.size
    dims = grid.dims
    b = buf if buf is not None else GradBuf(grid.n_rows)
    sums = np.zeros(2)
    lib().oracle_tv_grid(
        _p(grid.links), _i(dims[0]), _i(dims[1]), _i(dims[2]), _p(grid.table),
        _p(cells), _i(n), _d(dims[0] / 256.0), _d(dims[1] / 256.0),
        _d(dims[2] / 256.0), _d(eps), _d(lam_sigma / n), _d(lam_sh / n),
        ctypes.c_int(wrap[0]), ctypes.c_int(wrap[1]), ctypes.c_int(wrap[2]),
        _p(b.data), _p(b.touched_mask), _p(b.touched_ids), _p(b._count),
        ctypes.c_int(buf is not None), _p(sums))
    return lam_sigma * sums[0] / n, lam_sh * sums[1] / n


def opt_step(grid, buf, v, lr_sigma, lr_sh, method="rmsprop", beta=0.95, eps=1e-8):
    """optim.step (O:81-97) on (table, v) in place."""
    lib().oracle_opt_step(_p(grid.table), _p(v), _p(buf.data), _p(buf.touched_ids),
                          _i(buf.n_touched), _i(ROW), _d(lr_sigma), _d(lr_sh),
                          _d(beta), _d(eps), ctypes.c_int(method == "rmsprop"))


def prune(grid, criterion, threshold, weights=None):
    """SparseGrid.prune (G:228-258) -> (new_grid, kept_old)."""
    Dx, Dy, Dz = grid.dims
    new_links = np.empty(grid.dims, dtype=np.int32)
    kept = np.empty(max(grid.n_rows, 1), dtype=np.int64)
    w = None
    if criterion == "weight":
        w = _f64(weights)
    elif criterion != "density":
        raise ValueError(f"unknown prune criterion {criterion!r}")
    n = lib().oracle_prune(_p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table),
                           _p(w) if w is not None else None, _d(threshold),
                           _p(new_links), _p(kept))
    kept = kept[:n].copy()
    return Grid(new_links, grid.table[kept].copy(), grid.aabb_min, grid.aabb_max), kept


def upsample(grid, new_dims):
    """SparseGrid.upsample (G:260-285)."""
    Nx, Ny, Nz = (int(x) for x in new_dims)
    Dx, Dy, Dz = grid.dims
    new_links = np.empty((Nx, Ny, Nz), dtype=np.int32)
    args = (_p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table), _p(grid.aabb_min),
            _p(grid.aabb_max), _i(Nx), _i(Ny), _i(Nz), _p(new_links))
    n = lib().oracle_upsample(*args, None)
    table = np.empty((n, ROW))
    lib().oracle_upsample(*args, _p(table))
    return Grid(new_links, table, grid.aabb_min, grid.aabb_max)


# -- multi-sphere-image background (360 scenes): K:603-977, msi.py -----------

def layer_radii(n_layers):
    """msi.layer_radii (msi.py:63-67): inverse radii linear from 1 to 0."""
    inv = np.linspace(1.0, 0.0, n_layers)
    with np.errstate(divide="ignore"):
        return 1.0 / inv


class BgGradBuf:
    """Twin of msi.BgGradientBuffer (msi.py:111-127): (L*H*W, 4) f64."""

    def __init__(self, n_texels):
        self.data = np.zeros((n_texels, 4))
        self.touched_mask = np.zeros(n_texels, dtype=np.uint8)
        self.touched_ids = np.zeros(max(n_texels, 1), dtype=np.int64)
        self._count = np.zeros(1, dtype=np.int64)

    @property
    def n_touched(self):
        return int(self._count[0])

    def touched_rows(self):
        return np.sort(self.touched_ids[: self.n_touched])

    def clear(self):
        lib().oracle_clear_grad(_p(self.data), _p(self.touched_mask),
                                _p(self.touched_ids), _p(self._count), _i(4))


def bg_sample(bgdata, pts):
    """msi.sample_background (msi.py:75-108): (sigma (n,), rgb (n, 3))."""
    bgdata = _f64(bgdata)
    L, H, W, _ = bgdata.shape
    p = _f64(np.atleast_2d(pts))
    out = np.empty((p.shape[0], 4))
    if lib().oracle_bg_sample(_p(bgdata), _i(L), _i(H), _i(W), _p(p), _i(p.shape[0]),
                              _p(out)) != 0:
        raise ValueError("background sample inside the unit sphere")
    return out[:, 0], out[:, 1:]


def render_360(grid, bgdata, radii, origins, dirs, step_frac=0.5, stop_thresh=1e-4,
               interp="trilinear", gt_rgb=None, buf=None, bg_buf=None, n_total=1,
               lam_cauchy=0.0, lam_beta=0.0, beta_eps=1e-6):
    """msi.render_rays_with_background (msi.py:130-183) over render_backward_360
    (K:661-881).  Returns (rgb, trans_fg, trans_final, mse, cauchy_raw, beta_raw)."""
    bgdata = _f64(bgdata)
    L, H, W, _ = bgdata.shape
    o = _f64(np.atleast_2d(origins))
    d = _f64(np.atleast_2d(dirs))
    n = o.shape[0]
    with_grad = buf is not None
    tg = np.zeros((n, 3)) if gt_rgb is None else _f64(np.atleast_2d(gt_rgb))
    if not with_grad:
        buf, bg_buf = GradBuf(0), BgGradBuf(8)
    step, dmax, scale = _geom(grid, step_frac)
    nmax = _max_samples(grid, step) + L + 2
    rgb, tfg, trans = np.empty((n, 3)), np.empty(n), np.empty(n)
    sums = np.zeros(3)
    Dx, Dy, Dz = grid.dims
    lib().oracle_render_360(
        _p(grid.links), _i(Dx), _i(Dy), _i(Dz), _p(grid.table), _p(grid.aabb_min),
        _p(grid.aabb_max), _p(scale), _p(dmax), _d(step), _p(bgdata), _i(L), _i(H), _i(W),
        _p(_f64(radii)), _p(o), _p(d), _i(n), _d(stop_thresh),
        ctypes.c_int(interp == "nearest"), _p(tg), ctypes.c_int(1),
        _d(2.0 / max(n_total, 1)), _d(lam_cauchy), _d(lam_beta), _d(beta_eps),
        _p(buf.data), _p(buf.touched_mask), _p(buf.touched_ids), _p(buf._count),
        _p(bg_buf.data), _p(bg_buf.touched_mask), _p(bg_buf.touched_ids), _p(bg_buf._count),
        _p(rgb), _p(tfg), _p(trans), _i(nmax), ctypes.c_int(with_grad), _p(sums))
    return rgb, tfg, trans, float(sums[0]), float(sums[1]), float(sums[2])


def sample_bg_tv_cells(n_texels, fraction, rng):
    """msi.sample_bg_tv_cells (msi.py:186-190)."""
    count = max(1, int(round(fraction * n_texels)))
    start = int(rng.integers(0, n_texels))
    return ((start + np.arange(count)) % n_texels).astype(np.int64)


def tv_bg(bgdata, cells, lam_sigma, lam_rgb, bg_buf=None, eps=1e-6):
    """msi.bg_tv_loss (msi.py:193-208) over tv_bg (K:884-977)."""
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    if cells.size == 0:
        return 0.0, 0.0
    bgdata = _f64(bgdata)
    L, H, W, _ = bgdata.shape
    n = cells.size
    b = bg_buf if bg_buf is not None else BgGradBuf(L * H * W)
    sums = np.zeros(2)
    lib().oracle_tv_bg(_p(bgdata), _i(L), _i(H), _i(W), _p(cells), _i(n), _d(eps),
                       _d(lam_sigma / n), _d(lam_rgb / n), _p(b.data), _p(b.touched_mask),
                       _p(b.touched_ids), _p(b._count), ctypes.c_int(bg_buf is not None),
                       _p(sums))
    return lam_sigma * sums[0] / n, lam_rgb * sums[1] / n


def step_table(table, grad, touched_ids, n_touched, v, lr_first, lr_rest,
               method="rmsprop", beta=0.95, eps=1e-8):
    """optim.step_table (O:100-107): the sparse update of a bare (rows, cols)
    f64 table (the background), in place."""
    ncol = table.shape[1]
    lib().oracle_opt_step(_p(table), _p(v), _p(grad), _p(np.ascontiguousarray(touched_ids)),
                          _i(n_touched), _i(ncol), _d(lr_first), _d(lr_rest), _d(beta),
                          _d(eps), ctypes.c_int(method == "rmsprop"))


# ---------------------------------------------------------------- cameras --
def camera_array(c2w, focal, width, height):
    """{c2w[:3, :4] row-major, focal, width, height} as the C restatement's
    float64[15] camera record."""
    c = np.zeros(15)
    c[:12] = np.asarray(c2w, dtype=np.float64)[:3, :4].reshape(-1)
    c[12:] = (float(focal), float(width), float(height))
    return c


def generate_rays(c2w, focal, width, height, pixels=None):
    """camera.py:91-100 (all pixels, row-major, or the given pixel ids)."""
    cam = camera_array(c2w, focal, width, height)
    pix = None if pixels is None else np.ascontiguousarray(pixels, dtype=np.int64)
    n = int(width) * int(height) if pix is None else len(pix)
    o, d = np.empty((n, 3)), np.empty((n, 3))
    lib().oracle_generate_rays(_p(cam), None if pix is None else _p(pix), _i(n), _p(o), _p(d))
    return o, d


def to_ndc(origins, dirs, focal, width, height, near=0.0):
    """camera.py:103-134 -> (o_ndc, d_ndc, valid)."""
    o, d = _f64(np.atleast_2d(origins)).copy(), _f64(np.atleast_2d(dirs)).copy()
    valid = np.zeros(len(o), dtype=np.uint8)
    lib().oracle_to_ndc(_p(o), _p(d), _i(len(o)), _d(focal), _d(width), _d(height), _d(near),
                        _p(valid))
    return o, d, valid.astype(bool)


# ------------------------------------------------- trainer host logic --
class EpochBatcher:
    """trainer.py:233-255: without-replacement batches, one rng.permutation
    per epoch from the trainer's rng."""

    def __init__(self, n, batch_size, rng):
        self.n, self.batch_size, self.rng = n, batch_size, rng
        self.perm = rng.permutation(n)
        self.cursor = 0

    def next(self):
        chunks, need = [], self.batch_size
        while need > 0:
            if self.cursor >= self.n:
                self.perm = self.rng.permutation(self.n)
                self.cursor = 0
            take = min(need, self.n - self.cursor)
            chunks.append(self.perm[self.cursor:self.cursor + take])
            self.cursor += take
            need -= take
        return np.concatenate(chunks) if len(chunks) > 1 else chunks[0]


def lr_at(kind, lr_init, lr_final, total_steps, step, delay_steps=0, delay_mult=0.01):
    """optim.py:42-55 (same op order)."""
    if kind == "constant":
        return lr_init
    t = min(max(step / total_steps, 0.0), 1.0)
    lr = lr_init * (lr_final / lr_init) ** t
    if kind == "delayed_exponential" and delay_steps > 0:
        p = min(max(step / delay_steps, 0.0), 1.0)
        lr *= delay_mult + (1.0 - delay_mult) * math.sin(0.5 * math.pi * p)
    return lr


# ---------------------------------------------------------------- metrics --
def psnr(a, b):
    """losses.py:110-119."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    return math.inf if mse == 0.0 else -10.0 * math.log10(mse)


def ssim(a, b, k1=0.01, k2=0.03):
    """losses.py:122-165 (scipy correlate1d, zero padding, valid interior)."""
    from scipy.ndimage import correlate1d

    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    r = 5
    x = np.arange(-r, r + 1, dtype=np.float64)
    win = np.exp(-(x * x) / (2.0 * 1.5 * 1.5))
    win = win / win.sum()
    c1, c2 = k1 * k1, k2 * k2

    def filt(img):
        out = correlate1d(img, win, axis=0, mode="constant")
        out = correlate1d(out, win, axis=1, mode="constant")
        return out[r:-r, r:-r]

    vals = []
    for ch in range(a.shape[2]):
        x_, y_ = a[..., ch], b[..., ch]
        mx, my = filt(x_), filt(y_)
        vx, vy, cov = filt(x_ * x_) - mx * mx, filt(y_ * y_) - my * my, filt(x_ * y_) - mx * my
        vals.append(np.mean((2 * mx * my + c1) * (2 * cov + c2) /
                            ((mx * mx + my * my + c1) * (vx + vy + c2))))
    return float(np.mean(vals))
