"""Differentiable volume rendering on the B200 (drop-in for
pkg/src/plenoxel/render.py).

Same public surface and argument meaning as the reference: RenderOptions
(R:27-42), march (R:72-95), render_rays (R:114-140), render_ray (R:143-155),
render_rays_backward (R:205-239), render_ray_backward (R:242-250),
fused_mse_backward (R:253-279), render_image (R:282-293).  Each call enqueues
one sm_100a kernel through libplx.so.  Inputs may be numpy arrays (results
come back as numpy, like the reference) or CUDA tensors (results stay on the
device, no host synchronisation except for returned Python scalars).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grid import GradientBuffer, SparseGrid
from .sh import normalize_dirs


@dataclass
class RenderOptions:
    step_frac: float = 0.5
    stop_thresh: float = 1e-4
    background: tuple = (1.0, 1.0, 1.0)
    interp: str = "trilinear"
    formula: str = "relative"
    jitter: float = 0.0

    def __post_init__(self):
        if self.step_frac <= 0:
            raise ValueError("step_frac must be positive")
        if self.interp not in ("trilinear", "nearest"):
            raise ValueError(f"unknown interpolation mode {self.interp!r}")
        if self.formula not in ("relative", "absolute"):
            raise ValueError(f"unknown rendering formula {self.formula!r}")


@dataclass
class SamplePoint:
    """R:45-52: one composited sample of render_ray(record=True)."""

    position: np.ndarray
    delta: float
    sigma: float
    rgb: np.ndarray
    trans: float
    weight: float


@dataclass
class RenderResult:
    rgb: np.ndarray
    trans: float
    weight_sum: float
    samples: list = field(default_factory=list)


def _step_size(grid: SparseGrid, step_frac: float) -> float:
    return step_frac * float(np.min(grid.voxel_size))          # R:63-64


def _max_samples(grid: SparseGrid, step: float) -> int:
    return int(math.ceil(float(np.linalg.norm(grid.extent)) / step)) + 4   # R:67-69


def kernel_opts(grid: SparseGrid, opts: RenderOptions) -> _lib.PlxRenderOpts:
    return _lib.make_opts(_step_size(grid, opts.step_frac), opts.stop_thresh, opts.background,
                          opts.interp == "nearest", opts.formula == "absolute")


def march(grid: SparseGrid, origin, direction, step_frac: float = 0.5):
    """Uniform samples along the chord (R:72-95), host float64."""
    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    t0, t1 = 0.0, math.inf
    for a in range(3):
        if abs(d[a]) < 1e-15:
            if o[a] < grid.aabb_min[a] or o[a] > grid.aabb_max[a]:
                return np.empty(0), np.empty(0)
        else:
            ta = (grid.aabb_min[a] - o[a]) / d[a]
            tb = (grid.aabb_max[a] - o[a]) / d[a]
            ta, tb = min(ta, tb), max(ta, tb)
            t0, t1 = max(t0, ta), min(t1, tb)
    length = t1 - t0
    if length <= 0.0:
        return np.empty(0), np.empty(0)
    step = _step_size(grid, step_frac)
    n = max(1, int(math.ceil(length / step - 1e-9)))
    ts = t0 + np.arange(n) * step
    deltas = np.full(n, step)
    deltas[-1] = length - step * (n - 1)
    return ts, deltas


def _ray_tensor(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)).to(device)
    t = t.reshape(-1, 3) if t.dim() == 1 else t
    if t.dim() != 2 or t.shape[1] != 3:
        raise ValueError("origins and directions must both be (N, 3)")
    return t.contiguous()


def _jitter_offsets(n: int, jitter: float, rng):
    if jitter <= 0.0:
        return None
    if rng is None:
        rng = np.random.default_rng()
    return rng.random(n) * jitter                               # R:106-111


def _batch(grid, origins, dirs, viewdirs, target=None, jitter=None):
    dev = grid.device
    o = _ray_tensor(origins, dev)
    d = _ray_tensor(dirs, dev)
    if o.shape != d.shape:
        raise ValueError("origins and directions must both be (N, 3)")
    if viewdirs is None:
        if isinstance(dirs, torch.Tensor):
            v = (d / torch.linalg.norm(d, dim=-1, keepdim=True)).contiguous()
        else:
            v = _ray_tensor(normalize_dirs(np.atleast_2d(dirs)), dev)
    else:
        v = _ray_tensor(viewdirs, dev)
    tg = _ray_tensor(target, dev) if target is not None else None
    jt = None
    if jitter is not None:
        jt = torch.from_numpy(np.ascontiguousarray(jitter, np.float64)).to(dev)
    r = _lib.PlxRays()
    r.origins, r.dirs, r.viewdirs = o.data_ptr(), d.data_ptr(), v.data_ptr()
    r.target = _lib.ptr(tg)
    r.jitter = _lib.ptr(jt)
    r.idx = None
    r.n = o.shape[0]
    keep = (o, d, v, tg, jt)        # keep device buffers alive until launch
    return r, keep


def render_rays(grid: SparseGrid, origins, dirs, opts: RenderOptions | None = None,
                viewdirs=None, rng=None):
    """R:114-140 -> (rgb (N,3), trans (N,), weight_sum (N,)), float64."""
    opts = opts or RenderOptions()
    as_np = not isinstance(origins, torch.Tensor)
    n = int(np.atleast_2d(origins).shape[0]) if as_np else int(origins.reshape(-1, 3).shape[0])
    r, keep = _batch(grid, origins, dirs, viewdirs,
                     jitter=_jitter_offsets(n, opts.jitter, rng))
    dev = grid.device
    rgb = torch.empty((n, 3), dtype=torch.float64, device=dev)
    trans = torch.empty(n, dtype=torch.float64, device=dev)
    wsum = torch.empty(n, dtype=torch.float64, device=dev)
    if grid.n_rows == 0:
        rgb[:] = torch.as_tensor(np.asarray(opts.background, np.float64), device=dev)
        trans.fill_(1.0)
        wsum.zero_()
    else:
        c, ko = grid._c(with_occ=opts.interp == "trilinear"), kernel_opts(grid, opts)
        _lib.check(_lib.lib().plx_render_fwd(ctypes.byref(c), ctypes.byref(r), ctypes.byref(ko),
                                             rgb.data_ptr(), trans.data_ptr(), wsum.data_ptr(),
                                             _lib.stream_ptr()), "render_fwd")
    del keep
    if as_np:
        return rgb.cpu().numpy(), trans.cpu().numpy(), wsum.cpu().numpy()
    return rgb, trans, wsum


def render_ray(grid: SparseGrid, origin, direction, opts: RenderOptions | None = None,
               viewdir=None, record: bool = False) -> RenderResult:
    """R:143-155.  record=True also returns the per-sample terms (R:158-202):
    the march positions of `march`, their interpolated (sigma, SH) from ONE
    SparseGrid.sample call on the device, and the compositing of R:171-201
    done sample by sample in float64 on the host (a debugging / test path;
    the fast path is the kernel)."""
    opts = opts or RenderOptions()
    if record:
        return _render_ray_record(grid, origin, direction, opts, viewdir)
    vd = None if viewdir is None else np.atleast_2d(viewdir)
    rgb, trans, wsum = render_rays(grid, np.atleast_2d(origin), np.atleast_2d(direction),
                                   opts, vd)
    return RenderResult(rgb=rgb[0], trans=float(trans[0]), weight_sum=float(wsum[0]))


def _render_ray_record(grid, origin, direction, opts, viewdir) -> RenderResult:
    """R:158-202 with the interpolation on the device."""
    from .sh import eval_sh_basis, normalize_dirs
    o = np.asarray(origin, dtype=np.float64).reshape(3)
    d = np.asarray(direction, dtype=np.float64).reshape(3)
    basis = eval_sh_basis(normalize_dirs(d if viewdir is None else
                                         np.asarray(viewdir, dtype=np.float64).reshape(3)))
    bg = np.asarray(opts.background, dtype=np.float64)
    ts, deltas = march(grid, o, d, opts.step_frac)
    rgb, T, asum, wsum, samples = np.zeros(3), 1.0, 0.0, 0.0, []
    if len(ts) and grid.n_rows:
        pos = o[None, :] + ts[:, None] * d[None, :]
        # the stencil clamps to the lattice anyway; clipping keeps positions a
        # rounding error outside a face inside sample()'s AABB check
        sig, coeffs = grid.sample(np.clip(pos, grid.aabb_min, grid.aabb_max), opts.interp)
        for i, dlt in enumerate(deltas):
            s = float(sig[i])       # clamped at 0: skipped exactly when R:179 skips
            if s <= 0.0:
                continue
            att = math.exp(-s * dlt)
            if opts.formula == "absolute":
                t_next = max(0.0, 1.0 - (asum + (1.0 - att)))
                asum += 1.0 - att
            else:
                t_next = T * att
            w = T - t_next
            color = np.maximum(basis @ coeffs[i].reshape(3, 9).T, 0.0)
            rgb += w * color
            wsum += w
            samples.append(SamplePoint(position=pos[i], delta=float(dlt), sigma=s, rgb=color,
                                       trans=T, weight=w))
            T = t_next
            if T < opts.stop_thresh:
                break
    return RenderResult(rgb=rgb + T * bg, trans=T, weight_sum=wsum, samples=samples)


def _launch_bwd(grid, r, opts, mse_mode, up_scale, lam_cauchy, grads, rgb, sums):
    if grid.n_rows == 0:
        raise ValueError("cannot backpropagate into an empty grid")
    if grads.n_rows != grid.n_rows:
        raise ValueError("gradient buffer rows do not match the grid table")
    c, ko, gb = grid._c(with_occ=opts.interp == "trilinear"), kernel_opts(grid, opts), grads._c()
    sp, sn, _keep = _lib.render_scratch(c, ko, r.n, grid.device)
    _lib.check(_lib.lib().plx_render_fused_bwd(
        ctypes.byref(c), ctypes.byref(r), ctypes.byref(ko), int(mse_mode), float(up_scale),
        float(lam_cauchy), ctypes.byref(gb), _lib.ptr(rgb), sums.data_ptr(), sp, sn,
        _lib.stream_ptr()), "render_fused_bwd")


def render_rays_backward(grid: SparseGrid, origins, dirs, upstream, grads: GradientBuffer,
                         opts: RenderOptions | None = None, viewdirs=None,
                         lam_cauchy: float = 0.0, rng=None):
    """R:205-239: scatter dL/dC (N,3) -> grads.  Returns (rgb, cauchy_raw)."""
    opts = opts or RenderOptions()
    as_np = not isinstance(origins, torch.Tensor)
    r, keep = _batch(grid, origins, dirs, viewdirs, target=upstream)
    r.jitter = None
    jt = _jitter_offsets(r.n, opts.jitter, rng)
    if jt is not None:
        jtt = torch.from_numpy(jt).to(grid.device)
        r.jitter = jtt.data_ptr()
    rgb = torch.empty((r.n, 3), dtype=torch.float64, device=grid.device)
    sums = torch.zeros(2, dtype=torch.float64, device=grid.device)
    _launch_bwd(grid, r, opts, False, 0.0, lam_cauchy, grads, rgb, sums)
    del keep
    cauchy = float(sums[1].item())
    return (rgb.cpu().numpy() if as_np else rgb), cauchy


def render_ray_backward(grid: SparseGrid, origin, direction, upstream,
                        opts: RenderOptions | None = None, viewdir=None) -> GradientBuffer:
    """R:242-250."""
    grads = GradientBuffer(grid.n_rows, device=grid.device)
    vd = None if viewdir is None else np.atleast_2d(viewdir)
    render_rays_backward(grid, np.atleast_2d(origin), np.atleast_2d(direction),
                         np.atleast_2d(upstream), grads, opts, vd)
    return grads


def fused_mse_backward(grid: SparseGrid, origins, dirs, viewdirs, gt_rgb,
                       grads: GradientBuffer, opts: RenderOptions, n_total: int,
                       lam_cauchy: float = 0.0, rng=None, sums: torch.Tensor | None = None):
    """R:253-279: forward render + MSE upstream 2(C-gt)/n_total + reverse
    sweep in ONE kernel.  Returns (rgb, mse_sum, cauchy_raw).

    Pass a device float64[2] `sums` to accumulate the two scalars on the
    device instead (then they are returned as that tensor, no host sync)."""
    as_np = not isinstance(origins, torch.Tensor)
    r, keep = _batch(grid, origins, dirs, viewdirs, target=gt_rgb)
    jt = _jitter_offsets(r.n, opts.jitter, rng)
    if jt is not None:
        jtt = torch.from_numpy(jt).to(grid.device)
        r.jitter = jtt.data_ptr()
    rgb = torch.empty((r.n, 3), dtype=torch.float64, device=grid.device)
    dev_sums = sums if sums is not None else torch.zeros(2, dtype=torch.float64,
                                                         device=grid.device)
    _launch_bwd(grid, r, opts, True, 2.0 / n_total, lam_cauchy, grads, rgb, dev_sums)
    del keep
    out_rgb = rgb.cpu().numpy() if as_np else rgb
    if sums is not None:
        return out_rgb, dev_sums, None
    s = dev_sums.cpu().numpy()
    return out_rgb, float(s[0]), float(s[1])


class RayPool:
    """Device-resident training rays: origins, march dirs,
    view dirs and gt colours as float64 (N, 3) in HBM; a batch is a device
    int64 index vector gathered inside the kernel (no per-step host copy)."""

    def __init__(self, origins, dirs, viewdirs, rgb, device=None):
        dev = torch.device(device or "cuda")
        self.origins = _ray_tensor(origins, dev)
        self.dirs = _ray_tensor(dirs, dev)
        self.viewdirs = _ray_tensor(viewdirs, dev)
        self.rgb = _ray_tensor(rgb, dev)
        self.n = self.origins.shape[0]

    def rays(self, idx: torch.Tensor | None, n: int | None = None) -> _lib.PlxRays:
        r = _lib.PlxRays()
        r.origins, r.dirs = self.origins.data_ptr(), self.dirs.data_ptr()
        r.viewdirs, r.target = self.viewdirs.data_ptr(), self.rgb.data_ptr()
        r.jitter = None
        r.idx = _lib.ptr(idx)
        r.n = int(idx.numel()) if idx is not None else int(n if n is not None else self.n)
        return r


class CameraPool:
    """Device ray pool of a set of calibrated views: the
    camera records and the float32 ground-truth colours (12 B per ray instead
    of the reference's 96 B of host-built float64 rays, camera.py:292-314).
    Pool row p is pixel p of the views in all_rays order (view-major,
    row-major pixels); the kernels regenerate its ray in the reference's
    float64 operation order (plx_camera.cuh).  Forward-facing pools (ndc)
    march NDC-warped rays and drop the rays parallel to the image plane as
    all_rays does (camera.py:303-307); `scale` pre-scales origins (360
    scenes, T:375-377)."""

    def __init__(self, cameras, images=None, ndc: bool = False, scale: float = 1.0,
                 drop_invalid: bool = True, device=None):
        from .camera import camera_record

        dev = torch.device(device or "cuda")
        cams = list(cameras)
        if not cams:
            raise ValueError("dataset needs at least one view")
        W, H = int(cams[0].width), int(cams[0].height)
        if any((int(c.width), int(c.height)) != (W, H) for c in cams):
            raise ValueError("images have mixed resolutions")      # camera.py:196-198
        self.device = dev
        self.width, self.height, self.n_views = W, H, len(cams)
        self.cams = torch.from_numpy(np.stack([camera_record(c) for c in cams])).to(dev)
        self.rgb = None
        if images is not None:
            img = np.ascontiguousarray(np.asarray(images, dtype=np.float32).reshape(-1, 3))
            if img.shape[0] != len(cams) * W * H:
                raise ValueError("image/camera count mismatch")
            self.rgb = torch.from_numpy(img).to(dev)
        self.pixel = None
        self.ndc, self.scale = bool(ndc), float(scale)
        self.n = len(cams) * W * H
        self._sync()
        if self.ndc and drop_invalid:
            _, _, v, _ = self.materialize(None, origins=False, dirs=False, rgb=False)
            valid = v[:, 2].abs() > 1e-10
            if not bool(valid.all()):
                self.pixel = torch.nonzero(valid).flatten().to(torch.int64).contiguous()
                if self.rgb is not None:
                    self.rgb = self.rgb[valid].contiguous()
                self.n = int(self.pixel.numel())
                self._sync()

    def _sync(self) -> None:
        c = _lib.PlxCameras()
        c.cams = self.cams.data_ptr()
        c.rgb = _lib.ptr(self.rgb)
        c.pixel = _lib.ptr(self.pixel)
        c.n_views, c.width, c.height = self.n_views, self.width, self.height
        c.ndc = int(self.ndc)
        c.scale = self.scale
        self._c = c

    def rays(self, idx: torch.Tensor | None, n: int | None = None) -> _lib.PlxRays:
        r = _lib.PlxRays()
        r.cams = ctypes.pointer(self._c)
        r.jitter = None
        r.idx = _lib.ptr(idx)
        r.n = int(idx.numel()) if idx is not None else int(n if n is not None else self.n)
        return r

    def materialize(self, idx: torch.Tensor | None, origins: bool = True, dirs: bool = True,
                    viewdirs: bool = True, rgb: bool = True):
        """Pool rows idx (all rows if None) as float64 (n, 3) device tensors
        (origins, march dirs, view dirs, gt) -- None where not requested."""
        n = int(idx.numel()) if idx is not None else self.n
        mk = lambda want: (torch.empty((n, 3), dtype=torch.float64, device=self.device)  # noqa: E731
                           if want else None)
        out = (mk(origins), mk(dirs), mk(viewdirs), mk(rgb and self.rgb is not None))
        _lib.check(_lib.lib().plx_generate_rays(
            ctypes.byref(self._c), _lib.ptr(idx), n, *(_lib.ptr(t) for t in out),
            _lib.stream_ptr()), "generate_rays")
        return out


def fused_mse_backward_pool(grid: SparseGrid, pool: RayPool, idx: torch.Tensor,
                            grads: GradientBuffer, opts: RenderOptions, n_total: int,
                            lam_cauchy: float, sums: torch.Tensor, jitter=None,
                            kopts: _lib.PlxRenderOpts | None = None,
                            cgrid: _lib.PlxGrid | None = None,
                            cgrad: _lib.PlxGrad | None = None) -> None:
    """The trainer's form of fused_mse_backward (R:253-279, T:455-457): batch =
    pool rows `idx` (device int64), sums (device f64[2]) accumulated, no sync."""
    r = pool.rays(idx)
    if jitter is not None:
        r.jitter = jitter.data_ptr()
    c = cgrid if cgrid is not None else grid._c(with_occ=opts.interp == "trilinear")
    ko = kopts if kopts is not None else kernel_opts(grid, opts)
    gb = cgrad if cgrad is not None else grads._c()
    sp, sn, _keep = _lib.render_scratch(c, ko, r.n, grid.device)
    _lib.check(_lib.lib().plx_render_fused_bwd(
        ctypes.byref(c), ctypes.byref(r), ctypes.byref(ko), 1, 2.0 / n_total, float(lam_cauchy),
        ctypes.byref(gb), None, sums.data_ptr(), sp, sn, _lib.stream_ptr()), "render_fused_bwd")


def render_pool(grid: SparseGrid, pool: CameraPool, opts: RenderOptions, first: int = 0,
                count: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """render_forward (K:173-238) of pool rows [first, first + count) with the
    rays generated in the kernel -> (count, 3) float64 device tensor."""
    count = pool.n - first if count is None else int(count)
    out = out if out is not None else torch.empty((count, 3), dtype=torch.float64,
                                                  device=grid.device)
    idx = torch.arange(first, first + count, dtype=torch.int64, device=grid.device)
    r = pool.rays(idx)
    c = grid._c(with_occ=opts.interp == "trilinear")
    ko = kernel_opts(grid, opts)
    _lib.check(_lib.lib().plx_render_fwd(ctypes.byref(c), ctypes.byref(r), ctypes.byref(ko),
                                         out.data_ptr(), None, None, _lib.stream_ptr()),
               "render_fwd")
    return out


def render_image(grid: SparseGrid, camera, opts: RenderOptions | None = None,
                 chunk: int = 1 << 20) -> np.ndarray:
    """R:282-293: full camera view -> (H, W, 3) float64 image, rays generated
    on the device."""
    opts = opts or RenderOptions()
    pool = CameraPool([camera], None, device=grid.device)
    return render_pool(grid, pool, opts).cpu().numpy().reshape(camera.height, camera.width, 3)
