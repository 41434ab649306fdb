"""Synthetic scenes for benchmarks and tests.

A restatement of the reference's procedural oracle scene (pkg/src/plenoxel/
toy.py:25-162): four soft spheres baked into a ground-truth grid, viewed by
inward-facing cameras on a golden-angle hemisphere spiral.  Images are
rendered on the device with the same forward kernel used for training and,
like the reference's PNG round trip (toy.py:152-154, artifact_io.py:199-223),
quantised to 8 bits.  Not part of the optimisation hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .camera import Camera
from .sh import SH_C0

TOY_AABB = 1.1
TOY_SIGMA = 45.0

_SPHERES = [   # toy.py:29-34
    ((0.38, 0.05, 0.12), 0.42, (0.85, 0.25, 0.20), None),
    ((-0.40, 0.30, -0.12), 0.34, (0.20, 0.55, 0.90), (3, 0.20)),
    ((-0.05, -0.45, 0.30), 0.28, (0.95, 0.80, 0.25), (6, 0.15)),
    ((0.05, 0.42, 0.45), 0.22, (0.35, 0.85, 0.45), None),
]


@dataclass
class Dataset:
    """Calibrated views (camera.py:60-76): images float32 (N, H, W, 3)."""

    images: np.ndarray
    cameras: list
    scene_type: str = "bounded"
    background: np.ndarray = field(default_factory=lambda: np.ones(3))
    paths: list = field(default_factory=list)

    def __post_init__(self):
        if len(self.cameras) == 0:
            raise ValueError("dataset needs at least one view")
        if len(self.cameras) != len(self.images):
            raise ValueError("image/camera count mismatch")

    @property
    def n_views(self) -> int:
        return len(self.cameras)


def toy_grid_arrays(dims: int = 64, aabb: float = TOY_AABB):
    """build_toy_grid (toy.py:65-99) before its final density prune:
    (table float64 (dims^3, 28), dims).  Host numpy."""
    d = int(dims)
    axis = np.linspace(-aabb, aabb, d)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    pts = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    band = 2.0 * (2 * aabb / (d - 1))
    sigma = np.zeros(len(pts))
    weight_sum = np.zeros(len(pts))
    coeffs = np.zeros((len(pts), 27))
    for center, radius, rgb, viewdep in _SPHERES:
        dist = np.linalg.norm(pts - np.asarray(center), axis=1)
        s = np.clip((radius - dist) / band + 0.5, 0.0, 1.0)
        s = s * s * (3.0 - 2.0 * s)
        sigma = np.maximum(sigma, TOY_SIGMA * s)
        shade = 1.0 + 0.25 * (pts[:, 2] - center[2]) / radius
        c = np.zeros((len(pts), 27))
        for ch in range(3):
            c[:, 9 * ch] = rgb[ch] * shade / SH_C0
        if viewdep is not None:
            bidx, scale = viewdep
            for ch in range(3):
                c[:, 9 * ch + bidx] = rgb[ch] * scale / SH_C0
        coeffs += s[:, None] * c
        weight_sum += s
    occupied = weight_sum > 0
    coeffs[occupied] /= weight_sum[occupied, None]
    table = np.zeros((len(pts), 28))
    table[:, 0] = sigma
    table[:, 1:] = coeffs
    return table, (d, d, d)


def build_toy_grid(dims: int = 64, aabb: float = TOY_AABB, device=None):
    """toy.py:65-99 on the device: dense bake, then prune('density', 1e-6)."""
    from .grid import SparseGrid

    table, shape = toy_grid_arrays(dims, aabb)
    g = SparseGrid(np.arange(table.shape[0], dtype=np.int32).reshape(shape),
                   table.astype(np.float32), (-aabb,) * 3, (aabb,) * 3, device=device)
    g, _ = g.prune("density", 1e-6)
    return g


def hemisphere_cameras(n: int, res: int, radius: float = 3.0, fov_x: float = 0.6911112,
                       phase: float = 0.0):
    """toy.py:102-126."""
    cams = []
    golden = math.pi * (3.0 - math.sqrt(5.0))
    focal = 0.5 * res / math.tan(0.5 * fov_x)
    for i in range(n):
        elev = math.radians(8.0 + 55.0 * ((i + 0.5) / n))
        azim = phase + i * golden
        pos = radius * np.array([math.cos(azim) * math.cos(elev),
                                 math.sin(azim) * math.cos(elev), math.sin(elev)])
        zc = pos / np.linalg.norm(pos)
        xc = np.cross(np.array([0.0, 0.0, 1.0]), zc)
        xc /= np.linalg.norm(xc)
        yc = np.cross(zc, xc)
        c2w = np.eye(4)
        c2w[:3, 0], c2w[:3, 1], c2w[:3, 2], c2w[:3, 3] = xc, yc, zc, pos
        cams.append(Camera(c2w=c2w, focal=focal, width=res, height=res))
    return cams, fov_x


def make_toy_dataset(n_views: int = 25, res: int = 128, n_test: int = 10, grid_dim: int = 64,
                     step_frac: float = 0.5, seed: int = 0, device=None):
    """toy.py:129-162 without the files: (train Dataset, test Dataset, gt grid)."""
    from .render import RenderOptions, render_image

    grid = build_toy_grid(grid_dim, device=device)
    opts = RenderOptions(step_frac=step_frac, background=(1.0, 1.0, 1.0))
    rng = np.random.default_rng(seed)
    phase_train = float(rng.uniform(0, 2 * math.pi))
    out = []
    for count, phase in ((n_views, phase_train), (n_test, phase_train + 0.5)):
        cams, _ = hemisphere_cameras(count, res, phase=phase)
        imgs = []
        for cam in cams:
            img = render_image(grid, cam, opts)
            q = np.rint(np.clip(img, 0.0, 1.0) * 255.0)          # write_image quantisation
            imgs.append((q / 255.0).astype(np.float32))           # read_image + astype(f32)
        out.append(Dataset(np.stack(imgs), cams, "bounded", np.ones(3),
                           [f"mem://{id(out)}/{len(out)}/{i}" for i in range(count)]))
    return out[0], out[1], grid


def dataset_from_arrays(imgs_u8, c2w, focal, scene_type: str = "bounded", tag: str = "") -> Dataset:
    """Rebuild a Dataset from uint8 images + poses (tests/golden/*.npz)."""
    imgs = (np.asarray(imgs_u8, dtype=np.float64) / 255.0).astype(np.float32)
    h, w = imgs.shape[1:3]
    cams = [Camera(c2w=c, focal=float(f), width=w, height=h) for c, f in zip(c2w, focal)]
    return Dataset(imgs, cams, scene_type, np.ones(3),
                   [f"mem://{tag}/{i}" for i in range(len(cams))])
