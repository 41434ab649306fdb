"""Pinhole ray generation and the NDC warp (host side, float64), restating
pkg/src/plenoxel/camera.py:27-134 and 292-314.  These feed the device ray
pool once per dataset; they are not on the per-step hot path."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Camera:
    """camera.py:27-48 (OpenGL convention, looking down -z)."""

    c2w: np.ndarray
    focal: float
    width: int
    height: int
    near: float = 0.0
    far: float = math.inf

    def __post_init__(self):
        self.c2w = np.asarray(self.c2w, dtype=np.float64)
        if self.c2w.shape != (4, 4):
            raise ValueError("camera transform must be 4x4")
        r = self.c2w[:3, :3]
        if np.max(np.abs(r @ r.T - np.eye(3))) > 1e-4:
            raise ValueError("camera rotation is not orthonormal")
        if self.focal <= 0:
            raise ValueError("focal length must be positive")

    @property
    def position(self) -> np.ndarray:
        return self.c2w[:3, 3]


def generate_rays(cam: Camera):
    """All pixel-centre rays, row-major (camera.py:91-100)."""
    xs = (np.arange(cam.width) + 0.5 - cam.width / 2) / cam.focal
    ys = -(np.arange(cam.height) + 0.5 - cam.height / 2) / cam.focal
    gx, gy = np.meshgrid(xs, ys)
    d_cam = np.stack([gx, gy, -np.ones_like(gx)], axis=-1).reshape(-1, 3)
    d = d_cam @ cam.c2w[:3, :3].T
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    o = np.broadcast_to(cam.position, d.shape).copy()
    return o, np.ascontiguousarray(d)


def to_ndc(origins, dirs, cam: Camera, near: float | None = None):
    """Forward-facing NDC warp (camera.py:103-134)."""
    near = cam.near if near is None else near
    if near <= 0:
        near = 1.0
    o = np.atleast_2d(np.asarray(origins, dtype=np.float64)).copy()
    d = np.atleast_2d(np.asarray(dirs, dtype=np.float64)).copy()
    valid = np.abs(d[:, 2]) > 1e-10
    dz = np.where(valid, d[:, 2], 1.0)
    t = -(near + o[:, 2]) / dz
    o = o + t[:, None] * d
    oz = np.where(np.abs(o[:, 2]) > 1e-12, o[:, 2], -1e-12)
    fx = cam.focal / (cam.width / 2.0)
    fy = cam.focal / (cam.height / 2.0)
    o_ndc = np.stack([-fx * o[:, 0] / oz, -fy * o[:, 1] / oz, 1.0 + 2.0 * near / oz], -1)
    d_ndc = np.stack([-fx * (d[:, 0] / dz - o[:, 0] / oz),
                      -fy * (d[:, 1] / dz - o[:, 1] / oz),
                      -2.0 * near / oz], axis=-1)
    return o_ndc, d_ndc, valid


def all_rays(images, cameras, scene_type: str = "bounded"):
    """Flatten every pixel of every view (camera.py:292-314) ->
    (origins, march_dirs, view_dirs, rgb), each (N, 3) float64.

    `images` are float arrays in [0, 1]; the reference stores them as float32
    (camera.py:193) and widens to float64 here, so we do the same."""
    origins, mdirs, vdirs, rgb = [], [], [], []
    for img, cam in zip(images, cameras):
        o, d = generate_rays(cam)
        v = d
        img = np.asarray(img, dtype=np.float32).reshape(-1, 3)
        if scene_type == "forward_facing_ndc":
            o, d, valid = to_ndc(o, d, cam)
            if not np.all(valid):
                o, d, v, img = o[valid], d[valid], v[valid], img[valid]
        origins.append(o)
        mdirs.append(d)
        vdirs.append(v)
        rgb.append(np.asarray(img, dtype=np.float64))
    return (np.concatenate(origins), np.concatenate(mdirs), np.concatenate(vdirs),
            np.concatenate(rgb))
