"""Cameras and rays (drop-in for pkg/src/plenoxel/camera.py:27-134, 292-314).

The reference builds every training ray on the host (generate_rays, to_ndc,
all_rays: 96 bytes of float64 per ray).  Here rays are generated on the
device from (view, pixel) ids by libplx.so (plx_generate_rays / plx_to_ndc,
csrc/plx_camera.cuh), bit-identical to the reference's float64 arrays; the
trainer never materialises them at all (render.CameraPool feeds the kernels
the camera records).  The functions below keep the reference's API and
return numpy arrays like it does.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


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


def camera_record(cam: Camera) -> np.ndarray:
    """The PLX_CAM-double record of plx_cameras: c2w[:3, :4] row-major,
    focal, width, height, near."""
    r = np.zeros(_lib.CAM)
    r[:12] = cam.c2w[:3, :4].reshape(-1)
    r[12:] = (float(cam.focal), float(cam.width), float(cam.height), float(cam.near))
    return r


def generate_rays(cam: Camera, device=None):
    """All pixel-centre rays of a view, row-major (camera.py:91-100) ->
    (origins, dirs) float64 (H*W, 3) numpy arrays, generated on the device."""
    from .render import CameraPool

    pool = CameraPool([cam], None, device=device)
    o, d, _, _ = pool.materialize(None, rgb=False)
    return o.cpu().numpy(), d.cpu().numpy()


def to_ndc(origins, dirs, cam: Camera, near: float | None = None, device=None):
    """Forward-facing NDC warp (camera.py:103-134) on the device ->
    (o_ndc, d_ndc, valid) numpy arrays."""
    import torch

    rec = camera_record(cam)
    if near is not None:
        rec[15] = float(near)
    dev = torch.device(device or "cuda")
    o = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(origins), dtype=np.float64)).to(dev)
    d = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(dirs), dtype=np.float64)).to(dev)
    valid = torch.empty(o.shape[0], dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().plx_to_ndc(rec.ctypes.data_as(ctypes.c_void_p), o.data_ptr(),
                                     d.data_ptr(), valid.data_ptr(), o.shape[0],
                                     _lib.stream_ptr()), "to_ndc")
    return o.cpu().numpy(), d.cpu().numpy(), valid.cpu().numpy().astype(bool)


def all_rays(images, cameras, scene_type: str = "bounded", device=None):
    """Flatten every pixel of every view (camera.py:292-314) ->
    (origins, march_dirs, view_dirs, rgb), each (N, 3) float64 numpy, with
    forward-facing rays that are parallel to the image plane dropped.  The
    arrays are generated on the device (render.CameraPool); the trainer uses
    the pool directly and never calls this."""
    from .render import CameraPool

    pool = CameraPool(cameras, images, ndc=scene_type == "forward_facing_ndc", device=device)
    return tuple(t.cpu().numpy() for t in pool.materialize(None))
