#!/usr/bin/env python3
"""Golden vectors for pinhole ray generation and the NDC warp, produced by the
REFERENCE (camera.py:91-134, 292-314 imported from /root/reference/pkg/src;
build container only).  -> camera.npz:

  cam{k}_c2w, cam{k}_focal, cam{k}_wh     camera k (hemisphere toy poses,
                                          random rotations, odd sizes)
  cam{k}_d                                 generate_rays(cam) directions
  ndc{k}_o, ndc{k}_d, ndc{k}_valid, ndc{k}_near
                                          to_ndc(generate_rays(cam), cam, near)
  ff_o, ff_d, ff_v                         all_rays of a forward-facing dataset

Usage: python tests/golden/make_camera_golden.py
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from plenoxel.camera import Camera, Dataset, all_rays, generate_rays, to_ndc  # noqa: E402
from plenoxel.toy import _hemisphere_cameras  # noqa: E402

OUT = Path(__file__).resolve().parent


def rot(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def main():
    rng = np.random.default_rng(7)
    cams = list(_hemisphere_cameras(3, 41, phase=0.3)[0])
    cams = [Camera(c2w=c.c2w, focal=c.focal, width=41, height=41) for c in cams]
    for w, h in ((37, 23), (64, 48), (20, 31)):
        c2w = np.eye(4)
        c2w[:3, :3] = rot(rng)
        c2w[:3, 3] = rng.uniform(-3, 3, 3)
        cams.append(Camera(c2w=c2w, focal=float(rng.uniform(20, 90)), width=w, height=h))
    out = {}
    for k, c in enumerate(cams):
        o, d = generate_rays(c)
        assert np.all(o == c.position)
        out[f"cam{k}_c2w"] = c.c2w
        out[f"cam{k}_focal"] = np.float64(c.focal)
        out[f"cam{k}_wh"] = np.array([c.width, c.height])
        out[f"cam{k}_d"] = d
    # forward-facing cameras (identity-like LLFF poses looking down -z)
    ff = []
    for k in range(3):
        c2w = np.eye(4)
        ang = rng.uniform(-0.15, 0.15, 3)
        cx, sx = math.cos(ang[0]), math.sin(ang[0])
        cy, sy = math.cos(ang[1]), math.sin(ang[1])
        rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
        ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
        c2w[:3, :3] = rx @ ry
        c2w[:3, 3] = rng.uniform(-0.3, 0.3, 3)
        near = [0.0, 1.0, 0.7][k]
        c = Camera(c2w=c2w, focal=float(rng.uniform(30, 60)), width=33 + 4 * k, height=27,
                   near=near)
        ff.append(c)
        o, d = generate_rays(c)
        on, dn, valid = to_ndc(o, d, c)
        out[f"ndc{k}_c2w"] = c.c2w
        out[f"ndc{k}_focal"] = np.float64(c.focal)
        out[f"ndc{k}_wh"] = np.array([c.width, c.height])
        out[f"ndc{k}_near"] = np.float64(near)
        out[f"ndc{k}_o"], out[f"ndc{k}_d"], out[f"ndc{k}_valid"] = on, dn, valid
    imgs = np.stack([rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32)
                     for c in ff[:1]])
    ds = Dataset(images=imgs, cameras=ff[:1], scene_type="forward_facing_ndc",
                 background=np.zeros(3), paths=["a"])
    o, d, v, rgb = all_rays(ds)
    out["ff_o"], out["ff_d"], out["ff_v"], out["ff_rgb"] = o, d, v, rgb
    out["ff_img"] = imgs
    np.savez_compressed(OUT / "camera.npz", **out)
    print("wrote", OUT / "camera.npz", sum(a.nbytes for a in out.values()), "bytes raw")


if __name__ == "__main__":
    main()
