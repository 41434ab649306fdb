"""Device ray generation and device metrics (§8(f)-2):
plx_generate_rays / plx_to_ndc bit-exact against the reference's own
generate_rays / to_ndc / all_rays outputs (tests/golden/camera.npz, ndc.npz,
make_camera_golden.py), the camera pool driving the kernels exactly like the
materialised float64 ray arrays, and plx_image_metrics against the
reference's host PSNR / SSIM (losses.py:110-165, restated in oracle.py)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

from helpers import load, random_grid, ray_batch

pytestmark = pytest.mark.gpu


def _cam(z, key, near=0.0):
    from paper_2112_05131_b200.camera import Camera
    w, h = (int(x) for x in z[f"{key}_wh"])
    return Camera(c2w=z[f"{key}_c2w"], focal=float(z[f"{key}_focal"]), width=w, height=h,
                  near=near)


def test_generate_rays_bit_exact_vs_reference():
    from paper_2112_05131_b200.camera import generate_rays
    z = load("camera.npz")
    k = 0
    while f"cam{k}_c2w" in z:
        cam = _cam(z, f"cam{k}")
        o, d = generate_rays(cam)
        np.testing.assert_array_equal(d, z[f"cam{k}_d"])
        assert np.all(o == cam.position)
        k += 1
    assert k >= 6


def test_to_ndc_bit_exact_vs_reference():
    from paper_2112_05131_b200.camera import Camera, generate_rays, to_ndc
    z = load("camera.npz")
    for k in range(3):
        cam = _cam(z, f"ndc{k}", near=float(z[f"ndc{k}_near"]))
        o, d = generate_rays(cam)
        on, dn, valid = to_ndc(o, d, cam)
        np.testing.assert_array_equal(on, z[f"ndc{k}_o"])
        np.testing.assert_array_equal(dn, z[f"ndc{k}_d"])
        np.testing.assert_array_equal(valid, z[f"ndc{k}_valid"])
    # random rays incl. rays parallel to the image plane (ndc.npz)
    n = load("ndc.npz")
    w, h = (int(x) for x in n["cam_wh"])
    cam = Camera(c2w=np.eye(4), focal=float(n["cam_focal"][0]), width=w, height=h)
    on, dn, valid = to_ndc(n["o"], n["d"], cam, near=1.0)
    np.testing.assert_array_equal(valid, n["valid"])
    np.testing.assert_array_equal(on, n["on"])
    np.testing.assert_array_equal(dn, n["dn"])


def test_all_rays_forward_facing_pool_bit_exact():
    """all_rays of a forward-facing dataset (camera.py:292-314): NDC march
    rays, world view dirs, float32-widened colours."""
    from paper_2112_05131_b200.camera import all_rays
    z = load("camera.npz")
    cam = _cam(z, "ndc0", near=float(z["ndc0_near"]))
    o, d, v, rgb = all_rays(z["ff_img"], [cam], "forward_facing_ndc")
    np.testing.assert_array_equal(o, z["ff_o"])
    np.testing.assert_array_equal(d, z["ff_d"])
    np.testing.assert_array_equal(v, z["ff_v"])
    np.testing.assert_array_equal(rgb, z["ff_rgb"])


def test_camera_pool_drops_invalid_ndc_rays():
    """A forward-facing view with rays parallel to the image plane: the pool
    keeps exactly the valid rows, in all_rays order (camera.py:303-307)."""
    from paper_2112_05131_b200.camera import Camera
    from paper_2112_05131_b200.render import CameraPool
    c2w = np.eye(4)
    c2w[:3, :3] = np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0]])   # looks along +y: d_z = y
    cam = Camera(c2w=c2w, focal=20.0, width=16, height=15)
    img = np.random.default_rng(0).uniform(0, 1, (1, 15, 16, 3)).astype(np.float32)
    pool = CameraPool([cam], img, ndc=True)
    full = CameraPool([cam], img, ndc=True, drop_invalid=False)
    _, _, v, _ = full.materialize(None)
    keep = (v[:, 2].abs() > 1e-10).cpu().numpy()
    assert 0 < keep.sum() < 240
    assert pool.n == keep.sum()
    o, d, vv, rgb = pool.materialize(None)
    o2, d2, v2, rgb2 = full.materialize(None)
    np.testing.assert_array_equal(o.cpu().numpy(), o2.cpu().numpy()[keep])
    np.testing.assert_array_equal(rgb.cpu().numpy(), rgb2.cpu().numpy()[keep])


def test_camera_pool_step_equals_array_pool_step():
    """The fused backward on pool rows: rays generated inside the kernels
    (CameraPool) == the same rays materialised as float64 arrays (RayPool):
    identical rgb, touched rows and mse; gradients to f32-atomic order."""
    from paper_2112_05131_b200 import render, scenes
    from paper_2112_05131_b200.grid import GradientBuffer, SparseGrid

    rng = np.random.default_rng(3)
    og = random_grid(rng, dims=(12, 11, 13), holes=0.2)
    g = SparseGrid(og.links, og.table, og.aabb_min, og.aabb_max)
    cams, _ = scenes.hemisphere_cameras(3, 24, radius=2.5)
    imgs = rng.uniform(0, 1, (3, 24, 24, 3)).astype(np.float32)
    cp = render.CameraPool(cams, imgs)
    o, d, v, gt = cp.materialize(None)
    ap = render.RayPool(o, d, v, gt)
    idx = torch.from_numpy(rng.permutation(cp.n)[:700]).cuda()
    opts = render.RenderOptions(background=(0.3, 0.6, 0.9))
    outs = []
    for pool in (cp, ap):
        gb = GradientBuffer(g.n_rows)
        sums = torch.zeros(2, dtype=torch.float64, device="cuda")
        render.fused_mse_backward_pool(g, pool, idx, gb, opts, 700, 0.0, sums)
        rgb = render.render_rays(g, *(t[idx] for t in (o, d)), opts, viewdirs=v[idx])[0]
        outs.append((gb.dense(), gb.touched_rows(), float(sums[0]), rgb.cpu().numpy()))
    (ga, ra, ma, _), (gb_, rb, mb, _) = outs
    np.testing.assert_array_equal(ra, rb)
    assert ma == pytest.approx(mb, rel=1e-12)
    np.testing.assert_allclose(ga, gb_, rtol=1e-5, atol=1e-7 * np.abs(gb_).max())
    # forward render through the pool == through the arrays, bit for bit
    cam_rgb = render.render_pool(g, cp, opts).cpu().numpy()
    arr_rgb = render.render_rays(g, o, d, opts, viewdirs=v)[0].cpu().numpy()
    np.testing.assert_array_equal(cam_rgb, arr_rgb)


def test_image_metrics_match_reference_formulas():
    """plx_image_metrics vs losses.psnr / losses.ssim (losses.py:110-165) of
    the reference (restated in oracle.py with scipy) to 1e-9."""
    from paper_2112_05131_b200 import losses
    rng = np.random.default_rng(0)
    for shape in ((40, 37, 3), (11, 11, 3), (64, 48), (128, 200, 3)):
        a = rng.uniform(0, 1, shape)
        b = np.clip(a + rng.normal(0, 0.05, shape), 0, 1)
        p, s = losses.image_metrics(a, b)
        assert p == pytest.approx(orc.psnr(a, b), rel=1e-12)
        assert abs(s - orc.ssim(a, b)) < 1e-9
        assert losses.psnr(a, b) == pytest.approx(orc.psnr(a, b), rel=1e-12)
        assert abs(losses.ssim(a, b) - orc.ssim(a, b)) < 1e-9
    assert losses.psnr(a, a) == float("inf")
    assert losses.psnr(np.zeros((3, 2)), np.ones((3, 2))) == 0.0    # any size for psnr
    with pytest.raises(ValueError):
        losses.ssim(np.zeros((10, 30, 3)), np.zeros((10, 30, 3)))
    with pytest.raises(ValueError):
        losses.psnr(np.zeros((4, 4)), np.zeros((4, 5)))


def test_evaluate_on_device_matches_host_evaluation():
    """trainer.evaluate (T:309-347) renders and scores on the device; the same
    views rendered through materialised rays and scored on the host by the
    reference's formulas give the same numbers (1e-9)."""
    from paper_2112_05131_b200 import render, trainer
    from paper_2112_05131_b200.camera import generate_rays
    from paper_2112_05131_b200.scenes import build_toy_grid, make_toy_dataset

    _, test_ds, gt_grid = make_toy_dataset(n_views=2, res=32, n_test=3, grid_dim=24)
    g = gt_grid.upsample((20, 20, 20))
    opts = render.RenderOptions(background=(1.0, 1.0, 1.0))
    p, s, rows = trainer.evaluate(g, test_ds, opts)
    for r, img, cam in zip(rows, test_ds.images, test_ds.cameras):
        o, d = generate_rays(cam)
        pred = render.render_rays(g, o, d, opts, viewdirs=d)[0].reshape(img.shape)
        gt = np.asarray(img, dtype=np.float64)
        assert r["psnr"] == pytest.approx(orc.psnr(pred, gt), rel=1e-12)
        assert abs(r["ssim"] - orc.ssim(pred, gt)) < 1e-9
    assert p == pytest.approx(np.mean([r["psnr"] for r in rows]))
