"""Edge cases of the device path against the CPU oracle: empty and ragged
batches, rays that miss the box, axis-aligned rays and rays starting inside
it, every ray on the same samples (scatter collisions), grids with no
positive density, the smallest lattice, and an update with nothing touched.
The reference's own tests cover the same shapes (pkg/tests/test_render.py,
test_kernels.py: missing rays, grazing rays, zero-density grids); bars as in
test_gpu_parity.py."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

from helpers import grad_close, random_grid, ray_batch
from test_gpu_parity import RGB_TOL, _check_bwd, dev_grid, px

pytestmark = pytest.mark.gpu


def _fwd_close(g, o, d, kw):
    want = orc.render_rays(g, o, d, **kw)
    got = px().render_rays(dev_grid(g), o, d, px().RenderOptions(**kw))
    for a, b in zip(got, want):
        assert a.shape == b.shape
        if a.size:
            assert np.max(np.abs(a - b)) < RGB_TOL
    return got


def test_zero_rays_forward_and_backward():
    rng = np.random.default_rng(300)
    g = random_grid(rng, dims=(5, 6, 7))
    o = np.zeros((0, 3))
    rgb, trans, wsum = _fwd_close(g, o, o, dict(stop_thresh=1e-4))
    assert rgb.shape == (0, 3) and trans.shape == (0,)
    dg = dev_grid(g)
    buf = px().GradientBuffer(dg.n_rows)
    rgb, mse, cau = px().fused_mse_backward(dg, o, o, o, o, buf, px().RenderOptions(),
                                            n_total=1, lam_cauchy=1e-3)
    assert rgb.shape == (0, 3) and mse == 0.0 and cau == 0.0
    assert buf.n_touched == 0 and float(buf.data.abs().sum()) == 0.0
    rgb, cau = px().render_rays_backward(dg, o, o, o, buf, px().RenderOptions(), lam_cauchy=1e-3)
    assert rgb.shape == (0, 3) and cau == 0.0 and buf.n_touched == 0
    w = dg.max_weight_accumulate(o, o)
    assert float(np.max(w)) == 0.0


@pytest.mark.parametrize("n", [1, 31, 33, 257])
def test_ragged_batches_match_oracle(n):
    rng = np.random.default_rng(301 + n)
    g = random_grid(rng, dims=(6, 5, 7), holes=0.2)
    o, d = ray_batch(rng, n)
    gt = rng.uniform(0, 1, (n, 3))
    _check_bwd(g, o, d, gt, dict(stop_thresh=1e-4, background=(0.2, 0.4, 0.6)), lam=1e-3)


def test_rays_missing_the_box_return_background_and_touch_nothing():
    rng = np.random.default_rng(302)
    g = random_grid(rng, dims=(5, 5, 5))
    n = 48
    o = rng.uniform(-0.5, 0.5, (n, 3)) + np.array([4.0, 0.0, 0.0])
    d = np.tile([0.0, 1.0, 0.0], (n, 1)) + rng.normal(scale=0.05, size=(n, 3))
    d[:, 0] = 0.0                                   # parallel to the +x face, outside it
    d[n // 2:] = np.array([1.0, 0.2, 0.1])          # pointing away from the box
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    bg = (0.25, 0.5, 0.75)
    rgb, trans, wsum = _fwd_close(g, o, d, dict(background=bg))
    np.testing.assert_array_equal(rgb, np.tile(bg, (n, 1)))
    np.testing.assert_array_equal(trans, np.ones(n))
    gt = rng.uniform(0, 1, (n, 3))
    buf_d, _ = _check_bwd(g, o, d, gt, dict(background=bg), lam=1e-3)
    assert buf_d.n_touched == 0


@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_axis_aligned_and_interior_rays_match_oracle(interp):
    rng = np.random.default_rng(303)
    g = random_grid(rng, dims=(7, 6, 5), holes=0.1)
    dirs, origins = [], []
    for axis in range(3):
        for sgn in (1.0, -1.0):
            for _ in range(6):
                dv = np.zeros(3)
                dv[axis] = sgn
                ov = rng.uniform(-0.8, 0.8, 3)
                ov[axis] = -3.0 * sgn
                dirs.append(dv)
                origins.append(ov)
    for _ in range(24):   # starting inside the box, any direction
        origins.append(rng.uniform(-0.7, 0.7, 3))
        v = rng.normal(size=3)
        dirs.append(v / np.linalg.norm(v))
    for _ in range(8):    # on a lattice plane, parallel to it
        ov = rng.uniform(-0.9, 0.9, 3)
        ov[2] = 0.0
        origins.append(ov - np.array([3.0, 0.0, 0.0]))
        dirs.append(np.array([1.0, 0.0, 0.0]))
    o, d = np.array(origins), np.array(dirs)
    gt = rng.uniform(0, 1, (len(o), 3))
    kw = dict(stop_thresh=1e-4, background=(1.0, 1.0, 1.0), interp=interp)
    _fwd_close(g, o, d, kw)
    _check_bwd(g, o, d, gt, kw, lam=1e-3)


def test_identical_rays_collide_on_every_row():
    """64 copies of one ray: every sample's rows receive 64 concurrent adds."""
    rng = np.random.default_rng(304)
    g = random_grid(rng, dims=(6, 6, 6))
    o1, d1 = ray_batch(rng, 1)
    o, d = np.repeat(o1, 64, 0), np.repeat(d1, 64, 0)
    gt = np.repeat(rng.uniform(0, 1, (1, 3)), 64, 0)
    buf_d, buf_o = _check_bwd(g, o, d, gt, dict(stop_thresh=0.0), lam=1e-3)
    # and the batch gradient is 64x the single-ray one
    single = px().GradientBuffer(buf_d.n_rows)
    px().fused_mse_backward(dev_grid(g), o1, d1, orc.normalize_dirs(d1), gt[:1], single,
                            px().RenderOptions(stop_thresh=0.0), n_total=64, lam_cauchy=1e-3)
    ok, worst, _ = grad_close(buf_d.dense(), 64.0 * single.dense(), rel=1e-5)
    assert ok, worst


@pytest.mark.parametrize("formula", ["relative", "absolute"])
def test_grid_without_positive_density(formula):
    rng = np.random.default_rng(305)
    g = random_grid(rng, dims=(5, 5, 5), sigma_range=(-2.0, -0.1))
    o, d = ray_batch(rng, 40)
    bg = (0.1, 0.9, 0.3)
    rgb, trans, _ = _fwd_close(g, o, d, dict(background=bg, formula=formula))
    np.testing.assert_allclose(trans, 1.0)
    gt = rng.uniform(0, 1, (40, 3))
    _check_bwd(g, o, d, gt, dict(background=bg, formula=formula), lam=1e-3)


def test_smallest_lattice():
    rng = np.random.default_rng(306)
    g = random_grid(rng, dims=(2, 2, 2))
    o, d = ray_batch(rng, 64)
    gt = rng.uniform(0, 1, (64, 3))
    for interp in ("trilinear", "nearest"):
        kw = dict(stop_thresh=1e-4, interp=interp)
        _fwd_close(g, o, d, kw)
        _check_bwd(g, o, d, gt, kw, lam=1e-3)


def test_update_with_nothing_touched_is_a_no_op():
    g = px().SparseGrid.dense((6, 7, 8), (0, 0, 0), (1, 1, 1), sigma=0.3, rgb=0.2)
    before = g.table.clone()
    buf = px().GradientBuffer(g.n_rows)
    st = px().OptimState(g.n_rows)
    from paper_2112_05131_b200 import optim
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")   # the caller zeroes it (optim.step)
    optim.step(g, buf, st, 0.1, 0.01, clear=True, count_out=cnt)
    assert int(cnt.item()) == 0
    assert torch.equal(g.table, before)
    assert float(st.v.abs().sum()) == 0.0
