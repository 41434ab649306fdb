"""The reference's remaining 360 / multi-sphere-image behaviours
(pkg/tests/test_msi.py) on the device path -- above all the finite-
difference check of the composite's gradients, which exercises the 360
backward end to end (the bounded march / colour / scatter kernels in 360
mode plus msi_bg_kernel, with the Cauchy and beta terms) against float64
central differences of the reference's render_backward_360 (the oracle)."""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def msi():
    from paper_2112_05131_b200 import msi as m
    return m


def px():
    import paper_2112_05131_b200 as m
    return m


def _bg(n_layers=6, h=8, w=12, sigma=0.5, rgb=(0.3, 0.5, 0.7)):
    bg = msi().MsiBackground.create(n_layers, h, w)
    bg.data[..., 0] = sigma
    for c in range(3):
        bg.data[..., 1 + c] = rgb[c]
    return bg


def test_layers_and_background_sampling():
    m = msi()
    r = m.layer_radii(64)
    np.testing.assert_allclose(np.diff(1.0 / r), -1.0 / 63.0, atol=1e-12)
    assert r[0] == 1.0 and math.isinf(r[-1]) and np.all(np.diff(r) > 0)
    rng = np.random.default_rng(0)
    pts = rng.normal(size=(50, 3))
    pts *= rng.uniform(1.0, 30.0, (50, 1)) / np.linalg.norm(pts, axis=1, keepdims=True)
    sig, rgb = m.sample_background(_bg(), pts)
    np.testing.assert_allclose(sig, 0.5, atol=1e-12)
    np.testing.assert_allclose(rgb, np.tile([0.3, 0.5, 0.7], (50, 1)), atol=1e-12)
    with pytest.raises(ValueError):
        m.sample_background(_bg(), np.array([0.5, 0.0, 0.0]))
    bg = _bg(n_layers=5, h=6, w=8)
    bg.data[:] = torch.as_tensor(rng.uniform(0.1, 1.0, tuple(bg.data.shape)))
    lay, j, i = 2, 3, 5       # a texel centre returns the stored texel
    th, ph = (j + 0.5) * math.pi / 6, -math.pi + (i + 0.5) * 2 * math.pi / 8
    p = bg.radii[lay] * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph),
                                  math.cos(th)])
    s, c = m.sample_background(bg, p)
    want = bg.data[lay, j, i].cpu().numpy()
    assert s == pytest.approx(want[0], rel=1e-9)
    np.testing.assert_allclose(c, want[1:], rtol=1e-9)
    gaps = []                 # continuity across the phi seam
    for eps in (1e-3, 1e-5, 1e-7):
        pa = 2.0 * np.array([math.cos(math.pi - eps) * math.sin(1.1),
                             math.sin(math.pi - eps) * math.sin(1.1), math.cos(1.1)])
        pb = 2.0 * np.array([math.cos(-math.pi + eps) * math.sin(1.1),
                             math.sin(-math.pi + eps) * math.sin(1.1), math.cos(1.1)])
        (sa, ca), (sb, cb) = m.sample_background(bg, pa), m.sample_background(bg, pb)
        gaps.append(abs(sa - sb) + np.max(np.abs(ca - cb)))
    assert gaps[2] < 1e-5


def test_opaque_foreground_blocks_background():
    g = px().SparseGrid.dense((4, 4, 4), (-1, -1, -1), (1, 1, 1), sigma=500.0, rgb=0.5)
    rgb, tfg, _, _, _, _ = msi().render_rays_with_background(
        g, _bg(sigma=5.0, rgb=(1.0, 0.0, 0.0)), np.array([[-0.9, 0.05, 0.0]]),
        np.array([[1.0, 0.0, 0.0]]))
    assert tfg[0] < 1e-6 and rgb[0, 0] - rgb[0, 1] < 1e-6


@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_composite_gradients_match_finite_differences(interp):
    m = msi()
    rng = np.random.default_rng(5)
    og = orc.Grid.dense((4, 4, 4), (-1, -1, -1), (1, 1, 1))
    og.table[:, 0] = rng.uniform(0.2, 1.5, og.n_rows)
    for ch in range(3):
        og.table[:, 1 + 9 * ch] = rng.uniform(0.5, 1.5, og.n_rows)
    og.table[:] = og.table.astype(np.float32)
    bg = _bg(n_layers=5, h=6, w=8)
    bgd = rng.uniform(0.1, 1.0, tuple(bg.data.shape))
    bg.data[:] = torch.as_tensor(bgd)
    rays = [(np.array([0.05, -0.1, 0.08]), np.array([0.6, 0.5, -0.4])),
            (np.array([-0.3, 0.2, 0.1]), np.array([-0.2, 0.9, 0.3]))]
    o = np.array([r[0] for r in rays])
    d = np.array([r[1] / np.linalg.norm(r[1]) for r in rays])
    gt = np.array([[0.2, 0.4, 0.6], [0.7, 0.1, 0.3]])
    lam_c, lam_b = 1e-3, 1e-2
    dg = px().SparseGrid(og.links, og.table.astype(np.float32), og.aabb_min, og.aabb_max)
    grads = px().GradientBuffer(dg.n_rows)
    bgrads = m.BgGradientBuffer(bg)
    m.render_rays_with_background(dg, bg, o, d, px().RenderOptions(stop_thresh=0.0, interp=interp),
                                  gt_rgb=gt, grads=grads, bg_grads=bgrads, n_total=2,
                                  lam_cauchy=lam_c, lam_beta=lam_b)
    radii = m.layer_radii(5)

    def value():   # the objective the gradients belong to, reference (oracle) float64
        _, _, _, mse, craw, braw = orc.render_360(
            og, bgd, radii, o, d, stop_thresh=0.0, interp=interp, gt_rgb=gt,
            buf=orc.GradBuf(og.n_rows), bg_buf=orc.BgGradBuf(bgd.size // 4), n_total=2,
            lam_cauchy=lam_c, lam_beta=lam_b)
        # upstream 2 (C - gt) / n_total is the gradient of mse_sum / n_total
        return mse / 2 + lam_c * craw + lam_b * braw

    h = 1e-4
    dense = grads.dense()
    nz = np.argwhere(dense != 0)
    assert len(nz) > 0
    for row, col in nz[rng.permutation(len(nz))[:60]]:
        old = og.table[row, col]
        og.table[row, col] = old + h
        fp = value()
        og.table[row, col] = old - h
        fm = value()
        og.table[row, col] = old
        assert dense[row, col] == pytest.approx((fp - fm) / (2 * h), rel=2e-4, abs=1e-7)
    flat = bgrads.data.cpu().numpy()
    view = bgd.reshape(-1, 4)
    nzb = np.argwhere(flat != 0)
    assert len(nzb) > 0
    for r, c in nzb[rng.permutation(len(nzb))[:60]]:
        old = view[r, c]
        view[r, c] = old + h
        fp = value()
        view[r, c] = old - h
        fm = value()
        view[r, c] = old
        assert flat[r, c] == pytest.approx((fp - fm) / (2 * h), rel=2e-4, abs=1e-7)


def test_background_tv():
    m = msi()
    bg = _bg(n_layers=3, h=4, w=6, sigma=0.0, rgb=(0, 0, 0))
    bg.data[1, 2, 0, 1] = 1.0                     # a colour step across the phi seam only
    _, tv_rgb = m.bg_tv_loss(bg, np.array([(1 * 4 + 2) * 6 + 5], dtype=np.int64), 0.0, 1.0, eps=0.0)
    assert tv_rgb == pytest.approx(6 / 256.0, rel=1e-12)
    rng = np.random.default_rng(6)
    bg = _bg(n_layers=3, h=4, w=6)
    bgd = rng.uniform(0.0, 1.0, tuple(bg.data.shape))
    bg.data[:] = torch.as_tensor(bgd)
    cells = np.arange(72, dtype=np.int64)
    buf = m.BgGradientBuffer(bg)
    m.bg_tv_loss(bg, cells, 0.9, 1.1, buf)
    dense = buf.data.cpu().numpy()
    view = bgd.reshape(-1, 4)
    h = 1e-5
    for r, c in np.argwhere(dense != 0)[rng.permutation(int((dense != 0).sum()))[:100]]:
        old = view[r, c]
        view[r, c] = old + h
        fp = sum(orc.tv_bg(bgd, cells, 0.9, 1.1))
        view[r, c] = old - h
        fm = sum(orc.tv_bg(bgd, cells, 0.9, 1.1))
        view[r, c] = old
        assert dense[r, c] == pytest.approx((fp - fm) / (2 * h), rel=1e-4, abs=1e-8)
    run = np.asarray(m.sample_bg_tv_cells(_bg(n_layers=4, h=8, w=8), 0.05,
                                          np.random.default_rng(7)))
    assert len(run) == round(0.05 * 256) and np.all((run >= 0) & (run < 256))
