"""Device parity of the multi-sphere-image (360) path: plx_msi_render /
plx_msi_tv / plx_msi_opt_step through paper_2112_05131_b200.msi against the
REFERENCE's outputs on the golden cases (tests/golden/make_msi_golden.py;
the oracle reproduces them bit-for-bit, tests/test_oracle_msi.py), plus the
reference's own behavioural tests (pkg/tests/test_msi.py) restated.

Tolerances: positions, stencils, sigma, the sample set and the crossings are
f64 as in the reference; colours are f32 FMAs (<= 3e-7 relative);
transmittance is a warp product scan (~1e-15 per sample) and device
atan2 / acos are within 2 ulp; grid gradients accumulate with f32 atomics
(1e-3 relative, helpers.grad_close), background gradients with f64 atomics."""

import numpy as np
import pytest
import torch

from helpers import golden_grid, grad_close, load

pytestmark = pytest.mark.gpu


def _px():
    import paper_2112_05131_b200 as px
    return px


def _dev_grid(z, p):
    g = golden_grid(z, p)
    return _px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def _case(z, ci):
    from paper_2112_05131_b200.render import RenderOptions
    p = f"c{ci}_"
    nearest, lam_c, lam_b, stop = z[p + "opts"]
    opts = RenderOptions(background=(0.0, 0.0, 0.0), interp="nearest" if nearest else "trilinear",
                         stop_thresh=float(stop))
    return p, opts, float(lam_c), float(lam_b)


def test_msi_forward_matches_reference():
    from paper_2112_05131_b200 import msi
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p, opts, _, _ = _case(z, ci)
        g = _dev_grid(z, p)
        bg = msi.MsiBackground(z[p + "bg"], z[p + "radii"])
        rgb, tfg, trans, _, _, _ = msi.render_rays_with_background(g, bg, z[p + "o"], z[p + "d"],
                                                                   opts)
        np.testing.assert_allclose(rgb, z[p + "rgb"], rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(tfg, z[p + "tfg"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(trans, z[p + "trans"], rtol=1e-9, atol=1e-12)


def test_msi_backward_matches_reference():
    from paper_2112_05131_b200 import msi
    from paper_2112_05131_b200.grid import GradientBuffer
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p, opts, lam_c, lam_b = _case(z, ci)
        g = _dev_grid(z, p)
        bg = msi.MsiBackground(z[p + "bg"], z[p + "radii"])
        grads, bgg = GradientBuffer(g.n_rows), msi.BgGradientBuffer(bg)
        rgb, _, _, mse, craw, braw = msi.render_rays_with_background(
            g, bg, z[p + "o"], z[p + "d"], opts, gt_rgb=z[p + "gt"], grads=grads, bg_grads=bgg,
            n_total=len(z[p + "o"]), lam_cauchy=lam_c, lam_beta=lam_b)
        torch.cuda.synchronize()
        want = z[p + "sums"]
        assert mse == pytest.approx(want[0], rel=1e-6)
        assert craw == pytest.approx(want[1], rel=1e-6, abs=1e-12)
        assert braw == pytest.approx(want[2], rel=1e-9, abs=1e-12)
        np.testing.assert_array_equal(grads.touched_rows(), z[p + "touched"])
        ok, worst, nbad = grad_close(grads.dense(), z[p + "grad"])
        assert ok, (ci, worst, nbad)
        np.testing.assert_array_equal(bgg.touched_rows(), z[p + "bg_touched"])
        # f64 atomics, but the sigma gradients carry the f32 colour rounding
        # through S_i (cancellation in small entries): grad_close at 1e-4
        ok, worst, nbad = grad_close(bgg.data.cpu().numpy(), z[p + "bg_grad"], rel=1e-4)
        assert ok, ("bg", ci, worst, nbad)


def test_msi_tv_and_step_table_match_reference():
    from paper_2112_05131_b200 import msi
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p = f"c{ci}_"
        bg = msi.MsiBackground(z[p + "bg"], z[p + "radii"])
        b = msi.BgGradientBuffer(bg)
        tv = msi.bg_tv_loss(bg, z[p + "tv_cells"], 0.9, 1.1, b)
        np.testing.assert_allclose(np.array(tv), z[p + "tv"], rtol=1e-12)
        np.testing.assert_allclose(b.data.cpu().numpy(), z[p + "tv_grad"], rtol=1e-10,
                                   atol=1e-14)
        np.testing.assert_array_equal(b.touched_rows(), z[p + "tv_touched"])
        # step_table on the merged (render + TV) gradient of the golden case
        g = msi.BgGradientBuffer(bg)
        g.data.copy_(torch.from_numpy(z[p + "opt_grad"]))
        g.touched_mask[torch.from_numpy(z[p + "opt_ids"]).cuda()] = 1
        st = msi.BgOptimState(bg)
        st.v.copy_(torch.from_numpy(z[p + "opt_v0"]))
        msi.step_table(bg, g, st, 0.5, 0.1)
        torch.cuda.synchronize()
        np.testing.assert_allclose(bg.data.reshape(-1, 4).cpu().numpy(), z[p + "opt_table"],
                                   rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(st.v.cpu().numpy(), z[p + "opt_v"], rtol=1e-14, atol=1e-18)
        assert int(g.touched_mask.sum()) == 0 and float(g.data.abs().sum()) == 0.0


# -- the reference's own behavioural tests (pkg/tests/test_msi.py) ----------

def _empty_grid():
    px = _px()
    return px.SparseGrid(np.full((4, 4, 4), -1, dtype=np.int32), np.zeros((0, 28)),
                         (-0.5,) * 3, (0.5,) * 3)


def test_empty_everything_renders_black_with_full_transmittance():
    """test_msi.py:124-132."""
    from paper_2112_05131_b200 import msi
    bg = msi.MsiBackground(np.zeros((4, 4, 8, 4)))
    o = np.zeros((3, 3))
    d = np.eye(3)
    rgb, tfg, trans, _, _, _ = msi.render_rays_with_background(_empty_grid(), bg, o, d)
    np.testing.assert_array_equal(rgb, 0.0)
    np.testing.assert_array_equal(tfg, 1.0)
    np.testing.assert_array_equal(trans, 1.0)


def test_empty_foreground_opaque_inner_layer_hand_value():
    """test_msi.py:135-148: sigma on layer 0 only; the ray from the centre
    crosses layer 0 (radius 1) first, delta = distance to the next sphere."""
    from paper_2112_05131_b200 import msi
    L = 4
    data = np.zeros((L, 4, 8, 4))
    data[0, ..., 0] = 2.0
    data[0, ..., 1:] = (0.2, 0.4, 0.6)
    bg = msi.MsiBackground(data)
    radii = msi.layer_radii(L)
    rgb, tfg, trans, _, _, _ = msi.render_rays_with_background(
        _empty_grid(), bg, np.zeros((1, 3)), np.array([[0.0, 0.6, 0.8]]))
    dlt = radii[1] - radii[0]
    w = 1.0 - np.exp(-2.0 * dlt)
    np.testing.assert_allclose(rgb[0], w * np.array([0.2, 0.4, 0.6]), rtol=1e-12)
    assert tfg[0] == 1.0
    assert trans[0] == pytest.approx(np.exp(-2.0 * dlt), rel=1e-12)


def test_composite_weights_plus_residual_sum_to_one():
    """test_msi.py:163-178: with white colours everywhere the composite
    plus the final transmittance is 1."""
    from paper_2112_05131_b200 import msi
    rng = np.random.default_rng(3)
    px = _px()
    n = 6 ** 3
    table = np.zeros((n, 28))
    table[:, 0] = rng.uniform(0.0, 2.0, n)
    table[:, 1] = table[:, 10] = table[:, 19] = 1.0 / 0.28209479177387814
    g = px.SparseGrid(np.arange(n, dtype=np.int32).reshape(6, 6, 6), table.astype(np.float32),
                      (-0.5,) * 3, (0.5,) * 3)
    data = np.zeros((5, 6, 8, 4))
    data[..., 0] = rng.uniform(0.0, 1.0, (5, 6, 8))
    data[..., 1:] = 1.0
    bg = msi.MsiBackground(data)
    o = np.zeros((16, 3))
    d = rng.normal(size=(16, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    from paper_2112_05131_b200.render import RenderOptions
    rgb, _, trans, _, _, _ = msi.render_rays_with_background(
        g, bg, o, d, RenderOptions(background=(0.0, 0.0, 0.0), stop_thresh=0.0))
    np.testing.assert_allclose(rgb + trans[:, None], 1.0, atol=2e-6)


def test_sample_background_matches_reference_golden():
    from paper_2112_05131_b200 import msi
    z = load("msi.npz")
    p = "c0_"
    bg = msi.MsiBackground(z[p + "bg"], z[p + "radii"])
    sig, rgb = msi.sample_background(bg, z[p + "pts"])
    np.testing.assert_allclose(sig, z[p + "s_sig"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(rgb, z[p + "s_rgb"], rtol=1e-14, atol=1e-15)
