"""Pin the oracle's multi-sphere-image (360) restatement to the reference:
render_rays_with_background forward + backward (K:661-881), sample_background
(msi.py:75-108), bg_tv_loss (K:884-977) and step_table (O:100-107) on the
golden cases of tests/golden/make_msi_golden.py.  Bit-for-bit: the oracle
keeps the reference's operation order and libm calls."""

import numpy as np

from oracle import oracle as orc

from helpers import golden_grid, load


def _case(z, ci):
    p = f"c{ci}_"
    nearest, lam_c, lam_b, stop = z[p + "opts"]
    return p, dict(interp="nearest" if nearest else "trilinear", stop_thresh=float(stop)), \
        float(lam_c), float(lam_b)


def test_render_360_forward_matches_reference():
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p, opts, _, _ = _case(z, ci)
        g = golden_grid(z, p)
        rgb, tfg, trans, _, _, _ = orc.render_360(g, z[p + "bg"], z[p + "radii"], z[p + "o"],
                                                  z[p + "d"], **opts)
        np.testing.assert_array_equal(rgb, z[p + "rgb"])
        np.testing.assert_array_equal(tfg, z[p + "tfg"])
        np.testing.assert_array_equal(trans, z[p + "trans"])


def test_render_360_backward_matches_reference():
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p, opts, lam_c, lam_b = _case(z, ci)
        g = golden_grid(z, p)
        L, H, W, _ = z[p + "bg"].shape
        buf, bgb = orc.GradBuf(g.n_rows), orc.BgGradBuf(L * H * W)
        rgb, _, _, mse, craw, braw = orc.render_360(
            g, z[p + "bg"], z[p + "radii"], z[p + "o"], z[p + "d"], gt_rgb=z[p + "gt"],
            buf=buf, bg_buf=bgb, n_total=len(z[p + "o"]), lam_cauchy=lam_c, lam_beta=lam_b,
            **opts)
        np.testing.assert_array_equal(rgb, z[p + "rgb"])
        np.testing.assert_array_equal(np.array([mse, craw, braw]), z[p + "sums"])
        np.testing.assert_array_equal(buf.data, z[p + "grad"])
        np.testing.assert_array_equal(buf.touched_rows(), z[p + "touched"])
        np.testing.assert_array_equal(bgb.data, z[p + "bg_grad"])
        np.testing.assert_array_equal(bgb.touched_rows(), z[p + "bg_touched"])


def test_sample_background_matches_reference():
    """sample_background is numpy (vectorised arctan2 / arccos, which may
    differ from libm in the last ulp): 1e-14 relative."""
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p = f"c{ci}_"
        sig, rgb = orc.bg_sample(z[p + "bg"], z[p + "pts"])
        np.testing.assert_allclose(sig, z[p + "s_sig"], rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(rgb, z[p + "s_rgb"], rtol=1e-14, atol=1e-15)


def test_bg_tv_and_step_table_match_reference():
    z = load("msi.npz")
    for ci in range(int(z["n"])):
        p = f"c{ci}_"
        L, H, W, _ = z[p + "bg"].shape
        b = orc.BgGradBuf(L * H * W)
        tv = orc.tv_bg(z[p + "bg"], z[p + "tv_cells"], 0.9, 1.1, b)
        np.testing.assert_array_equal(np.array(tv), z[p + "tv"])
        np.testing.assert_array_equal(b.data, z[p + "tv_grad"])
        np.testing.assert_array_equal(b.touched_rows(), z[p + "tv_touched"])
        table = z[p + "bg"].reshape(-1, 4).copy()
        v = z[p + "opt_v0"].copy()
        ids = z[p + "opt_ids"]
        orc.step_table(table, z[p + "opt_grad"], ids, len(ids), v, 0.5, 0.1)
        np.testing.assert_array_equal(table, z[p + "opt_table"])
        np.testing.assert_array_equal(v, z[p + "opt_v"])
