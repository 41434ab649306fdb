"""Pin the CPU oracle (oracle/plx_oracle.c) to the reference's own outputs.

The golden vectors were produced by running the reference package
(/root/reference/pkg/src/plenoxel, numba kernels) -- see
tests/golden/make_golden.py.  The oracle must reproduce them bit-for-bit
(or to 1e-12 where the reference's numpy einsum order is unspecified)."""

import json
import zlib

import numpy as np
import pytest

from oracle import oracle as orc

from helpers import GOLDEN, golden_grid, load


def _opts(z, ci):
    stop, step_frac, nearest, absolute = z[f"c{ci}_opts"][:4]
    return dict(stop_thresh=float(stop), step_frac=float(step_frac),
                interp="nearest" if nearest else "trilinear",
                formula="absolute" if absolute else "relative",
                background=z[f"c{ci}_bg"])


def test_render_forward_matches_reference():
    z = load("render.npz")
    for ci in range(int(z["n"])):
        g = golden_grid(z, f"c{ci}_")
        rgb, trans, wsum = orc.render_rays(g, z[f"c{ci}_o"], z[f"c{ci}_d"], **_opts(z, ci))
        np.testing.assert_array_equal(rgb, z[f"c{ci}_rgb"])
        np.testing.assert_array_equal(trans, z[f"c{ci}_trans"])
        np.testing.assert_array_equal(wsum, z[f"c{ci}_wsum"])


def test_fused_backward_matches_reference():
    z = load("backward.npz")
    for ci in range(int(z["n"])):
        g = golden_grid(z, f"c{ci}_")
        o, d = z[f"c{ci}_o"], z[f"c{ci}_d"]
        buf = orc.GradBuf(g.n_rows)
        opts = _opts(z, ci)
        lam = float(z[f"c{ci}_opts"][4])
        rgb, mse, cauchy = orc.fused_mse_backward(g, o, d, orc.normalize_dirs(d),
                                                  z[f"c{ci}_gt"], buf, len(o),
                                                  lam_cauchy=lam, **opts)
        np.testing.assert_array_equal(rgb, z[f"c{ci}_rgb"])
        assert mse == z[f"c{ci}_sums"][0]
        assert cauchy == z[f"c{ci}_sums"][1]
        np.testing.assert_array_equal(buf.data, z[f"c{ci}_grad"])
        np.testing.assert_array_equal(buf.touched_rows(), z[f"c{ci}_touched"])
    # upstream mode, render_rays_backward (R:205-239)
    g = golden_grid(z, "c4_")
    buf = orc.GradBuf(g.n_rows)
    rgb, cs = orc.render_rays_backward(g, z["c4_o"], z["c4_d"], z["up_up"], buf,
                                       lam_cauchy=float(z["c4_opts"][4]), **_opts(z, 4))
    np.testing.assert_array_equal(rgb, z["up_rgb"])
    assert cs == z["up_cauchy"][0]
    np.testing.assert_array_equal(buf.data, z["up_grad"])
    np.testing.assert_array_equal(buf.touched_rows(), z["up_touched"])


def test_tv_matches_reference():
    z = load("tv.npz")
    for ci in range(int(z["n"])):
        g = golden_grid(z, f"c{ci}_")
        buf = orc.GradBuf(g.n_rows)
        a, b = orc.tv_loss(g, z[f"c{ci}_cells"], 0.7, 1.3, buf, eps=float(z[f"c{ci}_eps"][0]))
        assert (a, b) == tuple(z[f"c{ci}_loss"])
        np.testing.assert_array_equal(buf.data, z[f"c{ci}_grad"])
        np.testing.assert_array_equal(buf.touched_rows(), z[f"c{ci}_touched"])


def test_opt_step_matches_reference():
    z = load("optim.npz")
    lr_s, lr_c = z["lr"]
    for ci, method in enumerate(("rmsprop", "sgd")):
        table = z[f"c{ci}_table"].copy()
        g = orc.Grid(np.arange(table.shape[0], dtype=np.int32).reshape(4, 4, 4), table,
                     (0, 0, 0), (1, 1, 1))
        v = z[f"c{ci}_v"].copy()
        buf = orc.GradBuf(table.shape[0])
        buf.data[:] = z[f"c{ci}_grad"]
        t = z[f"c{ci}_touched"]
        buf.touched_ids[: len(t)] = t
        buf.touched_mask[t] = 1
        buf._count[0] = len(t)
        orc.opt_step(g, buf, v, lr_s, lr_c, method)
        np.testing.assert_array_equal(g.table, z[f"c{ci}_table_out"])
        np.testing.assert_array_equal(v, z[f"c{ci}_v_out"])
        buf.clear()
        assert buf.n_touched == 0 and not buf.data.any() and not buf.touched_mask.any()


def test_max_weight_matches_reference():
    z = load("maxw.npz")
    for ci, interp in enumerate(("trilinear", "nearest")):
        g = golden_grid(z, f"c{ci}_")
        w = orc.max_weight_accumulate(g, z[f"c{ci}_o"], z[f"c{ci}_d"], interp=interp)
        np.testing.assert_array_equal(w, z[f"c{ci}_w"])


def test_prune_matches_reference():
    z = load("structure.npz")
    g = golden_grid(z, "pd_")
    p, kept = orc.prune(g, "density", float(z["pd_thr"][0]))
    np.testing.assert_array_equal(p.links, z["pd_links_out"])
    np.testing.assert_array_equal(kept, z["pd_kept"])
    np.testing.assert_array_equal(p.table, g.table[kept])
    g = golden_grid(z, "pw_")
    p, kept = orc.prune(g, "weight", float(z["pw_thr"][0]), z["pw_w"])
    np.testing.assert_array_equal(p.links, z["pw_links_out"])
    np.testing.assert_array_equal(kept, z["pw_kept"])


def test_prune_lone_voxel_keeps_27():
    """pkg/tests/test_grid.py:185-193."""
    g = orc.Grid.dense((5, 5, 5), (0, 0, 0), (1, 1, 1), sigma=0.0)
    g.table[g.links[2, 2, 2], 0] = 10.0
    p, _ = orc.prune(g, "density", 1.0)
    assert p.n_rows == 27 and (p.links[1:4, 1:4, 1:4] >= 0).all()


def test_upsample_matches_reference():
    z = load("structure.npz")
    g = golden_grid(z, "up_")
    for ti in range(int(z["n_up"])):
        u = orc.upsample(g, tuple(z[f"up{ti}_dims"]))
        np.testing.assert_array_equal(u.links, z[f"up{ti}_links"])
        np.testing.assert_allclose(u.table, z[f"up{ti}_table"], rtol=1e-12, atol=1e-13)


def test_toy_render_golden():
    """pkg/tests/test_viewer_fixtures.py:42-53 through the oracle."""
    from paper_2112_05131_b200 import artifact_io

    ref = json.load(open(f"{GOLDEN}/toy_ref.json"))
    links, table, lo, hi = artifact_io.read_plnx(f"{GOLDEN}/{ref['file']}")
    g = orc.Grid(links, table.astype(np.float64), lo, hi)
    o, d = orc.generate_rays(np.asarray(ref["c2w"]), ref["focal"], ref["width"], ref["height"])
    rgb, _, _ = orc.render_rays(g, o, d, step_frac=ref["step_frac"],
                                stop_thresh=ref["stop_thresh"],
                                background=ref["background"])
    golden = np.fromfile(f"{GOLDEN}/toy_render.bin", dtype="<f4").reshape(-1, 3)
    assert np.max(np.abs(rgb - golden)) < 1e-6


@pytest.mark.parametrize("i", range(10))
def test_plnx_writer_crc_matches_reference_golden(i):
    """g00i.plnx round trip: our reader + writer reproduce the reference's bytes,
    whose CRC32 is pinned by pkg/frontend/test/fixtures/golden.json."""
    from paper_2112_05131_b200 import artifact_io

    gold = json.load(open(f"{GOLDEN}/plnx_golden.json"))[i]
    raw = open(f"{GOLDEN}/plnx/{gold['file']}", "rb").read()
    assert len(raw) == gold["size"]
    assert zlib.crc32(raw[:-4]) & 0xFFFFFFFF == gold["crc32"]
    if gold["has_background"]:
        return
    links, table, lo, hi = artifact_io.read_plnx(f"{GOLDEN}/plnx/{gold['file']}")
    assert artifact_io.plnx_bytes(links, table, lo, hi) == raw


def test_to_ndc_matches_reference():
    """camera.to_ndc (camera.py:103-134) on random rays incl. rays parallel to
    the image plane, against the reference's own output (ndc.npz)."""
    z = load("ndc.npz")
    w, h = (int(x) for x in z["cam_wh"])
    on, dn, valid = orc.to_ndc(z["o"], z["d"], float(z["cam_focal"][0]), w, h, near=1.0)
    np.testing.assert_array_equal(valid, z["valid"])
    np.testing.assert_array_equal(on, z["on"])
    np.testing.assert_array_equal(dn, z["dn"])


def test_oracle_generate_rays_matches_reference():
    """camera.py:91-100 restated (oracle_generate_rays) bit-for-bit, all
    pixels and a scattered pixel subset."""
    z = load("camera.npz")
    k = 0
    while f"cam{k}_c2w" in z:
        w, h = (int(x) for x in z[f"cam{k}_wh"])
        c2w, f = z[f"cam{k}_c2w"], float(z[f"cam{k}_focal"])
        o, d = orc.generate_rays(c2w, f, w, h)
        np.testing.assert_array_equal(d, z[f"cam{k}_d"])
        assert np.all(o == c2w[:3, 3])
        pix = np.random.default_rng(k).integers(0, w * h, 97)
        _, ds = orc.generate_rays(c2w, f, w, h, pixels=pix)
        np.testing.assert_array_equal(ds, z[f"cam{k}_d"][pix])
        k += 1
    assert k >= 6


def test_oracle_to_ndc_matches_reference():
    """camera.py:103-134 restated (oracle_to_ndc) bit-for-bit, incl. all_rays'
    forward-facing pool (camera.py:292-314)."""
    z = load("camera.npz")
    for k in range(3):
        w, h = (int(x) for x in z[f"ndc{k}_wh"])
        c2w, f = z[f"ndc{k}_c2w"], float(z[f"ndc{k}_focal"])
        o, d = orc.generate_rays(c2w, f, w, h)
        on, dn, valid = orc.to_ndc(o, d, f, w, h, float(z[f"ndc{k}_near"]))
        np.testing.assert_array_equal(on, z[f"ndc{k}_o"])
        np.testing.assert_array_equal(dn, z[f"ndc{k}_d"])
        np.testing.assert_array_equal(valid, z[f"ndc{k}_valid"])
    np.testing.assert_array_equal(z["ff_o"], z["ndc0_o"])
    np.testing.assert_array_equal(z["ff_d"], z["ndc0_d"])
