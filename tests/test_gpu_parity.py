"""Parity of the sm_100a path (through libplx.so) against the CPU oracle and
the reference's golden vectors.

Bars (north star): RGB within 1e-4 abs; gradients within 1e-3 rel (+ an abs
floor of 1e-6 * max|g|, f32 atomics); links / prune masks / upsampled index
bit-exact; touched-row sets identical."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

from helpers import golden_grid, grad_close, load, random_grid, ray_batch

pytestmark = pytest.mark.gpu

RGB_TOL = 1e-4
# The colour dot products are f32 FMAs (~3e-7 from float64, far inside
# RGB_TOL); sigma, transmittance and the sample set stay float64-exact, so the
# Cauchy sums keep 1e-9 while the MSE sum carries the colour rounding.
MSE_REL = 1e-6


def px():
    import paper_2112_05131_b200 as px_
    return px_


def dev_grid(g):
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def _opts(z, ci):
    stop, step_frac, nearest, absolute = z[f"c{ci}_opts"][:4]
    return dict(stop_thresh=float(stop), step_frac=float(step_frac),
                interp="nearest" if nearest else "trilinear",
                formula="absolute" if absolute else "relative",
                background=tuple(z[f"c{ci}_bg"]))


@pytest.fixture(params=[True, False], ids=["cellocc", "links"])
def cell_occ(request):
    from paper_2112_05131_b200 import grid as gmod
    old = gmod.USE_CELL_OCC
    gmod.USE_CELL_OCC = request.param
    yield request.param
    gmod.USE_CELL_OCC = old


# ----------------------------------------------------------------- forward --
def test_render_forward_golden(cell_occ):
    z = load("render.npz")
    for ci in range(int(z["n"])):
        g = dev_grid(golden_grid(z, f"c{ci}_"))
        opts = px().RenderOptions(**_opts(z, ci))
        rgb, trans, wsum = px().render_rays(g, z[f"c{ci}_o"], z[f"c{ci}_d"], opts)
        assert np.max(np.abs(rgb - z[f"c{ci}_rgb"])) < RGB_TOL
        assert np.max(np.abs(trans - z[f"c{ci}_trans"])) < RGB_TOL
        assert np.max(np.abs(wsum - z[f"c{ci}_wsum"])) < RGB_TOL


@pytest.mark.parametrize("formula", ["relative", "absolute"])
@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_render_forward_random_vs_oracle(formula, interp, cell_occ):
    rng = np.random.default_rng(100)
    worst = 0.0
    for gi in range(12):
        dims = tuple(int(x) for x in rng.integers(3, 12, 3))
        g = random_grid(rng, dims=dims, holes=float(rng.uniform(0, 0.5)),
                        sigma_range=(-0.5, 6.0))
        o, d = ray_batch(rng, 96)
        kw = dict(step_frac=float(rng.uniform(0.2, 1.0)), stop_thresh=[1e-4, 0.0, 1e-2][gi % 3],
                  background=tuple(rng.uniform(0, 1, 3)), interp=interp, formula=formula)
        want = orc.render_rays(g, o, d, **kw)
        got = px().render_rays(dev_grid(g), o, d, px().RenderOptions(**kw))
        for a, b in zip(got, want):
            worst = max(worst, float(np.max(np.abs(a - b))))
    assert worst < RGB_TOL, worst


def test_toy_render_matches_reference_golden():
    """pkg/tests/test_viewer_fixtures.py:42-53 on the device."""
    import json
    from helpers import GOLDEN

    ref = json.load(open(f"{GOLDEN}/toy_ref.json"))
    grid, _ = px().load_grid(f"{GOLDEN}/{ref['file']}")
    cam = px().Camera(c2w=np.asarray(ref["c2w"]), focal=ref["focal"], width=ref["width"],
                      height=ref["height"])
    opts = px().RenderOptions(step_frac=ref["step_frac"], stop_thresh=ref["stop_thresh"],
                              background=tuple(ref["background"]))
    img = px().render_image(grid, cam, opts)
    golden = np.fromfile(f"{GOLDEN}/toy_render.bin", dtype="<f4").reshape(
        ref["height"], ref["width"], 3)
    assert np.max(np.abs(img - golden)) < 1e-6


# ---------------------------------------------------------------- backward --
def _check_bwd(g, o, d, gt, kw, lam=0.0, upstream=None):
    buf_o = orc.GradBuf(g.n_rows)
    vd = orc.normalize_dirs(d)
    dg = dev_grid(g)
    buf_d = px().GradientBuffer(dg.n_rows)
    opts = px().RenderOptions(**kw)
    if upstream is None:
        rgb_o, mse_o, cau_o = orc.fused_mse_backward(g, o, d, vd, gt, buf_o, len(o),
                                                     lam_cauchy=lam, **kw)
        rgb_d, mse_d, cau_d = px().fused_mse_backward(dg, o, d, vd, gt, buf_d, opts,
                                                      n_total=len(o), lam_cauchy=lam)
        assert mse_d == pytest.approx(mse_o, rel=MSE_REL, abs=1e-12)
    else:
        rgb_o, cau_o = orc.render_rays_backward(g, o, d, upstream, buf_o, lam_cauchy=lam, **kw)
        rgb_d, cau_d = px().render_rays_backward(dg, o, d, upstream, buf_d, opts,
                                                 lam_cauchy=lam)
    assert np.max(np.abs(rgb_d - rgb_o)) < RGB_TOL
    assert cau_d == pytest.approx(cau_o, rel=1e-9, abs=1e-12)
    np.testing.assert_array_equal(buf_d.touched_rows(), buf_o.touched_rows())
    assert buf_d.n_touched == buf_o.n_touched
    ok, worst, nbad = grad_close(buf_d.dense(), buf_o.data)
    assert ok, (worst, nbad)
    return buf_d, buf_o


def test_fused_backward_golden(cell_occ):
    z = load("backward.npz")
    for ci in range(int(z["n"])):
        g = golden_grid(z, f"c{ci}_")
        dg = dev_grid(g)
        o, d = z[f"c{ci}_o"], z[f"c{ci}_d"]
        kw = _opts(z, ci)
        lam = float(z[f"c{ci}_opts"][4])
        buf = px().GradientBuffer(dg.n_rows)
        rgb, mse, cau = px().fused_mse_backward(dg, o, d, orc.normalize_dirs(d), z[f"c{ci}_gt"],
                                                buf, px().RenderOptions(**kw), n_total=len(o),
                                                lam_cauchy=lam)
        assert np.max(np.abs(rgb - z[f"c{ci}_rgb"])) < RGB_TOL
        assert mse == pytest.approx(z[f"c{ci}_sums"][0], rel=MSE_REL)
        assert cau == pytest.approx(z[f"c{ci}_sums"][1], rel=1e-9, abs=1e-15)
        np.testing.assert_array_equal(buf.touched_rows(), z[f"c{ci}_touched"])
        ok, worst, nbad = grad_close(buf.dense(), z[f"c{ci}_grad"])
        assert ok, (ci, worst, nbad)


@pytest.mark.parametrize("formula", ["relative", "absolute"])
@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_fused_backward_random_vs_oracle(formula, interp, cell_occ):
    rng = np.random.default_rng(200)
    for gi in range(8):
        dims = tuple(int(x) for x in rng.integers(3, 12, 3))
        sr = (-0.5, 4.0) if formula == "relative" else (-0.1, 0.8)
        g = random_grid(rng, dims=dims, holes=float(rng.uniform(0, 0.4)), sigma_range=sr)
        o, d = ray_batch(rng, 64)
        gt = rng.uniform(0, 1, (64, 3))
        kw = dict(stop_thresh=[1e-4, 0.0, 1e-3][gi % 3], background=tuple(rng.uniform(0, 1, 3)),
                  interp=interp, formula=formula)
        _check_bwd(g, o, d, gt, kw, lam=1e-3 if gi % 2 else 0.0)


def test_upstream_mode_vs_oracle():
    rng = np.random.default_rng(201)
    g = random_grid(rng, dims=(7, 6, 9), holes=0.2)
    o, d = ray_batch(rng, 40)
    up = rng.normal(size=(40, 3))
    _check_bwd(g, o, d, None, dict(stop_thresh=0.0, background=(0.3, 0.6, 0.1)), lam=0.0,
               upstream=up)


def test_backward_linear_in_upstream():
    """pkg/tests/test_render.py:247-255 (size-independent property)."""
    rng = np.random.default_rng(7)
    g = dev_grid(random_grid(rng, dims=(9, 9, 9)))
    o, d = ray_batch(rng, 32)
    up = rng.normal(size=(32, 3))
    opts = px().RenderOptions(stop_thresh=0.0)
    b1 = px().GradientBuffer(g.n_rows)
    px().render_rays_backward(g, o, d, up, b1, opts)
    b2 = px().GradientBuffer(g.n_rows)
    px().render_rays_backward(g, o, d, 2.5 * up, b2, opts)
    ok, worst, _ = grad_close(b2.dense(), 2.5 * b1.dense(), rel=1e-5)
    assert ok, worst


# ---------------------------------------------------------------------- TV --
def test_tv_golden():
    z = load("tv.npz")
    for ci in range(int(z["n"])):
        g = dev_grid(golden_grid(z, f"c{ci}_"))
        buf = px().GradientBuffer(g.n_rows)
        a, b = px().tv_loss(g, z[f"c{ci}_cells"], 0.7, 1.3, buf, eps=float(z[f"c{ci}_eps"][0]))
        assert a == pytest.approx(z[f"c{ci}_loss"][0], rel=1e-9)
        assert b == pytest.approx(z[f"c{ci}_loss"][1], rel=1e-9)
        np.testing.assert_array_equal(buf.touched_rows(), z[f"c{ci}_touched"])
        ok, worst, nbad = grad_close(buf.dense(), z[f"c{ci}_grad"])
        assert ok, (ci, worst, nbad)


def test_tv_contiguous_run_matches_oracle():
    rng = np.random.default_rng(300)
    g = random_grid(rng, dims=(13, 11, 17), holes=0.3, sigma_range=(-1, 1), dc_range=(-1, 1),
                    band_scale=0.8)
    dg = dev_grid(g)
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    cells_o = orc.sample_tv_cells(g.dims, 0.2, r1)
    run = px().sample_tv_cells(dg, 0.2, r2)
    np.testing.assert_array_equal(np.asarray(run), cells_o)
    bo = orc.GradBuf(g.n_rows)
    a0, b0 = orc.tv_loss(g, cells_o, 1e-5, 1e-3, bo)
    bd = px().GradientBuffer(dg.n_rows)
    a1, b1 = px().tv_loss(dg, run, 1e-5, 1e-3, bd)
    assert a1 == pytest.approx(a0, rel=1e-9) and b1 == pytest.approx(b0, rel=1e-9)
    np.testing.assert_array_equal(bd.touched_rows(), bo.touched_rows())
    ok, worst, _ = grad_close(bd.dense(), bo.data)
    assert ok, worst


# --------------------------------------------------------------- optimiser --
def test_opt_step_golden():
    z = load("optim.npz")
    lr_s, lr_c = (float(x) for x in z["lr"])
    for ci, method in enumerate(("rmsprop", "sgd")):
        t0 = z[f"c{ci}_table"]
        g = px().SparseGrid(np.arange(t0.shape[0], dtype=np.int32).reshape(4, 4, 4),
                            t0.astype(np.float32), (0, 0, 0), (1, 1, 1))
        st = px().OptimState(t0.shape[0])
        st.v.copy_(torch.as_tensor(z[f"c{ci}_v"], dtype=torch.float32))
        buf = px().GradientBuffer(t0.shape[0])
        buf.data.copy_(torch.as_tensor(z[f"c{ci}_grad"], dtype=torch.float32))
        buf.touched_mask[torch.as_tensor(z[f"c{ci}_touched"]).cuda()] = 1
        from paper_2112_05131_b200 import optim
        optim.step(g, buf, st, lr_s, lr_c, method)
        want_t = z[f"c{ci}_table_out"]
        got_t = g.table.double().cpu().numpy()
        # f32 storage: within 2 ulp of the reference's float64 result
        np.testing.assert_allclose(got_t, want_t, rtol=3e-7, atol=1e-12)
        if method == "rmsprop":
            np.testing.assert_allclose(st.v.double().cpu().numpy(), z[f"c{ci}_v_out"],
                                       rtol=3e-7, atol=1e-30)
        assert buf.n_touched == len(z[f"c{ci}_touched"])
        buf.clear()
        assert buf.n_touched == 0 and float(buf.data.abs().sum()) == 0.0


@pytest.mark.parametrize("method", ["rmsprop", "sgd"])
def test_opt_step_bitwise_after_f32_rounding(method):
    """The kernel's float64 update (MUFU-seeded Newton root/quotient, no IEEE
    div/sqrt subroutines) rounded to f32 equals the oracle's float64 result
    (K:572-590) rounded to f32 on ~1.8 M values spanning 12 decades; only
    f32 rounding ties may differ."""
    rng = np.random.default_rng(11)
    n = 64000
    t0 = rng.normal(size=(n, 28)).astype(np.float32).astype(np.float64)
    v0 = (10.0 ** rng.uniform(-12, 0, (n, 28))).astype(np.float32).astype(np.float64)
    gr = (rng.normal(size=(n, 28)) * 10.0 ** rng.uniform(-6, 2, (n, 28)))
    gr[rng.random((n, 28)) < 0.1] = 0.0       # stale-state entries (g == 0)
    gr = gr.astype(np.float32).astype(np.float64)
    touched = np.sort(rng.permutation(n)[: n // 2])
    gr[np.setdiff1d(np.arange(n), touched)] = 0.0
    g = px().SparseGrid(np.arange(n, dtype=np.int32).reshape(40, 40, 40), t0.astype(np.float32),
                        (0, 0, 0), (1, 1, 1))
    st = px().OptimState(n)
    st.v.copy_(torch.as_tensor(v0, dtype=torch.float32))
    buf = px().GradientBuffer(n)
    buf.data.copy_(torch.as_tensor(gr, dtype=torch.float32))
    buf.touched_mask[torch.as_tensor(touched).cuda()] = 1
    from paper_2112_05131_b200 import optim
    optim.step(g, buf, st, 30.0, 0.01, method)
    og = orc.Grid(np.arange(n, dtype=np.int32).reshape(40, 40, 40), t0.copy(), (0, 0, 0),
                  (1, 1, 1))
    ob = orc.GradBuf(n)
    ob.data[:] = gr
    ob.touched_ids[: len(touched)] = touched
    ob._count[0] = len(touched)
    vo = v0.copy()
    orc.opt_step(og, ob, vo, 30.0, 0.01, method)
    got = g.table.cpu().numpy()
    want = og.table.astype(np.float32)
    assert np.count_nonzero(got != want) <= 4, np.count_nonzero(got != want)
    if method == "rmsprop":
        assert np.count_nonzero(st.v.cpu().numpy() != vo.astype(np.float32)) == 0


def test_opt_step_fused_clear_counts():
    rng = np.random.default_rng(3)
    g = px().SparseGrid.dense((6, 7, 8), (0, 0, 0), (1, 1, 1), sigma=0.3, rgb=0.2)
    buf = px().GradientBuffer(g.n_rows)
    rows = rng.permutation(g.n_rows)[:57]
    for r in rows:
        buf.add(int(r), rng.normal(size=28))
    st = px().OptimState(g.n_rows)
    from paper_2112_05131_b200 import optim
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    optim.step(g, buf, st, 0.1, 0.01, clear=True, count_out=cnt)
    assert int(cnt.item()) == 57
    assert buf.n_touched == 0 and float(buf.data.abs().sum()) == 0.0


# -------------------------------------------------------------- max weight --
def test_max_weight_golden(cell_occ):
    z = load("maxw.npz")
    for ci, interp in enumerate(("trilinear", "nearest")):
        g = dev_grid(golden_grid(z, f"c{ci}_"))
        w = g.max_weight_accumulate(z[f"c{ci}_o"], z[f"c{ci}_d"], interp=interp)
        np.testing.assert_allclose(w, z[f"c{ci}_w"], rtol=1e-12, atol=1e-15)


# --------------------------------------------------------------- structure --
def test_prune_golden_bit_exact():
    z = load("structure.npz")
    g = dev_grid(golden_grid(z, "pd_"))
    p, kept = g.prune("density", float(z["pd_thr"][0]))
    np.testing.assert_array_equal(p.links.cpu().numpy(), z["pd_links_out"])
    np.testing.assert_array_equal(kept.cpu().numpy(), z["pd_kept"])
    np.testing.assert_array_equal(p.table.cpu().numpy(), g.table.cpu().numpy()[z["pd_kept"]])
    g = dev_grid(golden_grid(z, "pw_"))
    p, kept = g.prune("weight", float(z["pw_thr"][0]), z["pw_w"])
    np.testing.assert_array_equal(p.links.cpu().numpy(), z["pw_links_out"])
    np.testing.assert_array_equal(kept.cpu().numpy(), z["pw_kept"])
    p.validate()


def test_prune_random_vs_oracle_and_edge_cases():
    rng = np.random.default_rng(400)
    for _ in range(6):
        dims = tuple(int(x) for x in rng.integers(2, 20, 3))
        g = random_grid(rng, dims=dims, holes=float(rng.uniform(0, 0.7)), sigma_range=(0, 4))
        thr = float(rng.uniform(0, 4))
        po, ko = orc.prune(g, "density", thr)
        pd, kd = dev_grid(g).prune("density", thr)
        np.testing.assert_array_equal(pd.links.cpu().numpy(), po.links)
        np.testing.assert_array_equal(kd.cpu().numpy(), ko)
    # everything below threshold -> empty grid (test_grid.py:177-182)
    g = px().SparseGrid.dense((4, 4, 4), (0, 0, 0), (1, 1, 1), sigma=0.5)
    p, k = g.prune("density", 1.0)
    assert p.n_rows == 0 and k.numel() == 0
    p.validate()


def test_upsample_golden_bit_exact_links():
    z = load("structure.npz")
    g = dev_grid(golden_grid(z, "up_"))
    for ti in range(int(z["n_up"])):
        u = g.upsample(tuple(int(x) for x in z[f"up{ti}_dims"]))
        np.testing.assert_array_equal(u.links.cpu().numpy(), z[f"up{ti}_links"])
        want = z[f"up{ti}_table"]
        np.testing.assert_allclose(u.table.double().cpu().numpy(), want, rtol=2e-7,
                                   atol=1e-6 * np.abs(want).max())
        u.validate()


def test_upsample_random_vs_oracle():
    rng = np.random.default_rng(500)
    for _ in range(5):
        dims = tuple(int(x) for x in rng.integers(2, 12, 3))
        g = random_grid(rng, dims=dims, holes=float(rng.uniform(0, 0.8)))
        nd = tuple(int(x) for x in rng.integers(2, 30, 3))
        uo = orc.upsample(g, nd)
        ud = dev_grid(g).upsample(nd)
        np.testing.assert_array_equal(ud.links.cpu().numpy(), uo.links)


def test_upsample_empty_grid_is_graceful():
    g = px().SparseGrid.empty((4, 4, 4), (0, 0, 0), (1, 1, 1))
    u = g.upsample((8, 8, 8))
    assert u.n_rows == 0 and u.dims == (8, 8, 8)


@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_fused_backward_long_rays_vs_oracle(interp):
    """Rays of several hundred positions (many 32-position chunks, face, edge
    and corner crossings, holes) through a 40^3 grid: exercises the scatter
    accumulator's carried state across chunks against the oracle."""
    rng = np.random.default_rng(300)
    g = random_grid(rng, dims=(40, 37, 43), holes=0.3, sigma_range=(-0.3, 0.6))
    o, d = ray_batch(rng, 200)
    gt = rng.uniform(0, 1, (200, 3))
    _check_bwd(g, o, d, gt, dict(step_frac=0.37, stop_thresh=1e-4,
                                 background=(0.2, 0.5, 0.9), interp=interp), lam=1e-4)


def test_lattice_sigma_mirror_tracks_optimiser():
    """sigma_lat (the lattice-indexed density mirror, NaN at empty points) is
    kept current by the optimiser, equals a from-scratch rebuild bit for bit,
    and the march reading corner sigmas from it renders exactly like the
    march through links -> density."""
    from paper_2112_05131_b200 import optim
    rng = np.random.default_rng(17)
    g = dev_grid(random_grid(rng, dims=(13, 11, 12), holes=0.25, sigma_range=(-1.0, 1.0)))
    neg, _ = g.lattice_sigma()
    st = px().OptimState(g.n_rows)
    for it in range(4):
        buf = px().GradientBuffer(g.n_rows)
        rows = rng.permutation(g.n_rows)[: g.n_rows // 2]
        buf.data[torch.as_tensor(rows).cuda(), 0] = torch.as_tensor(
            rng.normal(size=len(rows)), dtype=torch.float32).cuda()
        buf.touched_mask[torch.as_tensor(rows).cuda()] = 1
        optim.step(g, buf, st, 0.5, 0.01, clear=True)
        kept = neg.clone()
        g.invalidate()                     # rebuild from scratch into the same buffer
        assert torch.equal(kept.view(torch.int32), neg.view(torch.int32)), it
    o, d = ray_batch(rng, 128)
    with_skip = px().render_rays(g, o, d, px().RenderOptions(stop_thresh=0.0))
    from paper_2112_05131_b200 import grid as gmod
    h = px().SparseGrid(g.links, g.table, g.aabb_min, g.aabb_max)   # fresh: no mirror
    old = gmod.USE_CELL_OCC
    gmod.USE_CELL_OCC = False
    try:
        plain = px().render_rays(h, o, d, px().RenderOptions(stop_thresh=0.0))
    finally:
        gmod.USE_CELL_OCC = old
    for a, b in zip(with_skip, plain):
        np.testing.assert_array_equal(a, b)
