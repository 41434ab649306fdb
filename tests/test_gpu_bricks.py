"""Dead-brick skipping (plx_grid.brick_dead): an 8^3-cell brick none of whose
positions can be composited -- every cell has no occupied corner or 8
occupied corners with sigma < 0, the two exits of _sigma_at before the
weights (K:126-135, K:211, K:293) -- is skipped by the march.  Skipping is
exact: the mask must equal its definition, and every render / backward /
max-weight result with it must equal the result without it, also after an
update revives bricks (a corner's sigma becomes >= 0)."""
import numpy as np
import pytest
import torch

from helpers import ray_batch

pytestmark = pytest.mark.gpu

DIMS = (41, 37, 45)


def _grid(seed=0):
    """Sparse grid: sigma < 0 almost everywhere, a few positive blobs, an
    empty slab, scattered holes in one region (cells mixing empty and
    negative corners are never skippable), and bricks of every kind (dead by
    emptiness, dead by negative sigma, mixed, live)."""
    import paper_2112_05131_b200 as px
    rng = np.random.default_rng(seed)
    D = DIMS
    x, y, z = np.meshgrid(*[np.linspace(-1, 1, d) for d in D], indexing="ij")
    occ = ~((x > 0.55) & (y < -0.3))           # an empty slab
    occ &= ~((rng.random(D) < 0.05) & (x < -0.6))   # scattered holes in one corner region
    links = np.full(D, -1, dtype=np.int32)
    links[occ] = np.arange(int(occ.sum()), dtype=np.int32)
    n = int(occ.sum())
    table = np.zeros((n, 28), dtype=np.float32)
    sig = np.full(D, -1.5)
    for c, r in (((0.3, 0.1, -0.2), 0.25), ((-0.5, -0.4, 0.4), 0.2), ((0.0, 0.6, 0.6), 0.15)):
        d2 = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2
        sig = np.where(d2 < r * r, rng.uniform(0.5, 4.0, D), sig)
    sig[rng.random(D) < 0.001] = 0.0           # a few exact zeros (recorded, K:293)
    table[:, 0] = sig[occ]
    table[:, 1:] = rng.uniform(-0.5, 1.0, (n, 27))
    return px.SparseGrid(torch.from_numpy(links).cuda(), torch.from_numpy(table).cuda(),
                         (-1.0,) * 3, (1.0,) * 3)


def _pair(seed=0):
    a = _grid(seed)
    b = a.copy()
    b.disable_bricks()
    a.lattice_sigma()
    b.lattice_sigma()
    assert a._bricks is not None and b._bricks is None
    return a, b


def _dead_bits_numpy(g):
    D = g.dims
    links = g.links.cpu().numpy()
    dens = g.density.cpu().numpy()
    lat = np.where(links >= 0, dens[np.maximum(links, 0)], np.nan).astype(np.float32)
    corners = [lat[i:D[0] - 1 + i, j:D[1] - 1 + j, k:D[2] - 1 + k]
               for i in (0, 1) for j in (0, 1) for k in (0, 1)]
    all_empty = np.logical_and.reduce([np.isnan(c) for c in corners])
    all_neg = np.logical_and.reduce([c < 0 for c in corners])
    skip = all_empty | all_neg
    nb = [(d - 2) // 8 + 1 for d in D]
    dead = np.ones(nb, dtype=bool)
    for bx in range(nb[0]):
        for by in range(nb[1]):
            for bz in range(nb[2]):
                dead[bx, by, bz] = skip[8 * bx:8 * bx + 8, 8 * by:8 * by + 8, 8 * bz:8 * bz + 8].all()
    return dead.reshape(-1)


def _mask_bits(g):
    w = g._bricks.cpu().numpy().view(np.uint32)
    nb = int(np.prod([(d - 2) // 8 + 1 for d in g.dims]))
    return ((w[np.arange(nb) >> 5] >> (np.arange(nb) & 31)) & 1).astype(bool)


def test_brick_mask_matches_definition():
    a, _ = _pair()
    want = _dead_bits_numpy(a)
    got = _mask_bits(a)
    assert want.any() and not want.all()
    np.testing.assert_array_equal(got, want)


def _compare(a, b, rng, interp="trilinear", formula="relative"):
    import paper_2112_05131_b200 as px
    o, d = ray_batch(rng, 3000)
    vd = d / np.linalg.norm(d, axis=1, keepdims=True)
    gt = rng.uniform(0, 1, (3000, 3))
    opts = px.RenderOptions(interp=interp, formula=formula)
    fa = px.render_rays(a, o, d, opts)
    fb = px.render_rays(b, o, d, opts)
    for x, y in zip(fa, fb):
        np.testing.assert_array_equal(x, y)
    ga, gb = px.GradientBuffer(a.n_rows), px.GradientBuffer(b.n_rows)
    ra, ma, ca = px.fused_mse_backward(a, o, d, vd, gt, ga, opts, n_total=3000, lam_cauchy=1e-3)
    rb, mb, cb = px.fused_mse_backward(b, o, d, vd, gt, gb, opts, n_total=3000, lam_cauchy=1e-3)
    np.testing.assert_array_equal(ra, rb)
    assert ma == pytest.approx(mb, rel=1e-12) and ca == pytest.approx(cb, rel=1e-12)
    np.testing.assert_array_equal(ga.touched_rows(), gb.touched_rows())
    da, db = ga.dense(), gb.dense()
    np.testing.assert_allclose(da, db, rtol=1e-5, atol=1e-7 * float(np.abs(db).max()))
    wa = a.max_weight_accumulate(o, d, interp=interp)
    wb = b.max_weight_accumulate(o, d, interp=interp)
    np.testing.assert_array_equal(wa, wb)
    return ga


@pytest.mark.parametrize("interp,formula", [("trilinear", "relative"), ("nearest", "relative"),
                                            ("trilinear", "absolute")])
def test_brick_skipping_is_exact(interp, formula):
    a, b = _pair()
    _compare(a, b, np.random.default_rng(1), interp, formula)


def test_revived_bricks_stay_exact():
    """An SGD step raises sigma >= 0 at lattice points inside dead bricks:
    the optimiser clears those bricks, and renders still match."""
    import paper_2112_05131_b200 as px
    from paper_2112_05131_b200 import optim
    a, b = _pair(2)
    dead0 = _mask_bits(a)
    D = a.dims
    links = a.links.cpu().numpy()
    nb = [(d - 2) // 8 + 1 for d in D]
    rng = np.random.default_rng(3)
    rows = []
    for bid in rng.permutation(np.flatnonzero(dead0)):   # one occupied point per brick
        bx, by, bz = np.unravel_index(bid, nb)
        pts = np.argwhere(links[8 * bx:8 * bx + 8, 8 * by:8 * by + 8, 8 * bz:8 * bz + 8] >= 0)
        if len(pts):
            p = pts[len(pts) // 2] + (8 * bx, 8 * by, 8 * bz)
            rows.append(int(links[tuple(p)]))
        if len(rows) == 6:
            break
    assert len(rows) == 6
    for g in (a, b):
        buf = px.GradientBuffer(g.n_rows)
        buf.data[rows, 0] = -10.0      # sigma -1.5 -> 8.5 under SGD with lr 1
        buf.touched_mask[rows] = 1
        st = optim.OptimState(g.n_rows)
        optim.step(g, buf, st, 1.0, 0.0, "sgd", clear=True)
    torch.cuda.synchronize()
    dead1 = _mask_bits(a)
    assert dead1.sum() < dead0.sum()
    assert not (dead1 & ~dead0).any()                # only clears
    assert not (dead1 & ~_dead_bits_numpy(a)).any()  # conservative
    _compare(a, b, np.random.default_rng(4))
    a.rebuild_bricks()                                # re-tightened = the definition
    np.testing.assert_array_equal(_mask_bits(a), _dead_bits_numpy(a))


def test_density_edit_rebuilds_bricks():
    a, b = _pair(5)
    t = a.table
    t[:, 0] = -2.0
    a.table = t
    b.table = t
    assert _mask_bits(a).sum() > 0
    np.testing.assert_array_equal(_mask_bits(a), _dead_bits_numpy(a))
    _compare(a, b, np.random.default_rng(6))


def test_trainer_steps_with_bricks_match(monkeypatch):
    """The trainer's graph step on a sparse grid: same loss trajectory with
    and without the mask (f32 atomic order aside), the mask rebuilt on its
    period."""
    from paper_2112_05131_b200 import grid as gmod, optim, scenes, trainer
    monkeypatch.setattr(trainer, "BRICK_REBUILD_EVERY", 4)
    train, _, _ = scenes.make_toy_dataset(n_views=4, res=48, n_test=1, grid_dim=16)
    out = []
    for use in (True, False):
        cfg = trainer.toy_config(grid_dim=16, total_steps=20, batch_size=2000)
        tr = trainer.Trainer(train, cfg)
        tr.grid = _grid(7)
        if not use:
            tr.grid.disable_bricks()
        tr.state = optim.OptimState(tr.grid.n_rows)
        tr.grads = gmod.GradientBuffer(tr.grid.n_rows)
        tr._refresh_cache()
        losses = [tr.step(s, sync=True)["loss"] for s in range(trainer.BRICK_REBUILD_EVERY + 3)]
        out.append(np.array(losses))
        assert (tr.grid._bricks is not None) == use
    np.testing.assert_allclose(out[0], out[1], rtol=1e-3)


def test_random_grids_bit_identical():
    """scripts/stress_bricks.py on 6 random grids (odd dims, hole slabs,
    negative regions, exact zeros, blobs; rays inside / outside / axis-aligned,
    jitter): every result with the mask equals the result without it."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts",
                        "stress_bricks.py")
    spec = importlib.util.spec_from_file_location("stress_bricks", path)
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert m.main(6) == 0
