"""The reference's structure-op behaviours (pkg/tests/test_grid.py:132-300:
max-weight, prune, upsample) and camera / SH behaviours (test_camera.py,
test_sh.py) on the device package.  Upsampled values are stored in f32, so
value comparisons that are 1e-12 between the reference's float64 grids are
at f32 resolution here; links, occupancy and row counts are exact."""

import math

import numpy as np
import pytest

from helpers import random_grid, random_hitting_ray

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as m
    return m


def dev(g):
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def set_sigma(g, rows, value):
    t = g.table.cpu().numpy()
    t[rows, 0] = value
    g.table = t


def np_(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def test_max_weight():
    m = px()
    g = m.SparseGrid.dense((4, 4, 4), (-1, -1, -1), (1, 1, 1), sigma=0.0)
    o, d = np.array([[-2.0, 0.0, 0.0]]), np.array([[1.0, 0.0, 0.0]])
    assert np.all(g.max_weight_accumulate(o, d) == 0.0)
    g = m.SparseGrid.dense((5, 5, 5), (-1, -1, -1), (1, 1, 1), sigma=0.0)
    row = int(np_(g.links)[2, 2, 2])
    set_sigma(g, row, 10.0)
    o = np.array([[-3.0, 0.0, 0.0]])
    w = g.max_weight_accumulate(o, d, step_frac=0.5)
    ts, dl = m.march(g, o[0], d[0], 0.5)        # the hand value: max over samples of T (1 - att)
    T, want = 1.0, 0.0
    for t, delta in zip(ts, dl):
        sig, _ = g.sample(o[0] + t * d[0])
        if sig > 0:
            want = max(want, T * (1 - math.exp(-sig * delta)))
            T *= math.exp(-sig * delta)
    assert want > 0 and w[row] == pytest.approx(want, rel=1e-12)
    set_sigma(g, row, 5.0)
    o2 = np.array([[-3.0, 0.0, 0.0], [0.0, 0.0, 3.0]])
    d2 = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -1.0]])
    np.testing.assert_allclose(g.max_weight_accumulate(o2, d2),
                               np.maximum(g.max_weight_accumulate(o2[:1], d2[:1]),
                                          g.max_weight_accumulate(o2[1:], d2[1:])), atol=1e-15)


def test_prune():
    m = px()
    g = m.SparseGrid.dense((4, 4, 4), (0, 0, 0), (1, 1, 1), sigma=0.5)
    pruned, kept = g.prune("density", 1.0)
    assert pruned.n_rows == 0 and len(kept) == 0
    pruned.validate()
    g = m.SparseGrid.dense((5, 5, 5), (0, 0, 0), (1, 1, 1), sigma=0.0)
    set_sigma(g, int(np_(g.links)[2, 2, 2]), 10.0)
    pruned, _ = g.prune("density", 1.0)             # the 26-neighbour dilation
    occ = np_(pruned.occupancy())
    assert pruned.n_rows == 27 and occ[1:4, 1:4, 1:4].all() and occ.sum() == 27
    rng = np.random.default_rng(7)
    g = dev(random_grid(rng, dims=(6, 6, 6), holes=0.3))
    weights = rng.uniform(0, 1, g.n_rows)
    pruned, kept = g.prune("weight", 0.5, weights)
    kept = np_(kept)
    assert pruned.n_rows <= g.n_rows and len(kept) == pruned.n_rows
    pruned.validate()
    np.testing.assert_array_equal(np_(pruned.table), np_(g.table)[kept])


def test_prune_at_the_least_occupied_weight_keeps_renders():
    m = px()
    rng = np.random.default_rng(8)
    g = dev(random_grid(rng, dims=(8, 8, 8), sigma_range=(0.0, 4.0)))
    rays = [random_hitting_ray(rng) for _ in range(64)]
    w = g.max_weight_accumulate(np.array([r[0] for r in rays]), np.array([r[1] for r in rays]))
    pruned, _ = g.prune("weight", w[w > 0].min(), w)
    rng2 = np.random.default_rng(9)
    held = [random_hitting_ray(rng2) for _ in range(64)]
    ho, hd = np.array([r[0] for r in held]), np.array([r[1] for r in held])
    assert np.mean((m.render_rays(g, ho, hd)[0] - m.render_rays(pruned, ho, hd)[0]) ** 2) < 1e-6


def test_upsample():
    m = px()
    rng = np.random.default_rng(10)
    g = dev(random_grid(rng, dims=(5, 5, 5), holes=0.3))
    up = g.upsample(g.dims)                          # identity dims
    np.testing.assert_array_equal(np_(up.links), np_(g.links))
    np.testing.assert_allclose(np_(up.table), np_(g.table), rtol=1e-7, atol=1e-12)
    up.validate()
    c = m.SparseGrid.dense((3, 3, 3), (0, 0, 0), (1, 1, 1), sigma=0.7, rgb=0.4)
    up = c.upsample((7, 5, 9))                        # a constant field stays constant
    assert up.n_rows == 7 * 5 * 9
    np.testing.assert_allclose(np_(up.table), np.broadcast_to(np_(c.table)[0], (315, 28)),
                               rtol=1e-7)
    g = dev(random_grid(rng, dims=(8, 8, 8)))
    up = g.upsample((15, 15, 15))                     # nested refinement: the same field
    pts = rng.uniform(-0.99, 0.99, (100, 3))
    for a, b in zip(g.sample(pts), up.sample(pts)):
        np.testing.assert_allclose(b, a, rtol=1e-6, atol=1e-6)
    up = dev(random_grid(rng, dims=(8, 8, 8)))
    up2 = up.upsample((16, 16, 16))                    # exact at the new lattice points
    up2.validate()
    ijk = np.stack(np.meshgrid(*(np.arange(16),) * 3, indexing="ij"), -1).reshape(-1, 3)
    pts = up2.lattice_to_world(ijk.astype(float))
    for a, b in zip(up.sample(pts), up2.sample(pts)):
        np.testing.assert_allclose(b, a, rtol=1e-6, atol=1e-6)


def test_upsample_occupancy_follows_the_stencil_rule():
    m = px()
    links = np.arange(64, dtype=np.int32).reshape(4, 4, 4)
    links[2:] = -1                                    # occupied: lattice x in {0, 1}
    keep = np.sort(links[links >= 0])
    remap = np.full(64, -1, dtype=np.int64)
    remap[keep] = np.arange(len(keep))
    table = np.zeros((len(keep), 28), dtype=np.float32)
    table[:, 0] = 1.0
    g = m.SparseGrid(np.where(links >= 0, remap[np.maximum(links, 0)], -1).astype(np.int32),
                     table, np.zeros(3), np.ones(3))
    occ = np_(g.upsample((7, 7, 7)).occupancy())
    for i in range(7):                                # nonzero stencil weight on x < 1/3
        assert occ[i].all() if i / 6.0 < 2.0 / 3.0 else not occ[i].any()


def test_camera_rays():
    m = px()
    cam = m.Camera(c2w=np.eye(4), focal=10.0, width=8, height=6)
    r = m.generate_ray(cam, 2, 1)                     # identity pose: ((px+.5-W/2)/f, -(py+.5-H/2)/f, -1)
    want = np.array([(2.5 - 4) / 10, -(1.5 - 3) / 10, -1.0])
    np.testing.assert_allclose(r.direction, want / np.linalg.norm(want), atol=1e-12)
    a, b = m.generate_ray(cam, 0, 2), m.generate_ray(cam, 7, 2)   # mirror pixels
    np.testing.assert_allclose(a.direction * [-1, 1, 1], b.direction, atol=1e-12)
    c2w = np.eye(4)
    c2w[:3, 3] = [1.0, -2.0, 0.5]
    o, d = m.generate_rays(m.Camera(c2w=c2w, focal=10.0, width=8, height=6))
    assert np.all(o == [1.0, -2.0, 0.5])
    np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)
    for bad in (dict(c2w=np.eye(3), focal=1.0, width=2, height=2),
                dict(c2w=np.diag([2.0, 1.0, 1.0, 1.0]), focal=1.0, width=2, height=2),
                dict(c2w=np.eye(4), focal=0.0, width=2, height=2)):
        with pytest.raises(ValueError):
            m.Camera(**bad)


def test_ndc_warp():
    m = px()
    cam = m.Camera(c2w=np.eye(4), focal=20.0, width=16, height=16, near=1.0)
    o, d, ok = m.to_ndc(np.array([0.1, -0.2, 0.0]), np.array([0.05, 0.02, -1.0]), cam)
    assert ok[0] and o[0, 2] == pytest.approx(-1.0, abs=1e-12)     # on the near plane
    # far along the ray the NDC depth approaches +1
    far = o[0] + 1.0 * d[0]
    assert far[2] == pytest.approx(1.0, abs=1e-9)
    _, _, ok = m.to_ndc(np.zeros(3), np.array([1.0, 0.0, 0.0]), cam)
    assert not ok[0]


def test_sh_properties():
    from paper_2112_05131_b200.sh import SH_C0, SH_C1, eval_sh_basis, normalize_dirs, sh_to_rgb
    rng = np.random.default_rng(12)
    dirs = normalize_dirs(rng.normal(size=(40, 3)))
    b = eval_sh_basis(dirs)
    assert np.all(b[:, 0] == SH_C0)
    np.testing.assert_allclose(eval_sh_basis(np.array([0.0, 0.0, 1.0]))[1:4], [0, SH_C1, 0])
    odd = [1, 2, 3]                                   # l = 1 flips sign, l = 2 does not
    np.testing.assert_allclose(eval_sh_basis(-dirs)[:, odd], -b[:, odd], atol=1e-15)
    np.testing.assert_allclose(eval_sh_basis(-dirs)[:, 4:], b[:, 4:], atol=1e-15)
    c = rng.normal(size=(40, 27))
    assert np.all(sh_to_rgb(c, dirs) >= 0)
    # d rgb / d coeff = basis (where positive): central differences
    c0 = 0.1 * rng.normal(size=27)
    c0[[0, 9, 18]] = 10.0                             # every channel well inside ReLU > 0
    d0 = dirs[0]
    for k in (0, 5, 13, 26):
        e = np.zeros(27)
        e[k] = 1e-6
        fd = (sh_to_rgb(c0 + e, d0) - sh_to_rgb(c0 - e, d0)) / 2e-6
        want = np.zeros(3)
        want[k // 9] = eval_sh_basis(d0)[k % 9]
        np.testing.assert_allclose(fd, want, atol=1e-8)
    with pytest.raises(ValueError):
        normalize_dirs(np.zeros(3))
