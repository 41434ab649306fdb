"""The reference's API behaviours beyond the render/step kernels, on the
device package: point sampling (SparseGrid.sample / sample_backward,
G:141-223, pkg/tests/test_grid.py:10-130), the beta prior (L:91-102,
test_losses.py:189-232), sh_to_rgb (sh.py:57-69, test_sh.py), the bare-table
optimiser step (O:100-107) and the single-ray camera helpers
(camera.py:52-142).  Each test states the property it checks; values are
compared with the reference's own tolerances where the device's f32 storage
allows it."""

import math

import numpy as np
import pytest
import torch

from helpers import random_grid

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as m
    return m


def dev(g):
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def numpy_sample(g, pts, mode="trilinear"):
    """G:154-200 on the oracle grid (float64 numpy), for comparison."""
    gl = (np.atleast_2d(pts) - g.aabb_min) * ((np.array(g.dims) - 1.0) / (g.aabb_max - g.aabb_min))
    gl = np.clip(gl, 0.0, np.array(g.dims) - 1.0)
    out = np.zeros((len(gl), 28))
    for n, p in enumerate(gl):
        if mode == "nearest":
            ijk = np.minimum(np.floor(p + 0.5).astype(int), np.array(g.dims) - 1)
            r = g.links[tuple(ijk)]
            if r >= 0:
                out[n] = g.table[r]
            continue
        i0 = np.minimum(np.floor(p).astype(int), np.array(g.dims) - 2)
        f = p - i0
        for di in (0, 1):
            for dj in (0, 1):
                for dk in (0, 1):
                    r = g.links[i0[0] + di, i0[1] + dj, i0[2] + dk]
                    w = (f[0] if di else 1 - f[0]) * (f[1] if dj else 1 - f[1]) * \
                        (f[2] if dk else 1 - f[2])
                    if r >= 0:
                        out[n] += w * g.table[r]
    out[:, 0] = np.maximum(out[:, 0], 0.0)
    return out


@pytest.mark.parametrize("mode", ["trilinear", "nearest"])
def test_sample_lattice_points_return_their_rows(mode):
    rng = np.random.default_rng(0)
    g = random_grid(rng, dims=(4, 5, 6), sigma_range=(-1.0, 2.0))
    dg = dev(g)
    ijk = np.stack([rng.integers(0, d, 20) for d in g.dims], -1)
    pts = dg.lattice_to_world(ijk.astype(float))
    sig, coeffs = dg.sample(pts, mode)
    rows = g.links[ijk[:, 0], ijk[:, 1], ijk[:, 2]]
    np.testing.assert_allclose(sig, np.maximum(g.table[rows, 0], 0.0), atol=1e-12)
    np.testing.assert_allclose(coeffs, g.table[rows, 1:], atol=1e-12)
    s1, c1 = dg.sample(pts[3], mode)          # a single (3,) point -> (float, (27,))
    assert isinstance(s1, float) and c1.shape == (27,)


def test_sample_cell_centre_is_corner_mean_and_linear_field_is_exact():
    rng = np.random.default_rng(1)
    g = random_grid(rng, dims=(4, 4, 4))
    dg = dev(g)
    c = np.array([1, 2, 0])
    corners = g.table[[g.links[c[0] + a, c[1] + b, c[2] + e]
                       for a in (0, 1) for b in (0, 1) for e in (0, 1)]]
    sig, coeffs = dg.sample(dg.lattice_to_world(c + 0.5))
    assert sig == pytest.approx(max(corners[:, 0].mean(), 0.0), abs=1e-12)
    np.testing.assert_allclose(coeffs, corners[:, 1:].mean(0), atol=1e-12)
    # sigma = i + 2j + 3k on the lattice is reproduced exactly in between
    lin = px().SparseGrid.dense((5, 5, 5), (0, 0, 0), (1, 1, 1))
    ii, jj, kk = np.meshgrid(*(np.arange(5),) * 3, indexing="ij")
    lin.density.copy_(torch.as_tensor((ii + 2 * jj + 3 * kk).reshape(-1), dtype=torch.float32))
    lin.invalidate()
    pts = rng.uniform(0, 1, (50, 3))
    lat = lin.world_to_lattice(pts)
    np.testing.assert_allclose(lin.sample(pts)[0], lat @ np.array([1.0, 2.0, 3.0]),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("mode", ["trilinear", "nearest"])
def test_sample_matches_the_reference_stencil_on_sparse_grids(mode):
    rng = np.random.default_rng(2)
    for _ in range(6):
        g = random_grid(rng, dims=tuple(int(x) for x in rng.integers(3, 9, 3)),
                        holes=float(rng.uniform(0, 0.5)), sigma_range=(-1.0, 3.0))
        pts = rng.uniform(-1, 1, (200, 3))
        pts[:4] = [[-1, -1, -1], [1, 1, 1], [1, -1, 0.3], [0, 0, 1]]   # faces and corners
        sig, coeffs = dev(g).sample(pts, mode)
        want = numpy_sample(g, pts, mode)
        np.testing.assert_allclose(sig, want[:, 0], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(coeffs, want[:, 1:], rtol=1e-12, atol=1e-12)


def test_sample_rejects_points_outside_the_aabb():
    dg = px().SparseGrid.dense((3, 3, 3), (0, 0, 0), (1, 1, 1))
    with pytest.raises(ValueError):
        dg.sample(np.array([1.5, 0.5, 0.5]))
    with pytest.raises(ValueError):
        dg.sample_backward(np.array([[0.5, -0.2, 0.5]]), np.zeros((1, 28)),
                           px().GradientBuffer(dg.n_rows))
    with pytest.raises(ValueError):
        dg.sample(np.array([0.5, 0.5, 0.5]), mode="cubic")
    dg.sample(np.array([1.0 + 1e-10, 0.5, 0.0]))   # within the 1e-9 * extent tolerance


def test_sample_is_continuous_across_a_lattice_plane():
    rng = np.random.default_rng(3)
    dg = dev(random_grid(rng, dims=(6, 6, 6)))
    base = dg.lattice_to_world(np.array([3.0, 2.3, 4.1]))
    gaps = []
    for eps in (1e-3, 1e-5, 1e-7):
        lo, hi = base.copy(), base.copy()
        lo[0] -= eps
        hi[0] += eps
        (s0, c0), (s1, c1) = dg.sample(lo), dg.sample(hi)
        gaps.append(abs(s1 - s0) + np.max(np.abs(c1 - c0)))
    assert gaps[0] > gaps[1] > gaps[2] and gaps[2] < 1e-5


def test_sample_backward_is_the_adjoint_of_sample():
    rng = np.random.default_rng(4)
    g = random_grid(rng, dims=(4, 4, 4), holes=0.2, sigma_range=(-1.0, 2.0))
    dg = dev(g)
    # a lattice point: the whole upstream lands on its one row
    p = dg.lattice_to_world(np.array([2.0, 1.0, 3.0]))
    row = int(g.links[2, 1, 3])
    up = rng.normal(size=28)
    buf = px().GradientBuffer(dg.n_rows)
    if row >= 0:
        dg.sample_backward(p, up, buf)
        d = buf.dense()
        want = up.copy()
        if g.table[row, 0] < 0:
            want[0] = 0.0   # clamped sigma: no sigma gradient
        np.testing.assert_allclose(d[row], want, rtol=1e-6, atol=1e-7)
        d[row] = 0
        assert np.all(d == 0) and buf.n_touched == 1
    # random points: <dL/dtable, e> equals the finite difference of
    # L = sum(upstream * sample(pts)) along a random perturbation e (linear
    # away from the sigma clamp: only coefficient columns are perturbed)
    pts = rng.uniform(-1, 1, (64, 3))
    ups = rng.normal(size=(64, 28))
    ups[:, 0] = 0.0
    buf = px().GradientBuffer(dg.n_rows)
    dg.sample_backward(pts, ups, buf)
    e = np.zeros_like(g.table)
    e[:, 1:] = rng.normal(size=(g.n_rows, 27))
    analytic = float(np.sum(buf.dense() * e))
    g2 = g.copy()
    g2.table[:] = g.table + 1e-3 * e
    fd = (np.sum(ups * numpy_sample(g2, pts)) - np.sum(ups * numpy_sample(g, pts))) / 1e-3
    assert analytic == pytest.approx(fd, rel=1e-5)


def test_beta_prior():
    beta_loss = px().beta_loss
    loss, grad = beta_loss(np.array([0.5]), lam=1.0)
    assert loss == pytest.approx(2 * math.log(0.5), rel=1e-12) and grad[0] == 0.0
    eps = 1e-6
    assert beta_loss(np.array([eps]), 1.0, eps)[1][0] > 1e5
    assert beta_loss(np.array([1 - eps]), 1.0, eps)[1][0] < -1e5
    assert beta_loss(np.array([eps / 2, 1 - eps / 2]), 1.0, eps)[1].tolist() == [0.0, 0.0]
    rng = np.random.default_rng(7)
    t = rng.uniform(0.05, 0.95, 40)
    lam = 0.3
    loss, grad = beta_loss(t, lam)
    assert loss == pytest.approx(lam * sum(math.log(v) + math.log(1 - v) for v in t), rel=1e-9)
    h = 1e-7
    for i in range(0, 40, 4):
        tp, tm = t.copy(), t.copy()
        tp[i] += h
        tm[i] -= h
        fd = (beta_loss(tp, lam)[0] - beta_loss(tm, lam)[0]) / (2 * h)
        assert grad[i] == pytest.approx(fd, rel=1e-4, abs=1e-7)
    # device tensors stay on the device with the same values
    lt, gt = beta_loss(torch.as_tensor(t, device="cuda"), lam)
    assert gt.is_cuda and lt == pytest.approx(loss, rel=1e-12)
    np.testing.assert_allclose(gt.cpu().numpy(), grad, rtol=1e-12)


def test_sh_to_rgb():
    from paper_2112_05131_b200.sh import SH_C0, eval_sh_basis, sh_to_rgb
    rng = np.random.default_rng(9)
    dirs = rng.normal(size=(30, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    coeffs = rng.normal(size=(30, 27))
    want = np.maximum(np.einsum("nb,ncb->nc", eval_sh_basis(dirs), coeffs.reshape(30, 3, 9)), 0)
    np.testing.assert_allclose(sh_to_rgb(coeffs, dirs), want, rtol=1e-12, atol=1e-15)
    dc = np.zeros(27)
    dc[[0, 9, 18]] = [1.0, -1.0, 2.0]                  # DC only: SH_C0 scale, negative clipped
    np.testing.assert_allclose(sh_to_rgb(dc, np.array([0.0, 0.0, 1.0])), [SH_C0, 0.0, 2 * SH_C0])
    assert np.all(sh_to_rgb(np.zeros(27), dirs[0]) == 0)
    with pytest.raises(ValueError):
        sh_to_rgb(np.zeros(26), dirs[0])


@pytest.mark.parametrize("method", ["rmsprop", "sgd"])
def test_step_table_on_a_bare_table(method):
    from paper_2112_05131_b200.optim import OptimState, step_table
    rng = np.random.default_rng(11)
    table = rng.normal(size=(50, 4))
    grads = rng.normal(size=(50, 4))
    grads[rng.random((50, 4)) < 0.3] = 0.0            # zero entries keep their state
    ids = np.array([3, 7, 8, 20, 41, 49], dtype=np.int64)
    st = OptimState(50, n_cols=4)
    v_ref = np.zeros((50, 4))
    t_ref = table.copy()
    for _ in range(3):
        step_table(table, grads, ids, len(ids), st, 0.1, 0.01, method)
        for r in ids:                                   # K:578-590 element by element
            for c in range(4):
                g = grads[r, c]
                if g == 0.0:
                    continue
                lr = 0.1 if c == 0 else 0.01
                if method == "rmsprop":
                    v_ref[r, c] = 0.95 * v_ref[r, c] + (1.0 - 0.95) * g * g
                    t_ref[r, c] -= lr * g / (math.sqrt(v_ref[r, c]) + 1e-8)
                else:
                    t_ref[r, c] -= lr * g
    np.testing.assert_array_equal(table, t_ref)
    if method == "rmsprop":
        np.testing.assert_array_equal(st.v.cpu().numpy(), v_ref)
    assert st.step_count == 3


def test_single_ray_camera_helpers():
    m = px()
    c2w = np.eye(4)
    c2w[:3, 3] = [0.1, -0.2, 3.0]
    cam = m.Camera(c2w=c2w, focal=50.0, width=16, height=12, near=1.0)
    o, d = m.generate_rays(cam)
    for px_, py_ in [(0, 0), (15, 11), (7, 5)]:
        r = m.generate_ray(cam, px_, py_)
        np.testing.assert_array_equal(r.origin, o[py_ * 16 + px_])
        np.testing.assert_array_equal(r.direction, d[py_ * 16 + px_])
        assert (r.px, r.py) == (px_, py_)
    with pytest.raises(ValueError):
        m.generate_ray(cam, 16, 0)
    r = m.ndc_ray(m.generate_ray(cam, 3, 4), cam)
    o2, d2, ok = m.to_ndc(o[4 * 16 + 3], d[4 * 16 + 3], cam)
    np.testing.assert_array_equal(r.origin, o2[0])
    np.testing.assert_array_equal(r.direction, d2[0])
    with pytest.raises(ValueError):   # parallel to the image plane
        m.ndc_ray(m.Ray(origin=np.zeros(3), direction=np.array([1.0, 0.0, 0.0])), cam)
