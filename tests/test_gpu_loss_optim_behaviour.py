"""The reference's loss, metric and optimiser behaviours
(pkg/tests/test_losses.py, test_optim.py) on the device path.  The device
table is float32 with float64 update arithmetic, so the optimiser's scalar
oracles here round the parameter and the second moment to float32 after
every step, exactly as the device does -- and then match bit for bit."""

import math

import numpy as np
import pytest

from helpers import random_grid
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

f32 = np.float32


def px():
    import paper_2112_05131_b200 as m
    return m


def dev(g):
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def set_table(g, fn):
    t = g.table.cpu().numpy()
    fn(t)
    g.table = t


def cell(dims, i, j, k):
    return np.array([(i * dims[1] + j) * dims[2] + k], dtype=np.int64)


def test_mse():
    m = px()
    x = np.random.default_rng(0).uniform(0, 1, (10, 3))
    loss, grad = m.mse_loss(x, x)
    assert loss == 0.0 and np.all(grad == 0.0)
    loss, grad = m.mse_loss(np.array([[0.6, 0.2, 0.9]]), np.array([[0.5, 0.2, 0.9]]))
    assert loss == pytest.approx(0.01, abs=1e-12)
    np.testing.assert_allclose(grad, [[0.2, 0.0, 0.0]], atol=1e-12)
    with pytest.raises(ValueError):
        m.mse_loss(np.zeros((0, 3)), np.zeros((0, 3)))


def test_tv_values():
    m = px()
    g = m.SparseGrid.dense((6, 6, 6), (0, 0, 0), (1, 1, 1), sigma=2.0, rgb=0.5)
    assert m.tv_loss(g, cell(g.dims, 2, 3, 2), 1.0, 1.0, eps=0.0) == (0.0, 0.0)   # interior
    sig, sh = m.tv_loss(g, cell(g.dims, 5, 5, 5), 1.0, 1.0, eps=0.0)   # off-lattice sigma = 0
    assert sig > 0.0 and sh == 0.0
    # a lone +1 step along x at D_x = 256 (Delta normalised by exactly 1): TV = 1
    g = m.SparseGrid.dense((256, 2, 2), (0, 0, 0), (1, 1, 1), sigma=3.0)
    links = g.links.cpu().numpy()
    set_table(g, lambda t: t.__setitem__((links[101].reshape(-1), 0), 4.0))
    assert m.tv_loss(g, cell(g.dims, 100, 0, 0), 1.0, 1.0, eps=0.0)[0] == pytest.approx(1.0, abs=1e-12)
    rng = np.random.default_rng(3)
    rg = dev(random_grid(rng, dims=(4, 4, 4)))
    sig, sh = m.tv_loss(rg, np.arange(64, dtype=np.int64), 1.0, 1.0, eps=0.0)
    assert sig > 0.0 and sh >= 0.0
    flat = m.SparseGrid.dense((4, 4, 4), (0, 0, 0), (1, 1, 1), sigma=0.0, rgb=0.3)
    assert m.tv_loss(flat, cell(flat.dims, 1, 1, 1), 1.0, 1.0, eps=0.0) == (0.0, 0.0)
    const = m.SparseGrid.dense((5, 5, 5), (0, 0, 0), (1, 1, 1), sigma=1.3, rgb=0.4)
    buf = m.GradientBuffer(const.n_rows)
    m.tv_loss(const, cell(const.dims, 2, 2, 2), 1.0, 1.0, buf)
    assert np.all(buf.dense() == 0.0)
    run = m.sample_tv_cells(m.SparseGrid.dense((8, 8, 8), (0, 0, 0), (1, 1, 1)), 0.01,
                            np.random.default_rng(4))
    cells = np.asarray(run)
    assert len(cells) == round(0.01 * 512) and np.all(np.diff(cells) % 512 == 1)


def test_tv_gradients_match_finite_differences():
    m = px()
    rng = np.random.default_rng(2)
    g = random_grid(rng, dims=(5, 5, 5), holes=0.3, sigma_range=(-1.0, 1.0),
                    dc_range=(-1.0, 1.0), band_scale=0.8)
    cells = np.arange(125, dtype=np.int64)
    buf = m.GradientBuffer(g.n_rows)
    m.tv_loss(dev(g), cells, 0.7, 1.3, buf)
    dense = buf.dense()
    nz = np.argwhere(dense != 0)
    h = 1e-5
    for row, col in nz[rng.permutation(len(nz))[:200]]:
        old = g.table[row, col]
        g.table[row, col] = old + h
        fp = sum(orc.tv_loss(g, cells, 0.7, 1.3))
        g.table[row, col] = old - h
        fm = sum(orc.tv_loss(g, cells, 0.7, 1.3))
        g.table[row, col] = old
        assert dense[row, col] == pytest.approx((fp - fm) / (2 * h), rel=1e-4, abs=1e-9)


def test_cauchy_prior():
    c = px().cauchy_sparsity_loss
    loss, grad = c(np.zeros(5), 1.0)
    assert loss == 0.0 and np.all(grad == 0.0)
    loss, grad = c(np.array([1.0]), 1.0)
    assert loss == pytest.approx(math.log(3.0), rel=1e-12) and grad[0] == pytest.approx(4 / 3, rel=1e-12)
    s = np.random.default_rng(6).uniform(0.1, 3.0, 20)
    _, grad = c(s, 0.7)
    for i in range(20):
        sp, sm = s.copy(), s.copy()
        sp[i] += 1e-6
        sm[i] -= 1e-6
        assert grad[i] == pytest.approx((c(sp, 0.7)[0] - c(sm, 0.7)[0]) / 2e-6, rel=1e-4, abs=1e-7)


def _ssim_loops(a, b, k1=0.01, k2=0.03):
    """Windowed SSIM written as explicit loops over the valid interior."""
    r, sg = 5, 1.5
    w1 = np.exp(-np.arange(-r, r + 1) ** 2 / (2 * sg * sg))
    win = np.outer(w1 / w1.sum(), w1 / w1.sum())
    c1, c2 = k1 * k1, k2 * k2
    per_ch = []
    for ch in range(a.shape[2]):
        vals = []
        for i in range(r, a.shape[0] - r):
            for j in range(r, a.shape[1] - r):
                x = a[i - r:i + r + 1, j - r:j + r + 1, ch]
                y = b[i - r:i + r + 1, j - r:j + r + 1, ch]
                mx, my = (win * x).sum(), (win * y).sum()
                vx = (win * x * x).sum() - mx * mx
                vy = (win * y * y).sum() - my * my
                cv = (win * x * y).sum() - mx * my
                vals.append((2 * mx * my + c1) * (2 * cv + c2) /
                            ((mx * mx + my * my + c1) * (vx + vy + c2)))
        per_ch.append(np.mean(vals))
    return float(np.mean(per_ch))


def test_image_metrics():
    m = px()
    img = np.random.default_rng(9).uniform(0, 1, (24, 24, 3))
    assert m.psnr(img, img) == math.inf
    assert m.ssim(img, img) == pytest.approx(1.0, abs=1e-12)
    assert m.psnr(np.full((8, 8, 3), 0.5), np.full((8, 8, 3), 0.6)) == pytest.approx(20.0, abs=1e-9)
    for f in (m.psnr, m.ssim):
        with pytest.raises(ValueError):
            f(np.zeros((24, 24, 3)), np.zeros((25, 24, 3)))
    rng = np.random.default_rng(11)
    base = rng.uniform(0.2, 0.8, (20, 22, 3))
    noisy = np.clip(base + rng.normal(0, 0.05, base.shape), 0, 1)
    s = m.ssim(base, noisy)
    assert s == pytest.approx(_ssim_loops(base, noisy), abs=1e-9) and 0.0 < s < 1.0


def _one_row_grid(sigma=0.5):
    return px().SparseGrid.dense((2, 2, 2), (-1, -1, -1), (1, 1, 1), sigma=sigma, rgb=0.2)


def _step(g, col_vals, lr_s, lr_c, state, method="rmsprop", row=0):
    m = px()
    from paper_2112_05131_b200 import optim
    grads = m.GradientBuffer(g.n_rows)
    up = np.zeros(28)
    for c, v in col_vals.items():
        up[c] = v
    grads.add(row, up)
    optim.step(g, grads, state, lr_s, lr_c, method)


def test_optimiser_semantics():
    m = px()
    from paper_2112_05131_b200 import optim
    g = _one_row_grid()
    before = g.table.cpu().numpy().copy()
    st = m.OptimState(g.n_rows)
    st.v.fill_(0.123)
    optim.step(g, m.GradientBuffer(g.n_rows), st, 1.0, 1.0)      # no gradient: nothing moves
    np.testing.assert_array_equal(g.table.cpu().numpy(), before)
    assert np.all(st.v.cpu().numpy() == f32(0.123))
    g = _one_row_grid(sigma=1.0)
    _step(g, {0: 0.5}, 0.1, 0.1, m.OptimState(g.n_rows), "sgd")
    assert g.table[0, 0].item() == f32(1.0 - 0.1 * 0.5)
    g = _one_row_grid(sigma=1.0)
    set_table(g, lambda t: t.__setitem__((slice(None), 1), 1.0))
    _step(g, {0: 1.0, 1: 1.0}, 0.2, 0.01, m.OptimState(g.n_rows), "sgd")   # own rates
    assert (g.table[0, 0].item(), g.table[0, 1].item()) == (f32(0.8), f32(0.99))
    with pytest.raises(ValueError):
        optim.step(g, m.GradientBuffer(g.n_rows), m.OptimState(g.n_rows + 1), 0.1, 0.1)


def test_rmsprop_recurrences_match_float32_scalar_oracles():
    m = px()
    from paper_2112_05131_b200 import optim
    # constant gradient 1 on one entry: v -> 1, the update size -> lr
    g = _one_row_grid()
    st = m.OptimState(g.n_rows)
    lr, v, th = 0.01, f32(0.0), f32(g.table[0, 0].item())
    for _ in range(300):
        _step(g, {0: 1.0}, lr, lr, st)
        nv = 0.95 * float(v) + (1.0 - 0.95) * 1.0       # K:586-589: the quotient uses nv
        th = f32(float(th) - lr * 1.0 / (math.sqrt(nv) + 1e-8))
        v = f32(nv)
        assert g.table[0, 0].item() == th and st.v[0, 0].item() == v
    assert float(v) == pytest.approx(1.0, abs=1e-4)
    # f(x) = (x - 2)^2 / 2 under a delayed-exponential schedule reaches 2
    g = _one_row_grid(sigma=0.0)
    st = m.OptimState(g.n_rows)
    sched = m.LrSchedule(kind="delayed_exponential", lr_init=0.5, lr_final=0.05,
                         total_steps=1000, delay_steps=100, delay_mult=0.01)
    x, v = f32(0.0), f32(0.0)
    for s in range(1000):
        lr = m.lr_at(sched, s)
        gv = f32(g.table[0, 0].item() - 2.0)                 # the f32 gradient the device sees
        _step(g, {0: float(gv)}, lr, lr, st)
        nv = 0.95 * float(v) + (1.0 - 0.95) * float(gv) * float(gv)
        x = f32(float(x) - lr * float(gv) / (math.sqrt(nv) + 1e-8))
        v = f32(nv)
        assert g.table[0, 0].item() == x
    assert abs(float(x) - 2.0) < 1e-3


def test_optimiser_finite_on_extreme_gradients_and_deterministic():
    m = px()
    from paper_2112_05131_b200 import optim
    g = m.SparseGrid.dense((3, 3, 3), (-1, -1, -1), (1, 1, 1), sigma=0.5, rgb=0.2)
    st = m.OptimState(g.n_rows)
    rng = np.random.default_rng(0)
    for _ in range(20):
        grads = m.GradientBuffer(g.n_rows)
        grads.add(0, rng.normal(size=28) * 1e12)
        grads.add(1, rng.normal(size=28) * 1e-12)
        optim.step(g, grads, st, 30.0, 0.01)
    assert np.all(np.isfinite(g.table.cpu().numpy())) and np.all(np.isfinite(st.v.cpu().numpy()))

    def run():
        gg = m.SparseGrid.dense((3, 3, 3), (-1, -1, -1), (1, 1, 1), sigma=0.5, rgb=0.2)
        s = m.OptimState(gg.n_rows)
        r = np.random.default_rng(7)
        for _ in range(50):
            grads = m.GradientBuffer(gg.n_rows)
            grads.add(int(r.integers(0, gg.n_rows)), r.normal(size=28))
            optim.step(gg, grads, s, 0.1, 0.01)
        return gg.table.cpu().numpy()
    np.testing.assert_array_equal(run(), run())
