"""The reference's render behaviours (pkg/tests/test_render.py) on the device
path: the march twin, closed forms of the forward render in both
compositing formulas, early termination, the record=True sample list, and
closed forms / linearity / finite differences of the backward.  Device
colours are f32 FMAs and gradients f32 atomics: where the reference compares
two float64 paths at 1e-12 these compare at 1e-6 (colour) or to the float64
oracle."""

import math

import numpy as np
import pytest

from helpers import random_grid, random_hitting_ray
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as m
    return m


def dev(g):
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def set_table(g, fn):
    t = g.table.cpu().numpy() if hasattr(g.table, "cpu") else np.array(g.table)
    fn(t)
    g.table = t


def test_march_twin():
    m = px()
    g = m.SparseGrid.dense((4, 4, 4), (0, 0, 0), (1, 1, 1))
    ts, dl = m.march(g, np.array([5.0, 5.0, 5.0]), np.array([1.0, 0.0, 0.0]))
    assert len(ts) == 0 and len(dl) == 0                       # a miss
    ts, dl = m.march(g, np.array([-1.0, 0.5, 0.5]), np.array([1.0, 0.0, 0.0]), 0.5)
    assert dl[0] == pytest.approx(0.5 / 3.0, abs=1e-12)      # step_frac x voxel edge
    assert ts[1] - ts[0] == pytest.approx(0.5 / 3.0, abs=1e-12)
    rng = np.random.default_rng(0)
    g = m.SparseGrid.dense((5, 7, 6), (-1, -0.8, -1.2), (1.0, 1.1, 0.9))
    for _ in range(50):
        o, d = random_hitting_ray(rng, aabb=1.2)
        ts, dl = m.march(g, o, d, 0.37)
        if len(ts) == 0:
            continue
        inv = 1.0 / d
        t1 = np.min(np.maximum((g.aabb_min - o) * inv, (g.aabb_max - o) * inv))
        t0 = np.max(np.minimum((g.aabb_min - o) * inv, (g.aabb_max - o) * inv))
        assert dl.sum() == pytest.approx(t1 - max(t0, 0.0), abs=1e-9) and np.all(dl > 0)


@pytest.mark.parametrize("formula", ["relative", "absolute"])
def test_empty_space_renders_background(formula):
    m = px()
    g = m.SparseGrid.dense((4, 4, 4), (-1, -1, -1), (1, 1, 1), sigma=0.0)
    res = m.render_ray(g, [-2.0, 0.1, 0.0], [1.0, 0.0, 0.0],
                       m.RenderOptions(background=(0.2, 0.4, 0.8), formula=formula))
    np.testing.assert_allclose(res.rgb, [0.2, 0.4, 0.8], atol=1e-12)
    assert res.trans == 1.0


def test_forward_closed_forms():
    m = px()
    c, k = 1.7, 0.6   # homogeneous medium over black: k (1 - exp(-c L))
    g = m.SparseGrid.dense((8, 8, 8), (-1, -1, -1), (1, 1, 1), sigma=c, rgb=k)
    res = m.render_ray(g, [-2.0, 0.05, -0.1], [1.0, 0.0, 0.0],
                       m.RenderOptions(step_frac=1 / 64, background=(0, 0, 0), stop_thresh=0.0))
    np.testing.assert_allclose(res.rgb, k * (1 - math.exp(-c * 2.0)), atol=1e-3)
    # one opaque first interval (sigma delta = 20) hides everything behind it
    g = m.SparseGrid.dense((4, 4, 4), (-1, -1, -1), (1, 1, 1), rgb=0.5)
    set_table(g, lambda t: t.__setitem__((slice(None), 0), 20.0 / (0.5 * 2.0 / 3.0)))
    res = m.render_ray(g, [-2.0, 0.0, 0.0], [1.0, 0.0, 0.0],
                       m.RenderOptions(step_frac=0.5, background=(0, 0, 0)))
    np.testing.assert_allclose(res.rgb, 0.5, atol=math.exp(-20.0) + 1e-6)
    # a single sample over the chord: the two formulas agree
    g = m.SparseGrid.dense((2, 2, 2), (-1, -1, -1), (1, 1, 1), sigma=0.4, rgb=0.7)
    base = dict(step_frac=4.0, background=(0.0, 0.0, 0.0), stop_thresh=0.0)
    o, d = np.array([-2.0, 0.1, 0.05]), np.array([1.0, 0.0, 0.0])
    rel = m.render_ray(g, o, d, m.RenderOptions(formula="relative", **base))
    ab = m.render_ray(g, o, d, m.RenderOptions(formula="absolute", **base))
    np.testing.assert_allclose(rel.rgb, ab.rgb, atol=1e-12)


def test_absolute_formula_clips_two_heavy_samples():
    from paper_2112_05131_b200.sh import SH_C0
    m = px()
    alpha, dl = 0.7, 0.3
    c1, c2 = np.array([1.0, 0.0, 0.5]), np.array([0.0, 1.0, 0.25])
    g = m.SparseGrid.dense((3, 2, 2), (0, -1, -1), (0.6, 1, 1), sigma=-math.log(1 - alpha) / dl)
    links = g.links.cpu().numpy()

    def fill(t):
        for i in range(3):
            for j in range(2):
                for kk in range(2):
                    t[links[i, j, kk], [1, 10, 19]] = (c1 if i == 0 else c2) / SH_C0
    set_table(g, fill)
    res = m.render_ray(g, np.array([0.0, 0.01, 0.02]), np.array([1.0, 0.0, 0.0]),
                       m.RenderOptions(formula="absolute", step_frac=1.0,
                                       background=(0, 0, 0), stop_thresh=0.0))
    np.testing.assert_allclose(res.rgb, alpha * c1 + (1 - alpha) * c2, rtol=1e-6, atol=1e-7)
    rng = np.random.default_rng(6)                  # overlapping heavy samples: they differ
    g = dev(random_grid(rng, dims=(6, 6, 6), sigma_range=(2.0, 8.0)))
    o, d = random_hitting_ray(rng)
    base = dict(background=(0, 0, 0), stop_thresh=0.0)
    rel = m.render_ray(g, o, d, m.RenderOptions(formula="relative", **base))
    ab = m.render_ray(g, o, d, m.RenderOptions(formula="absolute", **base))
    assert np.max(np.abs(rel.rgb - ab.rgb)) > 1e-3


def test_refinement_termination_and_weight_normalisation():
    m = px()
    rng = np.random.default_rng(1)
    g = dev(random_grid(rng, dims=(8, 8, 8), sigma_range=(0.0, 5.0)))
    o, d = random_hitting_ray(rng)
    vals = [m.render_ray(g, o, d, m.RenderOptions(step_frac=f, stop_thresh=0.0)).rgb
            for f in (0.5, 0.25, 0.125, 0.0625)]
    gaps = [np.max(np.abs(b - a)) for a, b in zip(vals, vals[1:])]
    assert gaps[2] < gaps[1] < gaps[0]
    g = dev(random_grid(rng, dims=(6, 6, 6), sigma_range=(0.0, 8.0)))
    rays = [random_hitting_ray(rng) for _ in range(200)]
    o, d = np.array([r[0] for r in rays]), np.array([r[1] for r in rays])
    _, trans, wsum = m.render_rays(g, o, d)
    np.testing.assert_allclose(wsum + trans, 1.0, atol=1e-6)
    g = dev(random_grid(rng, dims=(8, 8, 8), sigma_range=(0.5, 30.0)))
    full = m.render_rays(g, o, d, m.RenderOptions(stop_thresh=0.0))[0]
    fast = m.render_rays(g, o, d, m.RenderOptions(stop_thresh=1e-4))[0]
    assert np.max(np.abs(full - fast)) < 1e-3


@pytest.mark.parametrize("formula", ["relative", "absolute"])
@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_kernel_matches_the_record_path(formula, interp):
    m = px()
    rng = np.random.default_rng(4)
    g = dev(random_grid(rng, dims=(6, 6, 6), holes=0.25, sigma_range=(-0.5, 4.0)))
    opts = m.RenderOptions(formula=formula, interp=interp, background=(0.3, 0.1, 0.9))
    for _ in range(10):
        o, d = random_hitting_ray(rng)
        fast = m.render_ray(g, o, d, opts)
        rec = m.render_ray(g, o, d, opts, record=True)
        np.testing.assert_allclose(fast.rgb, rec.rgb, atol=1e-6)
        assert fast.trans == pytest.approx(rec.trans, abs=1e-12)
    o, d = random_hitting_ray(rng)
    res = m.render_ray(g, o, d, m.RenderOptions(stop_thresh=0.0), record=True)
    assert len(res.samples) > 0
    for s in res.samples:
        assert s.delta > 0 and 0.0 <= s.trans <= 1.0
        assert s.weight == pytest.approx(s.trans * (1 - math.exp(-s.sigma * s.delta)), rel=1e-12)
    assert sum(s.weight for s in res.samples) + res.trans == pytest.approx(1.0, abs=1e-9)


def test_backward_closed_forms_and_linearity():
    m = px()
    bgc = 0.25   # zero opacity: dC/dsigma summed over rows = sum(delta) (c - bg) . up
    g = m.SparseGrid.dense((3, 3, 3), (-1, -1, -1), (1, 1, 1), sigma=0.0, rgb=0.6)
    opts = m.RenderOptions(step_frac=1.0, stop_thresh=0.0, background=(bgc,) * 3)
    o, d, up = np.array([-2.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), np.ones(3)
    dense = m.render_ray_backward(g, o, d, up, opts).dense()
    _, dl = m.march(g, o, d, 1.0)
    assert dense[:, 0].sum() == pytest.approx(np.sum(dl) * (0.6 - bgc) * 3.0, rel=1e-6)
    g = m.SparseGrid.dense((3, 3, 3), (-1, -1, -1), (1, 1, 1), sigma=0.0)
    z = m.render_ray_backward(g, o, d, up, m.RenderOptions(stop_thresh=0.0, background=(0, 0, 0)))
    assert np.all(z.dense() == 0.0)
    sigma, k, bgc = 1.3, 0.8, 0.2   # one sample: dC/dsigma = delta e^(-s delta) (c - b)
    g = m.SparseGrid.dense((2, 2, 2), (-1, -1, -1), (1, 1, 1), sigma=sigma, rgb=k)
    up = np.array([1.0, 0.5, 0.25])
    dense = m.render_ray_backward(g, np.array([-2.0, 0.2, -0.3]), d, up,
                                  m.RenderOptions(step_frac=4.0, stop_thresh=0.0,
                                                  background=(bgc,) * 3)).dense()
    assert dense[:, 0].sum() == pytest.approx(2.0 * math.exp(-2.0 * sigma) * (k - bgc) * up.sum(),
                                              rel=1e-6)
    rng = np.random.default_rng(7)
    g = dev(random_grid(rng, dims=(5, 5, 5)))
    o, d = random_hitting_ray(rng)
    up = np.array([0.3, -0.7, 1.1])
    opts = m.RenderOptions(stop_thresh=0.0)
    g1 = m.render_ray_backward(g, o, d, up, opts).dense()
    g2 = m.render_ray_backward(g, o, d, 2.5 * up, opts).dense()
    np.testing.assert_allclose(g2, 2.5 * g1, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("formula", ["relative", "absolute"])
@pytest.mark.parametrize("interp", ["trilinear", "nearest"])
def test_backward_matches_finite_differences(formula, interp):
    m = px()
    rng = np.random.default_rng(8)
    g = random_grid(rng, dims=(5, 5, 5), holes=0.2,
                    sigma_range=(0.2, 3.0) if formula == "relative" else (0.05, 0.6))
    bg = (0.7, 0.2, 0.4)
    o, d = random_hitting_ray(rng)
    up = rng.normal(size=3)
    dense = m.render_ray_backward(dev(g), o, d, up,
                                  m.RenderOptions(stop_thresh=0.0, formula=formula,
                                                  interp=interp, background=bg)).dense()
    nz = np.argwhere(dense != 0)
    assert len(nz) > 0

    def value():   # the reference's own forward (oracle, float64)
        rgb, _, _ = orc.render_rays(g, o[None], d[None], stop_thresh=0.0, background=bg,
                                    interp=interp, formula=formula)
        return float(rgb[0] @ up)

    h = 1e-3
    for row, col in nz[rng.permutation(len(nz))[:150]]:
        old = g.table[row, col]
        g.table[row, col] = old + h
        fp = value()
        g.table[row, col] = old - h
        fm = value()
        g.table[row, col] = old
        assert dense[row, col] == pytest.approx((fp - fm) / (2 * h), rel=1e-4, abs=1e-7)


def test_fused_mse_backward_is_mse_upstream_through_the_render():
    m = px()
    rng = np.random.default_rng(9)
    g = dev(random_grid(rng, dims=(5, 5, 5)))
    opts = m.RenderOptions(stop_thresh=0.0)
    rays = [random_hitting_ray(rng) for _ in range(8)]
    o, d = np.array([r[0] for r in rays]), np.array([r[1] for r in rays])
    gt = rng.uniform(0, 1, (8, 3))
    buf = m.GradientBuffer(g.n_rows)
    rgb, mse_sum, _ = m.fused_mse_backward(g, o, d, orc.normalize_dirs(d), gt, buf, opts,
                                           n_total=8)
    loss, up = m.mse_loss(rgb, gt)
    assert mse_sum / 8 == pytest.approx(loss, rel=1e-12)
    buf2 = m.GradientBuffer(g.n_rows)
    rgb2, _ = m.render_rays_backward(g, o, d, up, buf2, opts)
    np.testing.assert_allclose(rgb, rgb2, atol=1e-12)
    np.testing.assert_allclose(buf.dense(), buf2.dense(), rtol=1e-5, atol=1e-9)


def test_jitter_is_deterministic_per_rng_and_moves_samples():
    m = px()
    rng = np.random.default_rng(10)
    g = dev(random_grid(rng, dims=(6, 6, 6)))
    o, d = random_hitting_ray(rng)
    opts = m.RenderOptions(jitter=1.0)
    r1 = m.render_rays(g, o[None], d[None], opts, rng=np.random.default_rng(42))[0]
    r2 = m.render_rays(g, o[None], d[None], opts, rng=np.random.default_rng(42))[0]
    r3 = m.render_rays(g, o[None], d[None], opts, rng=np.random.default_rng(7))[0]
    r0 = m.render_rays(g, o[None], d[None], m.RenderOptions())[0]
    np.testing.assert_array_equal(r1, r2)
    assert np.max(np.abs(r1 - r3)) > 0 and np.max(np.abs(r1 - r0)) > 0
