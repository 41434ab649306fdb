"""Shared test utilities: golden-case loaders and the reference's own test
fixtures (pkg/tests/conftest.py:10-42) restated for numpy."""

from __future__ import annotations

import os

import numpy as np

from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_grid(z, prefix):
    return orc.Grid(z[f"{prefix}links"], z[f"{prefix}table"], z[f"{prefix}aabb_min"],
                    z[f"{prefix}aabb_max"])


def random_grid(rng, dims=(5, 5, 5), aabb=1.0, sigma_range=(0.2, 3.0),
                dc_range=(0.5, 1.5), band_scale=0.05, holes=0.0, f32=True):
    """pkg/tests/conftest.py:10-31 (table quantised to f32 when f32=True)."""
    g = orc.Grid.dense(dims, (-aabb,) * 3, (aabb,) * 3)
    g.table[:, 0] = rng.uniform(*sigma_range, g.n_rows)
    for ch in range(3):
        g.table[:, 1 + 9 * ch] = rng.uniform(*dc_range, g.n_rows)
        for b in range(1, 9):
            g.table[:, 1 + 9 * ch + b] = rng.uniform(-band_scale, band_scale, g.n_rows)
    if holes > 0:
        links = g.links.copy()
        mask = rng.random(links.shape) < holes
        links[mask] = -1
        keep = np.sort(g.links[links >= 0])
        remap = np.full(g.n_rows, -1, dtype=np.int64)
        remap[keep] = np.arange(len(keep))
        links = np.where(links >= 0, remap[np.maximum(links, 0)], -1)
        g = orc.Grid(links.astype(np.int32), g.table[keep], g.aabb_min, g.aabb_max)
    if f32:
        g.table[:] = g.table.astype(np.float32)
    return g


def random_hitting_ray(rng, aabb=1.0):
    """pkg/tests/conftest.py:34-42."""
    target = rng.uniform(-0.6 * aabb, 0.6 * aabb, 3)
    theta = rng.uniform(0, 2 * np.pi)
    z = rng.uniform(-0.9, 0.9)
    r = np.sqrt(1 - z * z)
    origin = 3.0 * aabb * np.array([r * np.cos(theta), r * np.sin(theta), z])
    d = target - origin
    return origin, d / np.linalg.norm(d)


def ray_batch(rng, n, aabb=1.0):
    o, d = zip(*[random_hitting_ray(rng, aabb) for _ in range(n)])
    return np.array(o), np.array(d)


def grad_close(got, want, rel=1e-3, floor_frac=1e-6, abs_floor=1e-9):
    """Gradient comparator for f32-atomic results vs the f64 oracle: per entry
    |got-want| <= rel*|want| + max(floor_frac*max|want|, abs_floor).
    Returns (ok, worst_ratio, n_bad)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    tol = rel * np.abs(want) + max(floor_frac * scale, abs_floor)
    err = np.abs(got - want)
    ratio = err / tol
    bad = int(np.count_nonzero(ratio > 1.0))
    return bad == 0, float(ratio.max()) if ratio.size else 0.0, bad
