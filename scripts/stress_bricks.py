#!/usr/bin/env python3
"""Randomised self-consistency of dead-brick skipping: random sparse grids
(odd dims, slabs of holes, sigma fields with large negative regions, exact
zeros, a few positive blobs) and random rays (inside / outside the box,
axis-aligned directions, jitter); forward render, fused backward (relative /
absolute, trilinear / nearest, Cauchy) and max-weight with and without the
mask must agree bit for bit (gradients: same set of touched rows, values to
f32 atomic order)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_05131_b200 as px  # noqa: E402


def grid(rng):
    D = tuple(int(x) for x in rng.integers(9, 60, 3))
    x, y, z = np.meshgrid(*[np.linspace(-1, 1, d) for d in D], indexing="ij")
    occ = rng.random(D) > rng.choice([0.0, 0.0, 0.01, 0.2])
    a = rng.integers(0, 3)
    occ &= ~((np.stack([x, y, z])[a] > rng.uniform(-0.5, 0.8)))  | (rng.random() < 0.3)
    sig = np.full(D, -rng.uniform(0.1, 3.0))
    for _ in range(rng.integers(0, 4)):
        c = rng.uniform(-0.8, 0.8, 3)
        r = rng.uniform(0.05, 0.4)
        d2 = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2
        sig = np.where(d2 < r * r, rng.uniform(0.0, 5.0, D), sig)
    sig[rng.random(D) < 0.002] = 0.0
    links = np.full(D, -1, dtype=np.int32)
    links[occ] = np.arange(int(occ.sum()), dtype=np.int32)
    n = int(occ.sum())
    table = np.zeros((n, 28), dtype=np.float32)
    table[:, 0] = sig[occ]
    table[:, 1:] = rng.uniform(-0.5, 1.0, (n, 27))
    g = px.SparseGrid(torch.from_numpy(links).cuda(), torch.from_numpy(table).cuda(),
                      (-1.0,) * 3, (1.0,) * 3)
    h = g.copy()
    h.disable_bricks()
    g.lattice_sigma()
    h.lattice_sigma()
    return g, h


def rays(rng, n):
    o = rng.uniform(-1.6, 1.6, (n, 3))
    o[: n // 4] = rng.uniform(-0.9, 0.9, (n // 4, 3))          # inside
    d = rng.normal(size=(n, 3))
    k = rng.integers(0, 3, n // 8)
    d[: n // 8] = 0.0
    d[np.arange(n // 8), k] = rng.choice([-1.0, 1.0], n // 8)  # axis-aligned
    tgt = rng.uniform(-0.3, 0.3, (n, 3))
    d[n // 8:] = tgt[n // 8:] - o[n // 8:] + 0.3 * d[n // 8:]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


def main(trials):
    rng = np.random.default_rng(int(os.environ.get("SEED", 0)))
    bad = tested = 0
    for t in range(trials):
        g, h = grid(rng)
        if g._bricks is None or not int(g._bricks.ne(0).sum()):
            continue
        tested += 1
        o, d = rays(rng, 2000)
        vd = d
        gt = rng.uniform(0, 1, (2000, 3))
        for interp, formula in (("trilinear", "relative"), ("trilinear", "absolute"),
                                ("nearest", "relative")):
            opts = px.RenderOptions(interp=interp, formula=formula,
                                    jitter=float(rng.choice([0.0, 1.0])))
            fa = px.render_rays(g, o, d, opts, rng=np.random.default_rng(t))
            fb = px.render_rays(h, o, d, opts, rng=np.random.default_rng(t))
            ok = all(np.array_equal(x, y) for x, y in zip(fa, fb))
            ga, gb = px.GradientBuffer(g.n_rows), px.GradientBuffer(h.n_rows)
            ra, ma, _ = px.fused_mse_backward(g, o, d, vd, gt, ga, opts, n_total=2000,
                                              lam_cauchy=1e-3, rng=np.random.default_rng(t))
            rb, mb, _ = px.fused_mse_backward(h, o, d, vd, gt, gb, opts, n_total=2000,
                                              lam_cauchy=1e-3, rng=np.random.default_rng(t))
            ok &= np.array_equal(ra, rb) and np.array_equal(ga.touched_rows(), gb.touched_rows())
            da, db = ga.dense(), gb.dense()
            ok &= np.allclose(da, db, rtol=1e-5, atol=1e-7 * max(1e-30, float(np.abs(db).max())))
            if opts.jitter == 0.0:
                ok &= np.array_equal(g.max_weight_accumulate(o, d, interp=interp),
                                     h.max_weight_accumulate(o, d, interp=interp))
            if not ok:
                bad += 1
                print("MISMATCH trial", t, g.dims, interp, formula, opts.jitter, flush=True)
    print(f"{trials} trials ({tested} with dead bricks), {bad} mismatches", flush=True)
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 40) else 0)
