"""The data-parallel exchange kernels (dist.py modes "union" and "p2p") on
one GPU: N rank replicas of the grid live in one process and the peer
pointers of plx_dp_peers are simply the other replicas' buffers, so the
owner-computes NVLink kernel and the packed-union path run exactly as on N
GPUs (minus the transport).  Each is checked against the single-GPU update
of the whole batch (the sharded step must equal the full-batch
step up to the f32 gradient summation order)."""

import ctypes

import numpy as np
import pytest
import torch

from helpers import random_grid, ray_batch

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as px_
    return px_


def _setup(n_ranks, seed):
    rng = np.random.default_rng(seed)
    g = random_grid(rng, dims=(14, 12, 13), holes=0.2, sigma_range=(-0.6, 1.2))
    o, d = ray_batch(rng, 96)
    gt = rng.uniform(0, 1, (96, 3))
    vd = d / np.linalg.norm(d, axis=1, keepdims=True)

    def grid():
        return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)
    return grid, (o, d, vd, gt)


def _render(grid, buf, rays, s, e):
    o, d, vd, gt = rays
    px().fused_mse_backward(grid, o[s:e], d[s:e], vd[s:e], gt[s:e], buf, px().RenderOptions(),
                            n_total=len(o))


def _bounds(n, k, total=96):
    from paper_2112_05131_b200.dist import shard_range
    s, c = shard_range(total, k, n)
    return s, s + c


def _reference(grid_fn, rays, steps, method):
    from paper_2112_05131_b200 import optim
    g = grid_fn()
    g.lattice_sigma()
    st = px().OptimState(g.n_rows)
    touched = []
    for it in range(steps):
        buf = px().GradientBuffer(g.n_rows)
        _render(g, buf, rays, 0, 96)
        touched.append(buf.n_touched)
        optim.step(g, buf, st, 0.7, 0.02, method, clear=True)
    torch.cuda.synchronize()
    return g, st, touched


def _close(got, want, method):
    """SGD is linear in the gradient: the f32 summation-order difference
    stays ~1e-7.  RMSProp divides by the running RMS, which amplifies it for
    entries whose contributions nearly cancel (the single-GPU atomics are
    order-nondeterministic in the same way), so there a handful of entries
    may move by more."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    if method == "sgd":
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)
        return
    bad = np.abs(got - want) > 1e-5 + 1e-5 * np.abs(want)
    assert bad.mean() <= 0.01, bad.mean()
    assert np.max(np.abs(got - want)) < 1e-2


def _assert_same(got, want, method, st_got=None, st_want=None, rows=None):
    _close(got.density.cpu().numpy(), want.density.cpu().numpy(), method)
    _close(got.sh.cpu().numpy(), want.sh.cpu().numpy(), method)
    lat = got.lattice_sigma()[0].clone()
    got.invalidate()   # the mirror kept by the exchange kernels == a rebuild
    assert torch.equal(lat.view(torch.int32), got.lattice_sigma()[0].view(torch.int32))
    if st_got is not None and method == "rmsprop":
        lo, hi = rows
        _close(st_got.v[lo:hi].cpu().numpy(), st_want.v[lo:hi].cpu().numpy(), method)


@pytest.mark.parametrize("method", ["sgd", "rmsprop"])
@pytest.mark.parametrize("n_ranks", [2, 3])
def test_p2p_owner_update_equals_full_batch_step(n_ranks, method):
    from paper_2112_05131_b200 import _lib
    from paper_2112_05131_b200.dist import owner_slice
    grid_fn, rays = _setup(n_ranks, 40 + n_ranks)
    ref, ref_st, ref_touched = _reference(grid_fn, rays, steps=2, method=method)
    reps = [grid_fn() for _ in range(n_ranks)]
    states = [px().OptimState(reps[0].n_rows) for _ in range(n_ranks)]
    L = _lib.lib()
    for it in range(2):
        bufs = [px().GradientBuffer(reps[0].n_rows) for _ in range(n_ranks)]
        for k in range(n_ranks):
            _render(reps[k], bufs[k], rays, *_bounds(n_ranks, k))
        p = _lib.PlxDpPeers()
        p.n, p.rows = n_ranks, reps[0].n_rows
        for k in range(n_ranks):
            p.grad[k] = bufs[k].data.data_ptr()
            p.tmask[k] = bufs[k].touched_mask.data_ptr()
            p.table[k] = reps[k].sh.data_ptr()
            p.density[k] = reps[k].density.data_ptr()
            p.sigma_lat[k] = reps[k].lattice_sigma()[0].data_ptr()
        count = torch.zeros(1, dtype=torch.int64, device="cuda")
        for o in range(n_ranks):          # every owner reads all ranks' grads first
            p.rank = o
            _lib.check(L.plx_dp_owner_update(
                ctypes.byref(p), states[o].v.data_ptr(), reps[o].lattice_sigma()[1].data_ptr(),
                0.7, 0.02, 0.95, 1e-8, int(method == "rmsprop"), None, count.data_ptr(),
                _lib.stream_ptr()), "dp")
        torch.cuda.synchronize()
        assert int(count.item()) == ref_touched[it]
        for b in bufs:
            b.clear()
    for k in range(n_ranks):
        _assert_same(reps[k], ref, method)
    for o in range(n_ranks):   # each owner holds the RMSProp state of its slice
        _assert_same(reps[o], ref, method, states[o], ref_st,
                     owner_slice(reps[0].n_rows, o, n_ranks))


@pytest.mark.parametrize("method", ["sgd", "rmsprop"])
@pytest.mark.parametrize("n_ranks", [2, 4])
def test_union_packed_update_equals_full_batch_step(n_ranks, method):
    from paper_2112_05131_b200 import _lib
    grid_fn, rays = _setup(n_ranks, 60 + n_ranks)
    ref, ref_st, ref_touched = _reference(grid_fn, rays, steps=2, method=method)
    reps = [grid_fn() for _ in range(n_ranks)]
    for r in reps:
        r.lattice_sigma()
    states = [px().OptimState(reps[0].n_rows) for _ in range(n_ranks)]
    L, st = _lib.lib(), _lib.stream_ptr()
    R = reps[0].n_rows
    ids = torch.empty(R, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    scratch = torch.empty(int(L.plx_scan_scratch_bytes(R)), dtype=torch.uint8, device="cuda")
    for it in range(2):
        bufs = [px().GradientBuffer(R) for _ in range(n_ranks)]
        for k in range(n_ranks):
            _render(reps[k], bufs[k], rays, *_bounds(n_ranks, k))
        union = torch.stack([b.touched_mask for b in bufs]).amax(0)   # all_reduce(MAX)
        _lib.check(L.plx_touched_list(union.data_ptr(), R, ids.data_ptr(), cnt.data_ptr(),
                                      scratch.data_ptr(), st), "list")
        n = int(cnt.item())
        assert n == ref_touched[it]
        assert torch.equal(ids[:n].long(), torch.nonzero(union).flatten())   # ascending
        packs = []
        for b in bufs:
            pk = torch.empty(n * 28, dtype=torch.float32, device="cuda")
            _lib.check(L.plx_pack_rows(b.data.data_ptr(), ids.data_ptr(), cnt.data_ptr(), n,
                                       pk.data_ptr(), st), "pack")
            packs.append(pk)
        red = torch.stack(packs).sum(0)                                # all_reduce(SUM)
        for k in range(n_ranks):
            bufs[k].touched_mask.copy_(union)
            count = torch.zeros(1, dtype=torch.int64, device="cuda")
            _lib.check(L.plx_opt_step_list(
                ctypes.byref(reps[k]._c(with_occ=False)), states[k].v.data_ptr(),
                ctypes.byref(bufs[k]._c()), ids.data_ptr(), cnt.data_ptr(), red.data_ptr(),
                0.7, 0.02, 0.95, 1e-8, int(method == "rmsprop"), 1, None, count.data_ptr(),
                st), "opt_list")
            torch.cuda.synchronize()
            assert int(count.item()) == n
            assert bufs[k].n_touched == 0 and float(bufs[k].data.abs().sum()) == 0.0
    for k in range(n_ranks):
        _assert_same(reps[k], ref, method, states[k], ref_st, (0, R))
