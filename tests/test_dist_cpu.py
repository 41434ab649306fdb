"""The N>1 data-parallel path on CPU (gloo, world_size 2): ray sharding, TV
sub-runs and the gradient exchange of paper_2112_05131_b200.dist reproduce
the single-process (full batch) gradient.  Per-rank gradients come from the
oracle here -- the collective logic is the product code under test."""

import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc

from helpers import random_grid, ray_batch


def test_shard_range_partitions():
    from paper_2112_05131_b200.dist import shard_range

    for n in (0, 1, 7, 5000, 5001):
        for size in (1, 2, 3, 8):
            got = [shard_range(n, r, size) for r in range(size)]
            assert sum(c for _, c in got) == n
            pos = 0
            for s, c in got:
                assert s == pos
                pos += c


def test_tv_run_split_covers_run():
    from paper_2112_05131_b200.losses import CellRun

    run = CellRun(start=990, count=37, n_cells=1000)
    full = np.asarray(run)
    parts = np.concatenate([np.asarray(run.split(r, 4)) for r in range(4)])
    np.testing.assert_array_equal(parts, full)


def _worker(rank, size, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from paper_2112_05131_b200.dist import World, reduce_gradients, shard_range
    from paper_2112_05131_b200.losses import CellRun

    rng = np.random.default_rng(42)
    g = random_grid(rng, dims=(7, 8, 6), holes=0.2)
    o, d = ray_batch(rng, 50)
    gt = rng.uniform(0, 1, (50, 3))
    B = len(o)
    s, c = shard_range(B, rank, size)
    buf = orc.GradBuf(g.n_rows)
    _, mse, _ = orc.fused_mse_backward(g, o[s:s + c], d[s:s + c], d[s:s + c], gt[s:s + c], buf, B)
    run = CellRun(100, 120, int(np.prod(g.dims)))
    sub = run.split(rank, size)
    a, b = orc.tv_loss(g, np.asarray(sub), 0.3 * sub.count / run.count,
                       0.7 * sub.count / run.count, buf)
    grad = torch.from_numpy(buf.data.astype(np.float32))
    mask = torch.from_numpy(buf.touched_mask.copy())
    sums = torch.tensor([mse, a, b], dtype=torch.float64)
    reduce_gradients(World(rank, size), grad, mask, sums)
    if rank == 0:
        out.put((grad.numpy(), mask.numpy(), sums.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gradient_exchange_equals_full_batch():
    rng = np.random.default_rng(42)
    g = random_grid(rng, dims=(7, 8, 6), holes=0.2)
    o, d = ray_batch(rng, 50)
    gt = rng.uniform(0, 1, (50, 3))
    full = orc.GradBuf(g.n_rows)
    _, mse, _ = orc.fused_mse_backward(g, o, d, d, gt, full, len(o))
    cells = (100 + np.arange(120)) % int(np.prod(g.dims))
    a, b = orc.tv_loss(g, cells, 0.3, 0.7, full)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    grad, mask, sums = q.get(timeout=120)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_array_equal(mask, full.touched_mask)
    scale = np.abs(full.data).max()
    assert np.all(np.abs(grad - full.data) <= 1e-6 * np.abs(full.data) + 1e-6 * scale)
    assert sums[0] == np.float64(mse) or abs(sums[0] - mse) < 1e-12 * abs(mse)
    assert abs(sums[1] - a) < 1e-9 * abs(a) and abs(sums[2] - b) < 1e-9 * abs(b)


def test_owner_slices_tile_the_rows():
    """p2p mode: the owners' 128-row-aligned slices partition [0, rows)."""
    from paper_2112_05131_b200.dist import owner_slice
    for rows in (1, 127, 128, 129, 5000, 16777216, 18680476):
        for n in (1, 2, 3, 4, 8):
            spans = [owner_slice(rows, r, n) for r in range(n)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 % 128 == 0


def _gather_worker(rank, size, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from paper_2112_05131_b200.dist import World, gather_owned_rows, owner_slice

    rows = 1000
    v = torch.full((rows, 32), -1.0)          # stale everywhere ...
    lo, hi = owner_slice(rows, rank, size)
    v[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None] + 0.5   # ... but the owned slice
    full = gather_owned_rows(World(rank, size, mode="p2p"), v)
    out.put((rank, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_checkpoint_state_gathers_owner_slices():
    """in p2p mode only a row's owner holds its current RMSProp
    state; a checkpoint must gather every owner's slice (identical on all
    ranks)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() + 7) % 1000
    size = 3
    ps = [ctx.Process(target=_gather_worker, args=(r, size, port, q)) for r in range(size)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(size))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.broadcast_to(np.arange(1000, dtype=np.float32)[:, None] + 0.5, (1000, 32))
    for r in range(size):
        np.testing.assert_array_equal(got[r], want)
