"""The multi-rank training step end to end on ONE GPU: two processes share
cuda:0 (gloo for the host collectives -- NCCL refuses two ranks on one
device), each runs paper_2112_05131_b200.trainer.Trainer with World(rank, 2,
mode).  In "p2p" mode the ranks map each other's grid and gradient buffers
with CUDA IPC and run the owner-computes NVLink kernel exactly as on two
GPUs.  The sharded steps must reproduce the single-process full-batch steps
(SGD, so the update is linear in the gradient and the f32 summation order
is the only difference)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import load

pytestmark = pytest.mark.gpu

STEPS = 3


def _cfg():
    from paper_2112_05131_b200 import trainer
    cfg = trainer.toy_config(grid_dim=16, total_steps=50, batch_size=512)
    cfg.optimizer = "sgd"
    cfg.lr_sigma.lr_init = cfg.lr_sigma.lr_final = 5.0
    cfg.lr_sigma.kind = "constant"
    return cfg


def _ds():
    from paper_2112_05131_b200.scenes import dataset_from_arrays
    z = load("trainer_tiny.npz")
    return dataset_from_arrays(z["imgs"], z["c2w"], z["focal"], tag="train")


def _run(world):
    from paper_2112_05131_b200 import trainer
    tr = trainer.Trainer(_ds(), _cfg(), device="cuda:0", world=world)
    losses = []
    for s in range(STEPS):
        losses.append(tr.step(s, sync=True)["loss"])
    torch.cuda.synchronize()
    return tr.grid.table.cpu().numpy(), np.array(losses), int(tr.count.item())


def _worker(rank, size, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from paper_2112_05131_b200.dist import World
        table, losses, cnt = _run(World(rank, size, mode=mode))
        q.put((rank, table, losses, cnt))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["dense", "union", "p2p"])
def test_two_ranks_on_one_gpu_match_single_process(mode):
    from paper_2112_05131_b200.dist import World
    want_table, want_losses, want_cnt = _run(World())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, table, losses, cnt in got:
        np.testing.assert_allclose(losses, want_losses, rtol=1e-6)
        np.testing.assert_allclose(table, want_table, rtol=1e-5, atol=1e-6)
        assert cnt == want_cnt, (rank, cnt, want_cnt)
