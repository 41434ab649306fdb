"""Data-parallel sharding of the training step over GPUs.

Rays are independent, so each rank takes a contiguous slice of
the global batch drawn by the (replicated, identically seeded) host batcher,
and a contiguous sub-run of the TV cell run.  The grid, the RMSProp state and
the optimiser step are replicated; the one exchange per step is the gradient
reduction:

  v1 (this file): all_reduce(SUM) of the dense f32 gradient table, all_reduce
     (MAX) of the uint8 touched mask, all_reduce(SUM) of the loss sums --
     three NCCL collectives over NVLink/NVSwitch, then an identical optimiser
     step on every rank keeps the replicas bit-identical.

Everything here is plain torch.distributed on whatever device the tensors
live on, so the same code runs over NCCL on B200s and over gloo on CPU
(tests/test_dist_cpu.py, world_size 2).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class World:
    rank: int = 0
    size: int = 1
    group: object = None

    @property
    def active(self) -> bool:
        return self.size > 1

    @classmethod
    def from_env(cls) -> "World":
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(), dist.get_world_size(), None)
        return cls()


def shard_range(n: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous [start, start+count) slice of n items for `rank`; the first
    n % size ranks take one extra item."""
    base, rem = divmod(int(n), int(size))
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def reduce_gradients(world: World, grad: torch.Tensor, tmask: torch.Tensor,
                     sums: torch.Tensor | None = None) -> None:
    """In place: grad <- sum over ranks, tmask <- max (logical OR), sums <- sum."""
    if not world.active:
        return
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=world.group)
    dist.all_reduce(tmask, op=dist.ReduceOp.MAX, group=world.group)
    if sums is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=world.group)


def max_reduce(world: World, t: torch.Tensor) -> None:
    """Max-weight accumulation sharded over rays (G:287-302): out_w max-reduce."""
    if world.active:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=world.group)
