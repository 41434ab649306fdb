"""Data-parallel sharding of the training step over GPUs.

Rays are independent, so each rank takes a contiguous slice of
the global batch drawn by the (replicated, identically seeded) host batcher,
and a contiguous sub-run of the TV cell run.  The grid is replicated; the one
exchange per step is the touched rows' gradients, followed by the update
(T:483-486).  Three exchange modes (`World.mode`):

  dense  v1: all_reduce(SUM) of the whole f32 gradient table and all_reduce
         (MAX) of the touched mask, then the replicated single-GPU update.
         1.9 GB per step at 256^3 -- kept as the reference for tests.
  union  NCCL baseline: all_reduce(MAX) of the byte masks (the union of the
         touched rows), ordered compaction of the union (identical on every
         rank), the union's rows packed and all-reduced, and the replicated
         update straight from the packed buffer (plx_opt_step_list).
  p2p    NVLink peer memory: each rank owns 1/N of the rows and runs one
         kernel (plx_dp_owner_update) that ORs the N masks, sums the N
         gradient rows with peer loads, updates with its shard of the RMSProp
         state and stores the new rows into all N grids; two tiny NCCL
         all_reduces (loss sums, touched count) order it against the ranks'
         renders and clears.  Buffers are mapped once per grid with CUDA IPC.

Every mode computes the same update: the reduced gradient of a row is the
sum of the ranks' partial sums (f32), as in the single-GPU atomics.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import _lib

MODES = ("dense", "union", "p2p")


@dataclass
class World:
    rank: int = 0
    size: int = 1
    group: object = None
    mode: str = field(default_factory=lambda: os.environ.get("PLX_DP", "p2p"))

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"unknown data-parallel mode {self.mode!r} (one of {MODES})")

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


def owner_slice(rows: int, rank: int, size: int) -> tuple[int, int]:
    """Rows [lo, hi) rank updates in p2p mode (128-row aligned; mirrors
    plx_dp_owner_update)."""
    nseg = (int(rows) + 127) // 128
    s0, s1 = nseg * rank // size, nseg * (rank + 1) // size
    return s0 * 128, min(s1 * 128, int(rows))


def gather_owned_rows(world: World, v: torch.Tensor) -> torch.Tensor:
    """p2p mode keeps each row's RMSProp state current only on the row's
    owner (owner_slice): a copy of `v` whose every owner slice comes from
    its owner rank (checkpoints, T:435-439 / T:501-510)."""
    out = v.clone()
    if not world.active:
        return out
    for r in range(world.size):
        lo, hi = owner_slice(v.shape[0], r, world.size)
        if hi <= lo:
            continue
        part = out[lo:hi].contiguous()
        dist.broadcast(part, src=r, group=world.group)
        out[lo:hi] = part
    return out


def reduce_gradients(world: World, grad: torch.Tensor, tmask: torch.Tensor,
                     sums: torch.Tensor | None = None) -> None:
    """Mode "dense": grad <- sum over ranks, tmask <- max (logical OR),
    sums <- sum, all in place."""
    if not world.active:
        return
    if not grad.is_contiguous():   # a 28-column view of the 32-float-pitch rows
        grad = torch.as_strided(grad, (grad.shape[0], grad.stride(0)), (grad.stride(0), 1))
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=world.group)
    dist.all_reduce(tmask, op=dist.ReduceOp.MAX, group=world.group)
    if sums is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=world.group)


def union_rows(world: World, tmask: torch.Tensor, scratch: torch.Tensor, ids: torch.Tensor,
               count: torch.Tensor) -> int:
    """Mode "union", part 1: tmask <- OR over ranks (in place), ids[:n] <- the
    union's rows in ascending order (identical on every rank).  Returns n."""
    if world.active:
        dist.all_reduce(tmask, op=dist.ReduceOp.MAX, group=world.group)
    _lib.check(_lib.lib().plx_touched_list(tmask.data_ptr(), tmask.numel(), ids.data_ptr(),
                                           count.data_ptr(), scratch.data_ptr(),
                                           _lib.stream_ptr()), "touched_list")
    return int(count.item())


def max_reduce(world: World, t: torch.Tensor) -> None:
    """Max-weight accumulation sharded over rays (G:287-302): out_w max-reduce."""
    if world.active:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=world.group)


class PeerMap:
    """CUDA-IPC view of every rank's grid / gradient buffers (p2p mode).

    Built collectively after each (re)allocation of the grid: every rank
    exports its buffers, the handles travel with all_gather_object, and the
    peers' buffers are opened in this process.  `peers` is the plx_dp_peers
    descriptor for plx_dp_owner_update."""

    KEYS = ("grad", "tmask", "table", "density", "sigma_lat")

    def __init__(self, world: World, grid, grads):
        L = _lib.lib()
        if getattr(grid, "_bricks", None) is not None:
            # plx_dp_owner_update keeps every rank's sigma mirror, not its
            # dead-brick mask: the grid must be built without one
            raise ValueError("p2p exchange: call grid.disable_bricks() before building "
                             "descriptors (Trainer does this on N ranks)")
        mine = {}
        lat, _ = grid.lattice_sigma() if grid.n_rows else (None, None)
        if lat is not None and lat.data_ptr() == grid.density.data_ptr():
            lat = None   # aliased mirror (dense grid): updating density is enough
        local = {"grad": grads.data, "tmask": grads.touched_mask, "table": grid.sh,
                 "density": grid.density, "sigma_lat": lat}
        for k in self.KEYS:
            t = local[k]
            if t is None or t.numel() == 0:
                mine[k] = None
                continue
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64()
            _lib.check(L.plx_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "ipc_export")
            mine[k] = (h.raw, off.value)
        allh = [None] * world.size
        dist.all_gather_object(allh, mine, group=world.group)
        self._opened = []
        p = _lib.PlxDpPeers()
        p.n, p.rank, p.rows = world.size, world.rank, grid.n_rows
        for r in range(world.size):
            for k in self.KEYS:
                if r == world.rank:
                    ptr = local[k].data_ptr() if local[k] is not None else None
                elif allh[r][k] is None:
                    ptr = None
                else:
                    hb, off = allh[r][k]
                    base, ptr_out = ctypes.c_void_p(), ctypes.c_void_p()
                    _lib.check(L.plx_ipc_import(hb, off, ctypes.byref(base),
                                                ctypes.byref(ptr_out)), "ipc_import")
                    self._opened.append(base.value)
                    ptr = ptr_out.value
                getattr(p, k)[r] = ptr
        self.peers = p
        self._keep = local

    def close(self) -> None:
        L = _lib.lib()
        for b in self._opened:
            L.plx_ipc_close(b)
        self._opened = []
