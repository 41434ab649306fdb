"""Device-resident sparse voxel grid and gradient buffer.

Mirrors pkg/src/plenoxel/grid.py (SparseGrid G:71-320, GradientBuffer
G:25-68) with HBM-resident storage:

  links   torch.int32  (Dx, Dy, Dz) C-order, -1 = empty      4 B / cell
  table   torch.float32 (rows, 28): sigma, 27 SH (112 B, 7 x float4 / row)
  grad    torch.float32 (rows, 28)  (GradientBuffer.data)
  tmask   torch.uint8   (rows,)     (GradientBuffer.touched_mask)

Structure ops (prune, upsample, max_weight_accumulate) run on the device
through libplx.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from ._lib import ROW, STRIDE
from .sh import SH_C0

EMPTY = -1
ROW_SIZE = ROW


def row_array(n_rows: int, device, zero: bool = True) -> torch.Tensor:
    """(n_rows, 28) float32 view of a (n_rows, 32) allocation: the kernels'
    128-byte row pitch (plx.h PLX_STRIDE), columns 28..31 padding."""
    f = torch.zeros if zero else torch.empty
    return f((int(n_rows), STRIDE), dtype=torch.float32, device=device)[:, :ROW]

# Empty-space skipping through the per-cell occupancy bitmask (an exact
# shortcut: a cell whose 8 corners are all empty has occ == False, K:126-135).
USE_CELL_OCC = True
# Dead-brick skipping (plx_grid.brick_dead, an exact shortcut: an 8^3-cell
# brick none of whose positions can be composited is skipped by the march's
# sigma gathers); sparse grids with a sigma mirror only.  PLX_BRICKS=0: off.
USE_BRICKS = os.environ.get("PLX_BRICKS", "1") != "0"


def _dev(device):
    return torch.device(device if device is not None else "cuda")


class GradientBuffer:
    """Sparse accumulator of per-row gradients (G:25-68).

    `touched_mask` marks rows that received any contribution; the reference's
    insertion-ordered `touched_ids` list is not materialised (only its sorted
    view `touched_rows()` and its length `n_touched` are observable)."""

    def __init__(self, n_rows: int, device=None):
        dev = _dev(device)
        self.data = row_array(n_rows, dev)
        self.touched_mask = torch.zeros(int(n_rows), dtype=torch.uint8, device=dev)
        self._count = torch.zeros(1, dtype=torch.int64, device=dev)
        # touched_ids / _count (G:25-68): filled by the two-phase optimiser step
        self.touched_ids = torch.empty(max(int(n_rows), 1), dtype=torch.int32, device=dev)
        self._tcnt = torch.zeros(1, dtype=torch.int64, device=dev)

    @property
    def n_rows(self) -> int:
        return self.data.shape[0]

    def _c(self, with_ids: bool = True) -> _lib.PlxGrad:
        g = _lib.PlxGrad()
        g.grad = self.data.data_ptr()
        g.tmask = self.touched_mask.data_ptr()
        if with_ids:
            g.tids = self.touched_ids.data_ptr()
            g.tcnt = self._tcnt.data_ptr()
        return g

    def count_touched_async(self) -> torch.Tensor:
        """Device int64[1] holding n_touched (no host sync)."""
        self._count.zero_()
        if self.n_rows:
            _lib.check(_lib.lib().plx_count_touched(
                self.touched_mask.data_ptr(), self.n_rows, self._count.data_ptr(),
                _lib.stream_ptr()), "count_touched")
        return self._count

    @property
    def n_touched(self) -> int:
        return int(self.count_touched_async().item())

    def touched_rows(self) -> np.ndarray:
        return torch.nonzero(self.touched_mask).flatten().cpu().numpy().astype(np.int64)

    def nnz_fraction(self) -> float:
        return self.n_touched / max(self.n_rows, 1)

    def add(self, row: int, values) -> None:
        values = torch.as_tensor(np.asarray(values, dtype=np.float64),
                                 dtype=torch.float32, device=self.data.device)
        if values.shape != (ROW,):
            raise ValueError(f"expected {ROW} gradient values")
        self.touched_mask[row] = 1
        self.data[row] += values

    def clear(self) -> None:
        """clear_grad (K:593-600): zero touched rows, reset the mask."""
        if self.n_rows:
            _lib.check(_lib.lib().plx_clear_grad(ctypes.byref(self._c()), self.n_rows, None,
                                                 _lib.stream_ptr()), "clear_grad")

    def dense(self) -> np.ndarray:
        return self.data.double().cpu().numpy()


class SparseGrid:
    """Dense int32 pointer lattice + f32 data in HBM (G:71-320).

    The reference's (rows, 28) `table` (column 0 sigma, 1..27 SH) is stored
    as two arrays: `density` (rows,) and `sh` (rows, 28) with column 0 unused
    (kept zero; 16-byte rows for float4 access).  The sigma gathers of the
    march then read a compact 4 B/row array.  `table` is the reference's
    combined view, materialised as a COPY (assign `grid.table = t` to write
    it back)."""

    def __init__(self, links, table, aabb_min, aabb_max, device=None):
        dev = _dev(device if device is not None else
                   (links.device if isinstance(links, torch.Tensor) and links.is_cuda else None))
        links = torch.as_tensor(links) if not isinstance(links, torch.Tensor) else links
        table = torch.as_tensor(np.asarray(table)) if not isinstance(table, torch.Tensor) else table
        if links.dim() != 3:
            raise ValueError("links must be a 3-d lattice")
        if any(int(d) < 2 for d in links.shape):
            raise ValueError("grid needs at least 2 lattice points per axis")
        if table.dim() != 2 or table.shape[1] != ROW:
            raise ValueError(f"table must be (rows, {ROW})")
        self._links = links.to(device=dev, dtype=torch.int32).contiguous()
        self.table = table.to(device=dev, dtype=torch.float32)
        self.aabb_min = np.asarray(aabb_min, dtype=np.float64).reshape(3).copy()
        self.aabb_max = np.asarray(aabb_max, dtype=np.float64).reshape(3).copy()
        if np.any(self.aabb_max <= self.aabb_min):
            raise ValueError("degenerate AABB")
        if int(np.prod(self.dims)) >= 2 ** 31:
            raise ValueError("lattice too large for int32 cell ids")
        self._cell_occ = None
        self._lat = None
        self._row_cell = None
        self._bricks = None

    # -- constructors -------------------------------------------------------
    @classmethod
    def _from_parts(cls, links, n_rows, aabb_min, aabb_max, device) -> "SparseGrid":
        """Grid over device links with uninitialised density / sh of n_rows
        (filled by a structure-op kernel)."""
        g = cls.__new__(cls)
        g._links = links.to(torch.int32).contiguous()
        g.density = torch.empty(int(n_rows), dtype=torch.float32, device=device)
        g.sh = row_array(n_rows, device, zero=False)
        g.aabb_min = np.asarray(aabb_min, dtype=np.float64).reshape(3).copy()
        g.aabb_max = np.asarray(aabb_max, dtype=np.float64).reshape(3).copy()
        g._cell_occ = None
        g._lat = None
        g._row_cell = None
        g._bricks = None
        return g

    @classmethod
    def dense(cls, dims, aabb_min, aabb_max, sigma: float = 0.0, rgb: float | None = None,
              device=None) -> "SparseGrid":
        """G:96-109: fully occupied; DC coefficients = rgb / SH_C0."""
        dims = tuple(int(d) for d in dims)
        dev = _dev(device)
        n = dims[0] * dims[1] * dims[2]
        links = torch.arange(n, dtype=torch.int32, device=dev).reshape(dims)
        table = torch.zeros((n, ROW), dtype=torch.float32, device=dev)
        table[:, 0] = sigma
        if rgb is not None:
            for ch in range(3):
                table[:, 1 + 9 * ch] = rgb / SH_C0
        return cls(links, table, aabb_min, aabb_max, device=dev)

    @classmethod
    def empty(cls, dims, aabb_min, aabb_max, device=None) -> "SparseGrid":
        dims = tuple(int(d) for d in dims)
        dev = _dev(device)
        return cls(torch.full(dims, EMPTY, dtype=torch.int32, device=dev),
                   torch.zeros((0, ROW), dtype=torch.float32, device=dev),
                   aabb_min, aabb_max, device=dev)

    # -- storage ------------------------------------------------------------
    @property
    def links(self) -> torch.Tensor:
        return self._links

    @links.setter
    def links(self, value) -> None:
        self._links = torch.as_tensor(value).to(self._links.device, torch.int32).contiguous()
        self._cell_occ = None
        self._lat = None
        self._row_cell = None
        self._bricks = None

    @property
    def table(self) -> torch.Tensor:
        """The reference's (rows, 28) table: a fresh tensor, column 0 = sigma."""
        t = self.sh.clone()
        t[:, 0] = self.density
        return t

    @table.setter
    def table(self, value) -> None:
        t = torch.as_tensor(value)
        dev = self._links.device
        if t.dim() != 2 or t.shape[1] != ROW:
            raise ValueError(f"table must be (rows, {ROW})")
        same_rows = hasattr(self, "density") and int(self.density.shape[0]) == int(t.shape[0])
        if same_rows:   # in place: descriptors cached by callers stay valid
            self.density.copy_(t[:, 0])
            self.sh.copy_(t)
            self.sh[:, 0] = 0.0
            if getattr(self, "_lat", None) is not None:
                self.invalidate()
            return
        self.density = t[:, 0].to(device=dev, dtype=torch.float32).contiguous()
        self.sh = row_array(t.shape[0], dev, zero=False)
        self.sh.copy_(t)
        self.sh[:, 0] = 0.0
        self._lat = None
        self._row_cell = None
        self._bricks = None

    @property
    def device(self):
        return self._links.device

    @property
    def dims(self) -> tuple[int, int, int]:
        return tuple(int(d) for d in self._links.shape)

    @property
    def n_rows(self) -> int:
        return int(self.density.shape[0])

    @property
    def extent(self) -> np.ndarray:
        return self.aabb_max - self.aabb_min

    @property
    def voxel_size(self) -> np.ndarray:
        return self.extent / (np.array(self.dims, dtype=np.float64) - 1.0)

    @property
    def lattice_scale(self) -> np.ndarray:
        return (np.array(self.dims, dtype=np.float64) - 1.0) / self.extent

    def world_to_lattice(self, pts) -> np.ndarray:
        return (np.asarray(pts, dtype=np.float64) - self.aabb_min) * self.lattice_scale

    def lattice_to_world(self, ijk) -> np.ndarray:
        return self.aabb_min + np.asarray(ijk, dtype=np.float64) * self.voxel_size

    def invalidate(self) -> None:
        """Call after editing `links` or `density` in place: rebuilds the
        derived structures (cell occupancy bitmask, lattice sigma mirror,
        row -> cell map).  Density edits are absorbed in place (cached
        descriptors stay valid); after a links edit rebuild descriptors too
        (the mirror may stop or start aliasing `density`)."""
        c = self._c(with_occ=False, with_lat=False)
        L, s = _lib.lib(), _lib.stream_ptr()
        if self._cell_occ is not None:
            _lib.check(L.plx_build_cell_occ(ctypes.byref(c), self._cell_occ.data_ptr(), s),
                       "build_cell_occ")
        if self._lat is not None:
            aliased = self._lat.data_ptr() == self.density.data_ptr()
            ncell = int(np.prod(self.dims))
            identity = self.n_rows == ncell and bool(torch.equal(
                self._links.view(-1), torch.arange(ncell, dtype=torch.int32, device=self.device)))
            if aliased != identity:
                self._lat = None
                self._row_cell = None
                self._bricks = None
                self.lattice_sigma()
                return
            if self._row_cell is not None and self.n_rows and not aliased:
                _lib.check(L.plx_build_row_cell(ctypes.byref(c), self._row_cell.data_ptr(), s),
                           "build_row_cell")
            if not aliased:
                _lib.check(L.plx_build_sigma_lat(ctypes.byref(c), self._lat.data_ptr(), s),
                           "build_sigma_lat")
                self.rebuild_bricks()

    def cell_occ(self) -> torch.Tensor:
        if self._cell_occ is None:
            words = _lib.load().plx_cell_occ_words(_lib.dims_array(self.dims))
            occ = torch.empty(int(words), dtype=torch.int32, device=self.device)
            c = self._c(with_occ=False, with_lat=False)
            _lib.check(_lib.lib().plx_build_cell_occ(ctypes.byref(c), occ.data_ptr(),
                                                     _lib.stream_ptr()), "build_cell_occ")
            self._cell_occ = occ
        return self._cell_occ

    def lattice_sigma(self):
        """(sigma_lat, row_cell): the lattice-indexed density mirror (NaN at
        empty points) and the row -> lattice point map.  Built on first use;
        from then on every descriptor of this grid carries them, the march
        reads corner sigmas from the mirror in one gather level, and the
        optimisers keep it current."""
        if self._lat is None:
            ncell = int(np.prod(self.dims))
            if self.n_rows == ncell and bool(torch.equal(
                    self._links.view(-1), torch.arange(ncell, dtype=torch.int32,
                                                       device=self.device))):
                # identity-linked dense grid: the mirror IS the density array
                self._row_cell = torch.arange(ncell, dtype=torch.int32, device=self.device)
                self._lat = self.density
                return self._lat, self._row_cell
            c = self._c(with_occ=False, with_lat=False)
            L, s = _lib.lib(), _lib.stream_ptr()
            rc = torch.empty(max(self.n_rows, 1), dtype=torch.int32, device=self.device)
            if self.n_rows:
                _lib.check(L.plx_build_row_cell(ctypes.byref(c), rc.data_ptr(), s),
                           "build_row_cell")
            lat = torch.empty(int(np.prod(self.dims)), dtype=torch.float32, device=self.device)
            _lib.check(L.plx_build_sigma_lat(ctypes.byref(c), lat.data_ptr(), s),
                       "build_sigma_lat")
            self._row_cell, self._lat = rc, lat
            if USE_BRICKS and getattr(self, "use_bricks", True):
                self._bricks = torch.empty(int(L.plx_brick_words(_lib.dims_array(self.dims))),
                                           dtype=torch.int32, device=self.device)
                self.rebuild_bricks()
        return self._lat, self._row_cell

    def rebuild_bricks(self) -> None:
        """Recompute the dead-brick mask from the sigma mirror.  The
        optimisers only clear bits (a brick revives when a corner's sigma
        becomes >= 0), so the mask tightens only here: the trainer calls this
        periodically."""
        if getattr(self, "_bricks", None) is None:
            return
        c = self._c(with_occ=False, with_lat=False)
        _lib.check(_lib.lib().plx_build_brick_dead(ctypes.byref(c), self._bricks.data_ptr(),
                                                   _lib.stream_ptr()), "build_brick_dead")

    def disable_bricks(self) -> None:
        """No dead-brick mask on this grid (the N-GPU owner update keeps the
        peers' sigma mirrors but not their masks).  A mask already built is
        cleared (no brick dead) and kept alive, so descriptors made before
        this call stay valid; new descriptors carry none."""
        self.use_bricks = False
        if getattr(self, "_bricks", None) is not None:
            self._bricks.zero_()
            self._bricks_retired = self._bricks
        self._bricks = None

    def _c(self, with_occ: bool = True, with_lat: bool | None = None) -> _lib.PlxGrid:
        """Kernel descriptor.  with_lat (default: with_occ) builds the
        lattice sigma mirror; once built it is always attached, so that the
        optimisers keep it current."""
        g = _lib.PlxGrid()
        g.links = self._links.data_ptr()
        g.table = self.sh.data_ptr() if self.n_rows else None
        g.density = self.density.data_ptr() if self.n_rows else None
        g.dims = _lib.dims_array(self.dims)
        g.rows = self.n_rows
        g.lo = (ctypes.c_double * 3)(*self.aabb_min)
        g.hi = (ctypes.c_double * 3)(*self.aabb_max)
        g.scale = (ctypes.c_double * 3)(*self.lattice_scale)
        g.dmax = (ctypes.c_double * 3)(*(np.array(self.dims, dtype=np.float64) - 1.0))
        if with_lat is None:
            with_lat = with_occ and USE_CELL_OCC
        if (with_lat or self._lat is not None) and self.n_rows:
            lat, rc = self.lattice_sigma()
            g.sigma_lat = lat.data_ptr()
            g.row_cell = rc.data_ptr()
            bricks = getattr(self, "_bricks", None)
            g.brick_dead = bricks.data_ptr() if bricks is not None else None
        # the cell-occupancy bitmask skips empty space; a fully occupied
        # (identity-linked) grid has none, and with the sigma mirror the test
        # would only add a dependent load to every march position
        dense = self._lat is not None and self._lat.data_ptr() == self.density.data_ptr()
        g.cell_occ = (self.cell_occ().data_ptr() if (with_occ and USE_CELL_OCC and not dense)
                      else None)
        return g

    def to_numpy(self):
        """(links int32 (Dx,Dy,Dz), table float32 (rows, 28)) host copies."""
        return self._links.cpu().numpy(), self.table.cpu().numpy()

    def copy(self) -> "SparseGrid":
        return SparseGrid(self._links.clone(), self.table, self.aabb_min.copy(),
                          self.aabb_max.copy(), device=self.device)

    def occupancy(self) -> torch.Tensor:
        return self._links >= 0

    # -- structure ops ------------------------------------------------------
    def _compact(self, flags: torch.Tensor):
        """flags (ncell uint8) -> (new_links int32 (ncell), n) via plx_scan_ids."""
        n = flags.numel()
        L = _lib.lib()
        scratch = torch.empty(int(L.plx_scan_scratch_bytes(n)), dtype=torch.uint8,
                              device=self.device)
        ids = torch.empty(n, dtype=torch.int32, device=self.device)
        count = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(L.plx_scan_ids(flags.data_ptr(), n, ids.data_ptr(), count.data_ptr(),
                                  scratch.data_ptr(), _lib.stream_ptr()), "scan_ids")
        return ids, int(count.item())

    def prune(self, criterion: str, threshold: float, weights=None):
        """G:228-258 -> (new_grid, kept_old_rows torch.int64)."""
        if criterion == "weight":
            if weights is None:
                raise ValueError("weight criterion needs per-row max weights")
            w = torch.as_tensor(weights).to(self.device, torch.float64).contiguous()
            if tuple(w.shape) != (self.n_rows,):
                raise ValueError("weights must have one entry per data row")
        elif criterion == "density":
            w = None
        else:
            raise ValueError(f"unknown prune criterion {criterion!r}")
        L = _lib.lib()
        ncell = int(np.prod(self.dims))
        scratch = torch.empty(2 * ncell, dtype=torch.uint8, device=self.device)
        flags = torch.empty(ncell, dtype=torch.uint8, device=self.device)
        c = self._c(with_occ=False)
        s = _lib.stream_ptr()
        _lib.check(L.plx_prune_mark(ctypes.byref(c), _lib.ptr(w), float(threshold),
                                    scratch.data_ptr(), flags.data_ptr(), s), "prune_mark")
        del scratch
        ids, n_keep = self._compact(flags)
        kept = torch.empty(max(n_keep, 1), dtype=torch.int64, device=self.device)
        grid = SparseGrid._from_parts(ids.reshape(self.dims), n_keep, self.aabb_min,
                                      self.aabb_max, self.device)
        if n_keep:
            _lib.check(L.plx_prune_apply(ctypes.byref(c), ids.data_ptr(), kept.data_ptr(),
                                         grid.sh.data_ptr(), grid.density.data_ptr(), s),
                       "prune_apply")
        return grid, kept[:n_keep]

    def upsample(self, new_dims) -> "SparseGrid":
        """G:260-285.  A 0-row grid upsamples to an empty grid (the reference
        raises IndexError there, G:277-278)."""
        new_dims = tuple(int(d) for d in new_dims)
        if any(d < 2 for d in new_dims):
            raise ValueError("upsample needs at least 2 points per axis")
        if self.n_rows == 0:
            return SparseGrid.empty(new_dims, self.aabb_min, self.aabb_max, device=self.device)
        L = _lib.lib()
        nd = _lib.dims_array(new_dims)
        ncell = int(np.prod(new_dims))
        flags = torch.empty(ncell, dtype=torch.uint8, device=self.device)
        c = self._c(with_occ=False)
        s = _lib.stream_ptr()
        _lib.check(L.plx_upsample_mark(ctypes.byref(c), nd, flags.data_ptr(), s),
                   "upsample_mark")
        ids, n_new = self._compact(flags)
        del flags
        grid = SparseGrid._from_parts(ids.reshape(new_dims), n_new, self.aabb_min,
                                      self.aabb_max, self.device)
        if n_new:
            _lib.check(L.plx_upsample_apply(ctypes.byref(c), nd, ids.data_ptr(),
                                            grid.sh.data_ptr(), grid.density.data_ptr(), s),
                       "upsample_apply")
        return grid

    # -- point sampling (G:141-223) -------------------------------------------
    def _check_inside(self, pts: torch.Tensor) -> None:
        """G:147-151."""
        tol = 1e-9 * float(np.max(self.extent))
        lo = torch.as_tensor(self.aabb_min, dtype=torch.float64, device=pts.device)
        hi = torch.as_tensor(self.aabb_max, dtype=torch.float64, device=pts.device)
        if bool(torch.any(pts < lo - tol)) or bool(torch.any(pts > hi + tol)):
            raise ValueError("sample position outside the grid AABB")

    def _points(self, pts):
        as_np = not isinstance(pts, torch.Tensor)
        t = torch.as_tensor(np.asarray(pts, dtype=np.float64) if as_np else pts,
                            dtype=torch.float64).to(self.device)
        single = t.dim() == 1
        t = t.reshape(-1, 3).contiguous()
        self._check_inside(t)
        return t, as_np, single

    def sample(self, pts, mode: str = "trilinear"):
        """G:182-200: interpolated (sigma, coeffs) at world positions inside
        the AABB (plx_grid_sample); sigma clamped at zero, empty corners read
        zero.  A single (3,) point gives (float, (27,)); a batch (N, 3) gives
        ((N,), (N, 27)) float64 -- numpy for numpy input."""
        if mode not in ("trilinear", "nearest"):
            raise ValueError(f"unknown interpolation mode {mode!r}")
        t, as_np, single = self._points(pts)
        out = torch.zeros((t.shape[0], ROW_SIZE), dtype=torch.float64, device=self.device)
        if self.n_rows and t.shape[0]:
            c = self._c(with_occ=False)
            _lib.check(_lib.lib().plx_grid_sample(ctypes.byref(c), t.data_ptr(), t.shape[0],
                                                  int(mode == "nearest"), out.data_ptr(),
                                                  _lib.stream_ptr()), "grid_sample")
        sigma, coeffs = out[:, 0], out[:, 1:]
        if as_np:
            sigma, coeffs = sigma.cpu().numpy(), coeffs.cpu().numpy()
        if single:
            return float(sigma[0]), coeffs[0]
        return sigma, coeffs

    def sample_backward(self, pts, upstream, grads: GradientBuffer,
                        mode: str = "trilinear") -> None:
        """G:202-223: adjoint of sample() -- upstream (N, 28) dL/d(sigma,
        coeffs) times each stencil weight added to the occupied corner rows of
        `grads` (plx_grid_sample_backward); the sigma entry is dropped where
        the interpolated sigma was clamped (< 0)."""
        if mode not in ("trilinear", "nearest"):
            raise ValueError(f"unknown interpolation mode {mode!r}")
        if grads.n_rows != self.n_rows:
            raise ValueError("gradient buffer rows do not match the grid table")
        t, _, _ = self._points(pts)
        up = torch.as_tensor(np.asarray(upstream, dtype=np.float64)
                             if not isinstance(upstream, torch.Tensor) else upstream,
                             dtype=torch.float64).to(self.device).reshape(-1, ROW_SIZE)
        if up.shape[0] != t.shape[0]:
            raise ValueError("one upstream row of 28 values per point")
        up = up.contiguous()
        if self.n_rows and t.shape[0]:
            c, gb = self._c(with_occ=False), grads._c(with_ids=False)
            _lib.check(_lib.lib().plx_grid_sample_backward(
                ctypes.byref(c), t.data_ptr(), up.data_ptr(), t.shape[0],
                int(mode == "nearest"), ctypes.byref(gb), _lib.stream_ptr()),
                "grid_sample_backward")

    def max_weight_accumulate(self, origins, dirs, step_frac: float = 0.5,
                              stop_thresh: float = 1e-4, interp: str = "trilinear",
                              chunk: int = 1 << 22):
        """G:287-302: per-row max of T*(1-exp(-sigma*delta)) over the rays.
        Returns float64 weights (numpy if the inputs are numpy)."""
        from .render import _ray_tensor
        as_np = not isinstance(origins, torch.Tensor)
        o = _ray_tensor(origins, self.device)
        d = _ray_tensor(dirs, self.device)
        out = torch.zeros(self.n_rows, dtype=torch.float64, device=self.device)
        step = step_frac * float(np.min(self.voxel_size))
        opts = _lib.make_opts(step, stop_thresh, (0, 0, 0), interp == "nearest", False)
        c = self._c()
        L = _lib.lib()
        for s0 in range(0, o.shape[0], chunk):
            r = _lib.PlxRays()
            r.origins = o[s0:s0 + chunk].data_ptr()
            r.dirs = d[s0:s0 + chunk].data_ptr()
            r.n = min(chunk, o.shape[0] - s0)
            _lib.check(L.plx_max_weight(ctypes.byref(c), ctypes.byref(r), ctypes.byref(opts),
                                        out.data_ptr(), _lib.stream_ptr()), "max_weight")
        return out.cpu().numpy() if as_np else out

    def max_weight_accumulate_pool(self, pool, first: int = 0, count: int | None = None,
                                   step_frac: float = 0.5, stop_thresh: float = 1e-4,
                                   interp: str = "trilinear", chunk: int = 1 << 22):
        """max_weight_accumulate (G:287-302) over the rays of camera-pool rows
        [first, first + count), generated in the kernel.  -> device float64."""
        count = pool.n - first if count is None else int(count)
        out = torch.zeros(self.n_rows, dtype=torch.float64, device=self.device)
        step = step_frac * float(np.min(self.voxel_size))
        opts = _lib.make_opts(step, stop_thresh, (0, 0, 0), interp == "nearest", False)
        c = self._c()
        L = _lib.lib()
        for s0 in range(first, first + count, chunk):
            n = min(chunk, first + count - s0)
            idx = torch.arange(s0, s0 + n, dtype=torch.int64, device=self.device)
            r = pool.rays(idx)
            _lib.check(L.plx_max_weight(ctypes.byref(c), ctypes.byref(r), ctypes.byref(opts),
                                        out.data_ptr(), _lib.stream_ptr()), "max_weight")
        return out

    # -- consistency --------------------------------------------------------
    def validate(self) -> None:
        """G:306-316: links/table bijection and finite values."""
        rows = self._links[self._links >= 0].long()
        if rows.numel() != self.n_rows:
            raise AssertionError("row count does not match occupied cells")
        if rows.numel():
            counts = torch.bincount(rows, minlength=self.n_rows)
            if int(rows.max()) >= self.n_rows or not bool(torch.all(counts == 1)):
                raise AssertionError("links and table rows are not a bijection")
        if not (bool(torch.all(torch.isfinite(self.sh))) and
                bool(torch.all(torch.isfinite(self.density)))):
            raise AssertionError("non-finite values in data table")
