"""`.plnx` grid container and `.state` optimiser sidecar, byte-compatible with
the reference (pkg/src/plenoxel/artifact_io.py:1-191).

Layout (little-endian): "PLNX", u32 version=1, 3*u32 dims, 6*f64 aabb, u8 SH
degree (2), u64 rows, links Dx*Dy*Dz i32 in x-fastest order, table rows*28
f32, u8 background flag [, MSI block: u16 layers, u32 width, u32 height,
layers*f64 radii, layers*H*W*4 f32 texels], u32 CRC32 over everything before
it.  The `.state` sidecar carries the background's RMSProp state after the
grid's (flag 1).

The device grid already stores f32, so save -> load -> save is byte-identical
without the reference's f64 -> f32 quantisation step.
"""

from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np

MAGIC = b"PLNX"
STATE_MAGIC = b"PLNS"
VERSION = 1


class GridFileError(ValueError):
    pass


def plnx_bytes(links: np.ndarray, table: np.ndarray, aabb_min, aabb_max, bg_radii=None,
               bg_data=None) -> bytes:
    """Serialise (artifact_io.py:42-62) including the CRC; bg_radii (L,) and
    bg_data (L, H, W, 4) add the MSI background block."""
    links = np.asarray(links)
    buf = bytearray()
    buf += MAGIC
    buf += struct.pack("<I", VERSION)
    buf += struct.pack("<3I", *links.shape)
    buf += struct.pack("<6d", *np.asarray(aabb_min, np.float64).reshape(3),
                       *np.asarray(aabb_max, np.float64).reshape(3))
    buf += struct.pack("<B", 2)
    buf += struct.pack("<Q", int(table.shape[0]))
    buf += np.ravel(links, order="F").astype("<i4").tobytes()
    with np.errstate(over="ignore"):
        buf += np.asarray(table).astype("<f4").tobytes()
    if bg_data is None:
        buf += struct.pack("<B", 0)
    else:
        bg_data = np.asarray(bg_data)
        n_layers, height, width, _ = bg_data.shape
        buf += struct.pack("<B", 1)
        buf += struct.pack("<H", n_layers)
        buf += struct.pack("<2I", width, height)
        buf += np.asarray(bg_radii, np.float64).astype("<f8").tobytes()
        buf += bg_data.astype("<f4").tobytes()
    payload = bytes(buf)
    return payload + struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF)


class _Reader:
    def __init__(self, data: bytes, path):
        self.data, self.off, self.path = data, 0, path

    def take(self, n: int) -> bytes:
        if self.off + n > len(self.data):
            raise GridFileError(f"{self.path}: truncated file")
        out = self.data[self.off:self.off + n]
        self.off += n
        return out

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))


def read_plnx(path):
    """Parse a container (artifact_io.py:89-135) -> (links i32 C-order (Dx,Dy,Dz),
    table f32 (rows, 28), aabb_min, aabb_max).  Raises GridFileError."""
    return read_plnx_full(path)[:4]


def read_plnx_full(path):
    """read_plnx plus the MSI background block: (..., bg_radii f64 (L,) or
    None, bg_data f32 (L, H, W, 4) or None)."""
    data = Path(path).read_bytes()
    if len(data) < 8:
        raise GridFileError(f"{path}: truncated file")
    stored = struct.unpack("<I", data[-4:])[0]
    if zlib.crc32(data[:-4]) & 0xFFFFFFFF != stored:
        raise GridFileError(f"{path}: CRC32 mismatch (corrupt file)")
    r = _Reader(data[:-4], path)
    if r.take(4) != MAGIC:
        raise GridFileError(f"{path}: bad magic (not a grid file)")
    (version,) = r.unpack("<I")
    if version != VERSION:
        raise GridFileError(f"{path}: unsupported version {version}")
    dims = r.unpack("<3I")
    aabb = r.unpack("<6d")
    (degree,) = r.unpack("<B")
    if degree != 2:
        raise GridFileError(f"{path}: unsupported SH degree {degree}")
    (n_rows,) = r.unpack("<Q")
    n_cells = dims[0] * dims[1] * dims[2]
    links = np.frombuffer(r.take(4 * n_cells), dtype="<i4").reshape(dims, order="F")
    links = np.ascontiguousarray(links, dtype=np.int32)
    table = np.frombuffer(r.take(4 * 28 * n_rows), dtype="<f4").reshape(n_rows, 28)
    table = np.array(table, dtype=np.float32)
    if n_rows and (links.max() >= n_rows or np.count_nonzero(links >= 0) != n_rows):
        raise GridFileError(f"{path}: index lattice does not match row count")
    (bg_flag,) = r.unpack("<B")
    radii = bgdata = None
    if bg_flag == 1:
        (n_layers,) = r.unpack("<H")
        width, height = r.unpack("<2I")
        radii = np.frombuffer(r.take(8 * n_layers), dtype="<f8").astype(np.float64)
        bgdata = np.frombuffer(r.take(16 * n_layers * height * width), dtype="<f4")
        bgdata = bgdata.reshape(n_layers, height, width, 4).astype(np.float32)
    elif bg_flag != 0:
        raise GridFileError(f"{path}: bad background flag {bg_flag}")
    if r.off != len(r.data):
        raise GridFileError(f"{path}: {len(r.data) - r.off} trailing bytes")
    return links, table, np.array(aabb[:3]), np.array(aabb[3:]), radii, bgdata


def save_grid(grid, path, background=None) -> None:
    """Write a device SparseGrid (and MSI background) (artifact_io.py:65-69)."""
    links, table = grid.to_numpy()
    radii = data = None
    if background is not None:
        radii, data = background.radii, background.data.cpu().numpy()
    Path(path).write_bytes(plnx_bytes(links, table, grid.aabb_min, grid.aabb_max, radii, data))


def load_grid(path, device="cuda"):
    """Read a container into a device SparseGrid; returns (grid, background
    MsiBackground or None)."""
    from .grid import SparseGrid

    links, table, lo, hi, radii, bgdata = read_plnx_full(path)
    background = None
    if bgdata is not None:
        from .msi import MsiBackground
        background = MsiBackground(bgdata.astype(np.float64), radii, device=device)
    return SparseGrid(links, table, lo, hi, device=device), background


def state_bytes(v: np.ndarray, step: int, beta: float, eps: float, bg_v=None) -> bytes:
    """The `.state` sidecar (artifact_io.py:138-156); bg_v: the background's
    RMSProp state (L*H*W, 4)."""
    buf = bytearray()
    buf += STATE_MAGIC
    buf += struct.pack("<I", VERSION)
    buf += struct.pack("<Q", int(step))
    buf += struct.pack("<2d", beta, eps)
    buf += struct.pack("<2Q", *v.shape)
    buf += np.asarray(v).astype("<f4").tobytes()
    if bg_v is None:
        buf += struct.pack("<B", 0)
    else:
        bg_v = np.asarray(bg_v)
        buf += struct.pack("<B", 1)
        buf += struct.pack("<2Q", *bg_v.shape)
        buf += bg_v.astype("<f4").tobytes()
    return bytes(buf) + struct.pack("<I", zlib.crc32(bytes(buf)) & 0xFFFFFFFF)


def _host(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def save_checkpoint(path, grid, state, step: int, background=None, bg_state=None) -> None:
    """GridFile plus the optimiser-state sidecar (artifact_io.py:138-156)."""
    save_grid(grid, path, background)
    bg_v = _host(bg_state.v) if bg_state is not None else None
    Path(str(path) + ".state").write_bytes(state_bytes(_host(state.v), step, state.beta,
                                                       state.eps, bg_v))


def read_state(path):
    """Parse a `.state` sidecar -> (v f32 (rows, cols), step, beta, eps)."""
    data = Path(path).read_bytes()
    if len(data) < 8:
        raise GridFileError(f"{path}: truncated file")
    if zlib.crc32(data[:-4]) & 0xFFFFFFFF != struct.unpack("<I", data[-4:])[0]:
        raise GridFileError(f"{path}: CRC32 mismatch")
    r = _Reader(data[:-4], path)
    if r.take(4) != STATE_MAGIC:
        raise GridFileError(f"{path}: bad magic")
    (version,) = r.unpack("<I")
    if version != VERSION:
        raise GridFileError(f"{path}: unsupported version {version}")
    (step,) = r.unpack("<Q")
    beta, eps = r.unpack("<2d")
    rows, cols = r.unpack("<2Q")
    v = np.frombuffer(r.take(4 * rows * cols), dtype="<f4").reshape(rows, cols).copy()
    return v, step, beta, eps


def read_state_full(path):
    """read_state plus the background state: (v, step, beta, eps, bg_v or None)."""
    v, step, beta, eps = read_state(path)
    data = Path(path).read_bytes()[:-4]
    off = 4 + 4 + 8 + 16 + 16 + 4 * v.size
    (flag,) = struct.unpack("<B", data[off:off + 1])
    bg_v = None
    if flag == 1:
        rows, cols = struct.unpack("<2Q", data[off + 1:off + 17])
        bg_v = np.frombuffer(data[off + 17:off + 17 + 4 * rows * cols],
                             dtype="<f4").reshape(rows, cols).copy()
    elif flag != 0:
        raise GridFileError(f"{path}: bad background flag {flag}")
    return v, step, beta, eps, bg_v


def load_checkpoint(path, device="cuda"):
    """artifact_io.load_checkpoint (artifact_io.py:159-191): returns (grid,
    background, state, bg_state, step) on the device."""
    import torch

    from .optim import OptimState

    grid, background = load_grid(path, device=device)
    v, step, beta, eps, bg_v = read_state_full(str(path) + ".state")
    state = OptimState(grid.n_rows, beta=beta, eps=eps, device=device)
    state.v[:, :v.shape[1]].copy_(torch.from_numpy(v))
    state.step_count = step
    bg_state = None
    if bg_v is not None and background is not None:
        from .msi import BgOptimState
        bg_state = BgOptimState(background, beta=beta, eps=eps)
        bg_state.v.copy_(torch.from_numpy(bg_v.astype(np.float64)))
        bg_state.step_count = step
    return grid, background, state, bg_state, step
