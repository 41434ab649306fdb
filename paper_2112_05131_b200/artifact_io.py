"""`.plnx` grid container and `.state` optimiser sidecar, byte-compatible with
the reference (pkg/src/plenoxel/artifact_io.py:1-191).

Layout (little-endian): "PLNX", u32 version=1, 3*u32 dims, 6*f64 aabb, u8 SH
degree (2), u64 rows, links Dx*Dy*Dz i32 in x-fastest order, table rows*28
f32, u8 background flag, u32 CRC32 over everything before it.  The MSI
background block (flag 1) is parsed and skipped: no BASELINE config is 360°.

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


def plnx_bytes(links: np.ndarray, table: np.ndarray, aabb_min, aabb_max) -> bytes:
    """Serialise (artifact_io.py:42-62, no background) including the CRC."""
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
    buf += struct.pack("<B", 0)
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
    if bg_flag == 1:
        (n_layers,) = r.unpack("<H")
        width, height = r.unpack("<2I")
        r.take(8 * n_layers)
        r.take(16 * n_layers * height * width)
    elif bg_flag != 0:
        raise GridFileError(f"{path}: bad background flag {bg_flag}")
    if r.off != len(r.data):
        raise GridFileError(f"{path}: {len(r.data) - r.off} trailing bytes")
    return links, table, np.array(aabb[:3]), np.array(aabb[3:])


def save_grid(grid, path) -> None:
    """Write a device SparseGrid (artifact_io.py:65-69)."""
    links, table = grid.to_numpy()
    Path(path).write_bytes(plnx_bytes(links, table, grid.aabb_min, grid.aabb_max))


def load_grid(path, device="cuda"):
    """Read a container into a device SparseGrid; returns (grid, None)."""
    from .grid import SparseGrid

    links, table, lo, hi = read_plnx(path)
    return SparseGrid(links, table, lo, hi, device=device), None


def state_bytes(v: np.ndarray, step: int, beta: float, eps: float) -> bytes:
    """The `.state` sidecar (artifact_io.py:138-156), no background state."""
    buf = bytearray()
    buf += STATE_MAGIC
    buf += struct.pack("<I", VERSION)
    buf += struct.pack("<Q", int(step))
    buf += struct.pack("<2d", beta, eps)
    buf += struct.pack("<2Q", *v.shape)
    buf += np.asarray(v).astype("<f4").tobytes()
    buf += struct.pack("<B", 0)
    return bytes(buf) + struct.pack("<I", zlib.crc32(bytes(buf)) & 0xFFFFFFFF)


def save_checkpoint(path, grid, state, step: int) -> None:
    save_grid(grid, path)
    v = state.v.detach().cpu().numpy() if hasattr(state.v, "detach") else state.v
    Path(str(path) + ".state").write_bytes(state_bytes(v, step, state.beta, state.eps))


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
