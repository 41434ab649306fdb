"""The reference's `.plnx` artifact behaviours (pkg/tests/test_io.py:25-122)
on the device package: round trips (values, background, re-save byte
identity), the file-size arithmetic of an empty grid, detection of corrupt,
truncated and foreign files, and the checkpoint sidecar."""

import struct
import zlib

import numpy as np
import pytest
import torch

from helpers import random_grid

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as m
    return m


def _file_grid(rng):
    g = random_grid(rng, dims=tuple(int(x) for x in rng.integers(2, 7, 3)),
                    holes=float(rng.uniform(0, 0.6)), sigma_range=(-2.0, 5.0),
                    dc_range=(-1.0, 1.0), band_scale=1.0)
    return px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)


def test_round_trips_are_exact_and_resaves_byte_identical(tmp_path):
    m = px()
    rng = np.random.default_rng(0)
    for i in range(10):
        g = _file_grid(rng)
        path = tmp_path / f"g{i}.plnx"
        m.save_grid(g, path)
        g2, bg = m.load_grid(path)
        assert bg is None and g2.dims == g.dims
        np.testing.assert_array_equal(g2.links.cpu().numpy(), g.links.cpu().numpy())
        np.testing.assert_array_equal(g2.table.cpu().numpy(), g.table.cpu().numpy())
        np.testing.assert_array_equal(g2.aabb_min, g.aabb_min)
        m.save_grid(g2, tmp_path / "resave.plnx")
        assert (tmp_path / "resave.plnx").read_bytes() == path.read_bytes()
    bgd = m.msi.MsiBackground.create(5, 6, 8)
    bgd.data[:] = torch.as_tensor(rng.uniform(0, 1, tuple(bgd.data.shape)).astype(np.float32))
    m.save_grid(g, tmp_path / "b.plnx", bgd)
    _, bg2 = m.load_grid(tmp_path / "b.plnx")
    np.testing.assert_array_equal(bg2.data.cpu().numpy(), bgd.data.cpu().numpy())
    np.testing.assert_array_equal(bg2.radii, bgd.radii)


def test_empty_grid_file_size(tmp_path):
    m = px()
    m.save_grid(m.SparseGrid.empty((2, 2, 2), (0, 0, 0), (1, 1, 1)), tmp_path / "e.plnx")
    # magic, version, dims, aabb, degree, row count, 8 links, background flag, crc
    assert (tmp_path / "e.plnx").stat().st_size == 4 + 4 + 12 + 48 + 1 + 8 + 8 * 4 + 1 + 4


def test_damaged_and_foreign_files_are_rejected(tmp_path):
    m = px()
    rng = np.random.default_rng(2)
    path = tmp_path / "g.plnx"
    m.save_grid(_file_grid(rng), path)
    good = path.read_bytes()
    for _ in range(5):                                # any flipped byte fails the CRC
        raw = bytearray(good)
        raw[int(rng.integers(0, len(raw)))] ^= 0x5A
        path.write_bytes(bytes(raw))
        with pytest.raises(m.GridFileError):
            m.load_grid(path)
    path.write_bytes(good[:-9])
    with pytest.raises(m.GridFileError):
        m.load_grid(path)
    payload = b"NOPE" + b"\x00" * 40
    path.write_bytes(payload + struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF))
    with pytest.raises(m.GridFileError, match="magic"):
        m.load_grid(path)


def test_checkpoint_round_trip(tmp_path):
    m = px()
    rng = np.random.default_rng(5)
    g = _file_grid(rng)
    st = m.OptimState(g.n_rows)
    st.v.copy_(torch.as_tensor(rng.uniform(0, 1, tuple(st.v.shape)).astype(np.float32)))
    st.step_count = 7
    m.save_checkpoint(tmp_path / "c.plnx", g, st, step=123)
    g2, bg2, st2, bgs2, step = m.load_checkpoint(tmp_path / "c.plnx")
    assert step == 123 and st2.step_count == 123 and bg2 is None and bgs2 is None
    np.testing.assert_array_equal(st2.v.cpu().numpy(), st.v.cpu().numpy())
    np.testing.assert_array_equal(g2.table.cpu().numpy(), g.table.cpu().numpy())
