"""The MSI background block of the `.plnx` container and the background
state of the `.state` sidecar, byte-compatible with the reference
(artifact_io.py:42-62, 110-133, 138-191): a container written by the
reference (tests/golden/make_msi_golden.py) parses and re-serialises to the
identical bytes.  Host-only."""

import os

import numpy as np

from paper_2112_05131_b200 import artifact_io as aio

from helpers import GOLDEN


def test_background_container_roundtrip_is_byte_identical():
    path = os.path.join(GOLDEN, "msi_grid.plnx")
    links, table, lo, hi, radii, bgdata = aio.read_plnx_full(path)
    assert bgdata.shape == (3, 4, 6, 4) and radii.shape == (3,)
    assert np.isinf(radii[-1]) and np.all(np.diff(radii) > 0)
    raw = open(path, "rb").read()
    assert aio.plnx_bytes(links, table, lo, hi, radii, bgdata) == raw
    # the grid-only reader still accepts it
    l2, t2, _, _ = aio.read_plnx(path)
    np.testing.assert_array_equal(l2, links)
    np.testing.assert_array_equal(t2, table)


def test_background_state_roundtrip_is_byte_identical():
    path = os.path.join(GOLDEN, "msi_grid.plnx.state")
    v, step, beta, eps, bg_v = aio.read_state_full(path)
    assert step == 1234 and bg_v.shape == (3 * 4 * 6, 4)
    assert aio.state_bytes(v, step, beta, eps, bg_v) == open(path, "rb").read()
