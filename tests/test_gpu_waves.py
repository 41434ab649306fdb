"""Batches larger than one wave of records (the record budget, 64 GiB, is
reached at C5-size batches) render in waves; every wave-sliced entry point
(array rays, upstream mode with jitter, the 360 backward, the trainer's
camera-pool / CUDA-graph step) must give the single-wave results.  A small
PLX_RECORD_MB forces 1024-ray waves on 3000-ray batches; each run is its own
process (the budget is read once).  The spatial segment order of large
waves (PLX_SEG_ORDER=1 forces it at these sizes) and the unpacked record
layout of very large lattices (PLX_PACK=0) must not change results either."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, name, env_extra):
    out = str(tmp_path / f"{name}.npz")
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, os.path.join(HERE, "multiwave_case.py"), out], env=env,
                   check=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("variant", ["waves", "ordered", "ordered_waves", "unpacked"])
def test_multi_wave_batches_match_one_wave(tmp_path, variant):
    one = _run(tmp_path, "one", {"PLX_SEG_ORDER": "0"})
    env = {"waves": {"PLX_RECORD_MB": "1", "PLX_SEG_ORDER": "0"},
           "ordered": {"PLX_SEG_ORDER": "1"},
           "ordered_waves": {"PLX_RECORD_MB": "1", "PLX_SEG_ORDER": "1"},
           "unpacked": {"PLX_SEG_ORDER": "0", "PLX_PACK": "0"}}[variant]
    many = _run(tmp_path, variant, env)
    for k in one.files:
        a, b = one[k], many[k]
        if k.endswith("touched"):
            np.testing.assert_array_equal(a, b, err_msg=k)
        elif k.endswith("grad") or k.startswith("train"):
            scale = max(float(np.max(np.abs(a))), 1e-30)
            np.testing.assert_allclose(b, a, rtol=1e-4, atol=1e-6 * scale, err_msg=k)
        else:   # per-ray values: the same arithmetic in either wave layout
            np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-15, err_msg=k)
