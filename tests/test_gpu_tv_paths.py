"""Both TV kernels (tv_dense_kernel on identity-linked grids, the two-phase
tv_sparse_kernel otherwise) against the oracle's restatement of K:456-569
(L:50-77), at sizes where every block runs several iterations: a contiguous
wrapped run and an explicit cell list with repeats, with and without the
periodic boundaries."""
import numpy as np
import pytest

from oracle import oracle as orc

from helpers import grad_close, random_grid

pytestmark = pytest.mark.gpu


def px():
    import paper_2112_05131_b200 as m
    return m


def dev_grid(g):
    d = px().SparseGrid(g.links, g.table.astype(np.float32), g.aabb_min, g.aabb_max)
    d.lattice_sigma()   # identity-linked grids then take the dense kernel (mirror = density)
    return d


@pytest.mark.parametrize("holes", [0.0, 0.85])
@pytest.mark.parametrize("wrap", [(False, False, False), (True, False, True)])
def test_tv_kernels_match_oracle(holes, wrap):
    rng = np.random.default_rng(17)
    g = random_grid(rng, dims=(70, 64, 66), holes=holes, sigma_range=(-1, 1), dc_range=(-1, 1),
                    band_scale=0.8)
    dg = dev_grid(g)
    ncell = int(np.prod(g.dims))
    run = px().losses.CellRun(int(rng.integers(0, ncell)), int(0.4 * ncell), ncell)
    lists = {"run": run, "list": rng.integers(0, ncell, 50_000)}
    for name, cells in lists.items():
        bo = orc.GradBuf(g.n_rows)
        a0, b0 = orc.tv_loss(g, np.asarray(cells), 1e-5, 1e-3, bo, wrap=wrap)
        bd = px().GradientBuffer(dg.n_rows)
        a1, b1 = px().tv_loss(dg, cells, 1e-5, 1e-3, bd, wrap=wrap)
        assert a1 == pytest.approx(a0, rel=1e-9), name
        assert b1 == pytest.approx(b0, rel=1e-9), name
        np.testing.assert_array_equal(bd.touched_rows(), bo.touched_rows(), err_msg=name)
        ok, worst, nbad = grad_close(bd.dense(), bo.data)
        assert ok, (name, worst, nbad)
