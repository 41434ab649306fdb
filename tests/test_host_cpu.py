"""Host logic of the trainer that needs no GPU: the device mirror of the
reference's EpochBatcher (T:233-255) and the RNG draw order of the step body
(T:441-466)."""

import numpy as np
import pytest


@pytest.mark.parametrize("n,batch", [(10, 4), (409600, 3000), (7, 7), (5, 11), (12, 4)])
def test_epoch_batcher_device_mirror_across_epochs(n, batch):
    """next_slice()/next_device() return exactly next()'s indices, including
    batches that straddle an epoch boundary (the old epoch's tail is a view of
    the permutation buffer the new permutation is copied into)."""
    from paper_2112_05131_b200.trainer import EpochBatcher

    host = EpochBatcher(n, batch, np.random.default_rng(3))
    dev = EpochBatcher(n, batch, np.random.default_rng(3), device="cpu")
    steps = max(4, 3 * (n // batch + 1)) if n < 1000 else 300
    seen_cross = False
    for _ in range(steps):
        want = host.next()
        got, off = dev.next_slice()
        np.testing.assert_array_equal(got.numpy(), want)
        if off is None:
            seen_cross = True
        else:
            np.testing.assert_array_equal(dev._dev_perm()[off:off + batch].numpy(), want)
    if n % batch:
        assert seen_cross


def test_epoch_batcher_epoch_is_a_permutation():
    """Every index appears exactly once per epoch (T:233-235)."""
    from paper_2112_05131_b200.trainer import EpochBatcher

    n, batch = 10, 4
    b = EpochBatcher(n, batch, np.random.default_rng(0), device="cpu")
    drawn = np.concatenate([b.next_device().numpy().copy() for _ in range(5)])   # 20 = 2 epochs
    for e in range(2):
        assert sorted(drawn[e * n:(e + 1) * n]) == list(range(n))
