"""The reference's training-loop behaviours (pkg/tests/test_trainer.py:135-241)
on the device trainer, on the same tiny toy data (4 views at 32^2 of the
toy scene; the reference writes it to disk, make_toy_dataset here keeps it
in memory).  Not restated: bit-for-bit run-to-run determinism
(test_trainer.py:146-161) -- the device accumulates gradients with f32
atomics, whose order varies; trajectories match the reference's within the
tolerances of tests/test_gpu_trainer.py instead."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    from paper_2112_05131_b200 import scenes
    train, test, _ = scenes.make_toy_dataset(n_views=4, res=32, n_test=2, grid_dim=16)
    return train, test


def _cfg(grid=8, steps=20, batch=64):
    from paper_2112_05131_b200 import trainer
    return trainer.toy_config(grid_dim=grid, total_steps=steps, batch_size=batch)


def test_zero_steps_returns_the_initialised_grid(tiny):
    import paper_2112_05131_b200 as px
    from paper_2112_05131_b200.sh import SH_C0
    cfg = _cfg(steps=0, batch=16)
    g = px.train(tiny[0], cfg).grid
    t = g.table.cpu().numpy()
    assert g.dims == (8, 8, 8)
    np.testing.assert_allclose(t[:, 0], cfg.init_sigma, rtol=1e-7)
    np.testing.assert_allclose(t[:, 1::9], cfg.init_rgb / SH_C0, rtol=1e-7)
    assert np.all(t[:, 2:9] == 0)


def test_loss_and_gradient_sparsity_decrease(tiny):
    import paper_2112_05131_b200 as px
    cfg = _cfg(grid=16, steps=300, batch=256)
    cfg.log_every = 10
    res = px.train(tiny[0], cfg)
    losses = [m["loss"] for m in res.metrics if "loss" in m]
    fracs = [m["nnz_fraction"] for m in res.metrics if "nnz_fraction" in m]
    assert losses[12] < 0.5 * losses[0]          # by step 120, as the reference asserts
    assert fracs[-1] < fracs[0]


def test_ladder_event_prunes_then_upsamples(tiny):
    import paper_2112_05131_b200 as px
    cfg = _cfg(steps=40, batch=128)
    cfg.ladder = [px.LadderRung(0, (8, 8, 8)), px.LadderRung(20, (12, 12, 12))]
    cfg.prune_criterion, cfg.prune_threshold = "weight", 1e-5
    res = px.train(tiny[0], cfg, test_ds=tiny[1])
    assert res.grid.dims == (12, 12, 12)
    res.grid.validate()
    assert res.grid.n_rows < 12 ** 3


def test_upsample_resource_guard_names_the_dims(tiny):
    import paper_2112_05131_b200 as px
    from paper_2112_05131_b200.trainer import ResourceError
    cfg = _cfg(steps=40)
    cfg.ladder = [px.LadderRung(0, (8, 8, 8)), px.LadderRung(5, (4096, 4096, 4096))]
    with pytest.raises(ResourceError, match="4096"):
        px.train(tiny[0], cfg)


def test_eval_records_and_checkpoints(tiny, tmp_path):
    import paper_2112_05131_b200 as px
    cfg = _cfg(steps=20)
    cfg.eval_every = 10
    res = px.train(tiny[0], cfg, test_ds=tiny[1])
    evals = [m for m in res.metrics if "psnr" in m]
    assert [m["step"] for m in evals] == [10, 20]
    assert all(set(m) == {"step", "psnr", "ssim", "wall_time_s"} and m["wall_time_s"] > 0
               for m in evals)
    cfg = _cfg(steps=20)
    cfg.ladder = [px.LadderRung(0, (8, 8, 8)), px.LadderRung(10, (10, 10, 10))]
    cfg.prune_threshold = 1e-6
    out = tmp_path / "run"
    px.train(tiny[0], cfg, out_dir=out)
    assert (out / "checkpoint_0000010.plnx").exists() and (out / "final.plnx").exists()
    grid, bg, state, bg_state, step = px.load_checkpoint(out / "final.plnx")
    assert step == 20 and state.v.shape[0] == grid.n_rows


def test_trainer_accepts_any_dataset_with_the_reference_fields(tiny):
    """Dataset loading stays host-side (the reference's camera.load_nerf_dataset,
    camera.py:150-290): the trainer reads only `images`, `scene_type` and the
    cameras' c2w / focal / width / height / near / position, so the
    reference's own Dataset objects train as they are."""
    import types
    import paper_2112_05131_b200 as px
    train = tiny[0]
    cams = [types.SimpleNamespace(c2w=c.c2w.copy(), focal=c.focal, width=c.width,
                                  height=c.height, near=c.near, far=np.inf,
                                  position=c.c2w[:3, 3].copy()) for c in train.cameras]
    ds = types.SimpleNamespace(images=np.asarray(train.images), cameras=cams,
                               scene_type="bounded", background=np.ones(3), paths=[])
    cfg = _cfg(steps=30, batch=128)
    cfg.log_every = 10
    a = px.train(ds, cfg)
    b = px.train(train, cfg)
    la = [m["loss"] for m in a.metrics if "loss" in m]
    lb = [m["loss"] for m in b.metrics if "loss" in m]
    np.testing.assert_allclose(la, lb, rtol=1e-3)
