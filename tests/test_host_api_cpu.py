"""Host-side behaviours of the drop-in API that need no GPU: the trainer's
per-scene defaults (T:102-154, pkg/tests/test_trainer.py:16-104), config
(de)serialisation and overrides, learning-rate schedules (O:20-55,
test_optim.py:11-52), the epoch batcher (T:233-255) and sh_to_rgb."""

import json
import math

import numpy as np
import pytest

from paper_2112_05131_b200 import optim, trainer


def test_scene_type_defaults():
    b = trainer.default_config("bounded")
    assert [(r.step, r.dims) for r in b.ladder] == [(0, (256,) * 3), (38400, (512,) * 3)]
    assert (b.total_steps, b.batch_size, b.optimizer) == (128000, 5000, "rmsprop")
    assert (b.prune_criterion, b.prune_threshold) == ("weight", 0.256)
    assert (b.lambda_tv_sigma, b.lambda_tv_sh, b.tv_until_step) == (1e-5, 1e-3, 38400)
    assert (b.lambda_sparsity, b.lambda_beta, b.background) == (0.0, 0.0, (1.0, 1.0, 1.0))
    assert (b.lr_sigma.kind, b.lr_sigma.lr_init, b.lr_sigma.lr_final) == \
        ("delayed_exponential", 30.0, 0.05)
    assert (b.lr_sigma.total_steps, b.lr_sigma.delay_steps) == (250000, 15000)
    assert (b.lr_sh.kind, b.lr_sh.lr_init, b.lr_sh.lr_final) == ("exponential", 0.01, 5e-6)
    f = trainer.default_config("forward_facing_ndc")
    assert [(r.step, r.dims) for r in f.ladder] == [
        (0, (256, 256, 128)), (38400, (512, 512, 128)), (76800, (1408, 1156, 128))]
    assert (f.prune_criterion, f.prune_threshold, f.tv_until_step, f.ndc_z_pad) == \
        ("density", 5.0, -1, 0.0)
    assert (f.lambda_tv_sigma, f.lambda_tv_sh, f.lambda_sparsity) == (5e-4, 5e-3, 1e-12)
    u = trainer.default_config("unbounded_360")
    assert [(r.step, r.dims[0]) for r in u.ladder] == [(0, 128), (25600, 256), (51200, 512),
                                                       (76800, 640)]
    assert (u.total_steps, u.prune_threshold, u.lambda_sparsity, u.lambda_beta) == \
        (102400, 1.28, 1e-11, 1e-5)
    assert (u.bg_layers, u.bg_width, u.bg_height, u.bg_lr_sigma.kind) == \
        (64, 2048, 1024, "exponential")


def test_config_round_trip_validation_and_overrides(tmp_path):
    cfg = trainer.default_config("forward_facing_ndc")
    trainer.save_config(cfg, tmp_path / "c.yaml")
    assert trainer.load_config(tmp_path / "c.yaml") == cfg
    d = trainer.config_to_dict(trainer.default_config("bounded"))
    with pytest.raises(ValueError, match="not_a_key"):
        trainer.config_from_dict({**d, "not_a_key": 1})
    bad = trainer.config_to_dict(trainer.default_config("bounded"))
    bad["lr_sigma"]["warmup"] = 5
    with pytest.raises(ValueError, match="warmup"):
        trainer.config_from_dict(bad)
    trainer.apply_override(d, "optimizer", "sgd")
    trainer.apply_override(d, "lr_sh.lr_init", 0.5)
    assert (d["optimizer"], d["lr_sh"]["lr_init"]) == ("sgd", 0.5)
    for key in ("nope", "nope.nope", "lr_sh.nope"):
        with pytest.raises(KeyError):
            trainer.apply_override(d, key, 1)
    with pytest.raises(ValueError):
        trainer.TrainConfig(ladder=[trainer.LadderRung(10, (4, 4, 4))], total_steps=100)
    with pytest.raises(ValueError):
        trainer.TrainConfig(ladder=[trainer.LadderRung(0, (4, 4, 4)),
                                    trainer.LadderRung(200, (8, 8, 8))], total_steps=100)


def test_train_split_scene_scale(tmp_path):
    rng = np.random.default_rng(3)
    pos = rng.normal(size=(12, 3))
    frames = []
    for p in pos:
        m = np.eye(4)
        m[:3, 3] = p
        frames.append({"transform_matrix": m.tolist()})
    (tmp_path / "transforms_train.json").write_text(json.dumps({"frames": frames}))
    c = pos.mean(0)
    want = 1.0 / (1.1 * np.max(np.linalg.norm(pos - c, axis=1)))
    assert trainer.train_split_scene_scale(tmp_path) == pytest.approx(want, rel=1e-12)


def test_learning_rate_schedules():
    s = trainer.default_config("bounded").lr_sigma
    assert optim.lr_at(s, s.total_steps) == pytest.approx(s.lr_final, rel=1e-12)
    sh = trainer.default_config("bounded").lr_sh
    assert optim.lr_at(sh, 0) == sh.lr_init
    e = optim.LrSchedule(kind="exponential", lr_init=1.0, lr_final=0.01, total_steps=100)
    assert optim.lr_at(e, 50) == pytest.approx(0.1, rel=1e-12)   # geometric mean
    assert optim.lr_at(e, 1000) == pytest.approx(0.01, rel=1e-12)
    d = optim.LrSchedule(kind="delayed_exponential", lr_init=1.0, lr_final=1.0,
                         total_steps=100, delay_steps=10, delay_mult=0.1)
    ramp = [optim.lr_at(d, k) for k in range(0, 12)]
    assert ramp[0] == pytest.approx(0.1) and ramp[10] == pytest.approx(1.0)
    assert all(b >= a for a, b in zip(ramp, ramp[1:]))
    assert optim.lr_at(d, 5) == pytest.approx(0.1 + 0.9 * math.sin(0.25 * math.pi))
    c = optim.LrSchedule(kind="constant", lr_init=0.3, lr_final=0.3)
    assert {optim.lr_at(c, k) for k in (0, 7, 10 ** 6)} == {0.3}
    for kw in (dict(kind="cosine"), dict(lr_init=0.1, lr_final=0.2), dict(lr_final=0.0),
               dict(delay_steps=-1)):
        with pytest.raises(ValueError):
            optim.LrSchedule(**kw)
    with pytest.raises(ValueError):
        optim.lr_at(e, -1)


def test_epoch_batcher_epochs_and_oversized_batches():
    b = trainer.EpochBatcher(103, 10, np.random.default_rng(0))
    flat = np.concatenate([b.next() for _ in range(103)])   # exactly 10 epochs
    for ep in range(10):
        assert len(np.unique(flat[ep * 103:(ep + 1) * 103])) == 103
    big = trainer.EpochBatcher(7, 20, np.random.default_rng(1)).next()
    counts = np.bincount(big, minlength=7)
    assert len(big) == 20 and counts.min() >= 2 and counts.max() <= 3
