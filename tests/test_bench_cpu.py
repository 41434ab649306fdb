"""bench.py's host side on CPU: the launcher (N ranks without torchrun), the
shared workload config of both arms, and the reference arm's ray pool."""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_c2_hyperparameters_match_default_config():
    """bench.C2 (used by the oracle arms) is default_config('bounded')."""
    import bench
    from paper_2112_05131_b200 import trainer

    cfg = trainer.default_config("bounded")
    for k, v in bench.C2.items():
        if k in ("lr_sigma", "lr_sh"):
            s = getattr(cfg, k)
            assert (s.kind, s.lr_init, s.lr_final, s.total_steps) == v[:4], k
            if s.kind == "delayed_exponential":
                assert (s.delay_steps, s.delay_mult) == v[4:], k
        else:
            got = getattr(cfg, k)
            assert (tuple(got) if isinstance(got, (list, tuple)) else got) == v, k


def test_oracle_lr_at_matches_package():
    from oracle import oracle as orc
    from paper_2112_05131_b200 import optim, trainer

    cfg = trainer.default_config("bounded")
    for sched in (cfg.lr_sigma, cfg.lr_sh):
        for step in (0, 1, 7, 14999, 15000, 38400, 250000, 300000):
            assert orc.lr_at(sched.kind, sched.lr_init, sched.lr_final, sched.total_steps, step,
                             sched.delay_steps, sched.delay_mult) == optim.lr_at(sched, step)


def test_reference_arm_pool_is_the_same_pool():
    """The reference arm's lazily generated rays are the rows of the pool our
    arm builds (all_rays of the same 100-view hemisphere dataset)."""
    import math

    import bench
    from oracle import oracle as orc
    from paper_2112_05131_b200 import scenes

    class A:
        views, res, dims = 100, 200, 256

    rays_for, n = bench.oracle_pool(A)
    assert n == 100 * 200 * 200
    phase = float(np.random.default_rng(0).uniform(0, 2 * math.pi))
    cams, _ = scenes.hemisphere_cameras(100, 200, phase=phase)
    idx = np.array([0, 1, 39999, 40000, 123457, 3999999])
    o, d, v, gt = rays_for(idx)
    for r, i in enumerate(idx):
        c = cams[i // 40000]
        oo, dd = orc.generate_rays(c.c2w, c.focal, c.width, c.height)
        np.testing.assert_array_equal(o[r], oo[i % 40000])
        np.testing.assert_array_equal(d[r], dd[i % 40000])
    assert np.all((gt >= 0) & (gt <= 1))
    assert np.all(np.rint(gt * 255) == gt * 255) or np.allclose(np.rint(gt * 255), gt * 255,
                                                               atol=1e-4)


def test_launcher_spawns_ranks_without_torchrun():
    """`python bench.py --gpus 2` (no torchrun) launches 2 ranks itself; the
    dry run joins them over gloo and takes the max over ranks."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["ranks_joined"] == 2
    assert rec["config"]["global_batch"] == 10000 and rec["config"]["parallelism"] == "dp2"
