"""End-to-end optimisation on the B200 (drop-in for pkg/src/plenoxel/trainer.py:
bounded, forward-facing-NDC and unbounded-360 scenes; the 360 scenes add the
multi-sphere-image background of msi.py, stepped by Trainer._step_360).

The step body (T:411-492) keeps the reference's order and RNG consumption --
EpochBatcher permutations and sample_tv_cells draws come from the same
numpy default_rng(seed) -- while the data path is device-resident:

  batch   = pool rows idx (device permutation, uploaded once per epoch)
  render  = plx_render_fused_bwd            (one kernel, sums stay on device)
  TV      = plx_tv on (start, count)        (one kernel)
  check   = one 32-byte D2H of the loss sums (finiteness, T:473-480)
  update  = plx_opt_step with fused clear   (one kernel, counts n_touched)

With a World of size N (dist.py) each rank renders its contiguous slice of
the global batch and its sub-run of the TV cells, then the gradients are
all-reduced and the (replicated) update runs everywhere.
"""

from __future__ import annotations

import dataclasses
import math
import os
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch
import yaml

from . import _lib, artifact_io, losses, optim, render
import ctypes

import torch.distributed as dist

from .dist import PeerMap, World, max_reduce, reduce_gradients, shard_range, union_rows
from .grid import GradientBuffer, SparseGrid

SCENE_TYPES = ("bounded", "forward_facing_ndc", "unbounded_360")


class TrainingDiverged(RuntimeError):
    pass


class ResourceError(RuntimeError):
    pass


@dataclass
class LadderRung:
    step: int
    dims: tuple


@dataclass
class TrainConfig:
    """T:40-99 (same keys, same defaults)."""

    scene_type: str = "bounded"
    aabb: tuple = (-1.5, -1.5, -1.5, 1.5, 1.5, 1.5)
    ladder: list = field(default_factory=lambda: [LadderRung(0, (256, 256, 256))])
    total_steps: int = 128000
    batch_size: int = 5000
    step_frac: float = 0.5
    stop_thresh: float = 1e-4
    interp: str = "trilinear"
    formula: str = "relative"
    background: tuple = (1.0, 1.0, 1.0)
    prune_criterion: str = "weight"
    prune_threshold: float = 0.256
    lambda_tv_sigma: float = 1e-5
    lambda_tv_sh: float = 1e-3
    tv_sample_frac: float = 0.01
    tv_until_step: int = -1
    lambda_sparsity: float = 0.0
    lambda_beta: float = 0.0
    lr_sigma: optim.LrSchedule = field(default_factory=lambda: optim.LrSchedule(
        kind="delayed_exponential", lr_init=30.0, lr_final=0.05, total_steps=250000,
        delay_steps=15000, delay_mult=0.01))
    lr_sh: optim.LrSchedule = field(default_factory=lambda: optim.LrSchedule(
        kind="exponential", lr_init=0.01, lr_final=5e-6, total_steps=250000))
    optimizer: str = "rmsprop"
    rms_beta: float = 0.95
    rms_eps: float = 1e-8
    init_sigma: float = 0.1
    init_rgb: float = 0.1
    seed: int = 0
    eval_every: int = 1000
    log_every: int = 100
    checkpoint_every: int = 0
    jitter: float = 0.0
    ndc_z_pad: float = 0.0
    # unbounded_360 only (T:77-86)
    bg_layers: int = 64
    bg_height: int = 1024
    bg_width: int = 2048
    bg_lambda_tv: float = 1e-3
    bg_lr_sigma: optim.LrSchedule = field(default_factory=lambda: optim.LrSchedule(
        kind="exponential", lr_init=30.0, lr_final=0.05, total_steps=250000))
    bg_lr_rgb: optim.LrSchedule = field(default_factory=lambda: optim.LrSchedule(
        kind="exponential", lr_init=0.01, lr_final=5e-6, total_steps=250000))
    scene_margin: float = 1.1

    def __post_init__(self):
        if self.scene_type not in SCENE_TYPES:
            raise ValueError(f"unknown scene type {self.scene_type!r}")
        if self.batch_size < 1:
            raise ValueError("batch size must be >= 1")
        steps = [r.step for r in self.ladder]
        if steps != sorted(steps) or len(set(steps)) != len(steps):
            raise ValueError("ladder steps must be strictly increasing")
        if steps and steps[0] != 0:
            raise ValueError("first ladder rung must start at step 0")
        if any(s >= self.total_steps for s in steps[1:]):
            raise ValueError("ladder steps must be < total_steps")


def default_config(scene_type: str) -> TrainConfig:
    """T:102-154."""
    if scene_type == "bounded":
        return TrainConfig(scene_type="bounded", aabb=(-1.5, -1.5, -1.5, 1.5, 1.5, 1.5),
                           ladder=[LadderRung(0, (256, 256, 256)),
                                   LadderRung(38400, (512, 512, 512))],
                           total_steps=128000, prune_criterion="weight", prune_threshold=0.256,
                           lambda_tv_sigma=1e-5, lambda_tv_sh=1e-3, tv_until_step=38400,
                           background=(1.0, 1.0, 1.0))
    if scene_type == "forward_facing_ndc":
        return TrainConfig(scene_type="forward_facing_ndc", aabb=(-1.0, -1.0, -1.0, 1.0, 1.0, 1.0),
                           ladder=[LadderRung(0, (256, 256, 128)),
                                   LadderRung(38400, (512, 512, 128)),
                                   LadderRung(76800, (1408, 1156, 128))],
                           total_steps=128000, prune_criterion="density", prune_threshold=5.0,
                           lambda_tv_sigma=5e-4, lambda_tv_sh=5e-3, lambda_sparsity=1e-12,
                           background=(0.0, 0.0, 0.0))
    if scene_type == "unbounded_360":
        return TrainConfig(scene_type="unbounded_360", aabb=(-1.0, -1.0, -1.0, 1.0, 1.0, 1.0),
                           ladder=[LadderRung(0, (128, 128, 128)),
                                   LadderRung(25600, (256, 256, 256)),
                                   LadderRung(51200, (512, 512, 512)),
                                   LadderRung(76800, (640, 640, 640))],
                           total_steps=102400, prune_criterion="weight", prune_threshold=1.28,
                           lambda_tv_sigma=5e-5, lambda_tv_sh=5e-3, lambda_sparsity=1e-11,
                           lambda_beta=1e-5, bg_layers=64, bg_height=1024, bg_width=2048,
                           bg_lambda_tv=1e-3, background=(0.0, 0.0, 0.0))
    raise ValueError(f"unknown scene type {scene_type!r}")


def toy_config(grid_dim: int = 64, step_frac: float = 0.5, total_steps: int = 5000,
               batch_size: int = 3000, aabb: float = 1.1) -> TrainConfig:
    """toy.py:37-62."""
    return TrainConfig(
        scene_type="bounded", aabb=(-aabb,) * 3 + (aabb,) * 3,
        ladder=[LadderRung(0, (grid_dim,) * 3)], total_steps=total_steps,
        batch_size=batch_size, step_frac=step_frac, lambda_tv_sigma=1e-6, lambda_tv_sh=1e-4,
        tv_until_step=-1,
        lr_sigma=optim.LrSchedule(kind="delayed_exponential", lr_init=2.0, lr_final=0.1,
                                  total_steps=2 * total_steps, delay_steps=total_steps // 10,
                                  delay_mult=0.01),
        lr_sh=optim.LrSchedule(kind="exponential", lr_init=0.01, lr_final=1e-4,
                               total_steps=2 * total_steps),
        eval_every=0, log_every=100, background=(1.0, 1.0, 1.0))


def config_to_dict(cfg: TrainConfig) -> dict:
    d = dataclasses.asdict(cfg)
    d["ladder"] = [{"step": r.step, "dims": list(r.dims)} for r in cfg.ladder]
    d["aabb"], d["background"] = list(cfg.aabb), list(cfg.background)
    return d


def config_from_dict(d: dict) -> TrainConfig:
    known = {f.name for f in dataclasses.fields(TrainConfig)}
    unknown = set(d) - known
    if unknown:
        raise ValueError(f"unknown config keys: {sorted(unknown)}")
    kw = dict(d)
    if "ladder" in kw:
        kw["ladder"] = [LadderRung(int(r["step"]), tuple(int(x) for x in r["dims"]))
                        for r in kw["ladder"]]
    sched_keys = {f.name for f in dataclasses.fields(optim.LrSchedule)}
    for key in ("lr_sigma", "lr_sh", "bg_lr_sigma", "bg_lr_rgb"):
        if key in kw and isinstance(kw[key], dict):
            bad = set(kw[key]) - sched_keys
            if bad:
                raise ValueError(f"unknown {key} schedule keys: {sorted(bad)}")
            kw[key] = optim.LrSchedule(**kw[key])
    for key in ("aabb", "background"):
        if key in kw:
            kw[key] = tuple(float(x) for x in kw[key])
    return TrainConfig(**kw)


def apply_override(d: dict, dotted_key: str, value) -> None:
    """T:209-218: set a (possibly nested, dotted) key of a config dict;
    KeyError for a key the config does not have."""
    node = d
    parts = dotted_key.split(".")
    for p in parts[:-1]:
        if not isinstance(node.get(p), dict):
            raise KeyError(f"unknown config key {dotted_key!r}")
        node = node[p]
    if parts[-1] not in node:
        raise KeyError(f"unknown config key {dotted_key!r}")
    node[parts[-1]] = value


def train_split_scene_scale(data_dir, margin: float = 1.1) -> float:
    """T:291-301: the 360 camera pre-scale from a NeRF-format dataset's
    training split metadata (transforms_train.json camera positions)."""
    import json
    meta = json.loads((Path(data_dir) / "transforms_train.json").read_text())
    pos = np.array([np.asarray(f["transform_matrix"], dtype=np.float64)[:3, 3]
                    for f in meta["frames"]])
    return _scale_from_positions(pos, margin)


def load_config(path) -> TrainConfig:
    with open(path) as f:
        return config_from_dict(yaml.safe_load(f))


def save_config(cfg: TrainConfig, path) -> None:
    with open(path, "w") as f:
        yaml.safe_dump(config_to_dict(cfg), f, sort_keys=False)


# steps between rebuilds of the grid's dead-brick mask (SparseGrid.rebuild_bricks)
BRICK_REBUILD_EVERY = 100


class EpochBatcher:
    """T:233-255 (identical RNG use) with a device mirror of the permutation:
    next_device() returns the same indices as next() as a CUDA int64 tensor,
    uploading each permutation once per epoch."""

    def __init__(self, n: int, batch_size: int, rng, device=None):
        self.n = n
        self.batch_size = batch_size
        self.rng = rng
        self.device = device
        self.perm = rng.permutation(n)
        self.cursor = 0
        self._perm_dev = None

    def _dev_perm(self):
        """The device permutation, in ONE persistent buffer (a captured step
        graph reads batches as slices of it); a new epoch's permutation is
        copied in stream order, after every step that read the old one."""
        if self._perm_dev is None:
            buf = getattr(self, "_perm_buf", None)
            if buf is None or buf.numel() != self.n:
                buf = self._perm_buf = torch.empty(self.n, dtype=torch.int64,
                                                   device=self.device or "cuda")
            buf.copy_(torch.from_numpy(self.perm))
            self._perm_dev = buf
        return self._perm_dev

    def next(self) -> np.ndarray:
        chunks = []
        need = self.batch_size
        while need > 0:
            if self.cursor >= self.n:
                self.perm = self.rng.permutation(self.n)
                self._perm_dev = None
                self.cursor = 0
            take = min(need, self.n - self.cursor)
            chunks.append(self.perm[self.cursor:self.cursor + take])
            self.cursor += take
            need -= take
        return np.concatenate(chunks) if len(chunks) > 1 else chunks[0]

    def next_device(self) -> torch.Tensor:
        return self.next_slice()[0]

    def next_slice(self):
        """next_device() and, when the batch is ONE slice of the device
        permutation buffer (it does not cross an epoch), its offset there;
        None otherwise."""
        chunks, offs = [], []
        need = self.batch_size
        while need > 0:
            if self.cursor >= self.n:
                self.perm = self.rng.permutation(self.n)
                self._perm_dev = None
                self.cursor = 0
                # the old epoch's tail is a view of the permutation buffer the
                # new epoch's permutation is about to be copied into
                chunks = [c.clone() for c in chunks]
            take = min(need, self.n - self.cursor)
            chunks.append(self._dev_perm()[self.cursor:self.cursor + take])
            offs.append(self.cursor)
            self.cursor += take
            need -= take
        if len(chunks) > 1:
            return torch.cat(chunks), None
        return chunks[0], offs[0]


@dataclass
class TrainResult:
    grid: SparseGrid
    metrics: list
    config: TrainConfig
    background: object = None      # msi.MsiBackground (360 scenes)
    scene_scale: float = 1.0


def _grid_aabb(cfg: TrainConfig, dims):
    lo = np.array(cfg.aabb[:3], dtype=np.float64)
    hi = np.array(cfg.aabb[3:], dtype=np.float64)
    if cfg.scene_type == "forward_facing_ndc" and cfg.ndc_z_pad > 0:
        pad = cfg.ndc_z_pad * (hi[2] - lo[2]) / (dims[2] - 1)
        lo[2] -= pad
        hi[2] += pad
    return lo, hi


def _scale_from_positions(pos: np.ndarray, margin: float) -> float:
    """T:282-287: 1 / (margin * max camera distance from the centroid)."""
    centroid = pos.mean(axis=0)
    maxdist = float(np.max(np.linalg.norm(pos - centroid, axis=1)))
    if maxdist <= 0:
        return 1.0
    return 1.0 / (margin * maxdist)


def _scene_scale_360(dataset, margin: float) -> float:
    """T:278-279: the 360 camera pre-scale from the training cameras."""
    return _scale_from_positions(np.stack([c.position for c in dataset.cameras]), margin)


def _estimate_table_bytes(dims) -> int:
    """Device footprint of a dense rung: links + density + sh + grad + v (f32)
    + touched mask and id list."""
    cells = int(np.prod([int(d) for d in dims]))
    return cells * (4 + 4 + 3 * 28 * 4 + 1 + 4)


class Trainer:
    """Owns the device state of one training run (grid, RMSProp state,
    gradient buffer, ray pool, batcher) and executes steps."""

    def __init__(self, train_ds, config: TrainConfig, device=None, world: World | None = None):
        cfg = config
        self.cfg = cfg
        self.world = world or World()
        self.device = torch.device(device or "cuda")
        self.rng = np.random.default_rng(cfg.seed)
        self.scene_scale = 1.0
        self.is_360 = cfg.scene_type == "unbounded_360"
        if self.is_360:   # T:375-377: cameras pre-scaled into the unit sphere
            self.scene_scale = _scene_scale_360(train_ds, cfg.scene_margin)
        # the training rays (T:372, all_rays) as a device camera pool: the
        # kernels generate each ray from its (view, pixel) row
        self.pool = render.CameraPool(train_ds.cameras, train_ds.images,
                                      ndc=train_ds.scene_type == "forward_facing_ndc",
                                      scale=self.scene_scale, device=self.device)
        dims0 = cfg.ladder[0].dims
        lo, hi = _grid_aabb(cfg, dims0)
        self.grid = SparseGrid.dense(dims0, lo, hi, sigma=cfg.init_sigma, rgb=cfg.init_rgb,
                                     device=self.device)
        self.state = optim.OptimState(self.grid.n_rows, beta=cfg.rms_beta, eps=cfg.rms_eps,
                                      device=self.device)
        self.grads = GradientBuffer(self.grid.n_rows, device=self.device)
        self.opts = render.RenderOptions(step_frac=cfg.step_frac, stop_thresh=cfg.stop_thresh,
                                         background=(0.0, 0.0, 0.0) if self.is_360
                                         else tuple(cfg.background), interp=cfg.interp,
                                         formula=cfg.formula, jitter=cfg.jitter)
        # the MSI background of 360 scenes (T:386-397)
        self.background = self.bg_state = self.bg_grads = None
        if self.is_360:
            from . import msi
            self.background = msi.MsiBackground.create(cfg.bg_layers, cfg.bg_height,
                                                       cfg.bg_width, device=self.device)
            self.background.data[..., 0] = cfg.init_sigma
            self.background.data[..., 1:] = cfg.init_rgb
            self.bg_state = msi.BgOptimState(self.background, beta=cfg.rms_beta,
                                             eps=cfg.rms_eps)
            self.bg_grads = msi.BgGradientBuffer(self.background)
        self.batcher = EpochBatcher(self.pool.n, cfg.batch_size, self.rng, self.device)
        self.rung_events = {r.step: tuple(r.dims) for r in cfg.ladder[1:]}
        # {mse_sum, cauchy_sum, tv_sigma_sum, tv_sh_sum, halt}: the loss sums of
        # the current step and the sticky divergence flag of the device guard
        self.sums = torch.zeros(5, dtype=torch.float64, device=self.device)
        self.count = torch.zeros(1, dtype=torch.int64, device=self.device)
        # march counters of the fused kernel, accumulated over steps:
        # {positions, samples, chunks, rays} (plx_render_opts.stats)
        self.march_stats = torch.zeros(4, dtype=torch.int64, device=self.device)
        # pinned copies of the last steps' loss sums, checked two steps late
        self._host_sums = [torch.zeros(4, dtype=torch.float64).pin_memory() for _ in range(3)]
        self._sums_ready = [torch.cuda.Event() for _ in range(3)]
        self._pending = []
        self.diverged_step = None
        self._peers = None
        self._dp_pack = None
        self.step_events = None   # optional 4 torch.cuda.Events (plx_step_args.events)
        # single-GPU steps replay a captured CUDA graph (PLX_GRAPH=0 disables);
        # 360 scenes step through the public msi API instead
        self.use_graph = os.environ.get("PLX_GRAPH", "1") != "0" and not self.is_360
        # graph mode: per-step scalars {tv_start, lr_sigma, lr_sh (f64 bits),
        # batch offset} in 3 pinned slots, copied to _dparams by the graph
        self._dparams = torch.zeros(4, dtype=torch.int64, device=self.device)
        self._hparams = [torch.zeros(4, dtype=torch.int64).pin_memory() for _ in range(3)]
        self._hparams_np = [h.numpy() for h in self._hparams]
        self._graphs, self._graph_args = {}, {}
        self._rays_buf = None   # step_rays(): two device batch slots (2, 4, B, 3)
        self._rays_idx = None
        self._rays_slot = 0
        self._copy_stream = None
        self._eager_done = False
        self._refresh_cache()

    def _refresh_cache(self):
        if self.world.active:   # the N-GPU owner update does not keep the peers' brick masks
            self.grid.disable_bricks()
        self._cgrid = self.grid._c(with_occ=self.opts.interp == "trilinear")
        self._cgrid_plain = self.grid._c(with_occ=False)
        self._cgrad = self.grads._c()
        self._kopts = render.kernel_opts(self.grid, self.opts)
        self._kopts.stats = self.march_stats.data_ptr()
        # the native step descriptor (plx_train_step): static fields here,
        # per-step fields (batch slice, TV run, learning rates) in step()
        a = _lib.PlxStepArgs()
        a.rays = self.pool.rays(None)
        a.opts = self._kopts
        a.lam_cauchy = self.cfg.lambda_sparsity
        B_local = shard_range(self.cfg.batch_size, 0, self.world.size)[1]
        sp, sn, self._scratch_keep = _lib.render_scratch(self._cgrid, self._kopts, B_local,
                                                         self.device)
        a.scratch, a.scratch_bytes = sp, sn
        dims = self.grid.dims
        a.tv_fac = (ctypes.c_double * 3)(*(d / 256.0 for d in dims))
        a.tv_eps = losses.TV_EPS
        a.rmsprop = int(self.cfg.optimizer == "rmsprop")
        a.v = self.state.v.data_ptr()
        a.beta, a.eps = self.state.beta, self.state.eps
        a.sums = self.sums.data_ptr()
        a.count = self.count.data_ptr()
        self._step_args = a
        self._graphs, self._graph_args = {}, {}   # descriptors changed: re-capture
        w = self.world
        if w.active and w.mode == "union":
            R = self.grid.n_rows
            self._dp_ids = torch.empty(max(R, 1), dtype=torch.int32, device=self.device)
            self._dp_cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
            self._dp_scratch = torch.empty(int(_lib.load().plx_scan_scratch_bytes(R)),
                                           dtype=torch.uint8, device=self.device)
        if w.active and w.mode == "p2p":
            if self._peers is not None:
                torch.cuda.synchronize()
                self._peers.close()
            self._peers = PeerMap(w, self.grid, self.grads)
            self._cgrid = self.grid._c(with_occ=self.opts.interp == "trilinear")

    # -- ladder event (T:412-439) ---------------------------------------------
    def rung_event(self, new_dims, out_dir=None, step=0):
        cfg = self.cfg
        if cfg.prune_criterion == "weight":
            w = self.max_weights()
            self.grid, kept = self.grid.prune("weight", cfg.prune_threshold, w)
        else:
            self.grid, kept = self.grid.prune("density", cfg.prune_threshold)
        self.state.reindex(kept)
        need = _estimate_table_bytes(new_dims)
        free, _ = torch.cuda.mem_get_info(self.device)
        if need > free:
            raise ResourceError(f"upsampling to {tuple(new_dims)} needs ~{need >> 20} MiB, "
                                f"only {free >> 20} MiB free on the device")
        self.grid = self.grid.upsample(new_dims)
        self.state.reset(self.grid.n_rows)
        self.grads = GradientBuffer(self.grid.n_rows, device=self.device)
        self._refresh_cache()
        if out_dir is not None:
            self.save_checkpoint(Path(out_dir) / f"checkpoint_{step:07d}.plnx", step)

    def full_state(self) -> optim.OptimState:
        """The RMSProp state of every row.  In p2p mode each rank updates
        only the rows it owns (dist.owner_slice), so the other ranks' slices
        of `v` are gathered from their owners."""
        w = self.world
        if not (w.active and w.mode == "p2p"):
            return self.state
        from .dist import gather_owned_rows
        v = gather_owned_rows(w, self.state.v)
        st = optim.OptimState.__new__(optim.OptimState)
        st.__dict__.update(self.state.__dict__)
        st.v = v
        return st

    def save_checkpoint(self, path, step: int) -> None:
        """artifact_io.save_checkpoint of the whole run (rank 0 writes; the
        p2p state slices are gathered on every rank first)."""
        st = self.full_state()
        if self.world.rank == 0:
            artifact_io.save_checkpoint(path, self.grid, st, step, self.background,
                                        self.bg_state)

    def max_weights(self) -> torch.Tensor:
        """Max-weight over all training rays, sharded over ranks + max-reduce."""
        s, c = shard_range(self.pool.n, self.world.rank, self.world.size)
        w = self.grid.max_weight_accumulate_pool(self.pool, s, c, self.cfg.step_frac,
                                                 self.cfg.stop_thresh, self.cfg.interp)
        max_reduce(self.world, w)
        return w

    # -- one optimisation step (T:441-492) ------------------------------------
    def step(self, step: int, check_finite: bool = True, sync: bool = False) -> dict:
        """One step: batch, fused render+backward, TV, (exchange), update.

        The divergence check (T:473-480) runs on the device: plx_opt_step is
        handed the step's loss sums and skips the update (stickily) when one
        is non-finite, so the grid is left exactly as the reference leaves it
        when it raises.  The host learns of it one step later: each call
        checks the PREVIOUS step's sums (copied asynchronously), so the host
        never waits for the step it just enqueued and the GPU never idles
        between steps.  sync=True (logging steps) waits for this step's loss
        and returns it in the record."""
        if step and step % BRICK_REBUILD_EVERY == 0:
            # the optimisers only revive bricks; re-tighten the dead-brick mask
            self.grid.rebuild_bricks()
        if self.is_360:
            return self._step_360(step)
        idx, off = self.batcher.next_slice()
        return self._step(step, int(idx.numel()), idx, check_finite, sync, off)

    def step_rays(self, step: int, origins, dirs=None, viewdirs=None, target=None,
                  check_finite: bool = True, sync: bool = False) -> dict:
        """One step on a caller-supplied batch instead of the pool (the step
        body T:441-486 with the batch T:448-453 given): this rank's rays as
        (B,3) float64 arrays -- host tensors (pinned: asynchronous copy) or
        device tensors; viewdirs None = dirs.  The arrays are copied into a
        fixed device buffer, so on one GPU the step replays the same CUDA
        graph as step().  The global batch is B x world size (each rank
        passes its own rays).  A packed (4, B, 3) array [origins, dirs,
        viewdirs, target] as `origins` alone is copied in one transfer."""
        packed = dirs is None and origins.dim() == 3 and origins.shape[0] == 4
        B = int(origins.shape[1] if packed else origins.shape[0])
        buf = self._rays_buf
        if buf is None or buf.shape[2] != B:
            # two contiguous batch slots (2, 4, B, 3): slot p's arrays sit 4B
            # rows after slot 0's, so the graph reads slot p as rows
            # [4pB, 4pB + B) through the identity index + offset 4pB
            torch.cuda.synchronize()
            buf = self._rays_buf = torch.empty((2, 4, B, 3), dtype=torch.float64,
                                               device=self.device)
            self._rays_idx = torch.arange(5 * B, dtype=torch.int64, device=self.device)
            self._rays_free = [torch.cuda.Event(), torch.cuda.Event()]
            self._rays_copied = [torch.cuda.Event(), torch.cuda.Event()]
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=self.device)
            for k in [k for k in self._graphs if k[0] == "rays"]:
                del self._graphs[k]
        p = step % 2
        dst = buf[p]
        # the H2D of this batch runs on a copy stream, overlapping the step
        # still in flight; it waits for the step that last read slot p
        cs, main = self._copy_stream, torch.cuda.current_stream(self.device)
        cs.wait_event(self._rays_free[p])
        with torch.cuda.stream(cs):
            if packed:
                dst.copy_(torch.as_tensor(origins), non_blocking=True)
            else:
                for k, src in enumerate((origins, dirs, dirs if viewdirs is None else viewdirs,
                                         target)):
                    dst[k].copy_(torch.as_tensor(src), non_blocking=True)
            self._rays_copied[p].record(cs)
        main.wait_event(self._rays_copied[p])
        self._rays_slot = p
        rec = self._step(step, B, None, check_finite, sync)
        self._rays_free[p].record(main)
        return rec

    def _step(self, step: int, B: int, idx, check_finite: bool, sync: bool,
              idx_off: int | None = None) -> dict:
        """step()/step_rays() body: idx = pool rows of the global batch (at
        offset idx_off of the batcher's permutation buffer when it is one
        slice of it), or None for the rank-local batch in _rays_buf."""
        cfg = self.cfg
        pool_mode = idx is not None
        if pool_mode:
            s0, c0 = shard_range(B, self.world.rank, self.world.size)
            n_global = B
        else:
            s0, c0 = 0, B
            n_global = B * self.world.size
        a = self._step_args
        tv_on = (cfg.lambda_tv_sigma > 0 or cfg.lambda_tv_sh > 0) and (
            cfg.tv_until_step < 0 or step < cfg.tv_until_step)
        jt = None
        if self.opts.jitter > 0:
            # R:106-111 draws the jitter inside fused_mse_backward (T:453-457),
            # before sample_tv_cells (T:463)
            jt = torch.from_numpy(self.rng.random(n_global if pool_mode else B)
                                  * self.opts.jitter).to(self.device)
        n_tv = 0
        tv_start = 0
        if tv_on:
            run = losses.sample_tv_cells(self.grid, cfg.tv_sample_frac, self.rng)
            n_tv = run.count
            sub = run.split(self.world.rank, self.world.size)
            tv_start = sub.start
        lr_s, lr_c = optim.lr_at(cfg.lr_sigma, step), optim.lr_at(cfg.lr_sh, step)
        ev = self.step_events
        slot = step % 3
        graphed = self._graph_ok(B, ev, pool_mode) and (idx_off is not None or not pool_mode)
        if graphed:
            # CUDA-graph replay of the whole step: the graph for this slot
            # copies the per-step scalars (TV start, learning rates, batch
            # offset in the permutation buffer) from pinned slot `slot`, runs
            # the step and copies the loss sums to pinned slot `slot`; the
            # graph of step-3 used the slot last
            self._sums_ready[slot].synchronize()
            hp = self._hparams_np[slot]
            hp[0] = tv_start
            hp[1:3].view(np.float64)[:] = (lr_s, lr_c)
            hp[3] = idx_off + s0 if pool_mode else self._rays_slot * 4 * B
            self._replay(tv_on, pool_mode, slot, c0, sub.count if tv_on else 0, n_tv)
        else:
            if pool_mode:
                a.rays = self.pool.rays(None)
                a.rays.idx = idx.data_ptr() + 8 * s0
            else:
                a.rays = self._rays_desc(self._rays_slot)
            a.rays.n = c0
            a.rays.jitter = None
            if jt is not None:
                self._jt_keep = jt
                a.rays.jitter = jt.data_ptr() + 8 * s0
            a.up_scale = 2.0 / n_global
            a.tv_count = 0
            if tv_on:
                a.tv_start, a.tv_count = sub.start, sub.count
                a.tv_f_sigma, a.tv_f_sh = cfg.lambda_tv_sigma / n_tv, cfg.lambda_tv_sh / n_tv
            a.update = int(not self.world.active)
            a.lr_sigma, a.lr_sh = lr_s, lr_c
            a.dev_tv_start = None
            a.dev_lr = None
            for i in range(4):
                a.events[i] = ev[i].cuda_event if ev is not None else None
            _lib.check(_lib.lib().plx_train_step(ctypes.byref(self._cgrid),
                                                 ctypes.byref(self._cgrad), ctypes.byref(a),
                                                 _lib.stream_ptr()), "train_step")
        B = n_global
        if self.world.active:
            self.exchange_update(step, slot)
            if ev is not None:
                ev[3].record()    # "after update" = after the exchange + update
        else:
            if not graphed:
                self._host_sums[slot].copy_(self.sums[0:4], non_blocking=True)
            self._sums_ready[slot].record()
        rec = {"B": B, "n_tv": n_tv}
        if sync:
            self.check_pending()
            self._sums_ready[slot].synchronize()
            rec.update(self._loss(step, slot, B, n_tv))
        elif check_finite:
            self._pending.append((step, slot, B, n_tv))
            if len(self._pending) > 2:   # the host runs up to two steps ahead
                self.check_pending(keep=2)
        return rec

    def _step_360(self, step: int) -> dict:
        """The 360 step body (T:441-492 with the background): fused render of
        grid + sphere layers with the MSE, Cauchy and beta terms
        (msi.render_rays_with_background), grid TV then background TV (the
        reference's RNG order), the divergence check, the grid update with
        its fused clear and the background's step_table + clear.  Single GPU;
        the loss is read every step (the reference's order)."""
        from . import msi

        cfg = self.cfg
        if self.world.active:
            raise NotImplementedError("unbounded_360 runs on one GPU")
        idx = self.batcher.next_device()
        B = int(idx.numel())
        o, d, _, gt = self.pool.materialize(idx, viewdirs=False)
        _, _, _, mse_sum, cauchy_raw, beta_raw = msi.render_rays_with_background(
            self.grid, self.background, o, d, self.opts,
            gt_rgb=gt, grads=self.grads, bg_grads=self.bg_grads, n_total=B,
            lam_cauchy=cfg.lambda_sparsity, lam_beta=cfg.lambda_beta)
        loss_mse = mse_sum / B
        tv_on = (cfg.lambda_tv_sigma > 0 or cfg.lambda_tv_sh > 0) and (
            cfg.tv_until_step < 0 or step < cfg.tv_until_step)
        tv_sig = tv_sh = 0.0
        if tv_on:
            run = losses.sample_tv_cells(self.grid, cfg.tv_sample_frac, self.rng)
            tv_sig, tv_sh = losses.tv_loss(self.grid, run, cfg.lambda_tv_sigma, cfg.lambda_tv_sh,
                                           self.grads)
            if cfg.bg_lambda_tv > 0:
                bcells = msi.sample_bg_tv_cells(self.background, cfg.tv_sample_frac, self.rng)
                msi.bg_tv_loss(self.background, bcells, cfg.bg_lambda_tv, cfg.bg_lambda_tv,
                               self.bg_grads)
        loss = (loss_mse + tv_sig + tv_sh + cfg.lambda_sparsity * cauchy_raw
                + cfg.lambda_beta * beta_raw)
        if not math.isfinite(loss):
            self.diverged_step = step
            raise TrainingDiverged(f"non-finite loss at step {step}: mse={loss_mse!r} "
                                   f"tv=({tv_sig!r}, {tv_sh!r})")
        lr_s, lr_c = optim.lr_at(cfg.lr_sigma, step), optim.lr_at(cfg.lr_sh, step)
        self.count.zero_()
        optim.step(self.grid, self.grads, self.state, lr_s, lr_c, cfg.optimizer, clear=True,
                   count_out=self.count, _cgrid=self._cgrid, _cgrad=self._cgrad)
        msi.step_table(self.background, self.bg_grads, self.bg_state,
                       optim.lr_at(cfg.bg_lr_sigma, step), optim.lr_at(cfg.bg_lr_rgb, step),
                       cfg.optimizer)
        return {"B": B, "loss": loss, "mse": loss_mse}

    def exchange_update(self, step: int, slot: int | None = None) -> None:
        """After the ranks' renders + TV: reduce the loss sums, exchange the
        touched rows' gradients (World.mode, dist.py) and apply the update
        with the fused clear (T:483-486).  The loss sums are copied to the
        pinned slot `slot` for the asynchronous divergence check."""
        cfg, w = self.cfg, self.world
        lr_s, lr_c = optim.lr_at(cfg.lr_sigma, step), optim.lr_at(cfg.lr_sh, step)
        if w.active:
            dist.all_reduce(self.sums[0:4], group=w.group)
        if slot is not None:
            self._host_sums[slot].copy_(self.sums[0:4], non_blocking=True)
            self._sums_ready[slot].record()
        self.count.zero_()
        if not w.active or w.mode == "dense":
            reduce_gradients(w, self.grads.data, self.grads.touched_mask)
            optim.step(self.grid, self.grads, self.state, lr_s, lr_c, cfg.optimizer, clear=True,
                       count_out=self.count, guard=self.sums, _cgrid=self._cgrid,
                       _cgrad=self._cgrad)
            return
        L, st = _lib.lib(), _lib.stream_ptr()
        rms = int(cfg.optimizer == "rmsprop")
        if w.mode == "union":
            n = union_rows(w, self.grads.touched_mask, self._dp_scratch, self._dp_ids,
                           self._dp_cnt)
            if n == 0:
                return
            if self._dp_pack is None or self._dp_pack.numel() < n * 28:
                self._dp_pack = torch.empty(int(n * 1.25) * 28, dtype=torch.float32,
                                            device=self.device)
            _lib.check(L.plx_pack_rows(self.grads.data.data_ptr(), self._dp_ids.data_ptr(),
                                       self._dp_cnt.data_ptr(), n, self._dp_pack.data_ptr(),
                                       st), "pack_rows")
            dist.all_reduce(self._dp_pack[:n * 28], group=w.group)
            _lib.check(L.plx_opt_step_list(
                ctypes.byref(self._cgrid), self.state.v.data_ptr(), ctypes.byref(self._cgrad),
                self._dp_ids.data_ptr(), self._dp_cnt.data_ptr(), self._dp_pack.data_ptr(),
                lr_s, lr_c, self.state.beta, self.state.eps, rms, 1, self.sums.data_ptr(),
                self.count.data_ptr(), st), "opt_step_list")
            return
        # p2p: owner-computes update over NVLink peer memory, then local clear
        rc = self.grid.lattice_sigma()[1]
        _lib.check(L.plx_dp_owner_update(
            ctypes.byref(self._peers.peers), self.state.v.data_ptr(), rc.data_ptr(), lr_s, lr_c,
            self.state.beta, self.state.eps, rms, self.sums.data_ptr(), self.count.data_ptr(),
            st), "dp_owner_update")
        dist.all_reduce(self.count, group=w.group)   # orders every owner before any clear
        self.grads.clear()

    # -- CUDA-graph replay of the native step ------------------------------------
    def _graph_ok(self, B: int, events, pool_mode: bool = True) -> bool:
        ok = (self.use_graph and self._eager_done and events is None
              and self.opts.jitter == 0 and (B == self.cfg.batch_size or not pool_mode))
        self._eager_done = True   # the first step runs eagerly (one-time library queries)
        return ok

    def _rays_desc(self, slot: int | None = None) -> _lib.PlxRays:
        """Descriptor of the step_rays batch buffer: slot p's rays directly
        (eager), or slot None: slot 0's arrays through the identity index,
        the graph adding the slot's row offset 4pB (dev_idx_off)."""
        r = _lib.PlxRays()
        sb = self._rays_buf[0 if slot is None else slot]
        r.origins, r.dirs = sb[0].data_ptr(), sb[1].data_ptr()
        r.viewdirs, r.target = sb[2].data_ptr(), sb[3].data_ptr()
        r.jitter, r.n = None, int(sb.shape[1])
        r.idx = self._rays_idx.data_ptr() if slot is None else None
        return r

    def _replay(self, tv_on: bool, pool_mode: bool, slot: int, n_local: int, tv_local: int,
                n_tv: int) -> None:
        """Replay (capturing on first use) the graph of one whole step for
        this grid, batch source (a slice of the batcher's permutation buffer
        at the offset in _dparams[3], or the rays in _rays_buf), TV on/off and
        pinned slot: plx_train_step's prologue kernel copies the slot's
        scalars to _dparams, and its compaction kernel writes the loss sums
        to the slot's pinned sums.  With N ranks the graph holds this rank's
        render (n_local rays) and TV sub-run (tv_local of the n_tv cells);
        the exchange and update follow eagerly (exchange_update)."""
        key = ("pool" if pool_mode else "rays", tv_on, slot)
        g = self._graphs.get(key)
        if g is None:
            cfg = self.cfg
            a = _lib.PlxStepArgs()
            ctypes.pointer(a)[0] = self._step_args   # copy of the static fields
            if pool_mode:
                a.rays = self.pool.rays(None)
                a.rays.idx = self.batcher._dev_perm().data_ptr()
                n_global = cfg.batch_size
            else:
                a.rays = self._rays_desc(None)
                n_global = n_local * self.world.size
            a.rays.n = n_local
            a.dev_idx_off = self._dparams.data_ptr() + 24
            a.rays.jitter = None
            a.up_scale = 2.0 / n_global
            a.update = int(not self.world.active)
            a.tv_count = tv_local if tv_on else 0
            nt = max(n_tv, 1)
            a.tv_f_sigma, a.tv_f_sh = cfg.lambda_tv_sigma / nt, cfg.lambda_tv_sh / nt
            a.dev_tv_start = self._dparams.data_ptr()
            a.dev_lr = self._dparams.data_ptr() + 8
            # the kernels read the slot's scalars from / write the loss sums
            # to pinned host memory: the graph has kernel nodes only
            a.host_params = self._hparams[slot].data_ptr()
            a.dev_params = self._dparams.data_ptr()
            a.host_sums = self._host_sums[slot].data_ptr()
            for i in range(4):
                a.events[i] = None
            L = _lib.lib()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                _lib.check(L.plx_train_step(ctypes.byref(self._cgrid), ctypes.byref(self._cgrad),
                                            ctypes.byref(a), _lib.stream_ptr()), "train_step")
            self._graphs[key] = g
            self._graph_args[key] = a
        g.replay()

    def _loss(self, step, slot, B, n_tv) -> dict:
        cfg = self.cfg
        mse_sum, cauchy_raw, tv_s, tv_h = (float(x) for x in self._host_sums[slot])
        loss_mse = mse_sum / B
        tv_sig = cfg.lambda_tv_sigma * tv_s / n_tv if n_tv else 0.0
        tv_sh = cfg.lambda_tv_sh * tv_h / n_tv if n_tv else 0.0
        loss = loss_mse + tv_sig + tv_sh + cfg.lambda_sparsity * cauchy_raw
        if not math.isfinite(loss):
            self.diverged_step = step
            raise TrainingDiverged(f"non-finite loss at step {step}: mse={loss_mse!r} "
                                   f"tv=({tv_sig!r}, {tv_sh!r})")
        return {"loss": loss, "mse": loss_mse}

    def check_pending(self, keep: int = 0) -> None:
        """Check the losses of unchecked steps, oldest first, leaving the
        newest `keep` pending (waits for those steps only)."""
        while len(self._pending) > keep:
            step, slot, B, n_tv = self._pending.pop(0)
            self._sums_ready[slot].synchronize()
            self._loss(step, slot, B, n_tv)

    def nnz_fraction(self) -> float:
        """GradientBuffer.nnz_fraction of the last step (counted by the opt kernel)."""
        return int(self.count.item()) / max(self.grid.n_rows, 1)

    # -- evaluation (T:309-347) -------------------------------------------------
    def evaluate(self, dataset, chunk: int = 1 << 20):
        return evaluate(self.grid, dataset, self.opts, chunk, self.background, self.scene_scale)


def evaluate(grid: SparseGrid, dataset, opts: render.RenderOptions, chunk: int = 1 << 20,
             background=None, scene_scale: float = 1.0):
    """Mean PSNR/SSIM over a dataset's views (T:309-347) on the device: each
    view's rays are generated and rendered by the kernels (evaluation keeps
    every pixel: forward-facing rays are warped without dropping, as
    T:316-319 does), the metrics are computed on the device
    (plx_image_metrics) and only two scalars per view come back."""
    pool = render.CameraPool(dataset.cameras, dataset.images,
                             ndc=dataset.scene_type == "forward_facing_ndc",
                             scale=scene_scale if dataset.scene_type == "unbounded_360" else 1.0,
                             drop_invalid=False, device=grid.device)
    ppv = pool.width * pool.height
    pred = torch.empty((ppv, 3), dtype=torch.float64, device=grid.device)
    rows = []
    for vi in range(pool.n_views):
        first = vi * ppv
        if dataset.scene_type == "unbounded_360":
            from . import msi
            idx = torch.arange(first, first + ppv, dtype=torch.int64, device=grid.device)
            o, d, _, _ = pool.materialize(idx, viewdirs=False, rgb=False)
            for s in range(0, ppv, chunk):
                pred[s:s + chunk] = msi.render_rays_with_background(
                    grid, background, o[s:s + chunk], d[s:s + chunk], opts)[0]
        else:
            for s in range(0, ppv, chunk):
                render.render_pool(grid, pool, opts, first + s, min(chunk, ppv - s),
                                   out=pred[s:s + chunk])
        gt = pool.rgb[first:first + ppv].double()
        shape = (pool.height, pool.width, 3)
        p, ss = losses.image_metrics(pred.view(shape), gt.view(shape))
        rows.append({"view": vi, "psnr": p, "ssim": ss})
    return (float(np.mean([r["psnr"] for r in rows])), float(np.mean([r["ssim"] for r in rows])),
            rows)


def _checked(tr: Trainer, out_dir) -> None:
    """Check every step still unchecked (the host runs two steps ahead of
    the device's loss sums) before the grid is used outside the step loop."""
    try:
        tr.check_pending()
    except TrainingDiverged:
        if out_dir is not None and tr.world.rank == 0:
            artifact_io.save_grid(tr.grid, Path(out_dir) / "diverged.plnx", tr.background)
        raise


def train(train_ds, config: TrainConfig, test_ds=None, out_dir=None, metrics_sink=None,
          device=None, world: World | None = None) -> TrainResult:
    """T:350-518 on the device (bounded, forward-facing and 360 scenes)."""
    cfg = config
    tr = Trainer(train_ds, cfg, device=device, world=world)
    out_dir = Path(out_dir) if out_dir is not None else None
    if out_dir is not None:
        out_dir.mkdir(parents=True, exist_ok=True)
    metrics: list = []

    def emit(rec):
        metrics.append(rec)
        if metrics_sink is not None:
            metrics_sink(rec)

    t_start = time.perf_counter()
    last_eval = -1
    for step in range(cfg.total_steps):
        if step in tr.rung_events:
            _checked(tr, out_dir)     # the reference raises before any rung event
            tr.rung_event(tr.rung_events[step], out_dir, step)
        log_now = cfg.log_every > 0 and step % cfg.log_every == 0
        try:
            rec = tr.step(step, sync=log_now)
            if step == cfg.total_steps - 1:
                tr.check_pending()
        except TrainingDiverged:
            if out_dir is not None and tr.world.rank == 0:   # the device guard kept the pre-update grid
                artifact_io.save_grid(tr.grid, out_dir / "diverged.plnx", tr.background)
            raise
        if log_now:
            emit({"step": step, "loss": rec["loss"], "mse": rec["mse"],
                  "nnz_fraction": tr.nnz_fraction()})
        if test_ds is not None and cfg.eval_every > 0 and (step + 1) % cfg.eval_every == 0:
            _checked(tr, out_dir)
            p, s, _ = tr.evaluate(test_ds)
            last_eval = step + 1
            emit({"step": step + 1, "psnr": p, "ssim": s,
                  "wall_time_s": time.perf_counter() - t_start})
        if cfg.checkpoint_every > 0 and out_dir is not None and (step + 1) % cfg.checkpoint_every == 0:
            _checked(tr, out_dir)
            tr.save_checkpoint(out_dir / f"checkpoint_{step + 1:07d}.plnx", step + 1)
    if test_ds is not None and last_eval != cfg.total_steps:
        p, s, _ = tr.evaluate(test_ds)
        emit({"step": cfg.total_steps, "psnr": p, "ssim": s,
              "wall_time_s": time.perf_counter() - t_start})
    if out_dir is not None:
        tr.save_checkpoint(out_dir / "final.plnx", cfg.total_steps)
    return TrainResult(grid=tr.grid, metrics=metrics, config=cfg, background=tr.background,
                       scene_scale=tr.scene_scale)
