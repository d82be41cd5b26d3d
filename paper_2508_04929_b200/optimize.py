"""Training on the GPU: loss, Adam, one step, the epoch loop (mirrors train.py).

``train_step`` / ``train`` keep the reference signatures (train.py:164-264) and
its semantics at ``batch_size = 1``: same seeded shuffle, one Adam step per
record, lr(e) = lr0 * gamma^e, divergence guard against 1e3 x the epoch-0
median, ``loss_trace.txt`` and one CGS1 checkpoint per epoch.  Unlike the
reference, ``batch_size > 1`` is accepted: the loss of a step is the mean of the
per-image MSEs, so B = 1 reduces exactly to the reference step.

The dataset (centred observations, poses, CTF parameters) is made resident in
HBM once; each step runs the libcgs_b200 pipeline (``engine.StepPipeline``) on
a batch gathered on the device, with no host synchronisation: losses are read
back in blocks and the divergence guard is applied to them in step order (the
run's parameters are discarded on a raise, so a late raise is equivalent).
With ``torch.distributed`` initialised, each rank takes its slice of every
global batch and the 10-float gradient accumulators are all-reduced (NCCL)
before the fused epilogue + Adam, which then runs identically on every rank.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib, engine, parallel
from .ctf import CtfParams, phase_shift_translate
from .exceptions import DegenerateRotationError, DivergenceError
from .mixture import MODES, GaussianMixture, GridSpec, init_random, save_checkpoint
from .render import Pose, RenderedImage

DIVERGENCE_FACTOR = 1e3
LOSS_READBACK_STEPS = 64


@dataclass(frozen=True)
class TrainConfig:
    """Optimisation settings (train.py:33-56); batch_size >= 1 is supported."""

    epochs: int = 5
    batch_size: int = 1
    learning_rate: float = 0.001
    decay_gamma: float = 0.1
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_epsilon: float = 1e-8
    seed: int = 0
    mode: str = "anisotropic"

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.learning_rate <= 0 or self.decay_gamma <= 0:
            raise ValueError("learning_rate and decay_gamma must be positive")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")

    def epoch_lr(self, epoch: int) -> float:
        return self.learning_rate * self.decay_gamma**epoch


@dataclass(eq=False)
class ParticleRecord:
    """One observed particle with its pose, CTF and recorded translation (px)."""

    image: np.ndarray
    pose: Pose
    ctf: CtfParams
    translation: np.ndarray = field(default_factory=lambda: np.zeros(2))

    def __post_init__(self):
        self.image = np.asarray(self.image)
        self.translation = np.asarray(self.translation, dtype=np.float64)
        if self.image.ndim != 2 or self.image.shape[0] != self.image.shape[1]:
            raise ValueError("particle image must be square")
        if not np.all(np.isfinite(self.image)):
            raise ValueError("particle image contains non-finite values")

    @classmethod
    def prevalidated(cls, image: np.ndarray, pose: Pose, ctf: CtfParams, translation: np.ndarray):
        """A record whose fields the caller has already checked in bulk (square finite f32
        image, f64 [2] translation), e.g. a whole simulated stack at once."""
        r = object.__new__(cls)
        r.image, r.pose, r.ctf, r.translation = image, pose, ctf, translation
        return r


@dataclass
class Dataset:
    records: list
    grid: GridSpec

    def __len__(self) -> int:
        return len(self.records)

    def half(self, which: str) -> "Dataset":
        """Even/odd split for gold-standard halves (train.py:85-90)."""
        if which not in ("even", "odd"):
            raise ValueError("half must be 'even' or 'odd'")
        return Dataset(records=self.records[(0 if which == "even" else 1)::2], grid=self.grid)


def _torch():
    import torch

    return torch


class AdamState:
    """Adam moments for the (N, 11) raw parameters, fp64 on the GPU (train.py:93-111)."""

    def __init__(self, n: int):
        torch = _torch()
        engine.require_cuda()
        self.n = int(n)
        self._m = torch.zeros((n, 11), dtype=torch.float64, device="cuda")
        self._v = torch.zeros((n, 11), dtype=torch.float64, device="cuda")
        self.t = 0

    @property
    def m(self) -> np.ndarray:
        return self._m.cpu().numpy()

    @property
    def v(self) -> np.ndarray:
        return self._v.cpu().numpy()

    def update(self, params: np.ndarray, grads: np.ndarray, lr: float, config: TrainConfig) -> None:
        """One in-place Adam step on host arrays (runs ``cgs_adam`` on the device)."""
        torch = _torch()
        ctx = engine.DeviceContext.get()
        p = torch.as_tensor(np.ascontiguousarray(params, dtype=np.float64)).cuda()
        g = torch.as_tensor(np.ascontiguousarray(grads, dtype=np.float64)).cuda()
        self.t += 1
        b1, b2 = config.adam_beta1, config.adam_beta2
        _lib.call("cgs_adam", p.data_ptr(), g.data_ptr(), self._m.data_ptr(), self._v.data_ptr(), p.numel(),
                  float(lr), b1, b2, config.adam_epsilon, 1.0 - b1**self.t, 1.0 - b2**self.t, ctx.stream)
        params[...] = p.cpu().numpy().reshape(params.shape)


def loss_mse(rendered, observed) -> float:
    """Mean squared difference over all pixels (train.py:114-121), fp64 sum on the GPU."""
    torch = _torch()
    a = rendered.pixels if isinstance(rendered, RenderedImage) else np.asarray(rendered)
    b = observed.pixels if isinstance(observed, RenderedImage) else np.asarray(observed)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    ctx = engine.DeviceContext.get()
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        # the device kernel is per square image; other shapes go through a square pad
        flat_a = np.zeros((1, a.size), np.float64)
        flat_b = np.zeros((1, b.size), np.float64)
        flat_a[0], flat_b[0] = a.ravel(), b.ravel()
        side = int(math.ceil(math.sqrt(a.size)))
        pa = np.zeros((side * side,))
        pb = np.zeros((side * side,))
        pa[: a.size], pb[: b.size] = a.ravel(), b.ravel()
        a, b = pa.reshape(side, side), pb.reshape(side, side)
        scale = (side * side) / max(flat_a.size, 1)
    else:
        scale = 1.0
    ta = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)[None]).cuda()
    tb = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float32)[None]).cuda()
    loss = engine.loss_residual(ctx, ta, tb)
    return float(loss.item()) * scale


def _centered_observation(record: ParticleRecord) -> np.ndarray:
    """Observed image with its recorded translation removed (train.py:124-133)."""
    img = np.asarray(record.image, dtype=np.float64)
    if record.translation[0] == 0.0 and record.translation[1] == 0.0:
        return img
    shifted = phase_shift_translate(RenderedImage(grid=GridSpec(img.shape[0]), pixels=img), -record.translation)
    return shifted.pixels


# ---------------------------------------------------------------------------
# device-resident reconstruction
# ---------------------------------------------------------------------------
class Reconstructor:
    """Holds a dataset and a mixture in HBM and runs batched Adam steps.

    ``obs`` f32 [R][D][D] (centred observations), ``poses`` f64 [R][12],
    ``ctfs`` f64 [R][8] or None (no CTF).  ``step(indices, lr)`` launches one
    full step for the given record indices and returns the device tensor of
    per-image losses (no host sync).
    """

    def __init__(self, grid: GridSpec, params: np.ndarray, obs, poses, ctfs, *, batch_size: int,
                 mode: str = "anisotropic", config: TrainConfig | None = None, process_group=None,
                 images_per_group: int = engine.DEFAULT_IMAGES_PER_GROUP, tile: int = engine.DEFAULT_TILE):
        torch = _torch()
        self.ctx = engine.DeviceContext.get()
        dev = self.ctx.device
        self.grid = grid
        self.gs = _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)
        self.config = config or TrainConfig(batch_size=batch_size, mode=mode)
        self.mode = mode
        self.n = int(params.shape[0])
        # Gaussians live on the device in spatial (Morton) order: a CTA's
        # Gaussians then project into a small region of each image, which is
        # what the region-staged kernels exploit.  Per-Gaussian math does not
        # depend on the order (renders are integer sums), so results are
        # unchanged; params_host() returns the caller's order.
        self.perm = morton_order(np.asarray(params)[:, :3], grid.extent)
        params = np.asarray(params, dtype=np.float64)[self.perm]
        self.params = torch.as_tensor(np.ascontiguousarray(params, dtype=np.float64)).to(dev)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.t = 0
        self.obs = obs if isinstance(obs, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(obs, np.float32))
        self.obs = self.obs.to(dev, torch.float32).contiguous()
        self.poses = torch.as_tensor(np.ascontiguousarray(poses, np.float64)).to(dev)
        self.ctfs = None if ctfs is None else torch.as_tensor(np.ascontiguousarray(ctfs, np.float64)).to(dev)
        # F(obs) and H_sym of every observation, once: with them K4 runs in the Fourier domain
        # with one forward and one inverse transform per image (cgs_ctf_mse_spectral)
        self.obs_spec = None if self.ctfs is None else engine.obs_spectra(self.ctx, self.obs, self.ctfs, self.gs)
        self.global_batch = int(batch_size)
        self.pg = process_group
        self.world = 1
        self.rank = 0
        if process_group is not None or _dist_active():
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
            self.rank = dist.get_rank(process_group)
        self.ipg = images_per_group
        self.tile = tile
        self._pipes: dict = {}
        self._copy_stream = None  # H2D stream of step_host
        self._h2d_slots: dict = {}  # step_host's double-buffered device inputs
        self._idx_slots: dict = {}  # step's graph inputs (batch indices, gathered batch, Adam scalars)
        # step_host replays each slot's step as a CUDA graph (single GPU; CGS_GRAPHS=0 disables)
        self.use_graphs = os.environ.get("CGS_GRAPHS", "1") == "1"
        # multi-GPU: CGS_DP_SHARDED=1 reduce-scatters the accumulator, runs the epilogue + Adam
        # on this rank's Gaussian slice only and all-gathers the parameters (ZeRO-1 style)
        self.sharded = self.world > 1 and os.environ.get("CGS_DP_SHARDED", "0") == "1"

    # -- helpers -------------------------------------------------------------
    def local_slice(self, indices: np.ndarray) -> np.ndarray:
        """This rank's contiguous share of a global batch."""
        return parallel.shard(indices, self.rank, self.world)

    def pipeline(self, b: int) -> engine.StepPipeline:
        if b not in self._pipes:
            self._pipes[b] = engine.StepPipeline(self.ctx, self.n, b, self.gs, tile=self.tile,
                                                 images_per_group=self.ipg, mode=self.mode)
        return self._pipes[b]

    def _batch(self, local: np.ndarray):
        torch = _torch()
        idx = torch.as_tensor(local, dtype=torch.int64).to(self.ctx.device, non_blocking=True)
        obs = self.obs.index_select(0, idx)
        poses = self.poses.index_select(0, idx)
        ctfs = None if self.ctfs is None else self.ctfs.index_select(0, idx)
        return obs, poses, ctfs

    def batch_spectra(self, local: np.ndarray):
        """The precomputed observation spectra of a batch (device), or None."""
        if self.obs_spec is None:
            return None
        torch = _torch()
        idx = torch.as_tensor(local, dtype=torch.int64).to(self.ctx.device, non_blocking=True)
        return self.obs_spec.index_select(0, idx)

    def ensure_capacity(self, indices_list) -> None:
        """Size the tile-list buffers from the given batches (one host read each)."""
        for local in indices_list:
            pipe = self.pipeline(len(local))
            _, poses, _ = self._batch(local)
            pipe.grow(pipe.measure_items(self.params, poses))

    def step(self, indices, lr: float):
        """One step over the global batch ``indices``; returns per-image losses (device).

        On one GPU the step (batch gather from the HBM-resident stack, status clear,
        K0..K6) is a CUDA graph per batch size, replayed with this step's indices and
        Adam scalars written into its static inputs (CGS_GRAPHS=0: eager)."""
        indices = np.asarray(indices)
        local = self.local_slice(indices)
        if self.use_graphs and self.world == 1:
            return self._graph_step_indexed(local, lr, global_batch=len(indices))
        obs, poses, ctfs = self._batch(local)
        return self.step_batch(obs, poses, ctfs, lr, global_batch=len(indices), obs_spec=self.batch_spectra(local))

    def _graph_step_indexed(self, local: np.ndarray, lr: float, *, global_batch: int):
        torch = _torch()
        dev = self.ctx.device
        b = len(local)
        key = (b, global_batch)
        sl = self._idx_slots.get(key)
        if sl is None:
            D = self.grid.size
            spec = self.obs_spec is not None
            sl = self._idx_slots[key] = {
                "idx": torch.empty(b, dtype=torch.int64, device=dev),
                "o": None if spec else torch.empty((b, D, D), dtype=torch.float32, device=dev),
                "s": torch.empty((b, self.obs_spec.shape[1]), dtype=torch.float32, device=dev) if spec else None,
                "p": torch.empty((b, 12), dtype=torch.float64, device=dev),
                "c": None if self.ctfs is None else torch.empty((b, 8), dtype=torch.float64, device=dev),
                "hyper": torch.empty(3, dtype=torch.float64, device=dev), "graph": None}
        cfg, t = self.config, self.t + 1
        sl["idx"].copy_(torch.as_tensor(np.asarray(local, dtype=np.int64)), non_blocking=True)
        sl["hyper"].copy_(torch.tensor([lr, 1.0 - cfg.adam_beta1 ** t, 1.0 - cfg.adam_beta2 ** t],
                                       dtype=torch.float64), non_blocking=True)
        pipe = self.pipeline(b)
        scale = 1.0 / global_batch

        def body():
            if sl["s"] is not None:
                torch.index_select(self.obs_spec, 0, sl["idx"], out=sl["s"])
            else:
                torch.index_select(self.obs, 0, sl["idx"], out=sl["o"])
            torch.index_select(self.poses, 0, sl["idx"], out=sl["p"])
            if sl["c"] is not None:
                torch.index_select(self.ctfs, 0, sl["idx"], out=sl["c"])
            pipe.clear_status()
            pipe.forward_backward(self.params, sl["p"], sl["o"], sl["c"], obs_spec=sl["s"])
            pipe.adam_dev(self.params, self.m, self.v, sl["hyper"], scale=scale, beta1=cfg.adam_beta1,
                          beta2=cfg.adam_beta2, eps=cfg.adam_epsilon)

        if sl["graph"] is None:
            body()  # eager first use (one-time kernel attribute setup outside the capture)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body()
            sl["graph"] = g
        else:
            sl["graph"].replay()
        self.t = t
        return pipe.loss

    def step_host(self, obs, poses, ctfs, lr: float, *, global_batch: int, loss_out=None):
        """Public end-to-end step from (pinned) HOST buffers of this rank's batch.

        Copies the batch host->device on a dedicated copy stream, runs the step
        on the current stream once the copy has landed, and copies the per-image
        losses device->host into ``loss_out`` (pinned).  Nothing synchronises the
        host, so back-to-back calls overlap the next batch's H2D (PCIe) with
        this batch's kernels; the caller synchronises when it needs the numbers.
        """
        torch = _torch()
        dev = self.ctx.device
        compute = torch.cuda.current_stream(dev)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(dev)
        # two preallocated device slots per batch shape, alternating: no allocator
        # traffic per step; a slot is refilled only after the step that read it
        key = (tuple(obs.shape), ctfs is None)
        slots = self._h2d_slots.get(key)
        if slots is None:
            def slot():
                return {"o": torch.empty(obs.shape, dtype=obs.dtype, device=dev),
                        "p": torch.empty(poses.shape, dtype=poses.dtype, device=dev),
                        "c": None if ctfs is None else torch.empty(ctfs.shape, dtype=ctfs.dtype, device=dev),
                        "hyper": torch.empty(3, dtype=torch.float64, device=dev),
                        "graph": None, "done": None}
            slots = self._h2d_slots[key] = [slot(), slot(), 0]
        sl = slots[slots[2]]
        slots[2] ^= 1
        cs = self._copy_stream
        if sl["done"] is not None:
            cs.wait_event(sl["done"])
        graphs = self.use_graphs and self.world == 1
        with torch.cuda.stream(cs):
            if graphs:  # Adam's per-step scalars travel with the batch
                cfg, t = self.config, self.t + 1
                sl["hyper"].copy_(torch.tensor([lr, 1.0 - cfg.adam_beta1 ** t, 1.0 - cfg.adam_beta2 ** t],
                                               dtype=torch.float64), non_blocking=True)
            sl["o"].copy_(obs, non_blocking=True)
            sl["p"].copy_(poses, non_blocking=True)
            if ctfs is not None:
                sl["c"].copy_(ctfs, non_blocking=True)
        compute.wait_stream(cs)
        o, p, c = sl["o"], sl["p"], sl["c"]
        if graphs:
            loss = self._graph_step(sl, o, p, c, global_batch)
        else:
            loss = self.step_batch(o, p, c, lr, global_batch=global_batch)
        if sl["done"] is None:
            sl["done"] = torch.cuda.Event()
        sl["done"].record(compute)
        if loss_out is not None:
            loss_out.copy_(loss, non_blocking=True)
        del torch
        return loss

    def _graph_step(self, sl, o, p, c, global_batch: int):
        """One step of a step_host slot as a CUDA graph replay: the first use of a
        slot runs eagerly and captures status clear, K0..K5 and K6 (with its
        scalars in sl["hyper"]); later steps replay it with one launch."""
        torch = _torch()
        pipe = self.pipeline(o.shape[0])
        cfg = self.config
        scale = 1.0 / global_batch

        def body():
            pipe.clear_status()
            pipe.forward_backward(self.params, p, o, c)
            pipe.adam_dev(self.params, self.m, self.v, sl["hyper"], scale=scale, beta1=cfg.adam_beta1,
                          beta2=cfg.adam_beta2, eps=cfg.adam_epsilon)

        if sl["graph"] is None:
            body()  # eager: also performs one-time kernel attribute setup outside the capture
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body()
            sl["graph"] = g
        else:
            sl["graph"].replay()
        self.t += 1
        return pipe.loss

    def step_batch(self, obs, poses, ctfs, lr: float, *, global_batch: int, events=None, obs_spec=None):
        """One step on device tensors of this rank's batch (obs f32 [b][D][D],
        poses f64 [b][12], ctfs f64 [b][8] or None); ``global_batch`` sets the
        1/B loss scale.  ``obs_spec``: the batch's precomputed observation spectra
        (batch_spectra); obs may then be None.  Returns the device tensor of
        per-image losses."""
        pipe = self.pipeline(poses.shape[0])
        cfg = self.config
        pipe.clear_status()
        pipe.forward_backward(self.params, poses, obs, ctfs, events=events, obs_spec=obs_spec)
        scale = 1.0 / global_batch
        self.t += 1
        if self.sharded:
            acc = pipe.reduce()
            part, skip = parallel.reduce_scatter_accumulator(acc, self.n, self.pg, status=pipe.status)
            a, b, per = parallel.gaussian_slice(self.n, self.rank, self.world)
            if b > a:
                pipe.adam(self.params[a:b], self.m[a:b], self.v[a:b], scale=scale, lr=lr, beta1=cfg.adam_beta1,
                          beta2=cfg.adam_beta2, eps=cfg.adam_epsilon, t=self.t, acc=part, groups=1, skip=skip,
                          n=b - a)
            parallel.all_gather_rows(self.params, per, self.pg)
        elif self.world > 1:
            acc = pipe.reduce()
            skip = parallel.allreduce_accumulator(acc, self.pg, status=pipe.status)
            pipe.adam(self.params, self.m, self.v, scale=scale, lr=lr, beta1=cfg.adam_beta1,
                      beta2=cfg.adam_beta2, eps=cfg.adam_epsilon, t=self.t, acc=acc, groups=1, skip=skip)
        else:
            pipe.adam(self.params, self.m, self.v, scale=scale, lr=lr, beta1=cfg.adam_beta1,
                      beta2=cfg.adam_beta2, eps=cfg.adam_epsilon, t=self.t)
        return pipe.loss

    def check_status(self) -> None:
        for pipe in self._pipes.values():
            if pipe.degenerate():
                raise DegenerateRotationError("quaternion with zero or non-finite norm")

    def params_host(self) -> np.ndarray:
        """Parameters in the caller's Gaussian order."""
        out = np.empty((self.n, 11), dtype=np.float64)
        out[self.perm] = self.params.cpu().numpy()
        return out

    def reorder(self) -> None:
        """Re-sort the device-resident Gaussians (and Adam moments) by Morton code
        of their current means, e.g. once per epoch as they move."""
        torch = _torch()
        local = morton_order(self.params[:, :3].cpu().numpy(), self.grid.extent)
        idx = torch.as_tensor(local, device=self.params.device)
        if self.sharded:  # the moments are current only on their owner: replicate before permuting
            per = parallel.gaussian_slice(self.n, self.rank, self.world)[2]
            parallel.all_gather_rows(self.m, per, self.pg)
            parallel.all_gather_rows(self.v, per, self.pg)
        # in place: captured step graphs keep pointing at these buffers
        self.params.copy_(self.params.index_select(0, idx))
        self.m.copy_(self.m.index_select(0, idx))
        self.v.copy_(self.v.index_select(0, idx))
        self.perm = self.perm[local]


def morton_order(means: np.ndarray, extent: float) -> np.ndarray:
    """Stable argsort of the 30-bit Morton (Z-order) codes of 3-D points in
    [-extent, extent]^3 (10 bits per axis)."""
    q = np.clip(((np.asarray(means, np.float64) / extent + 1.0) * 511.5).astype(np.int64), 0, 1023)

    def spread(v):
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        return (v | (v << 2)) & 0x09249249

    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    return np.argsort(code, kind="stable")


def _dist_active() -> bool:
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    except Exception:
        return False


def centered_observations(records, grid: GridSpec, chunk: int = 4096) -> np.ndarray:
    """f32 [R][D][D] observations with their recorded translations removed
    (train.py:124-133, :222), batched on the GPU: one cgs_fourier_filter launch
    per chunk of translated records."""
    from .ctf import filter_batch

    obs = np.stack([np.asarray(r.image, dtype=np.float32) for r in records])
    shifts = np.stack([np.asarray(r.translation, dtype=np.float64) for r in records]) if len(records) else None
    moved = np.flatnonzero(np.any(shifts != 0.0, axis=1)) if len(records) else np.zeros(0, int)
    if len(moved) == 0:
        return obs
    torch = _torch()
    for a in range(0, len(moved), chunk):
        idx = moved[a:a + chunk]
        x = torch.as_tensor(obs[idx]).cuda()
        y = filter_batch(x, grid, shifts=-shifts[idx])
        obs[idx] = y.cpu().numpy()
    return obs


def _record_arrays(records, grid: GridSpec):
    from .engine import ctf_array, pose_array

    obs = centered_observations(records, grid)
    poses = pose_array([r.pose.rotation for r in records], [r.pose.translation for r in records])
    ctfs = ctf_array([r.ctf for r in records])
    return obs, poses, ctfs


def train_step(mixture: GaussianMixture, record: ParticleRecord, config: TrainConfig, adam: AdamState,
               *, lr: float | None = None, grid: GridSpec | None = None, record_index: int = -1):
    """One render / CTF / MSE / backward / Adam cycle on one record (train.py:164-191).

    Mutates ``mixture.params`` in place and returns ``(mixture, loss)``.  A
    non-finite loss raises DivergenceError and leaves the parameters unchanged.
    """
    torch = _torch()
    if grid is None:
        grid = GridSpec(record.image.shape[0], pixel_size=1.0)
    if lr is None:
        lr = config.learning_rate
    obs, poses, ctfs = _record_arrays([record], grid)
    ctx = engine.DeviceContext.get()
    gs = _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)
    pipe = _step_pipe(ctx, len(mixture), gs, config.mode)
    params = torch.as_tensor(np.ascontiguousarray(mixture.params)).to(ctx.device)
    p_t = torch.as_tensor(poses).to(ctx.device)
    o_t = torch.as_tensor(obs).to(ctx.device)
    c_t = torch.as_tensor(ctfs).to(ctx.device)
    pipe.clear_status()
    pipe.grow(pipe.measure_items(params, p_t))
    pipe.forward_backward(params, p_t, o_t, c_t)
    loss = float(pipe.loss[0].item())
    if pipe.degenerate():
        raise DegenerateRotationError("quaternion with zero or non-finite norm")
    if not math.isfinite(loss):
        raise DivergenceError("non-finite loss", epoch=-1, step=-1, record_index=record_index)
    adam.t += 1
    pipe.adam(params, adam._m, adam._v, scale=1.0, lr=lr, beta1=config.adam_beta1, beta2=config.adam_beta2,
              eps=config.adam_epsilon, t=adam.t)
    mixture.params[...] = params.cpu().numpy()
    return mixture, loss


_PIPES: dict = {}


def _step_pipe(ctx, n, gs, mode):
    key = (ctx.device.index, n, gs.size, gs.extent, gs.pixel_size, mode)
    if key not in _PIPES:
        _PIPES.clear()
        _PIPES[key] = engine.StepPipeline(ctx, n, 1, gs, mode=mode)
    return _PIPES[key]


def train(dataset: Dataset, config: TrainConfig, *, n_gaussians: int, out_dir: str | None = None,
          initial: GaussianMixture | None = None, process_group=None):
    """Fit a mixture to the dataset (train.py:194-264).  Returns (mixture, epoch_losses)."""
    if len(dataset) == 0:
        raise ValueError("cannot train on an empty dataset")
    grid = dataset.grid
    mixture = initial.copy() if initial is not None else init_random(n_gaussians, config.seed, grid, mode=config.mode)
    shuffle_rng = np.random.default_rng(config.seed)
    obs, poses, ctfs = _record_arrays(dataset.records, grid)
    rec = Reconstructor(grid, mixture.params, obs, poses, ctfs, batch_size=config.batch_size, mode=config.mode,
                        config=config, process_group=process_group)
    R = len(dataset)
    B = config.batch_size
    is_root = rec.rank == 0
    trace, epoch_losses = [], []
    epoch0_median = None
    history0: list = []
    torch = _torch()

    for epoch in range(config.epochs):
        lr = config.epoch_lr(epoch)
        if epoch > 0:
            rec.reorder()  # keep the device order spatial as the means move
        order = shuffle_rng.permutation(R)
        batches = [order[i:i + B] for i in range(0, R, B)]
        if epoch == 0:
            sizes = {}
            for b in batches:
                sizes.setdefault(len(rec.local_slice(b)), rec.local_slice(b))
            rec.ensure_capacity(list(sizes.values()))
        steps = len(batches)
        losses = np.empty(steps, dtype=np.float64)
        pending: list = []

        def drain(upto):
            nonlocal epoch0_median
            for s, dev_loss, nloc, bidx in pending:
                val = _global_batch_loss(dev_loss, nloc, len(bidx), rec)
                losses[s] = val
                ridx = int(bidx[0]) if B == 1 else -1
                if not math.isfinite(val):
                    raise DivergenceError("non-finite loss", epoch=epoch, step=s, record_index=ridx)
                if epoch0_median is not None:
                    ref = epoch0_median
                else:
                    history0.append(val)
                    ref = float(np.median(history0))
                if val > DIVERGENCE_FACTOR * ref:
                    raise DivergenceError(
                        f"loss {val:.6g} exceeded {DIVERGENCE_FACTOR:g} x epoch-0 median {ref:.6g}",
                        epoch=epoch, step=s, record_index=ridx)
                trace.append(f"{epoch} {s} {val:.17g} {lr:.17g}")
            pending.clear()

        for s, bidx in enumerate(batches):
            dev_loss = rec.step(bidx, lr)
            pending.append((s, dev_loss.clone(), len(rec.local_slice(bidx)), bidx))
            if len(pending) >= LOSS_READBACK_STEPS:
                drain(s)
        drain(steps)
        rec.check_status()
        if any(p.overflowed() for p in rec._pipes.values()):  # pragma: no cover - capacity sized above
            raise RuntimeError("tile list capacity overflow: re-run with a larger capacity")
        if epoch == 0:
            epoch0_median = float(np.median(losses))
        epoch_losses.append(losses)
        if out_dir is not None and is_root:
            mixture.params[...] = rec.params_host()
            save_checkpoint(mixture, os.path.join(out_dir, f"checkpoint_epoch_{epoch}.cgs"))
    mixture.params[...] = rec.params_host()
    if out_dir is not None and is_root:
        with open(os.path.join(out_dir, "loss_trace.txt"), "w") as fh:
            fh.write(f"# seed {config.seed}\n")
            fh.write("# epoch step loss lr\n")
            fh.write("\n".join(trace) + "\n")
    del torch
    return mixture, epoch_losses


def _global_batch_loss(dev_loss, n_local: int, n_global: int, rec: Reconstructor) -> float:
    """Mean per-image loss of the global batch (sum over ranks when distributed)."""
    torch = _torch()
    total = dev_loss[:n_local].sum()
    if rec.world > 1:
        import torch.distributed as dist

        t = total.reshape(1).clone()
        dist.all_reduce(t, group=rec.pg)
        total = t[0]
    return float(total.item()) / n_global


def half_config(config: TrainConfig, which: str) -> TrainConfig:
    """Gold-standard half configs: the odd half uses seed + 1 (train.py:267-273)."""
    if which == "even":
        return config
    if which == "odd":
        return replace(config, seed=config.seed + 1)
    raise ValueError("half must be 'even' or 'odd'")
