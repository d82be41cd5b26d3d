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
class _StepRunner:
    """One step shape as a list of segments: ("dev", fn) device work on the current stream,
    ("coll", fn) a collective.  With graphs the first run is eager (one-time kernel attribute
    setup, NCCL communicator warm-up) and the step is then captured: as one CUDA graph when
    every segment can be captured (single GPU, or NCCL collectives), else one graph per device
    segment with the collectives run eagerly between the replays (gloo)."""

    def __init__(self, segments, graphs: bool, whole: bool):
        self.segments, self.graphs, self.whole = segments, graphs, whole
        self._plan = None
        self._graphs = []

    @property
    def captured(self) -> bool:
        return self._plan is not None

    def run(self) -> None:
        if not self.graphs:
            for _, fn in self.segments:
                fn()
            return
        if self._plan is not None:
            for _, fn in self._plan:
                fn()
            return
        torch = _torch()
        for _, fn in self.segments:
            fn()
        plan = []
        if self.whole:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _, fn in self.segments:
                    fn()
            self._graphs.append(g)
            plan.append(("dev", g.replay))
        else:
            for kind, fn in self.segments:
                if kind == "dev":
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        fn()
                    self._graphs.append(g)
                    plan.append(("dev", g.replay))
                else:
                    plan.append((kind, fn))
        self._plan = plan


class Reconstructor:
    """Holds a dataset and a mixture in HBM and runs batched Adam steps.

    ``obs`` f32 [R][D][D] (centred observations), ``poses`` f64 [R][12],
    ``ctfs`` f64 [R][8] or None (no CTF).  ``step(indices, lr)`` launches one
    full step for the given global batch of record indices (this rank runs its
    shard of it) and returns the device tensor of this rank's per-image losses
    (no host sync).

    Data parallel (``process_group`` or an initialised default group with more
    than one rank): the step is K0..K5 on the local shard, the accumulator
    exchange (``parallel.Exchange``: all-reduce, or reduce-scatter + parameter
    all-gather with ``CGS_DP_SHARDED=1``) and the fused epilogue + Adam, all
    graph-captured (see ``_StepRunner``).  A rank whose shard of a short batch
    is empty still joins the exchange with a zero accumulator.

    Residency: ``"full"`` keeps every record (and its spectral-K4 record) in
    HBM; ``"epoch"`` (default with more than one rank) keeps only the records
    this rank touches in the current epoch, 1/world of the dataset, loaded by
    ``begin_epoch`` (and prefetched for the next epoch on a copy stream).
    """

    def __init__(self, grid: GridSpec, params: np.ndarray, obs, poses, ctfs, *, batch_size: int,
                 mode: str = "anisotropic", config: TrainConfig | None = None, process_group=None,
                 images_per_group: int | None = None, tile: int = engine.DEFAULT_TILE,
                 residency: str | None = None):
        torch = _torch()
        self.ctx = engine.DeviceContext.get()
        dev = self.ctx.device
        self.grid = grid
        self.gs = _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)
        self.config = config or TrainConfig(batch_size=batch_size, mode=mode)
        self.mode = mode
        self.n = int(params.shape[0])
        self.global_batch = int(batch_size)
        self.pg = process_group
        self.world, self.rank = 1, 0
        if process_group is not None or _dist_active():
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
            self.rank = dist.get_rank(process_group)
        # multi-GPU: CGS_DP_SHARDED=1 reduce-scatters the accumulator, runs the epilogue + Adam
        # on this rank's Gaussian slice only and all-gathers the parameters (ZeRO-1 style).
        # CGS_DP_EXCHANGE=1 keeps the exchange even in a 1-rank group (exercises the collective
        # path, e.g. NCCL graph capture, on a single GPU).
        # CGS_DP_PEER=1: the sharded exchange as one kernel over peer memory (parallel.PeerExchange).
        dp = self.world > 1 or (self.pg is not None and os.environ.get("CGS_DP_EXCHANGE", "0") == "1")
        self.peer = dp and os.environ.get("CGS_DP_PEER", "0") == "1"
        self.sharded = dp and (self.peer or os.environ.get("CGS_DP_SHARDED", "0") == "1")
        self.xch = None
        if dp:
            per = parallel.gaussian_slice(self.n, self.rank, self.world)[2] if self.sharded else self.n
            sf = int(self.ctx.lib.cgs_acc_slice_floats(self.n, per))
            if self.peer:
                self.xch = parallel.PeerExchange(self.n, process_group, device=dev, slice_floats=sf)
            else:
                self.xch = parallel.Exchange(self.n, process_group, sharded=self.sharded, device=dev, slice_floats=sf)
        # Gaussians live on the device in spatial (Morton) order: a CTA's
        # Gaussians then project into a small region of each image, which is
        # what the region-staged kernels exploit.  Per-Gaussian math does not
        # depend on the order (renders are integer sums), so results are
        # unchanged; params_host() returns the caller's order.  The fp64
        # parameters and moments sit in buffers padded to world x ceil(N / world)
        # rows in sharded mode, so the parameter all-gather runs in place.
        self.perm = morton_order(np.asarray(params)[:, :3], grid.extent)
        params = np.asarray(params, dtype=np.float64)[self.perm]
        rows = self.xch.per * self.world if self.sharded else self.n
        self._store = self.xch.store if self.peer else torch.zeros((rows, 11), dtype=torch.float64, device=dev)
        self._m_store = torch.zeros_like(self._store)
        self._v_store = torch.zeros_like(self._store)
        self._store[: self.n].copy_(torch.as_tensor(np.ascontiguousarray(params)))
        self.params, self.m, self.v = self._store[: self.n], self._m_store[: self.n], self._v_store[: self.n]
        self.t = 0
        # dataset
        self.residency = residency or ("epoch" if self.world > 1 else "full")
        if self.residency not in ("full", "epoch"):
            raise ValueError(f"unknown residency {self.residency!r}")
        R = len(poses)
        self.n_records = R
        self._poses_all = torch.as_tensor(np.ascontiguousarray(poses, np.float64)).to(dev)
        self._ctfs_all = None if ctfs is None else torch.as_tensor(np.ascontiguousarray(ctfs, np.float64)).to(dev)
        if self.residency == "full":
            o = obs if isinstance(obs, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(obs, np.float32))
            self.obs = o.to(dev, torch.float32).contiguous()
            self.poses, self.ctfs = self._poses_all, self._ctfs_all
            # F(obs) and H_sym of every observation, once: with them K4 runs in the Fourier domain
            # with one forward and one inverse transform per image (cgs_ctf_mse_spectral)
            self.obs_spec = None if self.ctfs is None else engine.obs_spectra(self.ctx, self.obs, self.ctfs, self.gs)
            self._slot = np.arange(R)
        else:
            o = obs.cpu() if isinstance(obs, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(obs, np.float32))
            self._obs_host = o.to(torch.float32).contiguous().pin_memory()
            self.obs = self.poses = self.ctfs = self.obs_spec = None
            self._slot = np.full(R, -1, dtype=np.int64)
            self._epoch_key = None
            self._staged = None
        self.ipg = images_per_group
        self.tile = tile
        self._pipes: dict = {}
        self._copy_stream = None  # H2D stream of step_host and of the epoch prefetch
        self._h2d_slots: dict = {}  # step_host's double-buffered device inputs
        self._idx_slots: dict = {}  # step's graph inputs (batch indices, gathered batch, Adam scalars)
        # each step shape is captured as a CUDA graph (CGS_GRAPHS=0: eager); with NCCL the
        # collectives are inside the graph (CGS_DP_GRAPH_COLLECTIVES=0 keeps them outside)
        self.use_graphs = os.environ.get("CGS_GRAPHS", "1") == "1"
        self._whole_graph = self.xch is None or (self.xch.capturable and
                                                 os.environ.get("CGS_DP_GRAPH_COLLECTIVES", "1") == "1")
        self._empty_loss = torch.zeros(0, dtype=torch.float64, device=dev)

    # -- helpers -------------------------------------------------------------
    def local_slice(self, indices: np.ndarray) -> np.ndarray:
        """This rank's contiguous share of a global batch."""
        return parallel.shard(indices, self.rank, self.world)

    def pipeline(self, b: int) -> engine.StepPipeline:
        if b < 1:
            raise ValueError("a step pipeline needs at least one image")
        if b not in self._pipes:
            self._pipes[b] = engine.StepPipeline(self.ctx, self.n, b, self.gs, tile=self.tile,
                                                 images_per_group=self.ipg, mode=self.mode)
        return self._pipes[b]

    def slots(self, records) -> np.ndarray:
        """Device rows of the given records in the resident set (raises if one is not resident)."""
        s = self._slot[np.asarray(records, dtype=np.int64)]
        if len(s) and s.min() < 0:
            raise RuntimeError("record not resident on this rank: call begin_epoch(order) first")
        return s

    def _batch(self, local: np.ndarray):
        torch = _torch()
        idx = torch.as_tensor(self.slots(local), dtype=torch.int64).to(self.ctx.device, non_blocking=True)
        obs = self.obs.index_select(0, idx)
        poses = self.poses.index_select(0, idx)
        ctfs = None if self.ctfs is None else self.ctfs.index_select(0, idx)
        return obs, poses, ctfs

    def batch_spectra(self, local: np.ndarray):
        """The precomputed observation spectra of a batch (device), or None."""
        if self.obs_spec is None:
            return None
        torch = _torch()
        idx = torch.as_tensor(self.slots(local), dtype=torch.int64).to(self.ctx.device, non_blocking=True)
        return self.obs_spec.index_select(0, idx)

    def ensure_capacity(self, indices_list) -> None:
        """Size the tile-list buffers from the given batches (one host read each)."""
        for local in indices_list:
            if len(local) == 0:
                continue
            pipe = self.pipeline(len(local))
            _, poses, _ = self._batch(local)
            pipe.grow(pipe.measure_items(self.params, poses))

    # -- particle residency --------------------------------------------------
    def _load_records(self, records, out, stream):
        """Device copies of ``records`` into the dict ``out`` (obs, poses, ctfs, spectra), on
        ``stream``, without blocking the host: the observations are gathered straight from the
        pinned host stack by a zero-copy kernel (cgs_gather_rows), then the spectral-K4 records
        are made from them."""
        torch = _torch()
        dev = self.ctx.device
        r = len(records)
        D = self.grid.size
        if out.get("obs") is None:
            out["obs"] = torch.empty((r, D, D), dtype=torch.float32, device=dev)
            out["poses"] = torch.empty((r, 12), dtype=torch.float64, device=dev)
            out["ctfs"] = None if self._ctfs_all is None else torch.empty((r, 8), dtype=torch.float64, device=dev)
            out["idx"] = torch.empty(r, dtype=torch.int64, device=dev)
            out["idx_host"] = torch.empty(r, dtype=torch.int64).pin_memory()
            out["spec"] = None
            per = engine.obs_record_elems(self.ctx, D)
            if out["ctfs"] is not None and per:
                out["spec"] = torch.empty((r, per), dtype=torch.float32, device=dev)
        with torch.cuda.stream(stream):
            if out.get("event") is not None:  # the pinned index buffer is reused: its last copy must be done
                out["event"].synchronize()
            out["idx_host"].copy_(torch.as_tensor(np.asarray(records, dtype=np.int64)))
            out["idx"].copy_(out["idx_host"], non_blocking=True)
            engine.gather_rows(self.ctx, self._obs_host, out["idx"], out["obs"])
            torch.index_select(self._poses_all, 0, out["idx"], out=out["poses"])
            if out["ctfs"] is not None:
                torch.index_select(self._ctfs_all, 0, out["idx"], out=out["ctfs"])
            if out["spec"] is not None:
                engine.obs_spectra(self.ctx, out["obs"], out["ctfs"], self.gs, out=out["spec"])
        out["records"] = np.asarray(records)
        out["event"] = torch.cuda.Event()
        out["event"].record(stream)
        return out

    def begin_epoch(self, order, next_order=None) -> None:
        """Make this rank's records of the epoch visiting ``order`` resident (residency "epoch";
        no-op for "full").  The records are this rank's shards of the epoch's global batches
        (parallel.epoch_records), 1/world of the dataset.  With ``next_order`` the next epoch's
        records are prefetched on a copy stream while this epoch runs.  The resident buffers are
        refilled in place, so captured step graphs stay valid."""
        if self.residency != "epoch":
            return
        torch = _torch()
        recs = parallel.epoch_records(order, self.global_batch, self.rank, self.world)
        compute = torch.cuda.current_stream(self.ctx.device)
        if self.obs is None:  # first epoch: allocate the live set
            live = self._load_records(recs, {}, compute)
            self.obs, self.poses, self.ctfs, self.obs_spec = live["obs"], live["poses"], live["ctfs"], live["spec"]
            self._live = live
        else:
            st = self._staged
            if st is not None and np.array_equal(st["records"], recs):
                compute.wait_event(st["event"])
                for k in ("obs", "poses", "ctfs", "spec"):
                    if self._live.get(k) is not None:
                        self._live[k].copy_(st[k])
            else:
                self._load_records(recs, self._live, compute)
                compute.wait_event(self._live["event"])
        self._slot.fill(-1)
        self._slot[recs] = np.arange(len(recs))
        if next_order is not None:
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(self.ctx.device)
            self._copy_stream.wait_stream(compute)
            nxt = parallel.epoch_records(next_order, self.global_batch, self.rank, self.world)
            self._staged = self._load_records(nxt, self._staged or {}, self._copy_stream)

    # -- one step --------------------------------------------------------------
    def _segments(self, b: int, global_batch: int, inputs, hyper, events=None, scalars=None):
        """The step for ``b`` local images (``inputs()`` -> obs, poses, ctfs, obs_spec on the
        device) as runner segments: K0..K5 (+ the accumulator in the exchange layout), the
        exchange, epilogue + Adam (+ the parameter all-gather when sharded)."""
        cfg = self.config
        pipe = self.pipeline(b) if b > 0 else None
        scale = 1.0 / global_batch
        mode = _lib.CGS_MODE[self.mode]
        xch = self.xch
        ptr = engine._ptr

        def local():
            if pipe is not None:
                o, p, c, s, *rows = inputs()
                pipe.clear_status()
                pipe.forward_backward(self.params, p, o, c, events=events, obs_spec=s,
                                      obs_rows=rows[0] if rows else None)
            if xch is not None:
                _lib.call("cgs_reduce_partials_sliced", ptr(pipe.partial) if pipe else 0, pipe.G if pipe else 0,
                          self.n, xch.per, ptr(pipe.status) if pipe else 0, ptr(xch.acc), self.ctx.stream)

        def update():
            if events is not None and "epi" in events:
                events["epi"][0].record()
            _update()
            if events is not None and "epi" in events:
                events["epi"][1].record()

        def _update():
            if xch is None:
                acc, G, a, bb, skip = pipe.partial, pipe.G, 0, self.n, pipe.status
            else:
                (acc, a, bb), G, skip = xch.own(), 1, xch.skip
            if bb <= a:
                return
            if scalars is not None:  # eager step: Adam's per-step scalars as kernel arguments
                lr, bc1, bc2 = scalars
                _lib.call("cgs_epilogue_adam", ptr(acc), G, bb - a, ptr(self.params[a:bb]), ptr(self.m[a:bb]),
                          ptr(self.v[a:bb]), mode, float(scale), float(lr), float(cfg.adam_beta1),
                          float(cfg.adam_beta2), float(cfg.adam_epsilon), float(bc1), float(bc2), ptr(skip),
                          self.ctx.stream)
            else:  # graph replay: read from the static device tensor hyper
                _lib.call("cgs_epilogue_adam_dev", ptr(acc), G, bb - a, ptr(self.params[a:bb]), ptr(self.m[a:bb]),
                          ptr(self.v[a:bb]), mode, float(scale), float(cfg.adam_beta1), float(cfg.adam_beta2),
                          float(cfg.adam_epsilon), ptr(hyper), ptr(skip), self.ctx.stream)

        def fused():  # PeerExchange: reduce-scatter + epilogue + Adam + parameter all-gather, one launch
            per, r = xch.per, self.rank
            h = hyper if hyper is not None else self._scalar_hyper(*scalars)
            _lib.call("cgs_peer_epilogue_adam", ptr(xch.acc_ptrs), ptr(xch.store_ptrs), ptr(xch.flag_ptrs), r,
                      self.world, self.n, per, ptr(self._m_store[r * per:(r + 1) * per]),
                      ptr(self._v_store[r * per:(r + 1) * per]), mode, float(scale), float(cfg.adam_beta1),
                      float(cfg.adam_beta2), float(cfg.adam_epsilon), ptr(h), self.ctx.stream)

        if self.peer:
            return [("dev", local), ("dev", fused)], pipe
        segs = [("dev", local)]
        if xch is not None:
            segs.append(("coll", xch.run))
        segs.append(("dev", update))
        if xch is not None and self.sharded:
            segs.append(("coll", lambda: xch.gather_rows(self._store)))
        return segs, pipe

    def _hyper(self, lr: float, t: int):
        """Adam's per-step scalars (lr, bc1, bc2) and the step counter t (the peer exchange's epoch)."""
        torch = _torch()
        cfg = self.config
        return torch.tensor([lr, 1.0 - cfg.adam_beta1 ** t, 1.0 - cfg.adam_beta2 ** t, float(t)],
                            dtype=torch.float64)

    def _scalar_hyper(self, lr: float, bc1: float, bc2: float):
        """Eager steps of the peer exchange: this step's scalars in a device tensor (stream-ordered)."""
        torch = _torch()
        if getattr(self, "_hyper_dev", None) is None:
            self._hyper_dev = torch.empty(4, dtype=torch.float64, device=self.ctx.device)
        self._hyper_dev.copy_(torch.tensor([lr, bc1, bc2, float(self.t + 1)], dtype=torch.float64))
        return self._hyper_dev

    def step(self, indices, lr: float):
        """One step over the global batch ``indices``; returns this rank's per-image losses (device).

        The step (batch gather from the HBM-resident set by a device index buffer, status clear,
        K0..K5, exchange, K6) is a CUDA graph per local batch size, replayed with this step's
        slots and Adam scalars written into its static inputs (CGS_GRAPHS=0: eager)."""
        torch = _torch()
        dev = self.ctx.device
        indices = np.asarray(indices)
        local = self.local_slice(indices)
        slots = self.slots(local)
        b = len(slots)
        key = (b, len(indices))
        sl = self._idx_slots.get(key)
        if sl is None:
            D = self.grid.size
            spec = self.obs_spec is not None
            sl = self._idx_slots[key] = {
                "idx": torch.zeros(max(b, 1), dtype=torch.int64, device=dev),
                "o": None if spec or b == 0 else torch.empty((b, D, D), dtype=torch.float32, device=dev),
                "p": torch.empty((max(b, 1), 12), dtype=torch.float64, device=dev),
                # the spectral K4 takes H from the records: the CTF rows are not gathered then
                "c": None if self.ctfs is None or spec else torch.empty((max(b, 1), 8), dtype=torch.float64,
                                                                         device=dev),
                "hyper": torch.empty(4, dtype=torch.float64, device=dev)}

            def inputs(sl=sl, spec=spec):
                i = sl["idx"]
                torch.index_select(self.poses, 0, i, out=sl["p"])
                if spec:  # K4 reads the batch's records in place, by row (no gathered copy)
                    return None, sl["p"], self.ctfs, self.obs_spec, i[:b]
                torch.index_select(self.obs, 0, i, out=sl["o"])
                if sl["c"] is not None:
                    torch.index_select(self.ctfs, 0, i, out=sl["c"])
                return sl["o"], sl["p"], sl["c"], None

            segs, pipe = self._segments(b, len(indices), inputs, sl["hyper"])
            sl["runner"] = _StepRunner(segs, self.use_graphs, self._whole_graph)
            sl["pipe"] = pipe
        t = self.t + 1
        if b:
            sl["idx"][:b].copy_(torch.as_tensor(slots, dtype=torch.int64), non_blocking=True)
        sl["hyper"].copy_(self._hyper(lr, t), non_blocking=True)
        sl["runner"].run()
        self.t = t
        return sl["pipe"].loss if sl["pipe"] is not None else self._empty_loss

    def step_host(self, obs, poses, ctfs, lr: float, *, global_batch: int, loss_out=None):
        """Public end-to-end step from (pinned) HOST buffers of this rank's batch.

        Copies the batch host->device on a dedicated copy stream (with a spectral
        K4 the batch's observation records are made there too, overlapping the
        previous step), runs the step on the current stream once the copy has
        landed, and copies the per-image
        losses device->host into ``loss_out`` (pinned).  Nothing synchronises the
        host, so back-to-back calls overlap the next batch's H2D (PCIe) with
        this batch's kernels; the caller synchronises when it needs the numbers.
        Each input slot's step is one CUDA graph (captured on first use).
        """
        torch = _torch()
        dev = self.ctx.device
        compute = torch.cuda.current_stream(dev)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(dev)
        # two preallocated device slots per (batch shape, global batch), alternating: no
        # allocator traffic per step; a slot is refilled only after the step that read it
        key = (tuple(obs.shape), ctfs is None, int(global_batch))
        slots = self._h2d_slots.get(key)
        if slots is None:
            # with a spectral K4 the batch's observation records are made on the copy stream right
            # after its H2D, so they overlap the previous step's kernels instead of running inside
            # this step; the step then reads them like a resident dataset's
            per = engine.obs_record_elems(self.ctx, self.grid.size) if ctfs is not None and obs.shape[0] else 0

            def slot():
                sl = {"o": torch.empty(obs.shape, dtype=obs.dtype, device=dev),
                      "p": torch.empty(poses.shape, dtype=poses.dtype, device=dev),
                      "c": None if ctfs is None else torch.empty(ctfs.shape, dtype=ctfs.dtype, device=dev),
                      "spec": torch.empty((obs.shape[0], per), dtype=torch.float32, device=dev) if per else None,
                      "hyper": torch.empty(4, dtype=torch.float64, device=dev), "done": None}
                if sl["spec"] is not None:
                    def inputs():
                        return None, sl["p"], sl["c"], sl["spec"]
                else:
                    def inputs():
                        return sl["o"], sl["p"], sl["c"], None
                segs, pipe = self._segments(obs.shape[0], global_batch, inputs, sl["hyper"])
                sl["runner"], sl["pipe"] = _StepRunner(segs, self.use_graphs, self._whole_graph), pipe
                return sl
            slots = self._h2d_slots[key] = [slot(), slot(), 0]
        sl = slots[slots[2]]
        slots[2] ^= 1
        cs = self._copy_stream
        if sl["done"] is not None:
            cs.wait_event(sl["done"])
        t = self.t + 1
        with torch.cuda.stream(cs):
            # Adam's per-step scalars travel with the batch
            sl["hyper"].copy_(self._hyper(lr, t), non_blocking=True)
            sl["o"].copy_(obs, non_blocking=True)
            sl["p"].copy_(poses, non_blocking=True)
            if ctfs is not None:
                sl["c"].copy_(ctfs, non_blocking=True)
            if sl["spec"] is not None:
                engine.obs_spectra(self.ctx, sl["o"], sl["c"], self.gs, out=sl["spec"])
        compute.wait_stream(cs)
        sl["runner"].run()
        self.t = t
        loss = sl["pipe"].loss if sl["pipe"] is not None else self._empty_loss
        if sl["done"] is None:
            sl["done"] = torch.cuda.Event()
        sl["done"].record(compute)
        if loss_out is not None and loss.numel():
            loss_out.copy_(loss, non_blocking=True)
        return loss

    def step_batch(self, obs, poses, ctfs, lr: float, *, global_batch: int, events=None, obs_spec=None):
        """One eager step on device tensors of this rank's batch (obs f32 [b][D][D],
        poses f64 [b][12], ctfs f64 [b][8] or None); ``global_batch`` sets the
        1/B loss scale.  ``obs_spec``: the batch's precomputed observation spectra
        (batch_spectra); obs may then be None.  ``events``: CUDA events per stage
        (bench).  Returns the device tensor of per-image losses."""
        b = 0 if poses is None else poses.shape[0]
        t = self.t + 1
        cfg = self.config
        segs, pipe = self._segments(b, global_batch, lambda: (obs, poses, ctfs, obs_spec), None, events=events,
                                    scalars=(lr, 1.0 - cfg.adam_beta1 ** t, 1.0 - cfg.adam_beta2 ** t))
        for _, fn in segs:
            fn()
        self.t = t
        return pipe.loss if pipe is not None else self._empty_loss

    def check_status(self) -> None:
        for pipe in self._pipes.values():
            if pipe.degenerate():
                raise DegenerateRotationError("quaternion with zero or non-finite norm")

    def params_host(self) -> np.ndarray:
        """Parameters in the caller's Gaussian order."""
        out = np.empty((self.n, 11), dtype=np.float64)
        out[self.perm] = self.params.cpu().numpy()
        return out

    def moments_host(self):
        """(m, v) in the caller's Gaussian order (gathered from their owners when sharded)."""
        if self.sharded:
            self.xch.gather_rows(self._m_store)
            self.xch.gather_rows(self._v_store)
        m = np.empty((self.n, 11))
        v = np.empty((self.n, 11))
        m[self.perm] = self.m.cpu().numpy()
        v[self.perm] = self.v.cpu().numpy()
        return m, v

    def reorder(self) -> None:
        """Re-sort the device-resident Gaussians (and Adam moments) by Morton code
        of their current means, e.g. once per epoch as they move."""
        torch = _torch()
        local = morton_order(self.params[:, :3].cpu().numpy(), self.grid.extent)
        idx = torch.as_tensor(local, device=self.params.device)
        if self.sharded:  # the moments are current only on their owner: replicate before permuting
            self.xch.gather_rows(self._m_store)
            self.xch.gather_rows(self._v_store)
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
    if rec.world > 1 and B < rec.world:
        raise ValueError(f"batch_size {B} is smaller than the {rec.world} data-parallel ranks")
    is_root = rec.rank == 0
    trace, epoch_losses = [], []
    epoch0_median = None
    history0: list = []
    torch = _torch()

    order = shuffle_rng.permutation(R)
    for epoch in range(config.epochs):
        lr = config.epoch_lr(epoch)
        if epoch > 0:
            rec.reorder()  # keep the device order spatial as the means move
        # the next epoch's order is drawn now (same rng sequence) so its records can be prefetched
        next_order = shuffle_rng.permutation(R) if epoch + 1 < config.epochs else None
        rec.begin_epoch(order, next_order)
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
                    rec.check_status()  # a degenerate rotation is the reference's first error (splat.py:191-193)
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
        if next_order is not None:
            order = next_order
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
    total = dev_loss[:n_local].sum() if n_local else torch.zeros((), dtype=torch.float64, device=rec.ctx.device)
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
