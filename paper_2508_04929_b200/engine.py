"""Device-resident execution of the splatting step over libcgs_b200.so.

PyTorch provides device memory, the current CUDA stream and (for multi-GPU)
``torch.distributed``; all compute runs in the hand-written sm_100a kernels of
``csrc/`` through the C ABI in ``include/cgs_b200.h``.  Nothing here computes on
the host, and nothing falls back to a CPU path: without a CUDA device or the
library every entry point raises ``CudaUnavailableError``.

Pipeline of one step (call stack A):
  K0 cgs_prepare -> K3 cgs_render (binning-free; or K2 cgs_bin_* + cgs_raster_fwd
  in tile mode) -> K4 cgs_ctf_mse (cuFFT R2C, H_sym, C2R, MSE, R2C,
  H_sym, C2R) -> K5 cgs_raster_bwd -> [NCCL all-reduce] -> K6
  cgs_epilogue_adam.  All launches are stream-ordered with no host sync.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import CudaUnavailableError

try:  # torch is the device-memory / stream / collective plumbing
    import torch
except ImportError:  # pragma: no cover - torch is in the image
    torch = None

DEFAULT_TILE = 32
# images per backward CTA (K5 partial groups): 10 balances the grid (5k CTAs on C2) against the
# partials the epilogue reads (measured 4..64 on C2, 6..12 within 1%; CGS_IMAGES_PER_GROUP
# overrides for A/B).  Large mixtures take more images per group (images_per_group()).
DEFAULT_IMAGES_PER_GROUP = int(os.environ.get("CGS_IMAGES_PER_GROUP", "10"))
# image-group heuristic in units of 256-Gaussian blocks at 4 per SM (raster_bwd.cu kRegThreads; the
# 128^2 kernel runs 128-thread CTAs, twice the blocks at up to 6 per SM: ~11 waves instead of 8)
_BWD_THREADS = 256
_BWD_TARGET_CTAS = 4736   # 8 waves of 148 SMs x 4 resident CTAs
_MAX_POSE_IMAGES = 64     # groups up to this size keep their poses in shared memory


def images_per_group_auto(n: int, B: int) -> int:
    """K5 image-group size for n Gaussians and B images: the default 10, raised for large n
    while the grid still has ~8 waves of CTAs, so the fp32 partials the epilogue reads
    (groups x n x 40 B: 1 GB at 1M Gaussians with groups of 10) stay few."""
    if "CGS_IMAGES_PER_GROUP" in os.environ:
        return DEFAULT_IMAGES_PER_GROUP
    blocks = -(-int(n) // _BWD_THREADS)
    groups = max(1, -(-_BWD_TARGET_CTAS // blocks))
    return int(min(_MAX_POSE_IMAGES, max(DEFAULT_IMAGES_PER_GROUP, -(-int(B) // groups))))


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise CudaUnavailableError(
            "a CUDA device is required: paper_2508_04929_b200 runs only on the GPU (no CPU fallback)"
        )
    return _lib.load()


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def pose_array(rotations, translations=None) -> np.ndarray:
    """Pack poses as f64 [B][12]: W row-major, tx, ty, 0 (include/cgs_b200.h)."""
    R = np.asarray(rotations, dtype=np.float64).reshape(-1, 3, 3)
    out = np.zeros((R.shape[0], 12), dtype=np.float64)
    out[:, :9] = R.reshape(-1, 9)
    if translations is not None:
        out[:, 9:11] = np.asarray(translations, dtype=np.float64).reshape(-1, 2)
    return out


def ctf_array(params_list) -> np.ndarray:
    """Pack CtfParams-like objects as f64 [B][8] (include/cgs_b200.h)."""
    out = np.zeros((len(params_list), 8), dtype=np.float64)
    for i, p in enumerate(params_list):
        out[i] = [p.defocus_u, p.defocus_v, p.astigmatism_angle, p.voltage, p.spherical_aberration,
                  p.amplitude_contrast, p.phase_shift, p.b_factor]
    return out


class DeviceContext:
    """Per-device library handle, grow-only scratch buffers and FFT plans."""

    _instances: dict = {}

    def __init__(self, device):
        self.lib = require_cuda()
        self.device = torch.device(device)
        self._bufs: dict = {}
        self._plans: dict = {}

    @classmethod
    def get(cls, device=None) -> "DeviceContext":
        require_cuda()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = dev.index if dev.index is not None else torch.cuda.current_device()
        if key not in cls._instances:
            cls._instances[key] = cls(torch.device("cuda", key))
        return cls._instances[key]

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def buf(self, name: str, numel: int, dtype) -> "torch.Tensor":
        """Grow-only scratch tensor (flat, at least ``numel`` elements; zeroed when allocated)."""
        t = self._bufs.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.zeros(max(int(numel), 1), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[: max(int(numel), 1)]

    def plan(self, size: int, batch: int, tag: str = "") -> int:
        """A cuFFT plan for (size, batch), cached; ``tag`` keeps separate plans (and cuFFT work
        areas) for users that may run on different streams."""
        key = (int(size), int(batch), tag)
        if key not in self._plans:
            h = ctypes.c_void_p()
            _lib.call("cgs_fft_plan_create", int(size), int(batch), ctypes.byref(h))
            self._plans[key] = h.value
        return self._plans[key]

    def __del__(self):  # pragma: no cover - best effort
        try:
            for h in self._plans.values():
                self.lib.cgs_fft_plan_destroy(h)
        except Exception:
            pass


@dataclass
class Binning:
    items: "torch.Tensor"   # int32 [capacity]
    offs: "torch.Tensor"    # int32 [B*T*S + 1]
    tile: int
    T: int
    S: int
    capacity: int


def prepare(ctx: DeviceContext, params, status, out=None):
    """K0: f64 [N][11] -> splat f32 [N][16]."""
    n = params.shape[0]
    splat = out if out is not None else ctx.buf("splat", n * 16, torch.float32)
    _lib.call("cgs_prepare", _ptr(params), n, _ptr(splat), _ptr(status), ctx.stream)
    return splat


def bin_count(ctx, params, poses, grid_s, tile, *, bbox_out=None, clamp=None, prefix="bin"):
    """K2 count + scan: returns (offs, rects, T, S)."""
    n = params.shape[0]
    B = poses.shape[0]
    T = int(ctx.lib.cgs_bin_tiles(grid_s.size, tile))
    S = int(ctx.lib.cgs_bin_segments(n))
    cnt = B * T * S + 1
    rects = ctx.buf(prefix + "_rects", B * n, torch.int32)
    counts = ctx.buf(prefix + "_counts", cnt, torch.int32)
    offs = ctx.buf(prefix + "_offs", cnt, torch.int32)
    ws = ctx.buf(prefix + "_scanws", ctx.lib.cgs_scan_workspace_bytes(cnt) // 4 + 1, torch.int32)
    _lib.call("cgs_bin_count", _ptr(params), n, _ptr(poses), B, grid_s, tile, _ptr(rects),
              _ptr(counts), _ptr(bbox_out), _ptr(clamp), ctx.stream)
    _lib.call("cgs_exclusive_scan", _ptr(counts), _ptr(offs), cnt, _ptr(ws), ctx.stream)
    return offs, rects, T, S


def bin_scatter(ctx, rects, n, B, grid_s, tile, offs, items, status):
    _lib.call("cgs_bin_scatter", _ptr(rects), n, B, grid_s.size, tile, _ptr(offs), _ptr(items),
              items.numel(), _ptr(status), ctx.stream)


def bin_full(ctx, params, poses, grid_s, tile, status, *, bbox_out=None, clamp=None, prefix="bin") -> Binning:
    """Count, scan, then size the item list exactly (one host read) and scatter."""
    offs, rects, T, S = bin_count(ctx, params, poses, grid_s, tile, bbox_out=bbox_out, clamp=clamp, prefix=prefix)
    total = int(offs[-1].item())
    items = ctx.buf(prefix + "_items", max(total, 1), torch.int32)
    bin_scatter(ctx, rects, params.shape[0], poses.shape[0], grid_s, tile, offs, items, status)
    return Binning(items, offs, tile, T, S, items.numel())


def raster_fwd(ctx, splat, n, poses, grid_s, binning: Binning, out, layout=_lib.CGS_LAYOUT_NATURAL):
    """K3: rendered images f32 [B][D][D]."""
    _lib.call("cgs_raster_fwd", _ptr(splat), n, _ptr(poses), poses.shape[0], grid_s, binning.tile,
              _ptr(binning.items), _ptr(binning.offs), binning.capacity, _ptr(out), layout, ctx.stream)
    return out


def render_direct(ctx, splat, n, poses, grid_s, out, clamp=None):
    """K3 binning-free render (cgs_render): images f32 [B][D][D], natural layout; ``clamp`` (device
    int64 [1], optional) accumulates the eigenvalue-floor clamp count."""
    ws = ctx.buf("render_ws", ctx.lib.cgs_render_workspace_bytes(n) // 4 + 1, torch.float32)
    _lib.call("cgs_render", _ptr(splat), n, _ptr(poses), poses.shape[0], grid_s, _ptr(out), _ptr(clamp), _ptr(ws),
              ctx.stream)
    return out


def raster_bwd(ctx, splat, n, poses, grid_s, upstream, ipg=None, out=None,
               layout=_lib.CGS_LAYOUT_NATURAL):
    """K5: partial world-frame accumulators f32 [G][N][10] (ipg: images per group, default
    images_per_group_auto(n, B))."""
    B = poses.shape[0]
    ipg = images_per_group_auto(n, B) if ipg is None else ipg
    G = int(ctx.lib.cgs_bwd_groups(B, ipg))
    partial = out if out is not None else ctx.buf("bwd_partial", G * n * 10, torch.float32)
    _lib.call("cgs_raster_bwd", _ptr(splat), n, _ptr(poses), B, grid_s, _ptr(upstream), layout,
              _ptr(partial), ipg, ctx.stream)
    return partial, G


def epilogue_grads(ctx, partial, G, params, mode, scale, out=None):
    n = params.shape[0]
    grads = out if out is not None else torch.empty((n, 11), dtype=torch.float64, device=ctx.device)
    _lib.call("cgs_epilogue_grads", _ptr(partial), G, n, _ptr(params), mode, float(scale), _ptr(grads), ctx.stream)
    return grads


def ctf_apply(ctx, images, grid_s, *, ctf=None, H=None, out=None):
    """apply_ctf on a device batch f32 [B][D][D]."""
    B = images.shape[0]
    D = grid_s.size
    out = out if out is not None else torch.empty_like(images)
    spec = ctx.buf("spectrum", 2 * int(ctx.lib.cgs_fft_spectrum_elems(D, B)), torch.float32)
    _lib.call("cgs_ctf_apply", ctx.plan(D, B), _ptr(images), _ptr(out), B, grid_s, _ptr(ctf), _ptr(H),
              _ptr(spec), _lib.CGS_LAYOUT_NATURAL, ctx.stream)
    return out


FILTER_SIZES = (32, 64, 128)


def fourier_filter(ctx, images, grid_s, *, ctf=None, shifts=None, out=None):
    """Re ifft2(H_sym . shift ramp . fft2(x)) on a device batch f32 [B][D][D]
    (apply_ctf then phase_shift_translate), one kernel; D in FILTER_SIZES.
    ctf f64 [B][8] and shifts f64 [B][2] (pixels) are optional device tensors."""
    B = images.shape[0]
    out = out if out is not None else torch.empty_like(images)
    _lib.call("cgs_fourier_filter", _ptr(images), _ptr(out), B, grid_s, _ptr(ctf), _ptr(shifts), ctx.stream)
    return out


def loss_residual(ctx, model, obs, resid=None):
    B, D = model.shape[0], model.shape[-1]
    loss = torch.empty(B, dtype=torch.float64, device=ctx.device)
    _lib.call("cgs_loss_residual", _ptr(model), _ptr(obs), B, D, _ptr(loss), _ptr(resid), 0, ctx.stream)
    return loss


def spectral_kind(ctx, D: int, render: str = "direct"):
    """Which spectral K4 a training step at image size D takes: "lf" (one CTA per image on line
    FFTs, D = 64 / 128), "fft" (cuFFT R2C, one filter/loss kernel, C2R: the other sizes, for the
    direct fixed-point render) or None (the real-space K4: D = 32, whose fused kernel is one
    launch; CGS_CTF_SPATIAL=1, or CGS_SPEC_FFT=0 for the cuFFT form, A/B)."""
    if os.environ.get("CGS_CTF_SPATIAL", "0") == "1":
        return None
    if int(ctx.lib.cgs_obs_spectrum_elems(D, 1)):
        return "lf"
    if render == "direct" and D >= 2 and D != 32 and os.environ.get("CGS_SPEC_FFT", "1") != "0":
        return "fft"
    return None


def obs_record_elems(ctx, D: int) -> int:
    """Floats per observation record of the spectral K4 at size D (0: no spectral K4)."""
    kind = spectral_kind(ctx, D)
    if kind == "lf":
        return int(ctx.lib.cgs_obs_spectrum_elems(D, 1))
    if kind == "fft":
        return int(ctx.lib.cgs_obs_spectrum_fft_elems(D, 1))
    return 0


def obs_spectra(ctx, obs, ctfs, grid_s, chunk: int = 4096, out=None):
    """Spectral-K4 records of a device stack (obs f32 [R][D][D], ctfs f64 [R][8]): F(obs) and
    H_sym / D^2 per observation, f32 [R][3 D (D/2+1)] (cgs_obs_spectrum, or cgs_obs_spectrum_fft
    with its own cuFFT plan and scratch), or None when the size has no spectral path.  ``out``:
    an existing [R][per] buffer to fill."""
    R, D = obs.shape[0], grid_s.size
    kind = spectral_kind(ctx, D)
    if kind is None:
        return None
    per = obs_record_elems(ctx, D)
    if out is None:
        out = torch.empty((R, per), dtype=torch.float32, device=ctx.device)
    if kind == "fft":  # cuFFT scratch of at most 256 MB per chunk
        chunk = max(1, min(chunk, (256 << 20) // (8 * D * (D // 2 + 1))))
        spectrum = torch.empty(2 * int(ctx.lib.cgs_fft_spectrum_elems(D, min(chunk, R))), dtype=torch.float32,
                               device=ctx.device)
    for a in range(0, R, chunk):
        b = min(R, a + chunk)
        if kind == "fft":
            _lib.call("cgs_obs_spectrum_fft", ctx.plan(D, b - a, tag="records"), _ptr(obs[a:b]), _ptr(ctfs[a:b]),
                      b - a, grid_s, _ptr(spectrum), _ptr(out[a:b]), ctx.stream)
        else:
            _lib.call("cgs_obs_spectrum", _ptr(obs[a:b]), _ptr(ctfs[a:b]), b - a, grid_s, _ptr(out[a:b]),
                      ctx.stream)
    return out


def gather_rows(ctx, src, idx, out):
    """out[i] = src[idx[i]] (rows of src's trailing shape); src on the device or in pinned host
    memory (zero-copy, cgs_gather_rows); idx int64 on the device."""
    rows = idx.numel()
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
    _lib.call("cgs_gather_rows", _ptr(src), _ptr(idx), rows, row_bytes, _ptr(out), ctx.stream)
    return out


def count_pairs(ctx, splat, n, poses, grid_s, cut_sq=None) -> "torch.Tensor":
    """Per-image (Gaussian, pixel) pairs with q < cut_sq (default 6.5^2: the reference's
    in-ellipse pairs)."""
    pairs = torch.zeros(poses.shape[0], dtype=torch.int64, device=ctx.device)
    if cut_sq is None:
        _lib.call("cgs_count_pairs", _ptr(splat), n, _ptr(poses), poses.shape[0], grid_s, _ptr(pairs), ctx.stream)
    else:
        _lib.call("cgs_count_pairs_cut", _ptr(splat), n, _ptr(poses), poses.shape[0], grid_s, float(cut_sq),
                  _ptr(pairs), ctx.stream)
    return pairs


class StepPipeline:
    """One fused training step over a device-resident batch, no host sync.

    Buffers are allocated once for (N, B, D); the step is stream-ordered and
    CUDA-Graph capturable.  ``render="direct"`` (default) renders with the
    binning-free fixed-point kernel (cgs_render); ``render="tiles"`` runs the
    reference's tile schedule (cgs_bin_* + cgs_raster_fwd), whose item buffer
    has a fixed capacity: an overflow only sets a status bit that makes the Adam
    epilogue skip the update (``overflowed``/``grow`` handle it on the host).
    """

    def __init__(self, ctx: DeviceContext, n: int, batch: int, grid_s, *, tile=DEFAULT_TILE,
                 images_per_group=None, mode="anisotropic", item_capacity=None,
                 render="direct"):
        self.ctx = ctx
        self.n, self.B, self.grid = int(n), int(batch), grid_s
        self.D = grid_s.size
        self.tile = tile
        self.ipg = images_per_group or images_per_group_auto(n, batch)
        self.mode = _lib.CGS_MODE[mode]
        self.render_mode = render
        dev = ctx.device
        D = self.D
        self.splat = torch.empty(n * 16, dtype=torch.float32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        # eigenvalue-floor clamps of every render, folded into CLAMP_EVENTS when it is read
        self.clamp = torch.zeros(1, dtype=torch.int64, device=dev)
        from .render import CLAMP_EVENTS

        CLAMP_EVENTS.track(self.clamp)
        self.render = torch.empty((self.B, D, D), dtype=torch.float32, device=dev)
        self.upstream = torch.empty((self.B, D, D), dtype=torch.float32, device=dev)
        self.spectrum = torch.empty(2 * int(ctx.lib.cgs_fft_spectrum_elems(D, self.B)), dtype=torch.float32, device=dev)
        self.loss = torch.empty(self.B, dtype=torch.float64, device=dev)
        self.G = int(ctx.lib.cgs_bwd_groups(self.B, self.ipg))
        self.partial = torch.empty(self.G * n * 10, dtype=torch.float32, device=dev)
        self.plan = ctx.plan(D, self.B)
        # zeroed once: the render's weight-bound pass keeps a self-resetting counter in it
        self.render_ws = torch.zeros(ctx.lib.cgs_render_workspace_bytes(n) // 4 + 1, dtype=torch.float32, device=dev)
        # per-step observation records of the spectral K4 (None: real-space K4)
        self.spectral_kind = spectral_kind(ctx, D, render)
        self.obs_spec = self.spec_ws = None
        if self.spectral_kind is not None:
            self.obs_spec = torch.empty(obs_record_elems(ctx, D) * self.B, dtype=torch.float32, device=dev)
        if self.spectral_kind == "fft":  # per-CTA loss sums + self-resetting counters, zeroed once
            self.spec_ws = torch.zeros(int(ctx.lib.cgs_spectral_fft_workspace_bytes(D, self.B)) // 8 + 1,
                                       dtype=torch.float64, device=dev)
        self.T = int(ctx.lib.cgs_bin_tiles(D, tile))
        self.S = int(ctx.lib.cgs_bin_segments(n))
        if render == "tiles":
            cnt = self.B * self.T * self.S + 1
            self.rects = torch.empty(self.B * n, dtype=torch.int32, device=dev)
            self.counts = torch.empty(cnt, dtype=torch.int32, device=dev)
            self.offs = torch.empty(cnt, dtype=torch.int32, device=dev)
            self.scan_ws = torch.empty(ctx.lib.cgs_scan_workspace_bytes(cnt) // 4 + 1, dtype=torch.int32, device=dev)
            self.items = torch.empty(max(int(item_capacity or 1), 1), dtype=torch.int32, device=dev)
        elif render != "direct":
            raise ValueError(f"unknown render mode {render!r}")

    @property
    def capacity(self) -> int:
        return self.items.numel() if self.render_mode == "tiles" else 0

    def grow(self, needed: int) -> None:
        if self.render_mode != "tiles":
            return
        cap = int(needed * 1.25) + 1024
        if cap > self.items.numel():
            self.items = torch.empty(cap, dtype=torch.int32, device=self.ctx.device)

    def measure_items(self, params, poses) -> int:
        """Tile mode: run the count pass once and read the item total (one host sync)."""
        if self.render_mode != "tiles":
            return 0
        self._prepare(params)
        self._count(params, poses)
        return int(self.offs[-1].item())

    def _prepare(self, params):
        _lib.call("cgs_prepare", _ptr(params), self.n, _ptr(self.splat), _ptr(self.status), self.ctx.stream)

    def _count(self, params, poses):
        s = self.ctx.stream
        _lib.call("cgs_bin_count", _ptr(params), self.n, _ptr(poses), self.B, self.grid, self.tile,
                  _ptr(self.rects), _ptr(self.counts), 0, 0, s)
        _lib.call("cgs_exclusive_scan", _ptr(self.counts), _ptr(self.offs), self.counts.numel(),
                  _ptr(self.scan_ws), s)

    # kernels of libcgs_b200 launched by one forward_backward + adam (bench accounting), direct mode:
    # wbound (+ prepare), raster_fwd_atomic, fixed_to_float, K4, raster_bwd,
    # epilogue_adam.  K4 is one ctf_mse_fused kernel for D = 32 / 64 / 128; otherwise ctf_multiply x2 +
    # loss_resid around cuFFT's own R2C/C2R kernels (library launches, not counted).
    def own_launches_per_step(self, ctf: bool = True, obs_spectrum: bool = False) -> int:
        """Kernels of this library per direct-mode step (bench accounting): the weight-bound pass
        (with K0 inside it when the spectral K4 follows, else after a separate prepare) +
        raster_fwd_atomic (+ fixed_to_float unless the spectral K4 converts on load); K4;
        raster_bwd; epilogue + Adam.  K4 is one kernel (spectral, plus obs_spectrum when the
        batch's records are not precomputed; or the real-space kernel for D = 32/64/128), or
        multiply x2 + loss around cuFFT's own transforms; without a CTF it is the loss/residual
        kernel."""
        spectral = ctf and self.spectral
        n = 2 + (0 if spectral else 2) + 1 + 1
        if not ctf:
            return n + 1
        if spectral and self.spectral_kind == "fft":  # fixed_scale, filter (+ interleave) around cuFFT's own
            k = 2 + (self.D % 2 == 0)
            return n + (k if obs_spectrum else k + 1)
        if spectral:
            return n + (1 if obs_spectrum else 2)
        fused = self.D in (32, 64, 128) and os.environ.get("CGS_CTF_CUFFT", "0") != "1"
        return n + (1 if fused else 3)

    @property
    def spectral(self) -> bool:
        """K4 runs in the Fourier domain with a CTF: cgs_ctf_mse_spectral* for D = 64 / 128,
        cgs_ctf_mse_spectral_fft for the other sizes but 32 (``spectral_kind``); CGS_CTF_SPATIAL=1
        keeps the real-space K4 (A/B)."""
        return self.obs_spec is not None

    def _render_scale(self):
        """Device view of the fixed-point render's scale (pixel = int / scale) in render_ws."""
        off = int(self.ctx.lib.cgs_render_scale_offset(self.n))
        return self.render_ws[off:off + 1]

    def render_image(self):
        """The last forward's rendered images as f32 [B][D][D] (converted from the fixed-point
        image when the step fed it to K4 unconverted)."""
        if not getattr(self, "_render_fixed", False):
            return self.render
        return self.render.view(torch.int32).to(torch.float32) / self._render_scale()

    def forward_backward(self, params, poses, obs, ctf, events=None, obs_spec=None, obs_rows=None):
        """K0..K5 for a batch; leaves partial accumulators in self.partial.

        ``obs_spec`` (spectral K4): this batch's observation records, or with ``obs_rows``
        (int64 [B] device) a dataset's resident records and the batch's rows in them.

        ``events`` (optional dict of name -> (start, end) torch.cuda.Event
        lists) records CUDA events around the fwd / ctf / bwd stages on the
        launching stream, for per-kernel timing inside the bench.
        """
        s = self.ctx.stream

        def mark(name, which):
            if events is not None and name in events:
                events[name][which].record()

        mark("fwd", 0)
        # direct render feeding the spectral K4: the int32 fixed-point image is converted as K4 loads it,
        # and K0 runs inside the render's weight-bound pass (cgs_prepare_render_fixed)
        fixed = self.render_mode == "direct" and ctf is not None and self.spectral
        self._render_fixed = fixed
        if fixed:
            _lib.call("cgs_prepare_render_fixed", _ptr(params), self.n, _ptr(self.splat), _ptr(self.status),
                      _ptr(poses), self.B, self.grid, _ptr(self.render), _ptr(self.clamp), _ptr(self.render_ws), s)
        elif self.render_mode == "direct":
            self._prepare(params)
            _lib.call("cgs_render", _ptr(self.splat), self.n, _ptr(poses), self.B, self.grid, _ptr(self.render),
                      _ptr(self.clamp), _ptr(self.render_ws), s)
        else:
            self._prepare(params)
            self._count(params, poses)
            _lib.call("cgs_bin_scatter", _ptr(self.rects), self.n, self.B, self.D, self.tile, _ptr(self.offs),
                      _ptr(self.items), self.items.numel(), _ptr(self.status), s)
            _lib.call("cgs_raster_fwd", _ptr(self.splat), self.n, _ptr(poses), self.B, self.grid, self.tile,
                      _ptr(self.items), _ptr(self.offs), self.items.numel(), _ptr(self.render),
                      _lib.CGS_LAYOUT_NATURAL, s)
        mark("fwd", 1)
        mark("ctf", 0)
        if ctf is not None and self.spectral:
            if obs_rows is not None and not fixed:  # only the fixed-point K4 reads records by row
                obs_spec, obs_rows = obs_spec.index_select(0, obs_rows), None
            fft = self.spectral_kind == "fft"
            if obs_spec is None:  # this batch's records (a dataset passes its precomputed ones)
                if fft:
                    _lib.call("cgs_obs_spectrum_fft", self.plan, _ptr(obs), _ptr(ctf), self.B, self.grid,
                              _ptr(self.spectrum), _ptr(self.obs_spec), s)
                else:
                    _lib.call("cgs_obs_spectrum", _ptr(obs), _ptr(ctf), self.B, self.grid, _ptr(self.obs_spec), s)
                obs_spec = self.obs_spec
            # the upstream goes out with row pairs interleaved: the backward's region staging is a copy
            # (after cuFFT's C2R an in-place interleave; odd sizes stay natural)
            up_layout = _lib.CGS_LAYOUT_NATURAL if fft and self.D % 2 else _lib.CGS_LAYOUT_ROWPAIR
            if fft:
                _lib.call("cgs_ctf_mse_spectral_fft", self.plan, _ptr(self.render), _ptr(self._render_scale()),
                          _ptr(obs_spec), _ptr(obs_rows), self.B, self.grid, _ptr(self.spectrum),
                          _ptr(self.spec_ws), _ptr(self.upstream), _ptr(self.loss), _ptr(self.status), up_layout, s)
            elif fixed and obs_rows is not None:
                _lib.call("cgs_ctf_mse_spectral_fixed_rows", _ptr(self.render), _ptr(self._render_scale()),
                          _ptr(obs_spec), _ptr(obs_rows), self.B, self.grid, _ptr(self.upstream), _ptr(self.loss),
                          _ptr(self.status), up_layout, s)
            elif fixed:
                _lib.call("cgs_ctf_mse_spectral_fixed", _ptr(self.render), _ptr(self._render_scale()), _ptr(obs_spec),
                          self.B, self.grid, _ptr(self.upstream), _ptr(self.loss), _ptr(self.status), up_layout, s)
            else:
                _lib.call("cgs_ctf_mse_spectral", _ptr(self.render), _ptr(obs_spec), self.B, self.grid,
                          _ptr(self.upstream), _ptr(self.loss), _ptr(self.status), up_layout, s)
        else:
            up_layout = _lib.CGS_LAYOUT_NATURAL
            _lib.call("cgs_ctf_mse", self.plan, _ptr(self.render), _ptr(obs), self.B, self.grid, _ptr(ctf),
                      _ptr(self.spectrum), 0, _ptr(self.upstream), _ptr(self.loss), _ptr(self.status),
                      _lib.CGS_LAYOUT_NATURAL, s)
        self.upstream_layout = up_layout
        mark("ctf", 1)
        mark("bwd", 0)
        _lib.call("cgs_raster_bwd", _ptr(self.splat), self.n, _ptr(poses), self.B, self.grid,
                  _ptr(self.upstream), up_layout, _ptr(self.partial), self.ipg, s)
        mark("bwd", 1)

    def adam(self, params, m, v, *, scale, lr, beta1, beta2, eps, t, acc=None, groups=None, skip=None, n=None):
        """K6 fused epilogue + Adam; acc defaults to this step's partials.  ``skip`` (int32 device
        status) decides whether the update is skipped; default: this pipeline's own status."""
        src = self.partial if acc is None else acc
        G = self.G if acc is None else (groups or 1)
        bc1 = 1.0 - beta1 ** t
        bc2 = 1.0 - beta2 ** t
        _lib.call("cgs_epilogue_adam", _ptr(src), G, self.n if n is None else n, _ptr(params), _ptr(m), _ptr(v),
                  self.mode,
                  float(scale), float(lr), float(beta1), float(beta2), float(eps), float(bc1), float(bc2),
                  _ptr(self.status if skip is None else skip), self.ctx.stream)

    def adam_dev(self, params, m, v, hyper, *, scale, beta1, beta2, eps):
        """K6 with (lr, bc1, bc2) read from the device tensor hyper f64 [3] (graph-capturable)."""
        _lib.call("cgs_epilogue_adam_dev", _ptr(self.partial), self.G, self.n, _ptr(params), _ptr(m), _ptr(v),
                  self.mode, float(scale), float(beta1), float(beta2), float(eps), _ptr(hyper), _ptr(self.status),
                  self.ctx.stream)

    def overflowed(self) -> bool:
        return bool(int(self.status.item()) & _lib.CGS_STATUS_BIN_OVERFLOW)

    def render_only(self, params, poses):
        """K0 + K3 (direct mode): rendered images in self.render."""
        self._prepare(params)
        self._render_fixed = False
        _lib.call("cgs_render", _ptr(self.splat), self.n, _ptr(poses), poses.shape[0], self.grid, _ptr(self.render),
                  _ptr(self.clamp), _ptr(self.render_ws), self.ctx.stream)
        return self.render

    def degenerate(self) -> bool:
        return bool(int(self.status.item()) & _lib.CGS_STATUS_DEGENERATE_ROTATION)

    def clear_status(self):
        self.status.zero_()
