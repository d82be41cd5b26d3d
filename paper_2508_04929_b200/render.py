"""Posed orthographic splatting on the GPU (mirrors the reference's splat.py).

``rasterize`` and ``rasterize_backward`` keep the reference signatures
(splat.py:263-381) and run K0/K2/K3 and K0/K5/K6 of libcgs_b200 on the current
CUDA device; host arrays are copied in and out around the kernels.  The batched
variants (``rasterize_batch``, ``rasterize_backward_batch``) take many poses per
call.  ``view_transform`` / ``orthographic_project`` are the per-Gaussian scalar
forms the reference exposes for tests (splat.py:150-168).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, engine
from .exceptions import DegenerateRotationError, DegenerateSplatError
from .mixture import (
    GaussianMixture,
    GaussianParams,
    GridSpec,
    build_covariance,
    normalize_quaternion,
    quaternion_to_matrix,
)

CULL_SIGMA = 6.5
_CUTOFF_SQ = CULL_SIGMA * CULL_SIGMA
_SUB = float(np.exp(-0.5 * _CUTOFF_SQ))
EIGEN_FLOOR_FRACTION = 0.1
DEFAULT_TILE_SIZE = 16


class ClampCounter:
    """Running count of Gaussians that hit the 2D eigenvalue floor (splat.py:60-70).

    The reference adds each rasterize's clamp count on the host (splat.py:276-277).
    Here the training step's render (K3, cgs_render) adds it into a device int64
    counter with no host sync; ``track`` registers such a counter and reading
    ``count`` folds every tracked counter into the host total (one device read per
    counter), so ``CLAMP_EVENTS.count`` means what it means in the reference."""

    def __init__(self):
        self._host = 0
        self._pending = []  # device int64 [1] counters (strong references: a count outlives its pipeline)

    def track(self, counter) -> None:
        self._pending.append(counter)

    def _drain(self) -> None:
        import sys

        live = []
        for t in self._pending:
            v = int(t.item())
            if v:
                self._host += v
                t.zero_()
            # keep counters someone else still holds; drop drained orphans
            if sys.getrefcount(t) > 3:
                live.append(t)
        self._pending = live

    @property
    def count(self) -> int:
        self._drain()
        return self._host

    @count.setter
    def count(self, value: int) -> None:
        self._drain()
        self._host = int(value)

    def reset(self):
        self.count = 0


CLAMP_EVENTS = ClampCounter()


@dataclass
class Pose:
    """Viewing pose: proper rotation plus in-plane translation (tx, ty, 0)."""

    rotation: np.ndarray
    translation: np.ndarray = field(default_factory=lambda: np.zeros(2))

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64)
        self.translation = np.asarray(self.translation, dtype=np.float64)
        if self.rotation.shape != (3, 3):
            raise ValueError("pose rotation must be a 3x3 matrix")
        if self.translation.shape != (2,):
            raise ValueError("pose translation must be a 2-vector")
        ortho = np.abs(self.rotation.T @ self.rotation - np.eye(3)).max()
        if ortho > 1e-9 or abs(np.linalg.det(self.rotation) - 1.0) > 1e-9:
            raise ValueError("pose rotation is not a proper rotation (orthonormal, det +1)")

    @classmethod
    def identity(cls) -> "Pose":
        return cls(np.eye(3))

    @classmethod
    def from_quaternion(cls, q, translation=(0.0, 0.0)) -> "Pose":
        return cls(quaternion_to_matrix(normalize_quaternion(q)), np.asarray(translation, float))

    @classmethod
    def from_quaternions(cls, qs) -> list:
        """Poses of many quaternions (K, 4) at zero translation: the same matrices as
        from_quaternion, validated in one vectorised check instead of one per pose."""
        R = quaternion_to_matrix(normalize_quaternion(np.asarray(qs, dtype=np.float64).reshape(-1, 4)))
        ortho = np.abs(np.einsum("kji,kjl->kil", R, R) - np.eye(3)).max(axis=(1, 2)) if len(R) else np.zeros(0)
        if np.any(ortho > 1e-9) or np.any(np.abs(np.linalg.det(R) - 1.0) > 1e-9):
            raise ValueError("pose rotation is not a proper rotation (orthonormal, det +1)")
        out = []
        for Rk in R:
            p = object.__new__(cls)
            p.rotation = Rk
            p.translation = np.zeros(2)
            out.append(p)
        return out

    @property
    def translation3(self) -> np.ndarray:
        return np.array([self.translation[0], self.translation[1], 0.0])


@dataclass
class CameraSpaceGaussian:
    mean3: np.ndarray
    cov3: np.ndarray


@dataclass
class SplatGaussian2D:
    """A z-marginalised Gaussian; integrates to ``amplitude``."""

    mean2: np.ndarray
    cov2: np.ndarray
    amplitude: float = 1.0

    def density(self, points) -> np.ndarray:
        pts = np.asarray(points, dtype=np.float64)
        d = pts - self.mean2
        P = np.linalg.inv(self.cov2)
        q = np.einsum("...i,ij,...j->...", d, P, d)
        return self.amplitude * np.exp(-0.5 * q) / (2.0 * np.pi * np.sqrt(np.linalg.det(self.cov2)))


@dataclass
class RenderedImage:
    """D x D samples of the projected density at pixel centres."""

    grid: GridSpec
    pixels: np.ndarray

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=np.float64)
        if self.pixels.shape != (self.grid.size, self.grid.size):
            raise ValueError("pixel array does not match grid size")


def view_transform(g: GaussianParams, pose: Pose) -> CameraSpaceGaussian:
    W = pose.rotation
    return CameraSpaceGaussian(W @ np.asarray(g.mean, float) + pose.translation3,
                               W @ build_covariance(g.quaternion, g.raw_scale) @ W.T)


def orthographic_project(cg: CameraSpaceGaussian, amplitude: float = 1.0) -> SplatGaussian2D:
    c2 = np.array(cg.cov3, dtype=np.float64)[:2, :2]
    if c2[0, 0] <= 0 or c2[0, 0] * c2[1, 1] - c2[0, 1] * c2[1, 0] <= 0:
        raise DegenerateSplatError("projected 2x2 covariance is not positive definite")
    return SplatGaussian2D(np.array(cg.mean3[:2], dtype=np.float64), c2, amplitude)


# ---------------------------------------------------------------------------
# GPU entry points
# ---------------------------------------------------------------------------
def _to_device(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda(non_blocking=False)


def _grid(grid: GridSpec):
    return _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)


def _check_status(status) -> None:
    if int(status.item()) & _lib.CGS_STATUS_DEGENERATE_ROTATION:
        raise DegenerateRotationError("quaternion with zero or non-finite norm")


def rasterize_batch(mixture: GaussianMixture, rotations, translations, grid: GridSpec, *,
                    tile_size: int = DEFAULT_TILE_SIZE, device_out: bool = False, method: str = "tiles"):
    """Render B poses at once -> (B, D, D) (float32 device tensor or float64 array).

    ``method="tiles"`` follows the reference schedule (fp64 bbox, tile lists,
    tiled forward); ``method="direct"`` uses the binning-free fixed-point render
    of the training step.  Both add the eigenvalue-floor clamp count to
    CLAMP_EVENTS (splat.py:276-277): the tile path from its fp64 projection, the
    direct path from the render's fp32 projection.
    """
    import torch

    ctx = engine.DeviceContext.get()
    params = _to_device(mixture.params, torch.float64)
    poses = _to_device(engine.pose_array(rotations, translations), torch.float64)
    B = poses.shape[0]
    gs = _grid(grid)
    status = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    splat = engine.prepare(ctx, params, status)
    out = torch.empty((B, grid.size, grid.size), dtype=torch.float32, device=ctx.device)
    if method == "direct":
        clamp = torch.zeros(1, dtype=torch.int64, device=ctx.device)
        engine.render_direct(ctx, splat, len(mixture), poses, gs, out, clamp=clamp)
        _check_status(status)
        CLAMP_EVENTS.count += int(clamp.item())
    elif method == "tiles":
        clamp = torch.zeros(B, dtype=torch.int32, device=ctx.device)
        binning = engine.bin_full(ctx, params, poses, gs, tile_size, status, clamp=clamp)
        engine.raster_fwd(ctx, splat, len(mixture), poses, gs, binning, out)
        _check_status(status)
        CLAMP_EVENTS.count += int(clamp.sum().item())
    else:
        raise ValueError(f"unknown method {method!r}")
    return out if device_out else out.double().cpu().numpy()


def rasterize(mixture: GaussianMixture, pose: Pose, grid: GridSpec, *,
              tile_size: int = DEFAULT_TILE_SIZE) -> RenderedImage:
    """Render the mixture at ``pose`` on the FFT-aligned grid (splat.py:263-298)."""
    img = rasterize_batch(mixture, pose.rotation[None], pose.translation[None], grid, tile_size=tile_size)
    return RenderedImage(grid=grid, pixels=img[0])


def rasterize_backward_batch(mixture: GaussianMixture, rotations, translations, grid: GridSpec,
                             dL_dpixels, *, scale: float = 1.0):
    """Sum over B poses of the raw-parameter gradients, times ``scale`` -> (N, 11)."""
    import torch

    ctx = engine.DeviceContext.get()
    params = _to_device(mixture.params, torch.float64)
    poses = _to_device(engine.pose_array(rotations, translations), torch.float64)
    up = dL_dpixels if isinstance(dL_dpixels, torch.Tensor) else _to_device(dL_dpixels, torch.float32)
    up = up.to(device=ctx.device, dtype=torch.float32).contiguous()
    status = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    gs = _grid(grid)
    splat = engine.prepare(ctx, params, status)
    partial, G = engine.raster_bwd(ctx, splat, len(mixture), poses, gs, up)
    grads = engine.epilogue_grads(ctx, partial, G, params, _lib.CGS_MODE["anisotropic"], scale)
    _check_status(status)
    return grads.cpu().numpy()


def rasterize_backward(mixture: GaussianMixture, pose: Pose, grid: GridSpec, dL_dpixels) -> np.ndarray:
    """Gradients of sum(dL_dpixels * rasterize(...)) w.r.t. the raw parameters (splat.py:301-381)."""
    dL = np.asarray(dL_dpixels, dtype=np.float64)
    if dL.shape != (grid.size, grid.size):
        raise ValueError("dL_dpixels shape does not match grid")
    return rasterize_backward_batch(mixture, pose.rotation[None], pose.translation[None], grid, dL[None])
