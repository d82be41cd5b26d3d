"""CPU oracle for the cryoGS splatting step -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker and the CPU baseline.  It is imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg.  The product package ``paper_2508_04929_b200`` never
imports it, and the product path fails loudly when its CUDA library is missing.

It restates the reference algorithm (``/root/reference/pkg/src/cryosplat``) in
NumPy fp64 plus the plain-C loops in ``oracle/loops.c``.  Each function cites the
reference ``file:line`` it follows.  Parity of this restatement is pinned by
``tests/test_oracle_golden.py`` against golden vectors that
``tests/golden/make_golden.py`` produced by running the reference itself.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# constants  (splat.py:49-57, gmm.py:25-29, train.py:29-30)
# ---------------------------------------------------------------------------
CULL_SIGMA = 6.5
CUTOFF_SQ = CULL_SIGMA * CULL_SIGMA
SUB = float(np.exp(-0.5 * CUTOFF_SQ))
EIGEN_FLOOR_FRACTION = 0.1
DEFAULT_TILE_SIZE = 16
PARAMS_PER_GAUSSIAN = 11
COL_MEAN = slice(0, 3)
COL_RAW_SCALE = slice(3, 6)
COL_QUAT = slice(6, 10)
COL_RAW_AMP = 10

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_loops.so")
_lib = None


def build_loops(force: bool = False) -> str:
    """Compile oracle/loops.c into oracle/liboracle_loops.so (gcc, fp64, no FMA)."""
    src = os.path.join(_HERE, "loops.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess

        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


def _loops():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_loops()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        F = ctypes.c_double
        lib.oracle_tile_counts.argtypes = [P, I, I, I, I, P]
        lib.oracle_tile_counts.restype = I
        lib.oracle_tile_scatter.argtypes = [P, I, I, I, I, P, P]
        lib.oracle_tile_scatter.restype = None
        lib.oracle_forward_tiles.argtypes = [P, I, P, P, I, I, I, P, P, P, P, F, F, F, F]
        lib.oracle_forward_tiles.restype = None
        lib.oracle_backward_pixels.argtypes = [P, I, I, P, P, P, F, F, F, F, P]
        lib.oracle_backward_pixels.restype = None
        lib.oracle_count_pairs.argtypes = [I, I, P, P, P, F, F, F]
        lib.oracle_count_pairs.restype = I
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# grid and activations  (gmm.py:38-98)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    """GridSpec (gmm.py:38-73): D pixels over [-extent, extent]."""

    size: int
    extent: float = 0.5
    pixel_size: float = 1.0

    @property
    def pixel_width(self) -> float:  # gmm.py:57-60
        return 2.0 * self.extent / self.size

    @property
    def origin_index(self) -> int:  # gmm.py:62-65
        return self.size // 2

    def coords(self) -> np.ndarray:  # gmm.py:67-69
        return (np.arange(self.size) - self.origin_index) * self.pixel_width

    def freq_indices(self) -> np.ndarray:  # gmm.py:71-73
        return np.arange(self.size) - self.origin_index


def activate(raw):
    """Softplus, overflow-safe (gmm.py:76-80)."""
    raw = np.asarray(raw, dtype=np.float64)
    return np.maximum(raw, 0.0) + np.log1p(np.exp(-np.abs(raw)))


def activate_derivative(raw):
    """Logistic sigmoid (gmm.py:83-88)."""
    raw = np.asarray(raw, dtype=np.float64)
    e = np.exp(-np.abs(raw))
    return np.where(raw >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def inverse_activate(value):
    """Inverse softplus (gmm.py:91-98)."""
    value = np.asarray(value, dtype=np.float64)
    if np.any(value <= 0):
        raise ValueError("inverse softplus requires strictly positive input")
    return value + np.log(-np.expm1(-value))


def normalize_quaternion(q):
    """gmm.py:101-107."""
    q = np.asarray(q, dtype=np.float64)
    norm = np.linalg.norm(q, axis=-1, keepdims=True)
    if not np.all(norm > 0) or not np.all(np.isfinite(norm)):
        raise ValueError("quaternion with zero or non-finite norm")
    return q / norm


def quaternion_to_matrix(q):
    """Scalar-first unit quaternion -> rotation matrix (gmm.py:110-124)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3), dtype=np.float64)
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


# ---------------------------------------------------------------------------
# synthetic inputs  (gmm.py:227-251, simulate.py:92-190, bench.py:34-40)
# ---------------------------------------------------------------------------
def init_random(n: int, seed: int, grid: Grid) -> np.ndarray:
    """init_random (gmm.py:227-251): returns the (n, 11) raw parameter array."""
    mean_std = 0.9 * grid.extent / 6.0
    scale_target = 0.1 * mean_std
    amp_target = 1.0 / (2.0 * n)
    rng = np.random.default_rng(seed)
    params = np.zeros((n, PARAMS_PER_GAUSSIAN), dtype=np.float64)
    params[:, COL_MEAN] = rng.normal(0.0, mean_std, size=(n, 3))
    params[:, COL_RAW_SCALE] = inverse_activate(scale_target)
    params[:, COL_QUAT.start] = 1.0
    params[:, COL_RAW_AMP] = inverse_activate(amp_target)
    return params


def bench_mixture(n: int, grid: Grid, seed: int) -> np.ndarray:
    """bench._bench_mixture (bench.py:34-40): scales U(0.8, 1.6) px."""
    params = init_random(n, seed, grid)
    rng = np.random.default_rng(seed + 1)
    scales = rng.uniform(0.8, 1.6, size=(n, 3)) * grid.pixel_width
    params[:, COL_RAW_SCALE] = inverse_activate(scales)
    return params


def pose_from_quaternion(q, translation=(0.0, 0.0)):
    """Pose.from_quaternion (splat.py:99-100) -> (W 3x3, t 2)."""
    return quaternion_to_matrix(normalize_quaternion(q)), np.asarray(translation, dtype=np.float64)


def sample_pose(rng: np.random.Generator, translation_range: float = 0.0, integer_translations=False):
    """sample_pose (simulate.py:92-106): rotation uniform over SO(3)."""
    q = rng.standard_normal(4)
    t = rng.uniform(-translation_range, translation_range, size=2) if translation_range else np.zeros(2)
    if integer_translations:
        t = np.rint(t)
    return pose_from_quaternion(q, t)


def make_helix(n: int) -> np.ndarray:
    """make_phantom('helix', n) (simulate.py:130-166)."""
    params = np.zeros((n, PARAMS_PER_GAUSSIAN), dtype=np.float64)
    params[:, COL_RAW_AMP] = inverse_activate(1.0 / n)
    t = np.linspace(0.0, 1.0, n)
    theta = 4.0 * np.pi * t
    radius, z_half = 0.15, 0.2
    params[:, 0] = radius * np.cos(theta)
    params[:, 1] = radius * np.sin(theta)
    params[:, 2] = -z_half + 2.0 * z_half * t
    tangent = np.stack(
        [-radius * 4.0 * np.pi * np.sin(theta), radius * 4.0 * np.pi * np.cos(theta), np.full(n, 2.0 * z_half)],
        axis=1,
    )
    tangent /= np.linalg.norm(tangent, axis=1, keepdims=True)
    x_axis = np.array([1.0, 0.0, 0.0])
    for i in range(n):
        axis = np.cross(x_axis, tangent[i])
        axis /= np.linalg.norm(axis)
        angle = math.acos(float(np.clip(np.dot(x_axis, tangent[i]), -1.0, 1.0)))
        params[i, COL_QUAT] = np.concatenate(([math.cos(angle / 2.0)], math.sin(angle / 2.0) * axis))
    params[:, 3] = inverse_activate(0.030)
    params[:, 4] = inverse_activate(0.015)
    params[:, 5] = inverse_activate(0.015)
    return params


# ---------------------------------------------------------------------------
# projection  (splat.py:176-260)
# ---------------------------------------------------------------------------
@dataclass
class Projection:
    mean2: np.ndarray
    prec: np.ndarray
    cnorm: np.ndarray
    amp: np.ndarray
    bbox: np.ndarray
    n_clamped: int
    s: np.ndarray
    qn: np.ndarray
    qnorm: np.ndarray
    R: np.ndarray
    B2: np.ndarray
    W: np.ndarray


def clamp_eigenvalues(cov2, floor):
    """_clamp_eigenvalues (splat.py:229-260)."""
    a = cov2[:, 0, 0]
    b = cov2[:, 0, 1]
    d = cov2[:, 1, 1]
    mid = 0.5 * (a + d)
    rad = np.sqrt(np.maximum(0.25 * (a - d) ** 2 + b * b, 0.0))
    lam1 = mid + rad
    lam2 = mid - rad
    mask = lam2 < floor
    if not mask.any():
        return cov2, lam1, mask
    cov2 = cov2.copy()
    for i in np.nonzero(mask)[0]:
        l1 = max(lam1[i], floor)
        l2 = max(lam2[i], floor)
        v1 = np.array([b[i], lam1[i] - a[i]])
        v1_alt = np.array([lam1[i] - d[i], b[i]])
        if np.dot(v1_alt, v1_alt) > np.dot(v1, v1):
            v1 = v1_alt
        nrm = np.sqrt(np.dot(v1, v1))
        v1 = np.array([1.0, 0.0]) if nrm == 0.0 else v1 / nrm
        v2 = np.array([-v1[1], v1[0]])
        cov2[i] = l1 * np.outer(v1, v1) + l2 * np.outer(v2, v2)
    return cov2, np.maximum(lam1, floor), mask


def project(params: np.ndarray, W: np.ndarray, t: np.ndarray, grid: Grid) -> Projection:
    """_Projection.__init__ (splat.py:184-226)."""
    raw = params
    s = activate(raw[:, COL_RAW_SCALE])
    amp = activate(raw[:, COL_RAW_AMP])
    q = raw[:, COL_QUAT]
    qnorm = np.sqrt((q * q).sum(axis=1))
    if not np.all(qnorm > 0) or not np.all(np.isfinite(qnorm)):
        raise ValueError("quaternion with zero or non-finite norm")
    qn = q / qnorm[:, None]
    R = quaternion_to_matrix(qn)
    M = R * s[:, None, :]
    B2 = W[:2, :] @ M
    mean2 = np.ascontiguousarray(raw[:, COL_MEAN] @ W[:2, :].T + t)
    n = len(raw)
    cov2 = np.empty((n, 2, 2), dtype=np.float64)
    cov2[:, 0, 0] = (B2[:, 0, :] * B2[:, 0, :]).sum(axis=1)
    cov2[:, 0, 1] = (B2[:, 0, :] * B2[:, 1, :]).sum(axis=1)
    cov2[:, 1, 0] = cov2[:, 0, 1]
    cov2[:, 1, 1] = (B2[:, 1, :] * B2[:, 1, :]).sum(axis=1)
    floor = (EIGEN_FLOOR_FRACTION * grid.pixel_width) ** 2
    cov2, lam_max, clamped = clamp_eigenvalues(cov2, floor)
    det = cov2[:, 0, 0] * cov2[:, 1, 1] - cov2[:, 0, 1] ** 2
    prec = np.empty((n, 3), dtype=np.float64)
    prec[:, 0] = cov2[:, 1, 1] / det
    prec[:, 1] = -cov2[:, 0, 1] / det
    prec[:, 2] = cov2[:, 0, 0] / det
    cnorm = 1.0 / (2.0 * np.pi * np.sqrt(det))
    radius_px = CULL_SIGMA * np.sqrt(lam_max) / grid.pixel_width
    c0 = grid.origin_index
    D = grid.size
    px = mean2 / grid.pixel_width + c0
    bbox = np.empty((n, 4), dtype=np.int64)
    bbox[:, 0] = np.maximum(np.ceil(px[:, 0] - radius_px), 0)
    bbox[:, 1] = np.minimum(np.floor(px[:, 0] + radius_px), D - 1)
    bbox[:, 2] = np.maximum(np.ceil(px[:, 1] - radius_px), 0)
    bbox[:, 3] = np.minimum(np.floor(px[:, 1] + radius_px), D - 1)
    return Projection(mean2, prec, cnorm, amp, bbox, int(clamped.sum()), s, qn, qnorm, R, B2, W)


# ---------------------------------------------------------------------------
# binning, forward, backward  (_kernels.py via loops.c; splat.py:263-381)
# ---------------------------------------------------------------------------
def build_tile_work(bbox: np.ndarray, tile_size: int, n_tiles_x: int, n_tiles_y: int):
    """build_tile_work (_kernels.py:17-63) -> (gauss_ids i64, tile_starts i64)."""
    lib = _loops()
    bbox = np.ascontiguousarray(bbox, dtype=np.int64)
    starts = np.zeros(n_tiles_x * n_tiles_y + 1, dtype=np.int64)
    total = lib.oracle_tile_counts(_ptr(bbox), len(bbox), tile_size, n_tiles_x, n_tiles_y, _ptr(starts))
    ids = np.empty(total, dtype=np.int64)
    lib.oracle_tile_scatter(_ptr(bbox), len(bbox), tile_size, n_tiles_x, n_tiles_y, _ptr(starts), _ptr(ids))
    return ids, starts


def rasterize(params, W, t, grid: Grid, tile_size: int = DEFAULT_TILE_SIZE):
    """rasterize (splat.py:263-298) -> (pixels (D, D) f64, n_clamped)."""
    proj = project(params, W, t, grid)
    D = grid.size
    pixels = np.zeros((D, D), dtype=np.float64)
    ntx = -(-D // tile_size)
    ids, starts = build_tile_work(proj.bbox, tile_size, ntx, ntx)
    weight = np.ascontiguousarray(proj.amp * proj.cnorm)
    _loops().oracle_forward_tiles(
        _ptr(pixels), D, _ptr(ids), _ptr(starts), ntx * ntx, ntx, tile_size,
        _ptr(proj.mean2), _ptr(np.ascontiguousarray(proj.prec)), _ptr(weight), _ptr(proj.bbox),
        grid.pixel_width, float(grid.origin_index), CUTOFF_SQ, SUB,
    )
    return pixels, proj.n_clamped


def backward_raw_sums(params, W, t, grid: Grid, dL_dpixels, proj: Projection | None = None):
    """backward_pixels (_kernels.py:128-190) -> (N, 6) raw sums."""
    proj = proj or project(params, W, t, grid)
    dL = np.ascontiguousarray(dL_dpixels, dtype=np.float64)
    sums = np.zeros((len(params), 6), dtype=np.float64)
    _loops().oracle_backward_pixels(
        _ptr(dL), grid.size, len(params), _ptr(proj.mean2), _ptr(np.ascontiguousarray(proj.prec)),
        _ptr(proj.bbox), grid.pixel_width, float(grid.origin_index), CUTOFF_SQ, SUB, _ptr(sums),
    )
    return sums


def count_pairs(params, W, t, grid: Grid) -> int:
    """In-ellipse (Gaussian, pixel) pairs for one image (SURVEY.md 8(d) work unit)."""
    proj = project(params, W, t, grid)
    return int(_loops().oracle_count_pairs(
        grid.size, len(params), _ptr(proj.mean2), _ptr(np.ascontiguousarray(proj.prec)),
        _ptr(proj.bbox), grid.pixel_width, float(grid.origin_index), CUTOFF_SQ,
    ))


def world_accumulator(proj: Projection, sums: np.ndarray) -> np.ndarray:
    """Per-image 10-float world-frame accumulator.

    [cnorm*sA, W2^T (ac*sx, ac*sy) (3), P = W2^T (ac*S) W2 (xx, xy, xz, yy, yz, zz)]
    so that dM = 2 P M and dmean = the 3-vector; both linear, summable over images.
    """
    ac = proj.amp * proj.cnorm
    W2 = proj.W[:2, :]
    n = len(ac)
    acc = np.empty((n, 10), dtype=np.float64)
    acc[:, 0] = proj.cnorm * sums[:, 0]
    dmean2 = ac[:, None] * sums[:, 1:3]
    acc[:, 1:4] = dmean2 @ W2
    S = np.empty((n, 2, 2))
    S[:, 0, 0] = ac * sums[:, 3]
    S[:, 0, 1] = S[:, 1, 0] = ac * sums[:, 4]
    S[:, 1, 1] = ac * sums[:, 5]
    P = np.einsum("ai,nab,bj->nij", W2, S, W2)
    acc[:, 4] = P[:, 0, 0]
    acc[:, 5] = P[:, 0, 1]
    acc[:, 6] = P[:, 0, 2]
    acc[:, 7] = P[:, 1, 1]
    acc[:, 8] = P[:, 1, 2]
    acc[:, 9] = P[:, 2, 2]
    return acc


def chain_from_sums(params, proj: Projection, sums: np.ndarray) -> np.ndarray:
    """Per-Gaussian chain of rasterize_backward (splat.py:332-381) -> (N, 11)."""
    raw = params
    ac = proj.amp * proj.cnorm
    n = len(raw)
    dA = proj.cnorm * sums[:, 0]
    dmean2 = ac[:, None] * sums[:, 1:3]
    dcov2 = np.empty((n, 2, 2), dtype=np.float64)
    dcov2[:, 0, 0] = ac * sums[:, 3]
    dcov2[:, 0, 1] = ac * sums[:, 4]
    dcov2[:, 1, 0] = ac * sums[:, 4]
    dcov2[:, 1, 1] = ac * sums[:, 5]
    dB2 = 2.0 * (dcov2 @ proj.B2)
    dM = proj.W[:2, :].T @ dB2
    return _chain_tail(raw, proj.s, proj.R, proj.qn, proj.qnorm, dM, dmean2 @ proj.W[:2, :], dA)


def _chain_tail(raw, s, R, qn, qnorm, dM, dmean, dA):
    """splat.py:346-381: dM -> dscale, dR -> dq; sigmoid factors."""
    n = len(raw)
    dscale = (R * dM).sum(axis=1)
    r = dM * s[:, None, :]
    qw, qx, qy, qz = qn[:, 0], qn[:, 1], qn[:, 2], qn[:, 3]
    dqn = np.empty((n, 4), dtype=np.float64)
    dqn[:, 0] = 2 * (-qz * r[:, 0, 1] + qy * r[:, 0, 2] + qz * r[:, 1, 0]
                     - qx * r[:, 1, 2] - qy * r[:, 2, 0] + qx * r[:, 2, 1])
    dqn[:, 1] = 2 * (qy * r[:, 0, 1] + qz * r[:, 0, 2] + qy * r[:, 1, 0]
                     - 2 * qx * r[:, 1, 1] - qw * r[:, 1, 2] + qz * r[:, 2, 0]
                     + qw * r[:, 2, 1] - 2 * qx * r[:, 2, 2])
    dqn[:, 2] = 2 * (-2 * qy * r[:, 0, 0] + qx * r[:, 0, 1] + qw * r[:, 0, 2]
                     + qx * r[:, 1, 0] + qz * r[:, 1, 2] - qw * r[:, 2, 0]
                     + qz * r[:, 2, 1] - 2 * qy * r[:, 2, 2])
    dqn[:, 3] = 2 * (-2 * qz * r[:, 0, 0] - qw * r[:, 0, 1] + qx * r[:, 0, 2]
                     + qw * r[:, 1, 0] - 2 * qz * r[:, 1, 1] + qy * r[:, 1, 2]
                     + qx * r[:, 2, 0] + qy * r[:, 2, 1])
    dq = (dqn - np.sum(dqn * qn, axis=1, keepdims=True) * qn) / qnorm[:, None]
    grads = np.empty_like(raw)
    grads[:, COL_MEAN] = dmean
    grads[:, COL_RAW_SCALE] = dscale * activate_derivative(raw[:, COL_RAW_SCALE])
    grads[:, COL_QUAT] = dq
    grads[:, COL_RAW_AMP] = dA * activate_derivative(raw[:, COL_RAW_AMP])
    return grads


def grads_from_world_accumulator(params, acc: np.ndarray) -> np.ndarray:
    """Batched epilogue: 10-float accumulator (summed over images) -> (N, 11) grads."""
    raw = params
    s = activate(raw[:, COL_RAW_SCALE])
    q = raw[:, COL_QUAT]
    qnorm = np.sqrt((q * q).sum(axis=1))
    qn = q / qnorm[:, None]
    R = quaternion_to_matrix(qn)
    M = R * s[:, None, :]
    P = np.empty((len(raw), 3, 3))
    P[:, 0, 0] = acc[:, 4]
    P[:, 0, 1] = P[:, 1, 0] = acc[:, 5]
    P[:, 0, 2] = P[:, 2, 0] = acc[:, 6]
    P[:, 1, 1] = acc[:, 7]
    P[:, 1, 2] = P[:, 2, 1] = acc[:, 8]
    P[:, 2, 2] = acc[:, 9]
    dM = 2.0 * (P @ M)
    return _chain_tail(raw, s, R, qn, qnorm, dM, acc[:, 1:4], acc[:, 0])


def rasterize_backward(params, W, t, grid: Grid, dL_dpixels) -> np.ndarray:
    """rasterize_backward (splat.py:301-381) -> (N, 11)."""
    proj = project(params, W, t, grid)
    sums = backward_raw_sums(params, W, t, grid, dL_dpixels, proj)
    return chain_from_sums(params, proj, sums)


# ---------------------------------------------------------------------------
# optics  (optics.py:30-141)
# ---------------------------------------------------------------------------
_PLANCK = 6.62607015e-34
_ELECTRON_MASS = 9.1093837015e-31
_ELEMENTARY_CHARGE = 1.602176634e-19
_LIGHT_SPEED = 299792458.0


def electron_wavelength(voltage_kv: float) -> float:
    """optics.py:30-36 (Angstrom)."""
    ev = _ELEMENTARY_CHARGE * voltage_kv * 1e3
    wavelength_m = _PLANCK / math.sqrt(
        2.0 * _ELECTRON_MASS * ev * (1.0 + ev / (2.0 * _ELECTRON_MASS * _LIGHT_SPEED**2))
    )
    return wavelength_m * 1e10


@dataclass(frozen=True)
class Ctf:
    """CtfParams (optics.py:39-62)."""

    defocus_u: float
    defocus_v: float
    astigmatism_angle: float = 0.0
    voltage: float = 300.0
    spherical_aberration: float = 2.7
    amplitude_contrast: float = 0.1
    phase_shift: float = 0.0
    b_factor: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.defocus_u, self.defocus_v, self.astigmatism_angle, self.voltage,
                         self.spherical_aberration, self.amplitude_contrast, self.phase_shift,
                         self.b_factor], dtype=np.float64)


def ctf_evaluate(ctf: Ctf, grid: Grid) -> np.ndarray:
    """optics.py:93-121: centered (D, D) CTF."""
    freqs = grid.freq_indices() / (grid.size * grid.pixel_size)
    kx = freqs[None, :]
    ky = freqs[:, None]
    k2 = kx * kx + ky * ky
    theta = np.arctan2(ky, kx)
    lam = electron_wavelength(ctf.voltage)
    cs_angstrom = ctf.spherical_aberration * 1e7
    defocus = 0.5 * ((ctf.defocus_u + ctf.defocus_v)
                     + (ctf.defocus_u - ctf.defocus_v) * np.cos(2.0 * (theta - ctf.astigmatism_angle)))
    chi = np.pi * lam * defocus * k2 - 0.5 * np.pi * cs_angstrom * lam**3 * k2 * k2 + ctf.phase_shift
    w = ctf.amplitude_contrast
    H = -(np.sqrt(1.0 - w * w) * np.sin(chi) + w * np.cos(chi))
    if ctf.b_factor > 0:
        H = H * np.exp(-ctf.b_factor * k2 / 4.0)
    return H


def fft_centered(pixels):
    """optics.py:78-84."""
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(pixels)))


def ifft_centered(values):
    """optics.py:87-90 (real part)."""
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(values))).real


def apply_ctf(pixels, H):
    """apply_ctf (optics.py:124-141) with a precomputed centered H."""
    return ifft_centered(fft_centered(pixels) * H)


def phase_shift_translate(pixels, translation_px):
    """optics.py:144-159."""
    tx, ty = float(translation_px[0]), float(translation_px[1])
    if tx == 0.0 and ty == 0.0:
        return np.array(pixels, dtype=np.float64, copy=True)
    D = pixels.shape[0]
    k = np.arange(D) - D // 2
    phase = np.exp(-2j * np.pi * (k[None, :] * tx + k[:, None] * ty) / D)
    return ifft_centered(fft_centered(pixels) * phase)


# ---------------------------------------------------------------------------
# loss, Adam, one batched step  (train.py:93-161)
# ---------------------------------------------------------------------------
def loss_mse(a, b) -> float:
    """train.py:114-121."""
    diff = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(diff * diff))


class Adam:
    """AdamState (train.py:93-111); eps outside sqrt(v_hat)."""

    def __init__(self, n, beta1=0.9, beta2=0.999, eps=1e-8):
        self.m = np.zeros((n, PARAMS_PER_GAUSSIAN))
        self.v = np.zeros((n, PARAMS_PER_GAUSSIAN))
        self.t = 0
        self.b1, self.b2, self.eps = beta1, beta2, eps

    def update(self, params, grads, lr):
        b1, b2, eps = self.b1, self.b2, self.eps
        self.t += 1
        self.m *= b1
        self.m += (1.0 - b1) * grads
        self.v *= b2
        self.v += (1.0 - b2) * grads * grads
        m_hat = self.m / (1.0 - b1**self.t)
        v_hat = self.v / (1.0 - b2**self.t)
        params -= lr * m_hat / (np.sqrt(v_hat) + eps)


def image_step(params, W, t, grid: Grid, H, observed):
    """_step body for one image without Adam (train.py:136-156).

    Returns (loss, grads (N, 11), rendered, model, upstream, raw sums, projection).
    ``H`` is the centered CTF array or None (no CTF: the identity operator).
    """
    rendered, _ = rasterize(params, W, t, grid)
    model = rendered if H is None else apply_ctf(rendered, H)
    loss = loss_mse(model, observed)
    d = grid.size
    dL_dmodel = (2.0 / (d * d)) * (model - observed)
    upstream = dL_dmodel if H is None else apply_ctf(dL_dmodel, H)
    proj = project(params, W, t, grid)
    sums = backward_raw_sums(params, W, t, grid, upstream, proj)
    grads = chain_from_sums(params, proj, sums)
    return loss, grads, rendered, model, upstream, sums, proj


def batch_step(params, poses, grid: Grid, Hs, observed, *, isotropic=False):
    """Batched semantics of the new framework: loss = mean over images of the
    per-image MSE, grads = mean of per-image ``rasterize_backward``.
    B = 1 reduces exactly to train._step (train.py:136-161)."""
    B = len(poses)
    losses = np.empty(B)
    grads = np.zeros_like(params)
    for i, (W, t) in enumerate(poses):
        H = None if Hs is None else Hs[i]
        loss, g, *_ = image_step(params, W, t, grid, H, observed[i])
        losses[i] = loss
        grads += g
    grads /= B
    if isotropic:
        grads[:, COL_RAW_SCALE] = grads[:, COL_RAW_SCALE].sum(axis=1, keepdims=True)
    return losses, grads
