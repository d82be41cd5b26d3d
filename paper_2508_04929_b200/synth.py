"""Synthetic particles on the GPU (the forward model of the reference's simulate.py).

``make_phantom``, ``sample_pose`` and every per-particle draw of ``simulate``
reproduce the reference's seeded generators (simulate.py:92-267) exactly, on
the host (a few numbers per particle).  The image work runs on the device in
batches: K0/K3 direct render of the truth, then one ``cgs_fourier_filter``
launch that applies the CTF and the sub-pixel translation together, then the
dataset-wide noise calibration.  Noise comes either from the reference's own
per-particle numpy streams (``noise="numpy"``, bit-compatible datasets) or
from the device Philox generator (``noise="device"``, for large sets).
``synthetic_stack`` is the device-resident variant used by bench.py.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib, engine
from .mixture import COL_MEAN, COL_QUAT, COL_RAW_AMP, COL_RAW_SCALE, PARAMS_PER_GAUSSIAN, GaussianMixture, GridSpec
from .mixture import inverse_activate, normalize_quaternion
from .render import Pose
from dataclasses import dataclass, replace

PHANTOM_KINDS = ("helix", "blob-cluster", "two-lobe")


def sample_rotation_quaternion(rng: np.random.Generator) -> np.ndarray:
    return rng.standard_normal(4)


def sample_pose(rng: np.random.Generator, translation_range: float = 0.0, integer_translations: bool = False) -> Pose:
    """Uniform SO(3) rotation, optional box-uniform translation (simulate.py:92-106)."""
    q = sample_rotation_quaternion(rng)
    t = rng.uniform(-translation_range, translation_range, size=2) if translation_range else np.zeros(2)
    if integer_translations:
        t = np.rint(t)
    return Pose.from_quaternion(q, t)


def make_phantom(kind: str, n: int, seed: int = 0) -> GaussianMixture:
    """Deterministic ground-truth mixtures (simulate.py:130-190)."""
    if n < 1:
        raise ValueError("phantom needs n >= 1")
    rng = np.random.default_rng(seed)
    p = np.zeros((n, PARAMS_PER_GAUSSIAN))
    p[:, COL_RAW_AMP] = inverse_activate(1.0 / n)
    if kind == "helix":
        u = np.linspace(0.0, 1.0, n)
        ang = 4.0 * np.pi * u
        r, zh = 0.15, 0.2
        p[:, 0], p[:, 1], p[:, 2] = r * np.cos(ang), r * np.sin(ang), -zh + 2.0 * zh * u
        tan = np.stack([-r * 4.0 * np.pi * np.sin(ang), r * 4.0 * np.pi * np.cos(ang), np.full(n, 2.0 * zh)], axis=1)
        tan /= np.linalg.norm(tan, axis=1, keepdims=True)
        ex = np.array([1.0, 0.0, 0.0])
        for i in range(n):
            axis = np.cross(ex, tan[i])
            axis /= np.linalg.norm(axis)
            half = 0.5 * math.acos(float(np.clip(np.dot(ex, tan[i]), -1.0, 1.0)))
            p[i, COL_QUAT] = np.concatenate(([math.cos(half)], math.sin(half) * axis))
        p[:, 3] = inverse_activate(0.030)
        p[:, 4] = inverse_activate(0.015)
        p[:, 5] = inverse_activate(0.015)
    elif kind == "two-lobe":
        centers = np.array([[-0.12, 0.0, 0.0], [0.12, 0.0, 0.0]])
        means = centers[np.arange(n) % 2] + rng.normal(0.0, 0.02, size=(n, 3))
        nrm = np.linalg.norm(means, axis=1)
        far = nrm > 0.245
        means[far] *= (0.245 / nrm[far])[:, None]
        p[:, COL_MEAN] = means
        p[:, COL_RAW_SCALE] = inverse_activate(0.04)
        p[:, COL_QUAT.start] = 1.0
    elif kind == "blob-cluster":
        means = np.empty((n, 3))
        got = 0
        while got < n:
            cand = rng.normal(0.0, 0.1, size=(n - got, 3))
            keep = cand[np.linalg.norm(cand, axis=1) <= 0.24]
            means[got:got + len(keep)] = keep
            got += len(keep)
        p[:, COL_MEAN] = means
        p[:, COL_RAW_SCALE] = inverse_activate(rng.uniform(0.02, 0.04, size=(n, 3)))
        p[:, COL_QUAT] = normalize_quaternion(rng.standard_normal((n, 4)))
    else:
        raise ValueError(f"unknown phantom kind {kind!r} (choose from {PHANTOM_KINDS})")
    return GaussianMixture(p)


def synthetic_stack(truth: GaussianMixture, rotations, grid: GridSpec, *, defocus=None, snr: float = 0.1,
                    noise_seed: int = 11, chunk: int = 256):
    """Observed particle stack on the device: render(truth) -> CTF -> + N(0, sigma^2).

    ``defocus`` (one per particle, Angstrom, non-astigmatic, 300 kV, Cs 2.7,
    w 0.1) or None for no CTF.  sigma^2 = var(clean stack) / snr.  Returns
    (obs f32 [K][D][D] device tensor, ctfs f64 [K][8] numpy or None, sigma).
    """
    import torch

    from .ctf import CtfParams
    from .render import rasterize_batch

    R = np.asarray(rotations, dtype=np.float64).reshape(-1, 3, 3)
    K = R.shape[0]
    ctfs = None
    if defocus is not None:
        ctfs = engine.ctf_array([CtfParams(float(d), float(d)) for d in defocus])
    ctx = engine.DeviceContext.get()
    out = torch.empty((K, grid.size, grid.size), dtype=torch.float32, device=ctx.device)
    gs = _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)
    for a in range(0, K, chunk):
        b = min(K, a + chunk)
        img = rasterize_batch(truth, R[a:b], None, grid, device_out=True, method="direct")
        if ctfs is not None:
            c = torch.as_tensor(ctfs[a:b]).to(ctx.device)
            img = engine.ctf_apply(ctx, img, gs, ctf=c)
        out[a:b] = img
    sigma = 0.0
    if math.isfinite(snr):
        sigma = float(math.sqrt(out.double().var().item() / snr))
        gen = torch.Generator(device=ctx.device)
        gen.manual_seed(int(noise_seed))
        out += sigma * torch.randn(out.shape, generator=gen, device=ctx.device, dtype=torch.float32)
    return out, ctfs, sigma


# ---------------------------------------------------------------------------
# simulate (simulate.py:35-267)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class NoiseModel:
    """Gaussian pixel noise with variance var(clean) / snr; snr = inf disables it (simulate.py:35-47)."""

    snr: float
    seed: int = 0

    def __post_init__(self):
        if not self.snr > 0:
            raise ValueError("snr must be positive (use math.inf to disable noise)")


def snr_from_db(db: float) -> float:
    """10**(db / 10) (simulate.py:50-52)."""
    return 10.0 ** (db / 10.0)


def _default_template():
    from .ctf import CtfParams

    return CtfParams(defocus_u=15000.0, defocus_v=15000.0)


@dataclass(frozen=True)
class DefocusRange:
    """Uniform defocus, defocus_v = defocus_u, no astigmatism (simulate.py:55-67)."""

    minimum: float
    maximum: float
    template: object = None

    def sample(self, rng: np.random.Generator):
        d = float(rng.uniform(self.minimum, self.maximum))
        t = self.template if self.template is not None else _default_template()
        return replace(t, defocus_u=d, defocus_v=d, astigmatism_angle=0.0)


@dataclass
class SimSpec:
    """simulate.py:70-86."""

    truth: GaussianMixture
    num_particles: int
    grid: GridSpec
    ctf_distribution: object
    noise: NoiseModel
    translation_range: float = 0.0
    integer_translations: bool = False
    pose_jitter_deg: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.num_particles < 2:
            raise ValueError("num_particles must be >= 2 (both half-splits must be non-empty)")


@dataclass
class SimulationResult:
    dataset: object
    quaternions: np.ndarray
    noise_sigma: float
    images: object = None  # device f32 [K][D][D] when simulate(..., keep_on_device=True)

    @property
    def records(self):
        return self.dataset.records


def _quaternion_multiply(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw])


def _jitter_quaternion(rng, degrees):
    axis = rng.standard_normal(3)
    axis /= np.linalg.norm(axis)
    angle = math.radians(degrees) * rng.standard_normal()
    return np.concatenate(([math.cos(angle / 2.0)], math.sin(angle / 2.0) * axis))


def _draws(spec: SimSpec):
    """The per-particle host draws of simulate.py:224-239, in the reference's order."""
    n = spec.num_particles
    true_q = np.empty((n, 4))
    rec_q = np.empty((n, 4))
    ctfs = []
    trans = np.zeros((n, 2))
    choices = None if isinstance(spec.ctf_distribution, DefocusRange) else list(spec.ctf_distribution)
    for i in range(n):
        rng = np.random.default_rng(spec.seed + i)
        q = sample_rotation_quaternion(rng)
        true_q[i] = q
        ctfs.append(spec.ctf_distribution.sample(rng) if choices is None else choices[int(rng.integers(len(choices)))])
        if spec.translation_range:
            t = rng.uniform(-spec.translation_range, spec.translation_range, size=2)
            if spec.integer_translations:
                t = np.rint(t)
            trans[i] = t
        if spec.pose_jitter_deg > 0:
            q = _quaternion_multiply(_jitter_quaternion(rng, spec.pose_jitter_deg), q)
        rec_q[i] = q
    return true_q, rec_q, ctfs, trans


def simulate(spec: SimSpec, *, noise: str = "numpy", chunk: int = 1024, keep_on_device: bool = False):
    """Render, modulate, translate and corrupt particles (simulate.py:204-267) on the GPU.

    noise="numpy" draws each particle's noise from default_rng(noise.seed + i)
    exactly as the reference (bit-compatible datasets); noise="device" uses the
    device generator seeded with noise.seed (same distribution, much faster
    for 1e5 particles).  Images are float32, as the reference stores them.
    """
    import torch

    from .ctf import filter_batch
    from .optimize import Dataset, ParticleRecord
    from .render import rasterize_batch

    if noise not in ("numpy", "device"):
        raise ValueError("noise must be 'numpy' or 'device'")
    grid = spec.grid
    n, D = spec.num_particles, grid.size
    true_q, rec_q, ctfs, trans = _draws(spec)
    R = np.stack([p.rotation for p in Pose.from_quaternions(true_q)])
    ctx = engine.DeviceContext.get()
    clean = torch.empty((n, D, D), dtype=torch.float32, device=ctx.device)
    carr = engine.ctf_array(ctfs)
    moved = bool(np.any(trans != 0.0))
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        img = rasterize_batch(spec.truth, R[a:b], None, grid, device_out=True, method="direct")
        filter_batch(img, grid, ctfs=carr[a:b], shifts=trans[a:b] if moved else None, out=clean[a:b])
    sigma = 0.0 if math.isinf(spec.noise.snr) else float(math.sqrt(clean.double().var(unbiased=False).item()
                                                                    / spec.noise.snr))
    if sigma > 0.0 and noise == "device":
        gen = torch.Generator(device=ctx.device)
        gen.manual_seed(int(spec.noise.seed))
        clean += sigma * torch.randn(clean.shape, generator=gen, device=ctx.device, dtype=torch.float32)
    if not bool(torch.isfinite(clean).all()):
        raise ValueError("simulated particle images contain non-finite values")
    host = clean.cpu().numpy()
    poses = Pose.from_quaternions(rec_q)
    trans = np.asarray(trans, dtype=np.float64)
    records = []
    for i in range(n):
        img = host[i]
        if sigma > 0.0 and noise == "numpy":
            img = (img.astype(np.float64)
                   + np.random.default_rng(spec.noise.seed + i).normal(0.0, sigma, size=img.shape)).astype(np.float32)
        records.append(ParticleRecord.prevalidated(img, poses[i], ctfs[i], trans[i]))
    images = None
    if keep_on_device:
        images = torch.as_tensor(np.stack([r.image for r in records])).to(ctx.device) if noise == "numpy" else clean
    return SimulationResult(dataset=Dataset(records=records, grid=grid), quaternions=rec_q, noise_sigma=sigma,
                            images=images)
