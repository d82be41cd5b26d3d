"""Synthetic particles on the GPU (the forward model of the reference's simulate.py).

``make_phantom`` and ``sample_pose`` reproduce the reference's seeded draws
(simulate.py:92-190) so that synthetic inputs match it exactly; rendering,
CTF modulation and noise for whole particle stacks run on the device
(``synthetic_stack``): K0/K2/K3 render, K4 CTF, ``torch.randn`` noise.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib, engine
from .mixture import COL_MEAN, COL_QUAT, COL_RAW_AMP, COL_RAW_SCALE, PARAMS_PER_GAUSSIAN, GaussianMixture, GridSpec
from .mixture import inverse_activate, normalize_quaternion
from .render import Pose

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
