"""CTF physics on the GPU (mirrors the reference's optics.py).

``ctf_evaluate`` (optics.py:93-121) and ``apply_ctf`` (optics.py:124-141) run
the K4 kernels of libcgs_b200 (cuFFT R2C/C2R around the H_sym multiply).
``fft_centered`` / ``ifft_centered`` / ``phase_shift_translate`` (optics.py:
78-90, 144-159) use cuFFT through ``torch.fft`` on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib, engine
from .mixture import GridSpec
from .render import RenderedImage

_H_PLANCK = 6.62607015e-34
_M_ELECTRON = 9.1093837015e-31
_Q_ELECTRON = 1.602176634e-19
_C_LIGHT = 299792458.0


def electron_wavelength(voltage_kv: float) -> float:
    """Relativistic electron wavelength in Angstrom (optics.py:30-36, CODATA 2018)."""
    if voltage_kv <= 0:
        raise ValueError("acceleration voltage must be positive")
    energy = _Q_ELECTRON * voltage_kv * 1e3
    momentum = math.sqrt(2.0 * _M_ELECTRON * energy * (1.0 + energy / (2.0 * _M_ELECTRON * _C_LIGHT**2)))
    return _H_PLANCK / momentum * 1e10


@dataclass(frozen=True)
class CtfParams:
    """Per-image microscope parameters (optics.py:39-62)."""

    defocus_u: float
    defocus_v: float
    astigmatism_angle: float = 0.0
    voltage: float = 300.0
    spherical_aberration: float = 2.7
    amplitude_contrast: float = 0.1
    phase_shift: float = 0.0
    b_factor: float = 0.0

    def __post_init__(self):
        if self.voltage <= 0:
            raise ValueError("voltage must be positive")
        if not 0.0 <= self.amplitude_contrast < 1.0:
            raise ValueError("amplitude contrast must lie in [0, 1)")
        if self.b_factor < 0:
            raise ValueError("b_factor must be non-negative")

    @property
    def wavelength(self) -> float:
        return electron_wavelength(self.voltage)


@dataclass
class Spectrum:
    grid: GridSpec
    values: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.complex128)
        if self.values.shape != (self.grid.size, self.grid.size):
            raise ValueError("spectrum array does not match grid size")


def _dev(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def ctf_evaluate(params: CtfParams, grid: GridSpec) -> np.ndarray:
    """Centred (D, D) CTF, evaluated in fp64 by ``cgs_ctf_evaluate``."""
    import torch

    if grid.pixel_size <= 0:
        raise ValueError("grid pixel_size must be positive to evaluate a CTF")
    ctx = engine.DeviceContext.get()
    c = _dev(engine.ctf_array([params]), torch.float64)
    H = torch.empty((1, grid.size, grid.size), dtype=torch.float64, device=ctx.device)
    _lib.call("cgs_ctf_evaluate", c.data_ptr(), 1, _lib.grid_struct(grid.size, grid.extent, grid.pixel_size),
              H.data_ptr(), ctx.stream)
    return H[0].cpu().numpy()


def apply_ctf_batch(images, grid: GridSpec, *, ctfs=None, H=None):
    """Batched apply_ctf on device: images f32 [B][D][D] (tensor) -> new tensor."""
    import torch

    ctx = engine.DeviceContext.get()
    ctf_t = None if ctfs is None else _dev(engine.ctf_array(ctfs), torch.float64)
    H_t = None if H is None else (H if isinstance(H, torch.Tensor) else _dev(H, torch.float64))
    return engine.ctf_apply(ctx, images, _lib.grid_struct(grid.size, grid.extent, grid.pixel_size),
                            ctf=ctf_t, H=H_t)


def apply_ctf(img: RenderedImage, ctf) -> RenderedImage:
    """Modulate by the CTF in Fourier space and invert (optics.py:124-141).

    ``ctf`` is a CtfParams or a precomputed centred (D, D) array.
    """
    import torch

    D = img.pixels.shape[0]
    if isinstance(ctf, CtfParams):
        ctfs, H = [ctf], None
    else:
        H = np.asarray(ctf, dtype=np.float64)
        if H.shape != img.pixels.shape:
            raise ValueError(f"CTF array shape {H.shape} does not match image shape {img.pixels.shape}")
        ctfs, H = None, H[None]
    x = _dev(img.pixels[None], torch.float32)
    out = apply_ctf_batch(x, img.grid, ctfs=ctfs, H=H)
    return RenderedImage(grid=img.grid, pixels=out[0].double().cpu().numpy().reshape(D, D))


def fft_centered(img: RenderedImage) -> Spectrum:
    """Forward FFT with the origin pixel at zero phase (optics.py:78-84)."""
    import torch

    px = img.pixels
    if px.ndim != 2 or px.shape[0] != px.shape[1] or px.shape[0] < 4:
        raise ValueError("fft_centered requires a square image with D >= 4")
    x = _dev(px, torch.float64)
    X = torch.fft.fftshift(torch.fft.fft2(torch.fft.ifftshift(x)))
    return Spectrum(grid=img.grid, values=X.cpu().numpy())


def ifft_centered(spectrum: Spectrum) -> RenderedImage:
    """Inverse of fft_centered, real part (optics.py:87-90)."""
    import torch

    X = _dev(spectrum.values, torch.complex128)
    x = torch.fft.fftshift(torch.fft.ifft2(torch.fft.ifftshift(X))).real
    return RenderedImage(grid=spectrum.grid, pixels=x.cpu().numpy())


def phase_shift_translate(img: RenderedImage, translation_px) -> RenderedImage:
    """Sub-pixel translation by a Fourier phase ramp (optics.py:144-159)."""
    import torch

    tx, ty = float(translation_px[0]), float(translation_px[1])
    if not (math.isfinite(tx) and math.isfinite(ty)):
        raise ValueError("translation must be finite")
    if tx == 0.0 and ty == 0.0:
        return RenderedImage(grid=img.grid, pixels=img.pixels.copy())
    D = img.grid.size
    if D in engine.FILTER_SIZES:
        out = filter_batch(_dev(img.pixels[None], torch.float32), img.grid, shifts=[(tx, ty)])
        return RenderedImage(grid=img.grid, pixels=out[0].double().cpu().numpy())
    k = torch.arange(D, dtype=torch.float64, device="cuda") - D // 2
    ramp = torch.exp(-2j * math.pi * (k[None, :] * tx + k[:, None] * ty) / D)
    x = _dev(img.pixels, torch.float64)
    X = torch.fft.fftshift(torch.fft.fft2(torch.fft.ifftshift(x))) * ramp
    y = torch.fft.fftshift(torch.fft.ifft2(torch.fft.ifftshift(X))).real
    return RenderedImage(grid=img.grid, pixels=y.cpu().numpy())


def filter_batch(images, grid: GridSpec, *, ctfs=None, shifts=None, out=None):
    """apply_ctf then phase_shift_translate for a device batch f32 [B][D][D] in
    one kernel (``cgs_fourier_filter``).  ``ctfs``: CtfParams list, f64 [B][8]
    array/tensor or None; ``shifts``: [B][2] pixels or None.  D in 32/64/128;
    other sizes go through cuFFT (CTF) and torch.fft (shift)."""
    import torch

    ctx = engine.DeviceContext.get()
    gs = _lib.grid_struct(grid.size, grid.extent, grid.pixel_size)
    c = None
    if ctfs is not None:
        c = ctfs if isinstance(ctfs, torch.Tensor) else _dev(
            engine.ctf_array(ctfs) if not isinstance(ctfs, np.ndarray) else ctfs, torch.float64)
    sh = None
    if shifts is not None:
        sh = shifts if isinstance(shifts, torch.Tensor) else _dev(np.asarray(shifts, np.float64).reshape(-1, 2),
                                                                  torch.float64)
    if grid.size in engine.FILTER_SIZES:
        return engine.fourier_filter(ctx, images, gs, ctf=c, shifts=sh, out=out)
    y = images if c is None else engine.ctf_apply(ctx, images, gs, ctf=c)
    if sh is not None:
        D = grid.size
        k = torch.arange(D, dtype=torch.float64, device=images.device) - D // 2
        ramp = torch.exp(-2j * math.pi * (k[None, None, :] * sh[:, 0, None, None] + k[None, :, None] * sh[:, 1, None, None]) / D)
        X = torch.fft.fftshift(torch.fft.fft2(torch.fft.ifftshift(y.double(), dim=(-2, -1))), dim=(-2, -1)) * ramp
        y = torch.fft.fftshift(torch.fft.ifft2(torch.fft.ifftshift(X, dim=(-2, -1))), dim=(-2, -1)).real.float()
    if out is not None:
        out.copy_(y)
        return out
    return y
