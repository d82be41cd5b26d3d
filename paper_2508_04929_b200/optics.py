"""Reference-compatible module path (cryosplat.optics) for the GPU CTF physics."""
from .ctf import (  # noqa: F401
    CtfParams, Spectrum, apply_ctf, apply_ctf_batch, ctf_evaluate, electron_wavelength, fft_centered,
    ifft_centered, phase_shift_translate,
)
