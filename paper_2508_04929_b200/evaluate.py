"""Voxelization and Fourier shell correlation (the reference's evaluate.py) on the GPU.

``voxelize`` samples a mixture at the D^3 voxel centres with the K8 kernel
(csrc/voxelize.cu: fp64, the rasterizer's q < 6.5^2 cull, deterministic
int64 fixed-point sums).  ``fsc`` transforms both volumes with a 3-D FFT on the
device (torch.fft over cuFFT, complex128), bins the cross and power spectra
into shells of rounded centred radius and reads the resolutions at 0.143 / 0.5
by linear interpolation of the first crossing (evaluate.py:125-197).  The
shell sums use a fixed voxel order per shell, so curves are reproducible.
``gold_standard_fsc`` trains the even/odd halves on the GPU and correlates them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, engine
from .mixture import GaussianMixture, GridSpec
from .optimize import Dataset, TrainConfig, half_config, train

FSC_GOLD_THRESHOLD = 0.143
FSC_HALF_THRESHOLD = 0.5


@dataclass
class VoxelVolume:
    """Density at voxel centres, [z, y, x], on an image grid (evaluate.py:35-49)."""

    grid: GridSpec
    voxels: np.ndarray

    def __post_init__(self):
        self.voxels = np.asarray(self.voxels, dtype=np.float64)
        d = self.grid.size
        if self.voxels.shape != (d, d, d):
            raise ValueError("voxel array does not match grid size")
        if not np.all(np.isfinite(self.voxels)):
            raise ValueError("voxel volume contains non-finite values")


@dataclass
class FscCurve:
    """Shell correlations and the 0.143 / 0.5 resolutions in Angstrom, None when
    never crossed (evaluate.py:52-73)."""

    shells: np.ndarray
    correlations: np.ndarray
    pixel_size: float
    grid_size: int
    resolution_0143: float | None
    resolution_05: float | None

    def spatial_frequencies(self) -> np.ndarray:
        return self.shells / (self.grid_size * self.pixel_size)

    def min_correlation(self, max_shell: int | None = None) -> float:
        top = self.shells.max() if max_shell is None else max_shell
        return float(self.correlations[self.shells <= top].min())


def voxelize_device(mixture: GaussianMixture, grid: GridSpec):
    """Device f64 [D][D][D] volume of the mixture (K8)."""
    import torch

    ctx = engine.DeviceContext.get()
    params = torch.as_tensor(np.ascontiguousarray(mixture.params, dtype=np.float64)).to(ctx.device)
    n = params.shape[0]
    D = grid.size
    out = torch.empty((D, D, D), dtype=torch.float64, device=ctx.device)
    ws = ctx.buf("voxelize_ws", int(ctx.lib.cgs_voxelize_workspace_bytes(n)), torch.uint8)
    status = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    _lib.call("cgs_voxelize", params.data_ptr(), n, _lib.grid_struct(D, grid.extent, grid.pixel_size),
              out.data_ptr(), ws.data_ptr(), status.data_ptr(), ctx.stream)
    if int(status.item()) & _lib.CGS_STATUS_DEGENERATE_ROTATION:
        from .exceptions import DegenerateRotationError

        raise DegenerateRotationError("quaternion with zero or non-finite norm")
    return out


def voxelize(mixture: GaussianMixture, grid: GridSpec) -> VoxelVolume:
    """evaluate.voxelize (evaluate.py:76-122)."""
    return VoxelVolume(grid=grid, voxels=voxelize_device(mixture, grid).cpu().numpy())


_SHELLS: dict = {}


def _shell_layout(D: int, device):
    """Voxel order grouped by shell (stable), shell sizes: fixed summation order."""
    import torch

    key = (D, str(device))
    if key not in _SHELLS:
        idx = torch.arange(D, dtype=torch.float64, device=device) - D // 2
        kz, ky, kx = torch.meshgrid(idx, idx, idx, indexing="ij")
        shell = torch.round(torch.sqrt(kx * kx + ky * ky + kz * kz)).to(torch.int64).reshape(-1)
        order = torch.argsort(shell, stable=True)
        counts = torch.bincount(shell)
        _SHELLS[key] = (order, counts)
    return _SHELLS[key]


def _shell_sums(values, order, counts):
    import torch

    v = values.reshape(-1)[order]
    return torch.segment_reduce(v, "sum", lengths=counts)


def _fft3_centered(v):
    import torch

    return torch.fft.fftshift(torch.fft.fftn(torch.fft.ifftshift(v)))


def _resolution_at(shells, corr, threshold, grid_size, pixel_size):
    """First drop below threshold, linearly interpolated from the previous shell
    (shell 0 counts as correlation 1); None if never (evaluate.py:128-136)."""
    s0, c0 = 0.0, 1.0
    for s, c in zip(shells, corr):
        if c < threshold:
            return grid_size * pixel_size / (s0 + (c0 - threshold) / (c0 - c) * (s - s0))
        s0, c0 = float(s), float(c)
    return None


def fsc(a: VoxelVolume, b: VoxelVolume) -> FscCurve:
    """Fourier shell correlation between two volumes on the same grid (evaluate.py:139-179)."""
    import torch

    if a.grid.size != b.grid.size:
        raise ValueError(f"grid mismatch: {a.grid.size} vs {b.grid.size}")
    if a.grid.pixel_size != b.grid.pixel_size:
        raise ValueError("grid mismatch: differing pixel sizes")
    D = a.grid.size
    dev = engine.DeviceContext.get().device
    fa = _fft3_centered(torch.as_tensor(a.voxels).to(dev))
    fb = _fft3_centered(torch.as_tensor(b.voxels).to(dev))
    order, counts = _shell_layout(D, dev)
    cross = fa * fb.conj()
    sums = [_shell_sums(x, order, counts) for x in (cross.real, cross.imag, fa.abs() ** 2, fb.abs() ** 2)]
    num_re, num_im, pa, pb = (s.cpu().numpy() for s in sums)
    shells = np.arange(1, D // 2 + 1)
    num_re, num_im = num_re[shells], num_im[shells]
    den = np.sqrt(pa[shells] * pb[shells])
    mag = np.hypot(num_re, num_im)
    if np.any(np.abs(num_im) > 1e-6 * mag + 1e-300):  # k and -k pair up inside each shell of a real volume
        raise ValueError("shell numerator has unexpectedly large imaginary part")
    with np.errstate(invalid="ignore", divide="ignore"):
        corr = np.clip(np.where(den > 0, num_re / den, 0.0), -1.0, 1.0)
    px = a.grid.pixel_size
    return FscCurve(shells=shells, correlations=corr, pixel_size=px, grid_size=D,
                    resolution_0143=_resolution_at(shells, corr, FSC_GOLD_THRESHOLD, D, px),
                    resolution_05=_resolution_at(shells, corr, FSC_HALF_THRESHOLD, D, px))


def gold_standard_fsc(dataset: Dataset, config: TrainConfig, *, n_gaussians: int,
                      voxel_grid: GridSpec | None = None) -> FscCurve:
    """Independent even/odd half reconstructions, correlated (evaluate.py:182-200);
    the odd half trains with seed + 1."""
    if len(dataset) < 2:
        raise ValueError("gold-standard FSC needs at least 2 records")
    grid = voxel_grid if voxel_grid is not None else dataset.grid
    vols = [voxelize(train(dataset.half(h), half_config(config, h), n_gaussians=n_gaussians)[0], grid)
            for h in ("even", "odd")]
    return fsc(vols[0], vols[1])


def _fmt_res(v):
    return "Nyquist (threshold never crossed)" if v is None else f"{v:.4f} A"


def fsc_table(curve: FscCurve) -> str:
    """shell_index spatial_freq_per_A correlation (evaluate.py:210-221)."""
    out = ["# shell_index spatial_freq_per_A correlation",
           f"# resolution at 0.5:   {_fmt_res(curve.resolution_05)}",
           f"# resolution at 0.143: {_fmt_res(curve.resolution_0143)}"]
    out += [f"{s} {f:.8f} {c:.8f}" for s, f, c in zip(curve.shells, curve.spatial_frequencies(), curve.correlations)]
    return "\n".join(out) + "\n"


def paired_fsc_report(curves: dict) -> str:
    """Several labelled curves on one grid, side by side (evaluate.py:224-238)."""
    labels = list(curves)
    first = curves[labels[0]]
    out = ["# shell spatial_freq_per_A " + " ".join(labels)]
    out += [f"# {lb}: resolution at 0.5 = {_fmt_res(curves[lb].resolution_05)}, "
            f"at 0.143 = {_fmt_res(curves[lb].resolution_0143)}" for lb in labels]
    for i, (s, f) in enumerate(zip(first.shells, first.spatial_frequencies())):
        out.append(" ".join([f"{s}", f"{f:.8f}"] + [f"{curves[lb].correlations[i]:.8f}" for lb in labels]))
    return "\n".join(out) + "\n"
