"""Dataset ingest: MRC2014 float32 stacks/volumes and the particle metadata table
(the reference's io.py:1-199), plus a device-resident loader.

``read_mrc`` / ``write_mrc`` / ``read_meta`` / ``write_meta`` / ``load_dataset``
/ ``write_simulation`` keep the reference's file layouts byte for byte
(tests/test_capi_and_host.py compares against files the reference wrote).
``load_dataset_device`` is the B200 path: the stack
payload is read straight into pinned host memory, copied to HBM
asynchronously, and the recorded translations are removed there by one
batched ``cgs_fourier_filter``; poses and CTFs become the step's f64 arrays.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .ctf import CtfParams
from .exceptions import DataError, UnsupportedModeError
from .mixture import GaussianMixture, GridSpec, normalize_quaternion, quaternion_to_matrix, save_checkpoint
from .optimize import Dataset, ParticleRecord
from .render import Pose

HEADER_BYTES = 1024
MODE_FLOAT32 = 2

META_COLUMNS = ("index", "qw", "qx", "qy", "qz", "tx_px", "ty_px", "defocus_u", "defocus_v", "astig_angle",
                "voltage_kv", "cs_mm", "amp_contrast", "phase_shift", "b_factor")

# MRC2014 header words used here: (byte offset, struct format)
_NXYZ, _MODE, _START, _MXYZ, _CELL, _ANGLES = (0, "<3i"), (12, "<i"), (16, "<3i"), (28, "<3i"), (40, "<3f"), (52, "<3f")
_AXES, _DSTATS, _ISPG, _NSYMBT, _MAP, _MACHST = (64, "<3i"), (76, "<3f"), (88, "<i"), (92, "<i"), 208, 212
_RMS, _NLABL = (216, "<f"), (220, "<i")


def _as_stack(data) -> np.ndarray:
    a = np.asarray(data)
    a = a[None] if a.ndim == 2 else a
    if a.ndim != 3:
        raise ValueError("MRC data must be 2D or 3D")
    if a.shape[1] != a.shape[2]:
        raise ValueError(f"MRC images must be square, got nx={a.shape[2]}, ny={a.shape[1]}")
    return a


def write_mrc(path, data, pixel_size: float, *, volume: bool | None = None) -> None:
    """Float32 little-endian MRC2014 (mode 2), data (nz, ny, nx); io.py:45-86.

    ``volume`` (default: cubic data) selects ISPG 1 (volume) vs 0 (image stack).
    """
    a = _as_stack(data)
    nz, ny, nx = a.shape
    volume = (nz == nx) if volume is None else volume
    if volume and nz != nx:
        raise ValueError("an MRC volume must be cubic")
    payload = np.ascontiguousarray(a, dtype="<f4")
    apix = np.float32(pixel_size)
    h = bytearray(HEADER_BYTES)
    fields = [
        (_NXYZ, (nx, ny, nz)), (_MODE, (MODE_FLOAT32,)), (_START, (0, 0, 0)), (_MXYZ, (nx, ny, nz)),
        (_CELL, (apix * nx, apix * ny, apix * nz)), (_ANGLES, (90.0, 90.0, 90.0)), (_AXES, (1, 2, 3)),
        (_DSTATS, (float(payload.min()), float(payload.max()), float(payload.mean()))),
        (_ISPG, (1 if volume else 0,)), (_NSYMBT, (0,)), (_RMS, (float(payload.std()),)), (_NLABL, (0,)),
    ]
    for (off, fmt), vals in fields:
        struct.pack_into(fmt, h, off, *vals)
    h[_MAP:_MAP + 4] = b"MAP "
    h[_MACHST:_MACHST + 4] = b"\x44\x44\x00\x00"  # little-endian machine stamp
    with open(path, "wb") as f:
        f.write(h)
        f.write(payload.tobytes())


def _header(path, blob):
    if len(blob) < HEADER_BYTES:
        raise DataError(f"{path}: truncated MRC file (no header)")
    nx, ny, nz = struct.unpack_from(_NXYZ[1], blob, _NXYZ[0])
    (mode,) = struct.unpack_from(_MODE[1], blob, _MODE[0])
    if mode != MODE_FLOAT32:
        raise UnsupportedModeError(mode)
    if min(nx, ny, nz) < 1:
        raise DataError(f"{path}: invalid MRC dimensions {nx} x {ny} x {nz}")
    if nx != ny:
        raise DataError(f"{path}: dimension mismatch, nx={nx} != ny={ny}")
    (nsymbt,) = struct.unpack_from(_NSYMBT[1], blob, _NSYMBT[0])
    (mx,) = struct.unpack_from("<i", blob, _MXYZ[0])
    (xlen,) = struct.unpack_from("<f", blob, _CELL[0])
    pixel_size = float(np.float32(xlen / mx)) if mx > 0 and xlen > 0 else 1.0
    return nx, ny, nz, HEADER_BYTES + nsymbt, pixel_size


def read_mrc(path):
    """(data (nz, ny, nx) float32, pixel_size) of a mode-2 MRC file; io.py:89-112."""
    with open(path, "rb") as f:
        blob = f.read()
    nx, ny, nz, off, apix = _header(path, blob)
    need = off + 4 * nx * ny * nz
    if len(blob) < need:
        raise DataError(f"{path}: truncated MRC payload ({len(blob)} < {need} bytes)")
    return np.frombuffer(blob, dtype="<f4", count=nx * ny * nz, offset=off).reshape(nz, ny, nx).copy(), apix


def read_mrc_pinned(path):
    """Like read_mrc, but the payload lands directly in a pinned host tensor
    (one readinto, no intermediate copy), ready for an async H2D copy."""
    import torch

    with open(path, "rb") as f:
        head = f.read(HEADER_BYTES)
        nx, ny, nz, off, apix = _header(path, head + b"\0" * max(0, HEADER_BYTES - len(head)))
        size = os.fstat(f.fileno()).st_size
        if size < off + 4 * nx * ny * nz:
            raise DataError(f"{path}: truncated MRC payload ({size} < {off + 4 * nx * ny * nz} bytes)")
        out = torch.empty((nz, ny, nx), dtype=torch.float32).pin_memory()
        f.seek(off)
        f.readinto(memoryview(out.numpy()).cast("B"))
    return out, apix


def write_meta(path, quaternions, translations, ctfs) -> None:
    """The metadata table, 17 significant digits (exact f64 round trip); io.py:115-133."""
    q = np.asarray(quaternions, dtype=np.float64)
    t = np.asarray(translations, dtype=np.float64)
    rows = ["# " + " ".join(META_COLUMNS)]
    for i, c in enumerate(ctfs):
        vals = (*q[i, :4], *t[i, :2], c.defocus_u, c.defocus_v, c.astigmatism_angle, c.voltage,
                c.spherical_aberration, c.amplitude_contrast, c.phase_shift, c.b_factor)
        rows.append(" ".join([str(i)] + [f"{float(v):.17g}" for v in vals]))
    with open(path, "w") as f:
        f.write("\n".join(rows) + "\n")


def read_meta(path) -> np.ndarray:
    """(n, 15) float64 rows, indices 0..n-1 in order; io.py:136-151."""
    try:
        rows = np.loadtxt(path, comments="#", dtype=np.float64, ndmin=2)
    except ValueError as exc:
        raise DataError(f"{path}: malformed metadata table ({exc})") from exc
    if rows.size == 0:
        raise DataError(f"{path}: empty metadata table")
    if rows.shape[1] != len(META_COLUMNS):
        raise DataError(f"{path}: expected {len(META_COLUMNS)} columns, found {rows.shape[1]}")
    if not np.array_equal(rows[:, 0].astype(np.int64), np.arange(len(rows))):
        raise DataError(f"{path}: metadata indices must run 0..{len(rows) - 1} in order")
    return rows


def _ctf(r) -> CtfParams:
    return CtfParams(defocus_u=r[7], defocus_v=r[8], astigmatism_angle=r[9], voltage=r[10],
                     spherical_aberration=r[11], amplitude_contrast=r[12], phase_shift=r[13], b_factor=r[14])


def load_dataset(stack_path, meta_path, extent: float = 0.5) -> Dataset:
    """Stack + metadata -> trainer records (io.py:154-184); counts checked first."""
    data, apix = read_mrc(stack_path)
    rows = read_meta(meta_path)
    if data.shape[0] != rows.shape[0]:
        raise DataError(f"stack has {data.shape[0]} images but metadata has {rows.shape[0]} rows")
    grid = GridSpec(data.shape[1], extent, apix)
    recs = [ParticleRecord(image=data[i], pose=Pose(quaternion_to_matrix(normalize_quaternion(r[1:5]))),
                           ctf=_ctf(r), translation=r[5:7].copy()) for i, r in enumerate(rows)]
    return Dataset(records=recs, grid=grid)


def load_dataset_device(stack_path, meta_path, extent: float = 0.5, chunk: int = 4096):
    """Stack + metadata straight into HBM for the Reconstructor.

    Returns (grid, obs f32 [R][D][D] device, centred: the recorded translations
    removed by a batched cgs_fourier_filter, poses f64 [R][12] numpy, ctfs
    f64 [R][8] numpy).  Same records as load_dataset + _centered_observation
    (train.py:124-133, :222), without a per-record host round trip.
    """
    import torch

    from . import engine
    from .ctf import filter_batch

    host, apix = read_mrc_pinned(stack_path)
    rows = read_meta(meta_path)
    if host.shape[0] != rows.shape[0]:
        raise DataError(f"stack has {host.shape[0]} images but metadata has {rows.shape[0]} rows")
    grid = GridSpec(host.shape[1], extent, apix)
    ctx = engine.DeviceContext.get()
    obs = host.to(ctx.device, non_blocking=True)
    shifts = rows[:, 5:7]
    moved = np.flatnonzero(np.any(shifts != 0.0, axis=1))
    for a in range(0, len(moved), chunk):
        idx = torch.as_tensor(moved[a:a + chunk], device=ctx.device)
        sub = obs.index_select(0, idx)
        filter_batch(sub, grid, shifts=-shifts[moved[a:a + chunk]], out=sub)
        obs.index_copy_(0, idx, sub)
    rot = np.stack([quaternion_to_matrix(normalize_quaternion(r[1:5])) for r in rows])
    poses = engine.pose_array(rot)
    ctfs = engine.ctf_array([_ctf(r) for r in rows])
    return grid, obs, poses, ctfs


def write_simulation(result, out_dir, prefix: str, truth: GaussianMixture):
    """Stack (.mrcs), metadata table and ground-truth checkpoint; io.py:187-199."""
    os.makedirs(out_dir, exist_ok=True)
    paths = tuple(os.path.join(out_dir, prefix + s) for s in (".mrcs", "_meta.txt", "_truth.cgs"))
    recs = result.records
    write_mrc(paths[0], np.stack([r.image.astype(np.float32) for r in recs]), result.dataset.grid.pixel_size,
              volume=False)
    write_meta(paths[1], result.quaternions, np.stack([r.translation for r in recs]), [r.ctf for r in recs])
    save_checkpoint(truth, paths[2])
    return paths
