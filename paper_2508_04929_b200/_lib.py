"""ctypes binding of libcgs_b200.so (declared in include/cgs_b200.h).

The product path has no fallback: if the library or a CUDA device is missing,
every call raises ``CudaUnavailableError`` (a RuntimeError).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CGS_B200_LIB selects an alternative in-tree build (kernel A/B experiments)
LIB_PATH = os.environ.get("CGS_B200_LIB") or os.path.join(_HERE, "libcgs_b200.so")

CGS_OK = 0
CGS_LAYOUT_NATURAL = 0
CGS_LAYOUT_FFT = 1
CGS_LAYOUT_ROWPAIR = 2
CGS_MODE = {"anisotropic": 0, "isotropic": 1}
CGS_SPLAT_STRIDE = 16
CGS_ACC_STRIDE = 10
CGS_BIN_CHUNK = 2048
CGS_STATUS_DEGENERATE_ROTATION = 1
CGS_STATUS_BIN_OVERFLOW = 2
CGS_STATUS_NONFINITE_LOSS = 4
CGS_STATUS_NONFINITE_PARAMS = 8


class CudaUnavailableError(RuntimeError):
    """libcgs_b200.so or the CUDA device is unavailable (no CPU fallback exists)."""


class CgsError(RuntimeError):
    """A libcgs_b200 entry point returned an error code."""


class cgs_grid(ctypes.Structure):
    _fields_ = [
        ("size", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("extent", ctypes.c_double),
        ("pixel_size", ctypes.c_double),
    ]


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double
G = cgs_grid

# name -> (restype, argtypes); mirrors include/cgs_b200.h
PROTOTYPES = {
    "cgs_version": (ctypes.c_char_p, []),
    "cgs_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "cgs_last_error_detail": (ctypes.c_char_p, []),
    "cgs_launch_state_entries": (I32, [I32]),
    "cgs_prepare": (ctypes.c_int, [P, I64, P, P, P]),
    "cgs_bin_segments": (I64, [I64]),
    "cgs_bin_tiles": (I64, [I32, I32]),
    "cgs_bin_count": (ctypes.c_int, [P, I64, P, I32, G, I32, P, P, P, P, P]),
    "cgs_bin_count_bbox": (ctypes.c_int, [P, I64, I32, I32, I32, P, P, P]),
    "cgs_scan_workspace_bytes": (ctypes.c_size_t, [I64]),
    "cgs_exclusive_scan": (ctypes.c_int, [P, P, I64, P, P]),
    "cgs_bin_scatter": (ctypes.c_int, [P, I64, I32, I32, I32, P, P, I64, P, P]),
    "cgs_raster_fwd": (ctypes.c_int, [P, I64, P, I32, G, I32, P, P, I64, P, I32, P]),
    "cgs_render_workspace_bytes": (ctypes.c_size_t, [I64]),
    "cgs_render": (ctypes.c_int, [P, I64, P, I32, G, P, P, P, P]),
    "cgs_render_fixed": (ctypes.c_int, [P, I64, P, I32, G, P, P, P, P]),
    "cgs_render_scale_offset": (I64, [I64]),
    "cgs_prepare_render_fixed": (ctypes.c_int, [P, I64, P, P, P, I32, G, P, P, P, P]),
    "cgs_ctf_evaluate": (ctypes.c_int, [P, I32, G, P, P]),
    "cgs_fft_plan_create": (ctypes.c_int, [I32, I32, ctypes.POINTER(ctypes.c_void_p)]),
    "cgs_fft_plan_destroy": (ctypes.c_int, [P]),
    "cgs_fft_spectrum_elems": (I64, [I32, I32]),
    "cgs_ctf_apply": (ctypes.c_int, [P, P, P, I32, G, P, P, P, I32, P]),
    "cgs_loss_residual": (ctypes.c_int, [P, P, I32, I32, P, P, P, P]),
    "cgs_ctf_mse": (ctypes.c_int, [P, P, P, I32, G, P, P, P, P, P, P, I32, P]),
    "cgs_fourier_filter": (ctypes.c_int, [P, P, I32, G, P, P, P]),
    "cgs_obs_spectrum_elems": (I64, [I32, I32]),
    "cgs_obs_spectrum": (ctypes.c_int, [P, P, I32, G, P, P]),
    "cgs_ctf_mse_spectral": (ctypes.c_int, [P, P, I32, G, P, P, P, I32, P]),
    "cgs_ctf_mse_spectral_fixed": (ctypes.c_int, [P, P, P, I32, G, P, P, P, I32, P]),
    "cgs_ctf_mse_spectral_fixed_rows": (ctypes.c_int, [P, P, P, P, I32, G, P, P, P, I32, P]),
    "cgs_obs_spectrum_fft_elems": (I64, [I32, I32]),
    "cgs_spectral_fft_workspace_bytes": (ctypes.c_size_t, [I32, I32]),
    "cgs_obs_spectrum_fft": (ctypes.c_int, [P, P, P, I32, G, P, P, P]),
    "cgs_ctf_mse_spectral_fft": (ctypes.c_int, [P, P, P, P, P, I32, G, P, P, P, P, P, I32, P]),
    "cgs_voxelize_workspace_bytes": (ctypes.c_size_t, [I64]),
    "cgs_voxelize": (ctypes.c_int, [P, I64, G, P, P, P, P]),
    "cgs_bwd_groups": (I64, [I32, I32]),
    "cgs_raster_bwd": (ctypes.c_int, [P, I64, P, I32, G, P, I32, P, I32, P]),
    "cgs_reduce_partials": (ctypes.c_int, [P, I32, I64, P, P]),
    "cgs_acc_slice_floats": (I64, [I64, I64]),
    "cgs_reduce_partials_sliced": (ctypes.c_int, [P, I32, I64, I64, P, P, P]),
    "cgs_peer_blocks": (I32, [I64]),
    "cgs_peer_epilogue_adam": (ctypes.c_int, [P, P, P, I32, I32, I64, I64, P, P, I32, F64, F64, F64, F64, P, P]),
    "cgs_epilogue_grads": (ctypes.c_int, [P, I32, I64, P, I32, F64, P, P]),
    "cgs_adam": (ctypes.c_int, [P, P, P, P, I64, F64, F64, F64, F64, F64, F64, P]),
    "cgs_epilogue_adam": (ctypes.c_int, [P, I32, I64, P, P, P, I32, F64, F64, F64, F64, F64, F64, F64, P, P]),
    "cgs_epilogue_adam_dev": (ctypes.c_int, [P, I32, I64, P, P, P, I32, F64, F64, F64, F64, P, P, P]),
    "cgs_count_pairs": (ctypes.c_int, [P, I64, P, I32, G, P, P]),
    "cgs_count_pairs_cut": (ctypes.c_int, [P, I64, P, I32, G, F64, P, P]),
    "cgs_bwd_cut_sq": (F64, []),
    "cgs_gather_rows": (ctypes.c_int, [P, P, I64, I64, P, P]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises CudaUnavailableError if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaUnavailableError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2508_04929_b200._build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Call an int-returning entry point and raise CgsError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != CGS_OK:
        detail = lib.cgs_last_error_detail().decode()
        raise CgsError(f"{name} failed: {lib.cgs_error_string(rc).decode()} ({detail})")


def grid_struct(size: int, extent: float, pixel_size: float) -> cgs_grid:
    return cgs_grid(int(size), 0, float(extent), float(pixel_size))
