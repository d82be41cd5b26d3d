"""B200-native cryoGS: differentiable orthographic Gaussian splatting for
known-pose cryo-EM reconstruction, as hand-written sm_100a CUDA behind a C ABI
(include/cgs_b200.h, libcgs_b200.so) with a PyTorch-plumbed host side.

The public names mirror the reference package ``cryosplat`` (its __init__.py
re-exports) for the render / reconstruct path, so ``import paper_2508_04929_b200
as cs`` is a drop-in for ``import cryosplat as cs`` there.  Every compute entry
point runs on the GPU; there is no CPU fallback.
"""

from .ctf import (
    CtfParams,
    Spectrum,
    apply_ctf,
    apply_ctf_batch,
    ctf_evaluate,
    electron_wavelength,
    fft_centered,
    ifft_centered,
    phase_shift_translate,
)
from .exceptions import (
    CgsError,
    CryosplatError,
    CudaUnavailableError,
    DataError,
    DegenerateRotationError,
    DegenerateSplatError,
    DivergenceError,
    UnsupportedModeError,
)
from .evaluate import FscCurve, VoxelVolume, fsc, gold_standard_fsc, voxelize
from .mixture import (
    GaussianMixture,
    GaussianParams,
    GridSpec,
    activate,
    build_covariance,
    init_random,
    inverse_activate,
    load_checkpoint,
    param_count,
    save_checkpoint,
)
from .optimize import (
    AdamState,
    Dataset,
    ParticleRecord,
    Reconstructor,
    TrainConfig,
    loss_mse,
    train,
    train_step,
)
from .render import (
    CameraSpaceGaussian,
    Pose,
    RenderedImage,
    SplatGaussian2D,
    orthographic_project,
    rasterize,
    rasterize_backward,
    rasterize_backward_batch,
    rasterize_batch,
    view_transform,
)
from .synth import DefocusRange, NoiseModel, SimSpec, make_phantom, sample_pose, simulate, snr_from_db

__version__ = "0.1.0"
