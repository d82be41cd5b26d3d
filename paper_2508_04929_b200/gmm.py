"""Reference-compatible module path (cryosplat.gmm) for the parameter model."""
from .mixture import (  # noqa: F401
    COL_MEAN, COL_QUAT, COL_RAW_AMP, COL_RAW_SCALE, MODES, PARAMS_PER_GAUSSIAN, GaussianMixture,
    GaussianParams, GridSpec, activate, activate_derivative, build_covariance, init_random,
    inverse_activate, load_checkpoint, normalize_quaternion, param_count, quaternion_to_matrix,
    save_checkpoint,
)
