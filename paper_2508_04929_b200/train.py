"""Reference-compatible module path (cryosplat.train) for GPU training."""
from .optimize import (  # noqa: F401
    DIVERGENCE_FACTOR, AdamState, Dataset, ParticleRecord, Reconstructor, TrainConfig, half_config,
    loss_mse, train, train_step,
)
