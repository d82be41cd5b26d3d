"""Reference module path ``cryosplat.simulate`` (simulate.py): the GPU implementations live in synth.py."""

from .synth import (  # noqa: F401
    PHANTOM_KINDS,
    DefocusRange,
    NoiseModel,
    SimSpec,
    SimulationResult,
    make_phantom,
    sample_pose,
    sample_rotation_quaternion,
    simulate,
    snr_from_db,
)
