"""Reference-compatible module path (cryosplat.splat) for the GPU rasterizer."""
from .render import (  # noqa: F401
    CLAMP_EVENTS, CULL_SIGMA, DEFAULT_TILE_SIZE, EIGEN_FLOOR_FRACTION, CameraSpaceGaussian, ClampCounter,
    Pose, RenderedImage, SplatGaussian2D, orthographic_project, rasterize, rasterize_backward,
    rasterize_backward_batch, rasterize_batch, view_transform,
)
