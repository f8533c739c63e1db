"""B200-native 2D Gaussian surfel render + refine path (drop-in for surfelslam's rasterizer/refine).

Modules:
  rasterizer  — reference-compatible API (render, grad_color_opacity, ...)
  mapper      — refine (reference backtracking GD) and AdamRefiner (multi-view Adam, NCCL)
  engine      — device-level API over the C ABI (include/surfel2d.h)
  geometry    — pose / quaternion value types
  scenes      — seeded synthetic workloads of BASELINE.json configs 1-5
  distributed — view sharding and the gradient all-reduce
"""

from .geometry import SE3Pose, Sim3Transform, UnitQuaternion  # noqa: F401
from .rasterizer import (  # noqa: F401
    DEFAULT_RASTER_CONFIG, CameraIntrinsics, LossWeights, RasterConfig, RenderBuffers, Surfel,
    SurfelArrays, grad_color_opacity, per_surfel_max_weight, project_surfel, render, render_loss,
    render_with_argmax,
)

__version__ = "0.1.0"
