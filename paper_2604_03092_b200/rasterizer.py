"""Drop-in replacement of ``surfelslam.rasterizer`` backed by sm_100a kernels.

Same names, argument order, return types and error behaviour as the reference
module (``pkg/src/surfelslam/rasterizer.py``):

* ``render``               — rasterizer.py:334-337
* ``render_with_argmax``   — rasterizer.py:340-343
* ``render_loss``          — rasterizer.py:346-357 (host numpy, as in the reference)
* ``grad_color_opacity``   — rasterizer.py:360-399
* ``per_surfel_max_weight``— rasterizer.py:402-428
* ``project_surfel``       — rasterizer.py:252-259 (host float64 utility)

Inputs are the reference's types (or this package's twins, duck-typed):
``list[Surfel]`` or ``SurfelArrays``, ``SE3Pose``/``Sim3Transform``,
``CameraIntrinsics``, ``RasterConfig``.  Outputs are numpy float64 arrays in
the reference's shapes, computed in float32 on the GPU; ``RenderBuffers``
additionally carries the alpha-blended camera-frame ``normal`` (H, W, 3).

Everything except ``render_loss``/``project_surfel`` runs through
``lib/libsurfel2d.so``; without it (or without a GPU) these functions raise
``NativeLibraryError`` — there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .engine import (DeviceContext, ImageBuffers, camera_struct, config_struct, forward_checked,
                     pack_params, unpack_params)
from .geometry import SE3Pose, Sim3Transform, UnitQuaternion, as_packed_pose, pk_inverse, quat_to_matrix

__all__ = [
    "CameraIntrinsics", "Surfel", "SurfelArrays", "RasterConfig", "DEFAULT_RASTER_CONFIG",
    "RenderBuffers", "SurfelFootprint", "LossWeights", "render", "render_with_argmax",
    "render_loss", "grad_color_opacity", "per_surfel_max_weight", "project_surfel",
]


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole intrinsics; pixel (row i, col j) samples the image plane at (j, i)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        # rasterizer.py:36-40
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point must lie inside the image")

    def scaled(self, factor: float) -> "CameraIntrinsics":
        return CameraIntrinsics(self.fx * factor, self.fy * factor, self.cx * factor, self.cy * factor,
                                max(1, int(round(self.width * factor))),
                                max(1, int(round(self.height * factor))))


@dataclass
class Surfel:
    """One 2D Gaussian primitive (disk spanned by the first two rotation axes)."""

    mean: np.ndarray
    rotation: UnitQuaternion
    scale: np.ndarray
    opacity: float
    color: np.ndarray
    confidence: float = 1.0
    keyframe_id: int = -1
    submap_id: int = -1

    def __post_init__(self):
        # rasterizer.py:62-68
        self.mean = np.asarray(self.mean, dtype=float)
        self.scale = np.asarray(self.scale, dtype=float)
        self.color = np.asarray(self.color, dtype=float)
        self.opacity = float(min(1.0, max(0.0, self.opacity)))
        if np.any(self.scale <= 0):
            raise ValueError("surfel scale components must be positive")


_FIELDS = ("means", "quats", "scales", "opacities", "colors", "confidences", "keyframe_ids",
           "submap_ids")


@dataclass
class SurfelArrays:
    """Structure-of-arrays surfel storage (rasterizer.py:71-147)."""

    means: np.ndarray
    quats: np.ndarray
    scales: np.ndarray
    opacities: np.ndarray
    colors: np.ndarray
    confidences: np.ndarray = None
    keyframe_ids: np.ndarray = None
    submap_ids: np.ndarray = None

    def __post_init__(self):
        n = len(np.asarray(self.means).reshape(-1, 3))
        if self.confidences is None:
            self.confidences = np.ones(n)
        if self.keyframe_ids is None:
            self.keyframe_ids = np.full(n, -1, np.int64)
        if self.submap_ids is None:
            self.submap_ids = np.full(n, -1, np.int64)

    def __len__(self):
        return np.asarray(self.means).reshape(-1, 3).shape[0]

    @classmethod
    def empty(cls):
        return cls(np.empty((0, 3)), np.empty((0, 4)), np.empty((0, 2)), np.empty(0), np.empty((0, 3)),
                   np.empty(0), np.empty(0, np.int64), np.empty(0, np.int64))

    @classmethod
    def from_surfels(cls, surfels) -> "SurfelArrays":
        if isinstance(surfels, SurfelArrays):
            return surfels
        if all(hasattr(surfels, f) for f in ("means", "quats", "scales", "opacities", "colors")):
            # the reference's own SurfelArrays (or any SoA twin)
            return cls(*[getattr(surfels, f, None) for f in _FIELDS])
        surfels = list(surfels)
        if not surfels:
            return cls.empty()
        return cls(
            np.stack([s.mean for s in surfels]),
            np.stack([np.asarray(s.rotation.array(), dtype=float) for s in surfels]),
            np.stack([s.scale for s in surfels]),
            np.array([s.opacity for s in surfels]),
            np.stack([s.color for s in surfels]),
            np.array([s.confidence for s in surfels]),
            np.array([s.keyframe_id for s in surfels], dtype=np.int64),
            np.array([s.submap_id for s in surfels], dtype=np.int64),
        )

    def to_surfels(self):
        return [Surfel(self.means[i], UnitQuaternion.from_array(self.quats[i]), self.scales[i],
                       float(self.opacities[i]), self.colors[i], float(self.confidences[i]),
                       int(self.keyframe_ids[i]), int(self.submap_ids[i])) for i in range(len(self))]

    def select(self, idx) -> "SurfelArrays":
        return SurfelArrays(*[np.asarray(getattr(self, f))[idx] for f in _FIELDS])

    @classmethod
    def concatenate(cls, parts):
        parts = [p for p in parts if len(p)]
        if not parts:
            return cls.empty()
        return cls(*[np.concatenate([getattr(p, f) for p in parts]) for f in _FIELDS])

    def copy(self) -> "SurfelArrays":
        return SurfelArrays(*[np.array(getattr(self, f), copy=True) for f in _FIELDS])


@dataclass(frozen=True)
class RasterConfig:
    """Rendering policy knobs (rasterizer.py:150-168).

    ``splat_mode`` is new: "affine" (default) is the reference's footprint model and the
    only one parity is claimed for; "ray" evaluates the exact ray / surfel-plane
    intersection (2D-Gaussian-splatting homography) and blends the per-pixel intersection
    depth (no reference counterpart)."""

    weight_clamp: float = 0.999
    termination_transmittance: float = 1e-4
    footprint_sigma: float = 3.0
    near_plane: float = 1e-3
    max_condition: float = 1e8
    max_view_angle_deg: float = 80.0
    center_margin_frac: float = 0.5
    splat_mode: str = "affine"

    def __post_init__(self):
        if self.splat_mode not in ("affine", "ray"):
            raise ValueError("splat_mode must be 'affine' or 'ray'")


DEFAULT_RASTER_CONFIG = RasterConfig()


@dataclass
class RenderBuffers:
    color: np.ndarray         # (H, W, 3)
    depth: np.ndarray         # (H, W) alpha-blended expected depth
    accumulation: np.ndarray  # (H, W)
    degenerate_skipped: int = 0
    normal: np.ndarray = field(default=None)  # (H, W, 3) camera-frame normal (new channel)


@dataclass(frozen=True)
class SurfelFootprint:
    center: np.ndarray
    covariance: np.ndarray
    z: float


@dataclass(frozen=True)
class LossWeights:
    mse: float = 1.0
    depth: float = 0.05


def _n(arrays) -> int:
    return len(np.asarray(arrays.means).reshape(-1, 3))


def _device_render(surfels, pose, intr, config, normal=True, argmax=False, max_weights=False,
                   mask=None):
    arrays = SurfelArrays.from_surfels(surfels)
    ctx = DeviceContext.get()
    dev = ctx.device
    n = _n(arrays)
    params = pack_params(arrays, dev) if n else torch.zeros(13, device=dev)
    img = ImageBuffers.allocate(intr.height, intr.width, dev, normal=normal, argmax=argmax)
    view = ctx.thread_view()
    cam = camera_struct(intr)
    cfg = config_struct(config)
    max_all = max_marked = mask_t = None
    if max_weights:
        max_all = torch.zeros(max(n, 1), device=dev)
        max_marked = torch.zeros(max(n, 1), device=dev)
        if mask is not None:
            mask_t = torch.from_numpy(np.ascontiguousarray(np.asarray(mask).astype(np.uint8))).to(dev)
    st = forward_checked(view, params, n, as_packed_pose(pose), cam, cfg, img, max_all, max_marked, mask_t)
    return arrays, params, img, st, view, (max_all, max_marked)


def _np64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def render(surfels, pose, intr: CameraIntrinsics, config: RasterConfig = DEFAULT_RASTER_CONFIG) -> RenderBuffers:
    """Alpha-blend surfels into color/depth/accumulation (+normal) buffers."""
    _, _, img, st, _, _ = _device_render(surfels, pose, intr, config)
    return RenderBuffers(_np64(img.color), _np64(img.depth), _np64(img.accumulation), int(st.degenerate),
                         _np64(img.normal))


def render_with_argmax(surfels, pose, intr, config=DEFAULT_RASTER_CONFIG):
    """Render plus the per-pixel input index of the max-blending-weight surfel (-1 if none)."""
    _, _, img, st, _, _ = _device_render(surfels, pose, intr, config, argmax=True)
    buf = RenderBuffers(_np64(img.color), _np64(img.depth), _np64(img.accumulation), int(st.degenerate),
                        _np64(img.normal))
    return buf, img.arg_w.cpu().numpy().astype(np.int64), _np64(img.max_w)


def render_loss(buffers: RenderBuffers, target_rgb, target_depth, weights: LossWeights = LossWeights()) -> float:
    """``mse * MSE(rgb) + depth * MSE(depth over accumulation > 0.5 pixels)`` (rasterizer.py:346-357)."""
    target_rgb = np.asarray(target_rgb, dtype=float)
    target_depth = np.asarray(target_depth, dtype=float)
    if target_rgb.shape != buffers.color.shape or target_depth.shape != buffers.depth.shape:
        raise ValueError("target dimensions do not match render buffers")
    loss = weights.mse * float(np.mean((buffers.color - target_rgb) ** 2))
    mask = buffers.accumulation > 0.5
    if weights.depth != 0.0 and np.any(mask):
        loss += weights.depth * float(np.mean((buffers.depth[mask] - target_depth[mask]) ** 2))
    return loss


def _targets(intr, target_rgb, target_depth, dev):
    target_rgb = np.asarray(target_rgb, dtype=float)
    target_depth = np.asarray(target_depth, dtype=float)
    if target_rgb.shape != (intr.height, intr.width, 3) or target_depth.shape != (intr.height, intr.width):
        raise ValueError("target dimensions do not match render buffers")
    return (torch.from_numpy(target_rgb.astype(np.float32)).to(dev),
            torch.from_numpy(target_depth.astype(np.float32)).to(dev))


def loss_struct(kind, weights_rgb, weights_depth, depth_mask, trgb, tdepth) -> N.Loss:
    return N.Loss(int(kind), int(depth_mask), float(weights_rgb), float(weights_depth), N.dptr(trgb),
                  N.dptr(tdepth), None, None, None, None)


def grad_all(surfels, pose, intr, target_rgb, target_depth, kind="mse", w_rgb=1.0, w_depth=0.05,
             depth_mask=True, config: RasterConfig = DEFAULT_RASTER_CONFIG):
    """Gradients of the loss w.r.t. ALL surfel parameters (new: geometry included).

    Returns (dict of numpy float64 arrays keyed like SurfelArrays fields, loss).
    """
    arrays, params, img, st, view, _ = _device_render(surfels, pose, intr, config)
    dev = params.device
    n = _n(arrays)
    trgb, tdepth = _targets(intr, target_rgb, target_depth, dev)
    grads = torch.zeros_like(params)
    loss_acc = torch.zeros(1, dtype=torch.float64, device=dev)
    k = N.LOSS_MSE if kind == "mse" else N.LOSS_L1
    view.backward(params, n, img, loss_struct(k, w_rgb, w_depth, depth_mask, trgb, tdepth), grads, loss_acc)
    g = {name: t.detach().cpu().numpy().astype(np.float64) for name, t in unpack_params(grads, n).items()} if n \
        else {name: np.zeros((0,) + ((k,) if k > 1 else ())) for name, k in
              (("means", 3), ("quats", 4), ("scales", 2), ("opacities", 1), ("colors", 3))}
    return g, float(loss_acc.item())


def grad_color_opacity(surfels, pose, intr, target_rgb, target_depth,
                       weights: LossWeights = LossWeights(),
                       config: RasterConfig = DEFAULT_RASTER_CONFIG):
    """d(render_loss)/d(color, opacity) (rasterizer.py:360-399): ``(grad_color (N,3), grad_opacity (N,), loss)``.

    The accumulation>0.5 depth mask is taken at the current state and held fixed.
    Culled or degenerate surfels get zero gradients.  The loss is computed by the
    fused backward kernel (float32 per pixel, float64 accumulation).
    """
    g, loss = grad_all(surfels, pose, intr, target_rgb, target_depth, "mse", weights.mse, weights.depth,
                       True, config)
    return g["colors"].reshape(-1, 3), g["opacities"].reshape(-1), loss


def per_surfel_max_weight(surfels, pose, intr, mask=None, config: RasterConfig = DEFAULT_RASTER_CONFIG):
    """Max per-pixel blending weight of each surfel, overall and over a pixel mask."""
    arrays = SurfelArrays.from_surfels(surfels)
    n = _n(arrays)
    if n == 0:
        return np.zeros(0), np.zeros(0)
    _, _, _, _, _, (max_all, max_marked) = _device_render(arrays, pose, intr, config, normal=False,
                                                          max_weights=True, mask=mask)
    return _np64(max_all[:n]), _np64(max_marked[:n])


def project_surfel(surfel: Surfel, pose, intr: CameraIntrinsics, config: RasterConfig = DEFAULT_RASTER_CONFIG):
    """Screen footprint of one surfel, or None when frustum-culled (host float64 utility).

    Restates _project_batch (rasterizer.py:201-236) for a single surfel; the device
    path computes the same quantities inside the projection kernel.
    """
    inv = pk_inverse(as_packed_pose(pose))
    mean = np.asarray(surfel.mean, dtype=float)
    from .geometry import quat_rotate
    p = inv[0] * quat_rotate(inv[4:8], mean) + inv[1:4]
    z = p[2]
    tan_max = np.tan(np.radians(config.max_view_angle_deg))
    if not (z > config.near_plane and np.hypot(p[0], p[1]) <= tan_max * z):
        return None
    rot = quat_to_matrix(np.asarray(surfel.rotation.array(), dtype=float))
    basis = rot[:, :2] * np.asarray(surfel.scale, dtype=float)[None, :]
    m_cw = inv[0] * quat_to_matrix(inv[4:8])
    bc = m_cw @ basis
    cov_cam = bc @ bc.T
    jac = np.array([[intr.fx / z, 0.0, -intr.fx * p[0] / z ** 2], [0.0, intr.fy / z, -intr.fy * p[1] / z ** 2]])
    cov2 = jac @ cov_cam @ jac.T
    cov2 = 0.5 * (cov2 + cov2.T)
    center = np.array([intr.fx * p[0] / z + intr.cx, intr.fy * p[1] / z + intr.cy])
    mx, my = config.center_margin_frac * intr.width, config.center_margin_frac * intr.height
    if not (-mx <= center[0] <= intr.width - 1 + mx and -my <= center[1] <= intr.height - 1 + my):
        return None
    return SurfelFootprint(center, cov2, float(z))
