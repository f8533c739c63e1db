"""Seeded synthetic workloads of BASELINE.json configs 1-5.

The paper's datasets are not available; these generators reproduce the
configs' shapes, sizes and value distributions.  All parameters are drawn in
float64 with ``numpy.random.default_rng(seed)`` in a fixed order and then
rounded to float32, so the GPU (float32) and the CPU oracle (float64) see
identical values.  Assumptions the configs leave open are marked [A] and
listed in DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import (Sim3Transform, UnitQuaternion, quat_canonicalize, quat_from_axis_angle,
                       quat_from_matrix, quat_mul, pk_act)
from .rasterizer import CameraIntrinsics, SurfelArrays

__all__ = ["Scene", "config1", "config2", "config3", "config4", "config5", "random_surfels",
           "depth_field_surfels", "f32"]


def f32(a):
    """Round to float32 and back (the values both sides compute on)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@dataclass
class Scene:
    surfels: SurfelArrays
    intr: CameraIntrinsics
    poses: list                      # camera->world Sim3Transform per view
    name: str = ""
    targets: list = field(default_factory=list)   # optional per-view (rgb, depth)
    gains: np.ndarray | None = None  # per-view exposure gain (config 5)
    extra: dict = field(default_factory=dict)


def _arrays(means, quats, scales, opac, colors):
    n = len(means)
    return SurfelArrays(f32(means), f32(quats), f32(scales), f32(opac), f32(colors), np.ones(n),
                        np.zeros(n, np.int64), np.zeros(n, np.int64))


def random_surfels(rng, n):
    """Config-1 distributions: x,y~U[-1,1], z~U[1,5]; scales log-U[.005,.05];
    uniform random unit quaternions; opacity sigmoid(N(0,1)); rgb U[0,1]."""
    means = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(1, 5, n)], axis=1)
    scales = np.exp(rng.uniform(np.log(0.005), np.log(0.05), (n, 2)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    opac = 1.0 / (1.0 + np.exp(-rng.normal(size=n)))
    colors = rng.uniform(0, 1, (n, 3))
    return _arrays(means, q, scales, opac, colors)


def config1(seed: int = 0) -> Scene:
    rng = np.random.default_rng(seed)
    s = random_surfels(rng, 2000)
    intr = CameraIntrinsics(100.0, 100.0, 64.0, 48.0, 128, 96)
    return Scene(s, intr, [Sim3Transform.identity()], "config1")


def perturbed(surfels: SurfelArrays, rng, mean_sigma=0.01, color_sigma=0.05) -> SurfelArrays:
    out = surfels.copy()
    n = len(out)
    out.means = f32(out.means + rng.normal(0, mean_sigma, (n, 3)))
    out.colors = f32(np.clip(out.colors + rng.normal(0, color_sigma, (n, 3)), 0, 1))  # [A] clip
    return out


def config2(seed: int = 0) -> Scene:
    """20k surfels, 320x240, fx=fy=250 ([A] cx=160, cy=120).  scene.extra['target_surfels'] is the
    perturbed copy whose render is the target (means + N(0,.01), rgb + N(0,.05))."""
    rng = np.random.default_rng(seed)
    s = random_surfels(rng, 20000)
    intr = CameraIntrinsics(250.0, 250.0, 160.0, 120.0, 320, 240)
    tgt = perturbed(s, rng)
    return Scene(s, intr, [Sim3Transform.identity()], "config2", extra={"target_surfels": tgt})


def _depth_field(rng, w, h, lo=0.5, hi=6.0, k=8):
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
    d = np.zeros((h, w))
    for _ in range(k):
        fx_, fy_ = rng.uniform(-2, 2, 2)       # [A] cycles per image
        a = rng.uniform(0.5, 1.0)
        ph = rng.uniform(0, 2 * np.pi)
        d += a * np.sin(2 * np.pi * (fx_ * xs / w + fy_ * ys / h) + ph)
    d = (d - d.min()) / max(d.max() - d.min(), 1e-12)
    return lo + (hi - lo) * d


def depth_field_surfels(rng, intr: CameraIntrinsics):
    """Pixel-aligned surfels of one keyframe (config 3): one per pixel of a smooth random
    depth map, oriented to the local depth-gradient normal, facing the camera (camera frame)."""
    w, h = intr.width, intr.height
    depth = _depth_field(rng, w, h)
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
    pts = np.stack([(xs - intr.cx) / intr.fx * depth, (ys - intr.cy) / intr.fy * depth, depth], axis=-1)
    t1 = np.gradient(pts, axis=1)
    t2 = np.gradient(pts, axis=0)
    nrm = np.cross(t1, t2)
    nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
    flip = np.sum(nrm * pts, axis=-1) > 0
    nrm[flip] = -nrm[flip]
    a = t1 - np.sum(t1 * nrm, axis=-1, keepdims=True) * nrm
    a /= np.linalg.norm(a, axis=-1, keepdims=True)
    b = np.cross(nrm, a)
    R = np.stack([a, b, nrm], axis=-1).reshape(-1, 3, 3)
    q = quat_from_matrix(R)
    n = w * h
    scales = (depth.reshape(-1, 1) / intr.fx) * rng.uniform(0.8, 1.5, (n, 2))
    opac = rng.uniform(0.5, 1.0, n)
    colors = rng.uniform(0, 1, (n, 3))
    return _arrays(pts.reshape(-1, 3), q, scales, opac, colors), depth


def _small_pose(rng, max_deg=5.0, max_t=0.2):
    axis = rng.normal(size=3)
    ang = np.radians(rng.uniform(0, max_deg))
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    t = d * rng.uniform(0, max_t)
    return Sim3Transform(1.0, UnitQuaternion.from_array(quat_from_axis_angle(axis, ang)), t)


def config3(seed: int = 0) -> Scene:
    """One 512x384 keyframe -> 196,608 pixel-aligned surfels; 8 nearby poses
    ([A] fx=fy=400, cx=256, cy=192; rotations <=5 deg, translations <=0.2 m)."""
    rng = np.random.default_rng(seed)
    intr = CameraIntrinsics(400.0, 400.0, 256.0, 192.0, 512, 384)
    s, _ = depth_field_surfels(rng, intr)
    poses = [_small_pose(rng) for _ in range(8)]
    return Scene(s, intr, poses, "config3")


def _trajectory_pose(t, rng=None, jitter=0.0, jitter_deg=0.0):
    """Smooth camera->world path: forward along z with lateral sway and yaw."""
    pos = np.array([0.6 * np.sin(2 * np.pi * 0.5 * t), 0.15 * np.sin(2 * np.pi * t), 1.2 * t])
    yaw = np.radians(12.0) * np.sin(2 * np.pi * 0.5 * t)
    pitch = np.radians(4.0) * np.sin(2 * np.pi * t + 0.3)
    q = quat_mul(quat_from_axis_angle([0, 1.0, 0], yaw), quat_from_axis_angle([1.0, 0, 0], pitch))
    if rng is not None and (jitter or jitter_deg):
        pos = pos + rng.normal(0, jitter, 3)
        q = quat_mul(q, quat_from_axis_angle(rng.normal(size=3), np.radians(rng.uniform(0, jitter_deg))))
    return Sim3Transform(1.0, UnitQuaternion.from_array(q), pos)


def transform_surfels(s: SurfelArrays, t: Sim3Transform) -> SurfelArrays:
    """Camera -> world as the reference's transform_surfels (mapper.py:184-197)."""
    q = t.rotation.array()
    return SurfelArrays(pk_act(t.packed(), s.means), quat_canonicalize(quat_mul(q[None, :], s.quats)),
                        t.scale * s.scales, s.opacities.copy(), s.colors.copy(), s.confidences.copy(),
                        s.keyframe_ids.copy(), s.submap_ids.copy())


def config4(seed: int = 0, n_keyframes: int = 8, per_keyframe: int = 125_000, n_views: int = 32,
            view_size=(640, 480), focal=500.0) -> Scene:
    """1,000,000 surfels from 8 config-3 keyframes fused in world frame ([A] seeded uniform
    subsample of 125,000 per keyframe); 32 training views 640x480, fx=fy=500 on a smooth
    trajectory near the keyframes ([A] cx=320, cy=240).  extra['perturbed'] is the c2-style
    perturbed copy to optimise; targets are renders of the unperturbed map."""
    rng = np.random.default_rng(seed)
    kintr = CameraIntrinsics(400.0, 400.0, 256.0, 192.0, 512, 384)
    parts = []
    kf_poses = []
    for k in range(n_keyframes):
        s, _ = depth_field_surfels(rng, kintr)
        sel = np.sort(rng.choice(len(s), size=per_keyframe, replace=False))
        s = s.select(sel)
        pose = _trajectory_pose(k / max(n_keyframes - 1, 1))
        kf_poses.append(pose)
        w = transform_surfels(s, pose)
        w.keyframe_ids[:] = k
        parts.append(w)
    surfels = SurfelArrays.concatenate(parts)
    for f in ("means", "quats", "scales", "opacities", "colors"):
        setattr(surfels, f, f32(getattr(surfels, f)))
    w_, h_ = view_size
    intr = CameraIntrinsics(focal, focal, w_ / 2.0, h_ / 2.0, w_, h_)
    poses = [_trajectory_pose(j / max(n_views - 1, 1), rng, jitter=0.05, jitter_deg=2.0) for j in range(n_views)]
    pert = perturbed(surfels, rng)
    return Scene(surfels, intr, poses, "config4", extra={"perturbed": pert, "keyframe_poses": kf_poses})


def config5(seed: int = 0, n_surfels: int = 4_000_000, n_views: int = 128) -> Scene:
    """4M surfels in 16 room clusters ([A] 4x4 grid of 4x4x3 m boxes, 1 m gaps), q uniform,
    scale = 3 m / fx x U(.8,1.5), opacity U(.5,1), rgb U; 128 views 1296x968, fx=fy=1000
    ([A] cx=648, cy=484) looking into the rooms; per-view exposure gain U(.7,1.3) on targets."""
    rng = np.random.default_rng(seed)
    fx = 1000.0
    per = n_surfels // 16
    means = []
    for i in range(4):
        for j in range(4):
            lo = np.array([5.0 * i, -3.0, 5.0 * j])
            means.append(lo + rng.uniform(0, 1, (per, 3)) * np.array([4.0, 3.0, 4.0]))
    means = np.concatenate(means)
    n = len(means)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scales = (3.0 / fx) * rng.uniform(0.8, 1.5, (n, 2))
    opac = rng.uniform(0.5, 1.0, n)
    colors = rng.uniform(0, 1, (n, 3))
    surfels = _arrays(means, q, scales, opac, colors)
    intr = CameraIntrinsics(fx, fx, 648.0, 484.0, 1296, 968)
    poses = []
    for v in range(n_views):
        room = v % 16
        i, j = divmod(room, 4)
        centre = np.array([5.0 * i + 2.0, -1.5, 5.0 * j + 2.0])
        ang = 2 * np.pi * (v // 16) / max(n_views // 16, 1) + rng.uniform(-0.1, 0.1)
        pos = centre + 2.6 * np.array([np.cos(ang), 0.0, np.sin(ang)])
        fwd = centre - pos
        fwd /= np.linalg.norm(fwd)
        right = np.cross([0.0, 1.0, 0.0], fwd)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd], axis=1)  # camera axes (x right, y down, z fwd) in world
        poses.append(Sim3Transform(1.0, UnitQuaternion.from_array(quat_from_matrix(R)), pos))
    gains = rng.uniform(0.7, 1.3, n_views)
    pert = perturbed(surfels, rng)
    return Scene(surfels, intr, poses, "config5", gains=gains, extra={"perturbed": pert})
