"""Pose and quaternion value types consumed by the render path.

Only the pieces of the reference's Lie-group layer that feed projection are
restated here (geometry row):

* ``quat_rotate``      — reference ``geometry.py:59-64``
* ``quat_to_matrix``   — reference ``geometry.py:132-142``
* ``pk_inverse``       — reference ``geometry.py:188-195``
* ``SE3Pose.as_sim3``  — reference ``geometry.py:426-427``
* ``Sim3Transform.packed`` — reference ``geometry.py:466-471``

The host-side pose inverse is evaluated in float64 with the same elementwise
operation order as the reference (no fused multiply-adds: numpy ufuncs never
fuse), so the 8 doubles handed to the device are bit-identical to the ones the
reference's ``_project_batch`` computes (``rasterizer.py:204``).

Packed Sim(3) layout: ``[s, tx, ty, tz, qw, qx, qy, qz]``; a pose maps camera
coordinates to world coordinates (camera->world), as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "quat_mul", "quat_conj", "quat_rotate", "quat_to_matrix", "quat_normalize",
    "quat_canonicalize", "quat_from_matrix", "quat_from_axis_angle",
    "pk_inverse", "pk_compose", "pk_act", "UnitQuaternion", "SE3Pose",
    "Sim3Transform", "as_packed_pose",
]


def quat_mul(q1, q2):
    """Hamilton product of (..., 4) wxyz arrays."""
    q1 = np.asarray(q1, dtype=float)
    q2 = np.asarray(q2, dtype=float)
    a, b, c, d = q1[..., 0], q1[..., 1], q1[..., 2], q1[..., 3]
    e, f, g, h = q2[..., 0], q2[..., 1], q2[..., 2], q2[..., 3]
    return np.stack([
        a * e - b * f - c * g - d * h,
        a * f + b * e + c * h - d * g,
        a * g - b * h + c * e + d * f,
        a * h + b * g - c * f + d * e,
    ], axis=-1)


def quat_conj(q):
    out = np.array(q, dtype=float, copy=True)
    out[..., 1:] = -out[..., 1:]
    return out


def _cross(a, b):
    # same association as numpy.cross: each component is one product minus another,
    # each product rounded separately
    a0, a1, a2 = a[..., 0], a[..., 1], a[..., 2]
    b0, b1, b2 = b[..., 0], b[..., 1], b[..., 2]
    return np.stack([a1 * b2 - a2 * b1, a2 * b0 - a0 * b2, a0 * b1 - a1 * b0], axis=-1)


def quat_rotate(q, v):
    """Rotate (..., 3) vectors by (..., 4) quaternions: ``v + 2(w (u x v) + u x (u x v))``.

    Reference ``geometry.py:59-64``; same operation order.
    """
    q = np.asarray(q, dtype=float)
    v = np.asarray(v, dtype=float)
    u = q[..., 1:]
    w = q[..., 0:1]
    uv = _cross(u, v)
    return v + 2.0 * (w * uv + _cross(u, uv))


def quat_to_matrix(q):
    """Rotation matrix of a (possibly non-unit) wxyz quaternion, used raw.

    Reference ``geometry.py:132-142`` (the render path never renormalises,
    ``rasterizer.py:212``).
    """
    q = np.asarray(q, dtype=float)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    r0 = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], axis=-1)
    r1 = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], axis=-1)
    r2 = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], axis=-1)
    return np.stack([r0, r1, r2], axis=-2)


def quat_normalize(q):
    q = np.asarray(q, dtype=float)
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def quat_canonicalize(q):
    """Sign-unique representative with w >= 0 (ties broken on x, y, z)."""
    q = np.asarray(q, dtype=float)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    neg = (w < 0) | ((w == 0) & ((x < 0) | ((x == 0) & ((y < 0) | ((y == 0) & (z < 0))))))
    return np.where(neg[..., None], -q, q) + 0.0


def quat_from_matrix(m):
    """Batched rotation matrix (..., 3, 3) -> unit wxyz quaternion (Shepperd's method)."""
    m = np.asarray(m, dtype=float)
    shape = m.shape[:-2]
    m = m.reshape(-1, 3, 3)
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    diag = np.stack([m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], axis=1)
    cand = np.stack([tr, diag[:, 0], diag[:, 1], diag[:, 2]], axis=1)
    pick = np.argmax(cand, axis=1)
    q = np.empty((m.shape[0], 4))
    # case w largest
    s = np.sqrt(np.maximum(1.0 + tr, 1e-300)) * 2.0
    qw = np.stack([0.25 * s, (m[:, 2, 1] - m[:, 1, 2]) / s, (m[:, 0, 2] - m[:, 2, 0]) / s,
                   (m[:, 1, 0] - m[:, 0, 1]) / s], axis=1)
    sx = np.sqrt(np.maximum(1.0 + m[:, 0, 0] - m[:, 1, 1] - m[:, 2, 2], 1e-300)) * 2.0
    qx = np.stack([(m[:, 2, 1] - m[:, 1, 2]) / sx, 0.25 * sx, (m[:, 0, 1] + m[:, 1, 0]) / sx,
                   (m[:, 0, 2] + m[:, 2, 0]) / sx], axis=1)
    sy = np.sqrt(np.maximum(1.0 + m[:, 1, 1] - m[:, 0, 0] - m[:, 2, 2], 1e-300)) * 2.0
    qy = np.stack([(m[:, 0, 2] - m[:, 2, 0]) / sy, (m[:, 0, 1] + m[:, 1, 0]) / sy, 0.25 * sy,
                   (m[:, 1, 2] + m[:, 2, 1]) / sy], axis=1)
    sz = np.sqrt(np.maximum(1.0 + m[:, 2, 2] - m[:, 0, 0] - m[:, 1, 1], 1e-300)) * 2.0
    qz = np.stack([(m[:, 1, 0] - m[:, 0, 1]) / sz, (m[:, 0, 2] + m[:, 2, 0]) / sz,
                   (m[:, 1, 2] + m[:, 2, 1]) / sz, 0.25 * sz], axis=1)
    for k, cand_q in enumerate((qw, qx, qy, qz)):
        sel = pick == k
        q[sel] = cand_q[sel]
    q = quat_canonicalize(quat_normalize(q))
    return q.reshape(shape + (4,))


def quat_from_axis_angle(axis, angle):
    axis = np.asarray(axis, dtype=float)
    axis = axis / np.linalg.norm(axis, axis=-1, keepdims=True)
    angle = np.asarray(angle, dtype=float)
    half = 0.5 * angle
    return np.concatenate([np.cos(half)[..., None], np.sin(half)[..., None] * axis], axis=-1)


def pk_inverse(a):
    """Inverse of packed Sim(3) ``[s, t, q]``: ``[1/s, -(1/s) q* t, q*]``.

    Reference ``geometry.py:188-195``; same operation order so the result is
    bit-identical.
    """
    a = np.asarray(a, dtype=float)
    out = np.empty_like(a)
    s_inv = 1.0 / a[..., 0]
    qc = quat_conj(a[..., 4:8])
    out[..., 0] = s_inv
    out[..., 1:4] = -s_inv[..., None] * quat_rotate(qc, a[..., 1:4])
    out[..., 4:8] = qc
    return out


def pk_compose(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    out = np.empty(np.broadcast_shapes(a.shape, b.shape))
    out[..., 0] = a[..., 0] * b[..., 0]
    out[..., 1:4] = a[..., 0, None] * quat_rotate(a[..., 4:8], b[..., 1:4]) + a[..., 1:4]
    out[..., 4:8] = quat_mul(a[..., 4:8], b[..., 4:8])
    return out


def pk_act(a, p):
    a = np.asarray(a, dtype=float)
    return a[..., 0, None] * quat_rotate(a[..., 4:8], np.asarray(p, dtype=float)) + a[..., 1:4]


@dataclass(frozen=True)
class UnitQuaternion:
    """Hamilton unit quaternion (w, x, y, z); normalised on construction."""

    w: float
    x: float
    y: float
    z: float

    def __post_init__(self):
        n = math.sqrt(self.w * self.w + self.x * self.x + self.y * self.y + self.z * self.z)
        if not math.isfinite(n) or n == 0.0:
            raise ValueError("quaternion must be finite and non-zero")
        if abs(n - 1.0) > 1e-12:
            for k in ("w", "x", "y", "z"):
                object.__setattr__(self, k, getattr(self, k) / n)

    @classmethod
    def identity(cls):
        return cls(1.0, 0.0, 0.0, 0.0)

    @classmethod
    def from_array(cls, q):
        return cls(float(q[0]), float(q[1]), float(q[2]), float(q[3]))

    @classmethod
    def from_axis_angle(cls, axis, angle):
        return cls.from_array(quat_from_axis_angle(axis, angle))

    @classmethod
    def from_matrix(cls, m):
        return cls.from_array(quat_from_matrix(m))

    def array(self):
        return np.array([self.w, self.x, self.y, self.z])

    def conjugate(self):
        return UnitQuaternion(self.w, -self.x, -self.y, -self.z)

    def __mul__(self, other):
        return UnitQuaternion.from_array(quat_mul(self.array(), other.array()))

    def rotate(self, v):
        return quat_rotate(self.array(), np.asarray(v, dtype=float))

    def matrix(self):
        return quat_to_matrix(self.array())


@dataclass(frozen=True)
class SE3Pose:
    """Rigid transform x -> R x + t (camera -> world when used as a view pose)."""

    rotation: UnitQuaternion
    translation: np.ndarray

    def __post_init__(self):
        t = np.array(self.translation, dtype=float)
        if t.shape != (3,):
            raise ValueError("translation must be a 3-vector")
        object.__setattr__(self, "translation", t)

    @classmethod
    def identity(cls):
        return cls(UnitQuaternion.identity(), np.zeros(3))

    def as_sim3(self) -> "Sim3Transform":
        return Sim3Transform(1.0, self.rotation, self.translation)

    def compose(self, other: "SE3Pose") -> "SE3Pose":
        return SE3Pose(self.rotation * other.rotation,
                       self.rotation.rotate(other.translation) + self.translation)

    def inverse(self) -> "SE3Pose":
        qc = self.rotation.conjugate()
        return SE3Pose(qc, -qc.rotate(self.translation))

    def act(self, p):
        return self.rotation.rotate(np.asarray(p, dtype=float)) + self.translation

    def __matmul__(self, other):
        return self.compose(other)


@dataclass(frozen=True)
class Sim3Transform:
    """Similarity x -> s R x + t."""

    scale: float
    rotation: UnitQuaternion
    translation: np.ndarray

    def __post_init__(self):
        if not (self.scale > 0 and math.isfinite(self.scale)):
            raise ValueError(f"scale must be positive and finite, got {self.scale}")
        t = np.array(self.translation, dtype=float)
        if t.shape != (3,):
            raise ValueError("translation must be a 3-vector")
        object.__setattr__(self, "translation", t)

    @classmethod
    def identity(cls):
        return cls(1.0, UnitQuaternion.identity(), np.zeros(3))

    @classmethod
    def from_packed(cls, a):
        a = np.asarray(a, dtype=float)
        return cls(float(a[0]), UnitQuaternion.from_array(a[4:8]), a[1:4])

    def packed(self):
        out = np.empty(8)
        out[0] = self.scale
        out[1:4] = self.translation
        out[4:8] = self.rotation.array()
        return out

    def compose(self, other: "Sim3Transform") -> "Sim3Transform":
        return Sim3Transform.from_packed(pk_compose(self.packed(), other.packed()))

    def inverse(self) -> "Sim3Transform":
        return Sim3Transform.from_packed(pk_inverse(self.packed()))

    def act(self, p):
        return pk_act(self.packed(), p)

    def __matmul__(self, other):
        return self.compose(other)


def as_packed_pose(pose) -> np.ndarray:
    """Packed camera->world Sim(3) of any pose-like object.

    Accepts this module's ``SE3Pose``/``Sim3Transform``, the reference's own
    classes (duck-typed through ``as_sim3()``/``packed()``, mirroring
    ``rasterizer._as_camera_packed`` ``rasterizer.py:195-198``) or a raw (8,) array.
    """
    if hasattr(pose, "as_sim3"):
        pose = pose.as_sim3()
    if hasattr(pose, "packed"):
        return np.asarray(pose.packed(), dtype=float)
    a = np.asarray(pose, dtype=float)
    if a.shape != (8,):
        raise TypeError("pose must be SE3Pose, Sim3Transform or a packed (8,) array")
    return a
