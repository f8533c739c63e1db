"""Surfel PLY I/O: drop-in for ``surfelslam.io.write_surfel_ply`` /
``read_surfel_ply`` (io.py:118-190), the on-disk map format the reference's render and
evaluate commands read.

Binary little-endian PLY, one vertex per surfel, float64 throughout (so round trips are
exact) plus int32 keyframe / submap ids.  The written normal is the third column of the
surfel's rotation matrix, as in the reference.  Host-side code: it moves bytes between a
file and :class:`~paper_2604_03092_b200.rasterizer.SurfelArrays`.
"""

from __future__ import annotations

import numpy as np

from .geometry import quat_to_matrix
from .rasterizer import SurfelArrays

__all__ = ["write_surfel_ply", "read_surfel_ply", "PLY_FIELDS"]

# vertex layout, in file order (io.py:121-130)
PLY_FIELDS = [
    ("x", "<f8"), ("y", "<f8"), ("z", "<f8"),
    ("nx", "<f8"), ("ny", "<f8"), ("nz", "<f8"),
    ("qw", "<f8"), ("qx", "<f8"), ("qy", "<f8"), ("qz", "<f8"),
    ("sx", "<f8"), ("sy", "<f8"),
    ("opacity", "<f8"),
    ("red", "<f8"), ("green", "<f8"), ("blue", "<f8"),
    ("confidence", "<f8"),
    ("kf_id", "<i4"), ("submap_id", "<i4"),
]
_TYPE_NAME = {"<f8": "double", "<i4": "int"}
_NAME_TYPE = {"double": "<f8", "float": "<f4", "int": "<i4"}
_REQUIRED = {"x", "y", "z", "qw", "qx", "qy", "qz", "sx", "sy", "opacity", "red", "green", "blue"}


def _normals(quats: np.ndarray) -> np.ndarray:
    if len(quats) == 0:
        return np.empty((0, 3))
    return quat_to_matrix(quats)[:, :, 2]


def write_surfel_ply(path, surfels) -> None:
    """Write ``surfels`` (SurfelArrays or list of Surfel) to ``path``."""
    s = SurfelArrays.from_surfels(surfels)
    n = len(s)
    v = np.empty(n, dtype=PLY_FIELDS)
    means = np.asarray(s.means, dtype=float).reshape(-1, 3)
    quats = np.asarray(s.quats, dtype=float).reshape(-1, 4)
    for k, name in enumerate(("x", "y", "z")):
        v[name] = means[:, k]
    nrm = _normals(quats)
    for k, name in enumerate(("nx", "ny", "nz")):
        v[name] = nrm[:, k]
    for k, name in enumerate(("qw", "qx", "qy", "qz")):
        v[name] = quats[:, k]
    scales = np.asarray(s.scales, dtype=float).reshape(-1, 2)
    v["sx"], v["sy"] = scales[:, 0], scales[:, 1]
    v["opacity"] = np.asarray(s.opacities, dtype=float)
    cols = np.asarray(s.colors, dtype=float).reshape(-1, 3)
    for k, name in enumerate(("red", "green", "blue")):
        v[name] = cols[:, k]
    v["confidence"] = np.asarray(s.confidences, dtype=float)
    v["kf_id"] = np.asarray(s.keyframe_ids)
    v["submap_id"] = np.asarray(s.submap_ids)
    lines = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    lines += [f"property {_TYPE_NAME[t]} {name}" for name, t in PLY_FIELDS]
    lines.append("end_header")
    with open(path, "wb") as f:
        f.write(("\n".join(lines) + "\n").encode("ascii"))
        f.write(v.tobytes())


def read_surfel_ply(path) -> SurfelArrays:
    """Read a surfel PLY (any property order; float/double/int properties).  ValueError on
    a non-PLY file, an unterminated header or missing surfel properties."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ValueError(f"{path} is not a PLY file")
        n = None
        props = []
        while True:
            raw = f.readline()
            if not raw:
                raise ValueError("unterminated PLY header")
            line = raw.decode("ascii").strip()
            if line == "end_header":
                break
            words = line.split()
            if words[:2] == ["element", "vertex"]:
                n = int(words[-1])
            elif words and words[0] == "property":
                props.append((words[2], _NAME_TYPE[words[1]]))
        data = np.fromfile(f, dtype=props, count=n)
    names = {name for name, _ in props}
    if not _REQUIRED <= names:
        raise ValueError(f"PLY missing surfel properties: {sorted(_REQUIRED - names)}")
    m = len(data)

    def cols(*fields):
        return np.stack([data[x].astype(float) for x in fields], axis=1)

    return SurfelArrays(
        cols("x", "y", "z"), cols("qw", "qx", "qy", "qz"), cols("sx", "sy"),
        data["opacity"].astype(float), cols("red", "green", "blue"),
        data["confidence"].astype(float) if "confidence" in names else np.ones(m),
        data["kf_id"].astype(np.int64) if "kf_id" in names else np.full(m, -1, np.int64),
        data["submap_id"].astype(np.int64) if "submap_id" in names else np.full(m, -1, np.int64),
    )
