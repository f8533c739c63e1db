"""The ray-splat oracle (oracle/raysplat.py) on the CPU: its homography form of the
ray / surfel-plane intersection against the first-principles intersection, and its
render's basic invariants.  The mode has no reference counterpart."""
import numpy as np
import pytest
import torch

import oracle.raysplat as RS
from oracle import DEFAULTS
from oracle.oracle import pose_inverse
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.geometry import Sim3Transform, UnitQuaternion, quat_to_matrix


def _axes(s, i, pose):
    inv, m_cw, _ = pose_inverse(pose)
    R = quat_to_matrix(np.asarray(s.quats[i], float))
    a = m_cw @ R[:, 0] * s.scales[i, 0]
    b = m_cw @ R[:, 1] * s.scales[i, 1]
    p = m_cw @ s.means[i] + inv[1:4]
    return a, b, p


def test_homography_equals_ray_plane_intersection():
    sc = scenes.config1(0)
    pose = Sim3Transform(1.2, UnitQuaternion.from_axis_angle([0.2, 1.0, 0.1], 0.3), np.array([0.1, -0.2, 0.3]))
    rng = np.random.default_rng(0)
    K = np.array([[sc.intr.fx, 0, sc.intr.cx], [0, sc.intr.fy, sc.intr.cy], [0, 0, 1.0]])
    for i in rng.choice(len(sc.surfels), 50, replace=False):
        a, b, p = _axes(sc.surfels, i, pose)
        Hi = np.linalg.inv(K @ np.stack([a, b, p], 1))
        for px, py in rng.uniform(0, [128, 96], (5, 2)):
            U, V, S = Hi @ [px, py, 1.0]
            u, v, lam = RS.intersect_uv(a, b, p, sc.intr, px, py)
            assert np.allclose([U / S, V / S, 1 / S], [u, v, lam], rtol=1e-9, atol=1e-9)


def test_ray_render_invariants_and_autograd():
    sc = scenes.config1(0)
    sub = sc.surfels.select(np.arange(300))
    pr = RS.params_from_arrays(sub)
    out = RS.render_ray(pr, sc.poses[0], sc.intr)
    acc = out["accumulation"].detach().numpy()
    assert acc.min() >= 0 and acc.max() < 1
    assert out["on"].sum() > 250
    # depth / accumulation is a convex combination of intersection depths: within the scene's z range
    d = out["depth"].detach().numpy()
    m = acc > 0.05
    assert np.all(d[m] / acc[m] > 0.5) and np.all(d[m] / acc[m] < 6.0)
    loss = out["color"].sum() + out["depth"].sum()
    loss.backward()
    for k in ("means", "quats", "scales", "opacities", "colors"):
        g = pr[k].grad
        assert g is not None and torch.isfinite(g).all() and g.abs().max() > 0, k
