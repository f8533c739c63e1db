"""Generate golden vectors by running the REFERENCE itself (surfelslam, /root/reference).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Inputs are produced by this repo's seeded generators (paper_2604_03092_b200.scenes)
and by small hand-built known-answer scenes; outputs come from the reference's
public functions (rasterizer._project_batch, _footprint_boxes, render,
render_with_argmax, grad_color_opacity, per_surfel_max_weight) and are stored
as .npz next to this script.  Nothing here is copied from the reference: it is
only called.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from surfelslam import rasterizer as R  # noqa: E402  (the reference)
from surfelslam.geometry import Sim3Transform, UnitQuaternion, SE3Pose  # noqa: E402

from paper_2604_03092_b200 import scenes  # noqa: E402


def ref_arrays(s):
    n = len(s.means)
    return R.SurfelArrays(np.asarray(s.means, float), np.asarray(s.quats, float), np.asarray(s.scales, float),
                          np.asarray(s.opacities, float), np.asarray(s.colors, float), np.ones(n),
                          np.zeros(n, np.int64), np.zeros(n, np.int64))


def ref_intr(i):
    return R.CameraIntrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height)


def ref_pose(p):
    return Sim3Transform(float(p.scale), UnitQuaternion.from_array(p.rotation.array()), np.asarray(p.translation))


def capture(name, surf, pose, intr, cfg=R.DEFAULT_RASTER_CONFIG, images_f32=False, grads=True, seed=0,
            extra=None):
    arr = ref_arrays(surf)
    ri = ref_intr(intr)
    centers, cov2, inv_abc, z, valid, degenerate, in_front = R._project_batch(arr, pose, ri, cfg)
    bbox, on_screen = R._footprint_boxes(centers, inv_abc, valid, ri, cfg.footprint_sigma)
    keep = np.flatnonzero(on_screen)
    order = keep[np.lexsort((keep, z[keep]))]
    buf, arg_w, max_w = R.render_with_argmax(arr, pose, ri, cfg)
    out = dict(
        means=arr.means, quats=arr.quats, scales=arr.scales, opacities=arr.opacities, colors=arr.colors,
        pose=np.asarray(pose.as_sim3().packed() if hasattr(pose, "as_sim3") else pose.packed()),
        intr=np.array([ri.fx, ri.fy, ri.cx, ri.cy, ri.width, ri.height], float),
        cfg=np.array([cfg.weight_clamp, cfg.termination_transmittance, cfg.footprint_sigma, cfg.near_plane,
                      cfg.max_condition, cfg.max_view_angle_deg, cfg.center_margin_frac]),
        centers=centers, cov2=np.stack([cov2[:, 0, 0], cov2[:, 0, 1], cov2[:, 1, 1]], 1), inv_abc=inv_abc, z=z,
        valid=valid, in_front=in_front, degenerate=np.int64(degenerate), bbox=bbox, on_screen=on_screen,
        order=order, arg_w=arg_w, degenerate_skipped=np.int64(buf.degenerate_skipped),
    )
    img_dt = np.float32 if images_f32 else np.float64
    out.update(color=buf.color.astype(img_dt), depth=buf.depth.astype(img_dt),
               accumulation=buf.accumulation.astype(img_dt), max_w=max_w.astype(img_dt))
    if grads:
        rng = np.random.default_rng(1000 + seed)
        trgb = np.clip(buf.color + rng.normal(0, 0.1, buf.color.shape), 0, 1)
        tdep = np.abs(buf.depth + rng.normal(0, 0.1, buf.depth.shape))
        w = R.LossWeights(1.0, 0.2)
        gc, go, loss = R.grad_color_opacity(arr, pose, ri, trgb, tdep, w, cfg)
        out.update(target_rgb=trgb, target_depth=tdep, loss_weights=np.array([w.mse, w.depth]), grad_color=gc,
                   grad_opacity=go, loss=np.float64(loss),
                   render_loss=np.float64(R.render_loss(buf, trgb, tdep, w)))
        mask = buf.accumulation > 0.3
        ma, mm = R.per_surfel_max_weight(arr, pose, ri, mask, cfg)
        out.update(mw_mask=mask, max_all=ma, max_marked=mm)
    if extra:
        out.update(extra)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: n={len(arr.means)} V={len(order)} -> {os.path.getsize(path) / 1e3:.0f} kB")


def kat_scenes():
    """Known-answer constructions (restated from the reference's own test intents)."""
    from paper_2604_03092_b200.rasterizer import SurfelArrays
    intr = scenes.CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)

    def arrays(rows):
        # inputs rounded to float32 so the GPU (float32 parameters) sees the very same values
        means, quats, scales, ops, cols = zip(*rows)
        f = scenes.f32
        return SurfelArrays(f(np.array(means, float)), f(np.array(quats, float)), f(np.array(scales, float)),
                            f(np.array(ops, float)), f(np.array(cols, float)))

    ident = [1.0, 0, 0, 0]
    # two-surfel compositing: near (opacity .5) in front of far (opacity .5) at the principal point
    two = arrays([([0, 0, 2.0], ident, [0.10, 0.10], 0.5, [0.0, 0.8, 0.4]),
                  ([0, 0, 1.0], ident, [0.05, 0.05], 0.5, [0.9, 0.1, 0.2])])
    # edge-on surfel: q = (.5,.5,.5,.5) maps the tangent axes to world y and z exactly; with
    # scales (1e-9, 0.1) the screen covariance has an exactly-zero eigenvalue -> degenerate
    edge = arrays([([0, 0, 2.0], [0.5, 0.5, 0.5, 0.5], [1e-9, 0.1], 1.0, [1, 1, 1])])
    # big opaque occluder in front of a random cloud
    rng = np.random.default_rng(11)
    rows = [([0, 0, 1.0], ident, [1.5, 1.5], 1.0, [0.2, 0.5, 0.7])]
    for _ in range(15):
        ax = rng.normal(size=3)
        rows.append(([rng.uniform(-0.8, 0.8), rng.uniform(-0.6, 0.6), rng.uniform(1.5, 3.5)],
                     UnitQuaternion.from_axis_angle(ax, rng.uniform(0, 0.6)).array(), rng.uniform(0.05, 0.18, 2),
                     rng.uniform(0.3, 0.8), rng.uniform(0.1, 0.9, 3)))
    occl = arrays(rows)
    # random scene of the reference's rasterizer-test style (64x48, fx=60)
    rng = np.random.default_rng(7)
    rows = []
    for _ in range(40):
        ax = rng.normal(size=3)
        rows.append(([rng.uniform(-0.8, 0.8), rng.uniform(-0.6, 0.6), rng.uniform(1.5, 3.5)],
                     UnitQuaternion.from_axis_angle(ax, rng.uniform(0, 0.6)).array(), rng.uniform(0.05, 0.18, 2),
                     rng.uniform(0.5, 1.0), rng.uniform(0.1, 0.9, 3)))
    rnd = arrays(rows)
    return intr, {"kat_two": two, "kat_edge": edge, "kat_occluder": occl, "kat_random40": rnd}


def main():
    exact = R.RasterConfig(weight_clamp=1.0)
    intr, kats = kat_scenes()
    ident = SE3Pose.identity()
    capture("kat_two_exact", kats["kat_two"], ident, intr, exact, grads=False)
    capture("kat_edge", kats["kat_edge"], ident, intr, grads=False)
    capture("kat_occluder_exact", kats["kat_occluder"], ident, intr, exact, grads=False)
    capture("kat_occluder_clamp", kats["kat_occluder"], ident, intr, grads=False)
    capture("kat_random40", kats["kat_random40"], ident, intr, seed=7)
    # config 1 (identity pose) and a posed variant (Sim3 with scale, rotation, translation)
    c1 = scenes.config1(0)
    capture("c1", c1.surfels, ident, c1.intr, seed=1)
    posed = Sim3Transform(1.25, UnitQuaternion.from_axis_angle([0.3, 1.0, -0.2], 0.35), np.array([0.2, -0.15, 0.4]))
    capture("c1_posed", c1.surfels, posed, c1.intr, seed=2)
    # config 2: binning pins at scale, images stored float32
    c2 = scenes.config2(0)
    capture("c2", c2.surfels, ident, c2.intr, images_f32=True, grads=False)


if __name__ == "__main__":
    main()
