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


def capture_map_ops():
    """transform_surfels / fuse / prune (mapper.py:184-260) and the surfel PLY writer (io.py:118-150)
    of the reference on seeded inputs (float32-representable, so the GPU sees the same values)."""
    from surfelslam import mapper as M
    from surfelslam import io as RIO
    f = scenes.f32
    rng = np.random.default_rng(31)
    out = {}
    # transform_surfels on random surfels; a Sim(3) with scale, rotation and translation
    s = scenes.random_surfels(rng, 500)
    arr = ref_arrays(s)
    t = Sim3Transform(1.3, UnitQuaternion.from_axis_angle([0.2, -1.0, 0.4], 0.9), np.array([0.5, -0.25, 1.5]))
    w = M.transform_surfels(arr, t)
    out.update(tr_means=arr.means, tr_quats=arr.quats, tr_scales=arr.scales, tr_pose=t.packed(),
               tr_out_means=w.means, tr_out_quats=w.quats, tr_out_scales=w.scales)
    # fuse: a map (config-1 cloud bound to keyframe 0 at pose p0) and camera-frame candidates from
    # keyframe 1 at pose p1
    c1 = scenes.config1(0)
    intr = ref_intr(c1.intr)
    p0 = Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0, 1, 0], 0.05), np.array([0.05, 0.0, 0.0]))
    p1 = Sim3Transform(1.0, UnitQuaternion.from_axis_angle([1, 0, 0.3], 0.08), np.array([-0.1, 0.05, 0.1]))
    m = M.GlobalSurfelMap()
    map_arr = ref_arrays(c1.surfels)
    M.fuse(m, map_arr, 0, p0, intr)                       # empty map: everything inserted
    # round the world map to float32 so both sides render the very same map
    for fld in ("means", "quats", "scales", "opacities", "colors"):
        setattr(m.surfels, fld, f(getattr(m.surfels, fld)))
    cand = ref_arrays(scenes.random_surfels(np.random.default_rng(32), 1500))
    m_before = m.surfels.copy()
    stats = M.fuse(m, cand, 1, p1, intr)
    n0 = len(m_before.means)
    out.update(fu_intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], float),
               fu_map_means=m_before.means, fu_map_quats=m_before.quats, fu_map_scales=m_before.scales,
               fu_map_opacities=m_before.opacities, fu_map_colors=m_before.colors,
               fu_p1=p1.packed(), fu_cand_means=cand.means, fu_cand_quats=cand.quats, fu_cand_scales=cand.scales,
               fu_cand_opacities=cand.opacities, fu_cand_colors=cand.colors,
               fu_inserted=np.int64(stats["inserted"]), fu_new_means=m.surfels.means[n0:],
               fu_new_quats=m.surfels.quats[n0:], fu_new_scales=m.surfels.scales[n0:],
               fu_new_kf=m.surfels.keyframe_ids[n0:],
               fu_acc=R.render(m_before, p1, intr).accumulation)
    # prune: observations = the map's own render at keyframe 0 with a corrupted block
    for fld in ("means", "quats", "scales", "opacities", "colors"):
        setattr(m.surfels, fld, f(getattr(m.surfels, fld)))
    buf = R.render(m.surfels, m.keyframe_poses[0], intr)
    orgb = f(buf.color.copy())
    odep = f(buf.depth / np.maximum(buf.accumulation, 1e-12))
    orgb[30:60, 40:90] = f(np.clip(1.0 - orgb[30:60, 40:90], 0, 1))
    odep[10:25, 10:50] *= np.float32(1.5)
    m_pr = m.copy()
    victims_n = M.prune(m_pr, 0, orgb, odep, intr)
    keep = np.ones(len(m.surfels.means), bool)
    # victims as indices: the surfels missing from the pruned map (prune keeps order)
    cfg = M.FusionConfig()
    covered = buf.accumulation > 0.5
    rgb_err = np.max(np.abs(buf.color - orgb), axis=2) > cfg.prune_rgb_error
    dn = buf.depth / np.maximum(buf.accumulation, 1e-12)
    depth_err = (odep > 0) & (np.abs(dn - odep) > cfg.prune_depth_error_frac * odep)
    marked = covered & (rgb_err | depth_err)
    _, mm = R.per_surfel_max_weight(m.surfels, m.keyframe_poses[0], intr, marked)
    victims = np.flatnonzero(mm > cfg.prune_contribution_floor)
    keep[victims] = False
    assert victims_n == len(victims) and np.array_equal(m_pr.surfels.means, m.surfels.means[keep])
    out.update(pr_map_means=m.surfels.means, pr_map_quats=m.surfels.quats, pr_map_scales=m.surfels.scales,
               pr_map_opacities=m.surfels.opacities, pr_map_colors=m.surfels.colors, pr_p0=p0.packed(),
               pr_obs_rgb=orgb, pr_obs_depth=odep, pr_marked=marked, pr_victims=victims, pr_max_marked=mm)
    # surfel PLY bytes written by the reference
    import tempfile
    small = m.surfels.select(np.arange(20))
    small.confidences = np.linspace(0.1, 1.0, 20)
    small.submap_ids = np.arange(20, dtype=np.int64) % 3
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.ply")
        RIO.write_surfel_ply(path, small)
        with open(path, "rb") as fh:
            ply = np.frombuffer(fh.read(), np.uint8)
    out.update(ply_bytes=ply, ply_means=small.means, ply_quats=small.quats, ply_scales=small.scales,
               ply_opacities=small.opacities, ply_colors=small.colors, ply_conf=small.confidences,
               ply_kf=small.keyframe_ids, ply_submap=small.submap_ids)
    path = os.path.join(HERE, "map_ops.npz")
    np.savez_compressed(path, **out)
    print(f"map_ops: inserted {stats['inserted']}/{len(cand.means)}, victims {len(victims)}, "
          f"marked px {int(marked.sum())} -> {os.path.getsize(path) / 1e3:.0f} kB")


def _random_rows(rng, n, op_lo=0.3, op_hi=0.8):
    """The reference rasterizer tests' random-scene distribution (test_rasterizer.py random_scene,
    restated): means in [-.8,.8]x[-.6,.6]x[1.5,3.5], axis-angle rotations up to 0.6 rad, tangent
    scales U(.05,.18), opacity U(op_lo, op_hi), colour U(.1,.9); float32-representable."""
    rows = []
    for _ in range(n):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        rows.append(([rng.uniform(-0.8, 0.8), rng.uniform(-0.6, 0.6), rng.uniform(1.5, 3.5)],
                     UnitQuaternion.from_axis_angle(ax, rng.uniform(0, 0.6)).array(), rng.uniform(0.05, 0.18, 2),
                     rng.uniform(op_lo, op_hi), rng.uniform(0.1, 0.9, 3)))
    means, quats, scales, ops, cols = zip(*rows)
    f = scenes.f32
    return R.SurfelArrays(f(np.array(means)), f(np.array(quats)), f(np.array(scales)), f(np.array(ops)),
                          f(np.array(cols)), np.ones(n), np.zeros(n, np.int64), np.zeros(n, np.int64))


def capture_fd():
    """The reference's gradient checks (test_rasterizer.py:263-291, test_acceptance.py:207-243,
    criterion 2): 20 seeded 12-surfel scenes at 64x48 whose accumulation stays 1e-3 clear of the
    0.5 mask edge, LossWeights(1.0, 0.2); the reference's grad_color_opacity and its central
    finite differences (h = 1e-4) of render_loss(render()) per colour channel and opacity."""
    intr = R.CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
    pose = SE3Pose.identity()
    w = R.LossWeights(mse=1.0, depth=0.2)
    out = {"intr": np.array([60.0, 60.0, 32.0, 24.0, 64, 48]), "loss_weights": np.array([w.mse, w.depth])}
    done, seed, checked = 0, 100, 0
    while done < 20:
        rng = np.random.default_rng(seed)
        seed += 1
        arr = _random_rows(rng, 12)
        buf = R.render(arr, pose, intr)
        if np.min(np.abs(buf.accumulation - 0.5)) <= 1e-3:
            continue
        trng = np.random.default_rng(seed + 5000)
        trgb = np.clip(buf.color + trng.normal(scale=0.1, size=buf.color.shape), 0, 1)
        tdep = np.abs(buf.depth + trng.normal(scale=0.1, size=buf.depth.shape))
        gc, go, loss = R.grad_color_opacity(arr, pose, intr, trgb, tdep, w)
        h = 1e-4
        fdc = np.zeros_like(gc)
        fdo = np.zeros_like(go)
        for i in range(len(arr)):
            for ch in range(3):
                orig = arr.colors[i, ch]
                arr.colors[i, ch] = orig + h
                lp = R.render_loss(R.render(arr, pose, intr), trgb, tdep, w)
                arr.colors[i, ch] = orig - h
                lm = R.render_loss(R.render(arr, pose, intr), trgb, tdep, w)
                arr.colors[i, ch] = orig
                fdc[i, ch] = (lp - lm) / (2 * h)
            orig = arr.opacities[i]
            arr.opacities[i] = orig + h
            lp = R.render_loss(R.render(arr, pose, intr), trgb, tdep, w)
            arr.opacities[i] = orig - h
            lm = R.render_loss(R.render(arr, pose, intr), trgb, tdep, w)
            arr.opacities[i] = orig
            fdo[i] = (lp - lm) / (2 * h)
        checked += int((np.abs(gc) > 1e-8).sum() + (np.abs(go) > 1e-8).sum())
        k = f"s{done:02d}_"
        out.update({k + "means": arr.means, k + "quats": arr.quats, k + "scales": arr.scales,
                    k + "opacities": arr.opacities, k + "colors": arr.colors, k + "target_rgb": trgb,
                    k + "target_depth": tdep, k + "grad_color": gc, k + "grad_opacity": go,
                    k + "loss": np.float64(loss), k + "fd_color": fdc, k + "fd_opacity": fdo})
        done += 1
    path = os.path.join(HERE, "fd_scenes.npz")
    np.savez_compressed(path, **out)
    print(f"fd_scenes: 20 scenes, {checked} checked gradients -> {os.path.getsize(path) / 1e3:.0f} kB")


def capture_refine():
    """The reference's mapper.refine (mapper.py:276-349) on a seeded three-keyframe map: the
    config-1 cloud bound round-robin to keyframes 0, 5, 10 at nearby poses, colours perturbed
    by U(-.15,.15) and clipped (test_acceptance.py:385-411 style), observations = the
    unperturbed map's renders (depth normalised by the accumulation).  Two runs: 10
    iterations over all three keyframes, and 3 iterations over keyframe 0 only (untargeted
    surfels)."""
    from surfelslam import mapper as M
    f = scenes.f32
    c1 = scenes.config1(3)
    intr = ref_intr(c1.intr)
    arr = ref_arrays(c1.surfels)
    n = len(arr.means)
    frames = [0, 5, 10]
    poses = {0: Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0, 1, 0], 0.04), np.array([0.03, 0.0, 0.0])),
             5: Sim3Transform(1.0, UnitQuaternion.from_axis_angle([1, 0, 0.2], 0.05), np.array([-0.05, 0.02, 0.05])),
             10: Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0.3, 1, 0], -0.06), np.array([0.0, -0.04, -0.06]))}
    arr.keyframe_ids = np.array([frames[i % 3] for i in range(n)], np.int64)
    obs = {}
    for k in frames:
        buf = R.render(arr, poses[k], intr)
        obs[k] = (buf.color, buf.depth / np.maximum(buf.accumulation, 1e-12))
    rng = np.random.default_rng(8)
    pert = arr.copy()
    pert.colors = f(np.clip(arr.colors + rng.uniform(-0.15, 0.15, arr.colors.shape), 0, 1))
    out = {"means": pert.means, "quats": pert.quats, "scales": pert.scales, "opacities": pert.opacities,
           "colors": pert.colors, "keyframe_ids": pert.keyframe_ids, "frames": np.array(frames),
           "intr": np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], float)}
    for k in frames:
        out[f"pose_{k}"] = poses[k].packed()
        out[f"obs_rgb_{k}"], out[f"obs_depth_{k}"] = obs[k]
    for tag, kfs, iters in (("all", frames, 10), ("kf0", [0], 3)):
        m = M.GlobalSurfelMap(pert.copy(), dict(poses))
        rep = M.refine(m, kfs, obs, intr, M.RefinementConfig(iterations=iters))
        out.update({f"{tag}_losses": np.array(rep.losses), f"{tag}_psnr": np.array([rep.psnr_before, rep.psnr_after]),
                    f"{tag}_accepted": np.int64(rep.accepted_steps), f"{tag}_colors": m.surfels.colors,
                    f"{tag}_opacities": m.surfels.opacities, f"{tag}_iters": np.int64(iters)})
        print(f"refine[{tag}]: losses {len(rep.losses)}, accepted {rep.accepted_steps}, "
              f"psnr {rep.psnr_before:.3f} -> {rep.psnr_after:.3f}")
    path = os.path.join(HERE, "refine_ref.npz")
    np.savez_compressed(path, **out)
    print(f"refine_ref -> {os.path.getsize(path) / 1e3:.0f} kB")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "map_ops":
        capture_map_ops()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "fd":
        capture_fd()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "refine":
        capture_refine()
        return
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
    capture_map_ops()
    capture_fd()
    capture_refine()


if __name__ == "__main__":
    main()
