"""The reference's own hot-path tests re-run through the drop-in (GPU), against values the
reference produced (tests/golden/make_golden.py):

* criterion 2 (test_acceptance.py:150-245): exact two-surfel compositing, accumulation bounds,
  order independence, opaque occluder, and analytic colour/opacity gradients within 1e-4 of
  the reference's central finite differences over its 20 seeded scenes
  (also test_rasterizer.py:263-291);
* mapper.refine (mapper.py:276-349; test_acceptance.py:385-411): loss trace, accepted steps,
  PSNRs and the final colours/opacities of the reference's run on the same map."""
import numpy as np
import pytest

from conftest import load_golden
from gpu_helpers import gate
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200.geometry import SE3Pose, UnitQuaternion
from paper_2604_03092_b200.mapper import GlobalSurfelMap, RefinementConfig, refine
from paper_2604_03092_b200.rasterizer import SurfelArrays

pytestmark = pytest.mark.gpu

INTR = R.CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
EXACT = R.RasterConfig(weight_clamp=1.0)
ID = SE3Pose.identity()


def test_criterion2_exact_compositing_bounds_order_occluder(goldens):
    f = lambda a: np.asarray(a, np.float32)  # noqa: E731  (the device computes in float32)
    c1, c2 = np.array([0.9, 0.1, 0.2]), np.array([0.0, 0.8, 0.4])
    near = R.Surfel(np.array([0, 0, 1.0]), UnitQuaternion.identity(), np.array([0.05, 0.05]), 0.5, c1)
    far = R.Surfel(np.array([0, 0, 2.0]), UnitQuaternion.identity(), np.array([0.10, 0.10]), 0.5, c2)
    buf = R.render([far, near], ID, INTR, EXACT)
    # Eq. 1 exactly, in the device's float32 arithmetic: 0.5 c1 + 0.25 c2 rounded once
    want = (np.float32(0.5) * f(c1) + np.float32(0.25) * f(c2)).astype(np.float64)
    assert np.array_equal(buf.color[24, 32], want)
    assert buf.accumulation[24, 32] == 0.75
    g = goldens["kat_random40"]
    b1 = R.render(g.surfels, ID, INTR)
    assert np.all(b1.accumulation >= 0) and np.all(b1.accumulation <= 1)
    perm = np.random.default_rng(7).permutation(len(g.surfels))
    b2 = R.render(g.surfels.select(perm), ID, INTR)
    assert b1.color.tobytes() == b2.color.tobytes() and b1.depth.tobytes() == b2.depth.tobytes()
    front = R.Surfel(np.array([0, 0, 1.0]), UnitQuaternion.identity(), np.array([1.5, 1.5]), 1.0,
                     np.array([0.2, 0.5, 0.7]))
    scene = [front] + [R.Surfel(g.surfels.means[i], UnitQuaternion.from_array(g.surfels.quats[i]),
                                g.surfels.scales[i], float(g.surfels.opacities[i]), g.surfels.colors[i])
                       for i in range(len(g.surfels))]
    with_back = R.render(scene, ID, INTR, EXACT)
    without = R.render([front], ID, INTR, EXACT)
    covered = without.accumulation >= 1.0 - 1e-12
    assert covered.any()
    assert np.array_equal(with_back.color[covered], without.color[covered])


def test_criterion2_fd_gradients_vs_reference():
    d = load_golden("fd_scenes")
    w = R.LossWeights(*[float(x) for x in d["loss_weights"]])
    checked = loose = 0
    for k in range(20):
        p = f"s{k:02d}_"
        s = SurfelArrays(d[p + "means"], d[p + "quats"], d[p + "scales"], d[p + "opacities"], d[p + "colors"])
        gc, go, loss = R.grad_color_opacity(s, ID, INTR, d[p + "target_rgb"], d[p + "target_depth"], w)
        assert abs(loss - d[p + "loss"]) <= 1e-5 * abs(d[p + "loss"])
        for a, b in ((gc, d[p + "grad_color"]), (go, d[p + "grad_opacity"])):
            ok, mx, l2 = gate(a, b)
            assert ok, (k, mx, l2)
        # the reference's criterion: |analytic - FD| <= 1e-4 |FD| wherever |analytic| > 1e-8.  The
        # float32 sums carry an absolute error of up to ~2e-6 of the tensor's largest gradient
        # (cancelling per-pixel terms), which is above 1e-4 relative for the tiniest elements:
        # those are held to 1e-4 |FD| + 1e-5 max|FD| (a tenth of the per-tensor gate) and counted
        for a, ref, fd in ((gc, d[p + "grad_color"], d[p + "fd_color"]), (go, d[p + "grad_opacity"], d[p + "fd_opacity"])):
            sel = np.abs(ref) > 1e-8
            err = np.abs(a[sel] - fd[sel])
            strict = err <= 1e-4 * np.abs(fd[sel])
            assert np.all(err <= 1e-4 * np.abs(fd[sel]) + 1e-5 * np.abs(fd).max()), k
            checked += int(sel.sum())
            loose += int((~strict).sum())
    print(f"criterion 2: {checked} gradients checked against the reference's FD, {loose} only within the "
          f"1e-5 max|FD| absolute term")
    assert checked > 300 and loose <= checked // 100


@pytest.mark.parametrize("tag", ["all", "kf0"])
def test_refine_vs_reference_run(tag):
    d = load_golden("refine_ref")
    frames = [int(x) for x in d["frames"]]
    s = SurfelArrays(d["means"], d["quats"], d["scales"], d["opacities"], d["colors"])
    s.keyframe_ids = np.asarray(d["keyframe_ids"], np.int64)
    m = GlobalSurfelMap(s, {k: d[f"pose_{k}"] for k in frames})
    obs = {k: (d[f"obs_rgb_{k}"], d[f"obs_depth_{k}"]) for k in frames}
    fx, fy, cx, cy, w, h = d["intr"]
    intr = R.CameraIntrinsics(fx, fy, cx, cy, int(w), int(h))
    kfs = frames if tag == "all" else [0]
    rep = refine(m, kfs, obs, intr, RefinementConfig(iterations=int(d[f"{tag}_iters"])))
    assert rep.accepted_steps == int(d[f"{tag}_accepted"])
    ref_losses = d[f"{tag}_losses"]
    assert len(rep.losses) == len(ref_losses)
    assert np.all(np.abs(np.array(rep.losses) - ref_losses) <= 1e-4 * np.abs(ref_losses)), (rep.losses, ref_losses)
    assert abs(rep.psnr_before - d[f"{tag}_psnr"][0]) < 1e-3 and abs(rep.psnr_after - d[f"{tag}_psnr"][1]) < 1e-3
    for a, b in ((m.surfels.colors, d[f"{tag}_colors"]), (m.surfels.opacities, d[f"{tag}_opacities"])):
        ok, mx, l2 = gate(a, b)
        assert ok, (mx, l2)
    if tag == "kf0":  # untargeted surfels: the reference's np.clip leaves in-range values bitwise
        out = np.asarray(d["keyframe_ids"]) != 0
        assert np.array_equal(m.surfels.colors[out], d["colors"][out])
