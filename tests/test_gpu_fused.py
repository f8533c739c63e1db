"""s2d_forward_backward: compositing, loss seeds and the reverse traversal in ONE raster kernel
(the losses without the whole-image depth mask: L1 as BASELINE configs 2/4/5 use it, MSE with
w_depth = 0).  Every parameter group within the 1e-4 gate of the float64 oracle, the loss
within 1e-5, the images (when requested) equal to the two-kernel path's, and the losses that
need the depth mask routed through s2d_forward + s2d_backward."""
import numpy as np
import pytest
import torch

import oracle as O
import oracle.raysplat as RS
from gpu_helpers import Run, far_targets, fused_grads, gate, l1_oracle_grads
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.rasterizer import SurfelArrays

pytestmark = pytest.mark.gpu

GROUPS = ("colors", "opacities", "means", "quats", "scales")


def _check_vs_oracle(s, pose, intr, kind, trgb, tdep, w_depth=0.1):
    g, loss, im, st = fused_grads(s, pose, intr, kind, trgb, tdep, 1.0, w_depth, False, image=True)
    oloss, og, _ = O.loss_and_grads(s, pose, intr, trgb, tdep, kind, 1.0, w_depth, mask_depth=False)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss), (loss, oloss)
    for f in GROUPS:
        ref = getattr(og, f)
        if np.abs(ref).max() < 1e-15:
            # analytically zero (e.g. the quaternion of an isotropic splat seen head-on, when no
            # other surfel is on screen): float rounding noise on both sides, compared absolutely
            assert np.abs(g[f]).max() < 1e-15, (kind, f, np.abs(g[f]).max())
            continue
        ok, mx, l2 = gate(g[f], ref)
        assert ok, (kind, f, mx, l2)
    return g, loss, im, st


@pytest.mark.parametrize("seed", range(8))
def test_config2_l1_fused_vs_oracle(seed):
    """BASELINE config 2's loss (L1 RGB + 0.1 L1 depth, no mask): all five groups, seeds 0-7."""
    sc = scenes.config2(seed)
    pose = sc.poses[0]
    ref = O.render(sc.surfels, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(300 + seed))
    g, loss, im, st = _check_vs_oracle(sc.surfels, pose, sc.intr, "l1", trgb, tdep)
    for k in ("color", "depth", "accumulation"):
        ok, mx, l2 = gate(im[k], getattr(ref, k))
        assert ok, (k, mx, l2)


def test_config2_perturbed_target_fused():
    """Config 2 exactly as BASELINE states it: the target rendered from the perturbed copy
    (residuals cross zero; sign-ambiguous channels take the GPU render's sign)."""
    sc = scenes.config2(0)
    pose = sc.poses[0]
    tb = O.render(sc.extra["target_surfels"], pose, sc.intr)
    g, loss, im, _ = fused_grads(sc.surfels, pose, sc.intr, "l1", tb.color, tb.depth, 1.0, 0.1, False, image=True)
    oloss, og, amb = l1_oracle_grads(sc.surfels, pose, sc.intr, tb.color, tb.depth, 1.0, 0.1, im["color"], im["depth"])
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2, amb)


def test_mse_without_depth_term_fused_vs_oracle():
    sc = scenes.config2(5)
    pose = sc.poses[0]
    ref = O.render(sc.surfels, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(8))
    _check_vs_oracle(sc.surfels, pose, sc.intr, "mse", trgb, tdep, w_depth=0.0)


def test_saturated_and_clamped_opacities_fused():
    """Opacities at 1 and around the weight clamp: the clamp decisions cross from the forward
    half of the kernel to its backward half in the blend stream."""
    sc = scenes.config2(3)
    s = sc.surfels
    rng = np.random.default_rng(5)
    op = np.asarray(s.opacities, dtype=np.float64).copy()
    pick = rng.random(len(op))
    op[pick < 0.4] = 1.0
    band = (pick >= 0.4) & (pick < 0.5)
    op[band] = np.float32(0.999) + rng.integers(-40, 40, band.sum()) * 1e-6
    s = SurfelArrays(s.means, s.quats, s.scales, op.astype(np.float32).astype(np.float64), s.colors)
    pose = sc.poses[0]
    ref = O.render(s, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(19))
    _check_vs_oracle(s, pose, sc.intr, "l1", trgb, tdep)


def test_needle_splat_fused():
    """config2(4) head-on holds a needle-like splat (kappa(M) ~ 620): an accurate slot, its
    whitened offsets taken from the float64 Minv in both halves of the kernel."""
    from paper_2604_03092_b200.geometry import SE3Pose
    sc = scenes.config2(4)
    pose = SE3Pose.identity()
    intr = R.CameraIntrinsics(250.0, 250.0, 160.0, 120.0, 320, 240)
    ref = O.render(sc.surfels, pose, intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(29))
    _check_vs_oracle(sc.surfels, pose, intr, "l1", trgb, tdep)


def test_config3_fused_matches_two_kernel_path():
    """Config 3 (196,608 pixel-aligned surfels, 512x384): the one-kernel path and
    s2d_forward + s2d_backward agree within the gate on every group, the images and counters
    are identical."""
    sc = scenes.config3(0)
    pose = sc.poses[3]
    run = Run(sc.surfels, pose, sc.intr, normal=False, argmax=False)
    im2 = run.images()
    rng = np.random.default_rng(11)
    trgb, tdep = far_targets(im2["color"], im2["depth"], rng)
    g2, l2loss = run.backward("l1", trgb, tdep, 1.0, 0.1, False)
    st2 = run.view.stats()
    g, loss, im, st = fused_grads(sc.surfels, pose, sc.intr, "l1", trgb, tdep, 1.0, 0.1, False, image=True)
    for k in ("color", "depth", "accumulation"):
        assert np.array_equal(im[k], im2[k]), k
    assert (st.pairs, st.visible, st.blended, st.guard_hits) == (st2.pairs, st2.visible, st2.blended, st2.guard_hits)
    assert abs(loss - l2loss) <= 1e-6 * abs(l2loss)
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], g2[f], 1e-5)
        assert ok, (f, mx, l2)


@pytest.mark.parametrize("kind", ["mse", "l1"])
def test_depth_mask_losses_fall_back_to_two_kernels(kind):
    """MSE with a depth term and L1 over the depth mask need the image's mask count before any
    seed: s2d_forward_backward runs them as forward + backward, equal to the oracle."""
    sc = scenes.config2(2)
    pose = sc.poses[0]
    ref = O.render(sc.surfels, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(13))
    g, loss, _, st = fused_grads(sc.surfels, pose, sc.intr, kind, trgb, tdep, 1.0, 0.1, True, image=True)
    oloss, og, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=True)
    assert st.n_mask == int((ref.accumulation > 0.5).sum())
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


def test_ray_mode_fused_vs_autograd():
    sc = scenes.config1(2)
    s, intr = sc.surfels.select(np.arange(300)), sc.intr
    from test_gpu_raysplat import POSE
    cfg = R.RasterConfig(splat_mode="ray", footprint_sigma=6.0)
    pr = RS.params_from_arrays(s)
    ref = RS.render_ray(pr, POSE, intr, cfg)
    trgb, tdep = far_targets(ref["color"].detach().numpy(), ref["depth"].detach().numpy(), np.random.default_rng(4))
    g, loss, _, _ = fused_grads(s, POSE, intr, "l1", trgb, tdep, 1.0, 0.1, False, cfg=cfg)
    npx = intr.width * intr.height
    L = ((ref["color"] - torch.as_tensor(trgb)).abs().sum() / (3 * npx)
         + 0.1 * (ref["depth"] - torch.as_tensor(tdep)).abs().sum() / npx)
    L.backward()
    assert abs(loss - L.item()) <= 1e-5 * abs(L.item())
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], pr[f].grad.numpy())
        assert ok, (f, mx, l2)


def test_empty_scene_and_no_image():
    sc = scenes.config1(0)
    s = sc.surfels.select(np.arange(0))
    h, w = sc.intr.height, sc.intr.width
    g, loss, _, st = fused_grads(s, sc.poses[0], sc.intr, "l1", np.full((h, w, 3), 0.5), np.ones((h, w)))
    assert st.pairs == 0
    # loss = mean |0 - 0.5| + 0.1 mean |0 - 1|
    assert abs(loss - (0.5 + 0.1)) <= 1e-6


def test_adam_refiner_fused_matches_two_kernel_trajectory():
    """Config-2 multi-view Adam: the default (fused) refiner and fused=False follow the same loss
    trajectory over 10 iterations (float32 atomics reorder: 1e-5)."""
    from paper_2604_03092_b200.mapper import AdamConfig, AdamRefiner, ViewLoss
    sc = scenes.config2(0)
    tgt = sc.extra["target_surfels"]
    bufs = [R.render(tgt, p, sc.intr) for p in sc.poses]
    out = []
    for fused in (True, False):
        ref = AdamRefiner(sc.surfels, sc.intr, sc.poses, [b.color for b in bufs], [b.depth for b in bufs],
                          ViewLoss("l1", 1.0, 0.1), AdamConfig(), inflight=4, fused=fused)
        assert ref.fused == fused
        out.append([ref.step() for _ in range(10)])
    a, b = np.array(out[0]), np.array(out[1])
    assert np.all(np.abs(a - b) <= 1e-5 * np.abs(b)), (a, b)
    assert a[-1] < a[0]


@pytest.mark.parametrize("n", [1, 257, 4097])
def test_ragged_image_and_counts_with_huge_splat_fused(n):
    """37x23 image (partial tiles at both edges), ragged surfel counts, one splat covering the
    whole image, identity and rotated poses: the one-kernel path against the oracle."""
    from paper_2604_03092_b200.geometry import Sim3Transform, UnitQuaternion
    rng = np.random.default_rng(n)
    intr = R.CameraIntrinsics(30.0, 30.0, 18.0, 11.0, 37, 23)
    s = scenes.random_surfels(rng, n)
    big = SurfelArrays(np.array([[0.0, 0.0, 1.5]]), np.array([[1.0, 0, 0, 0]]), np.array([[2.0, 2.0]]),
                       np.array([0.3]), np.array([[0.2, 0.4, 0.6]]))
    s = SurfelArrays.concatenate([s, big])
    s = SurfelArrays(*[np.asarray(getattr(s, k), np.float32).astype(np.float64)
                       for k in ("means", "quats", "scales", "opacities", "colors")])
    for pose in (Sim3Transform.identity(), Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0, 0, 1.0], 0.3),
                                                         np.zeros(3))):
        ref = O.render(s, pose, intr)
        trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(n + 1))
        _, _, im, _ = _check_vs_oracle(s, pose, intr, "l1", trgb, tdep)
        for k in ("color", "depth", "accumulation"):
            ok, mx, l2 = gate(im[k], getattr(ref, k))
            assert ok, (k, mx, l2)
