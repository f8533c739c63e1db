"""GPU parity through the C ABI: binning bit-exact, images/gradients within the 1e-4
relative gate, against golden vectors of the reference and against the CPU oracle."""
import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN_NAMES
from gpu_helpers import Run, drawn_order, far_targets, gate
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.geometry import SE3Pose, Sim3Transform, UnitQuaternion
from paper_2604_03092_b200.rasterizer import RasterConfig, SurfelArrays

pytestmark = pytest.mark.gpu


def check_binning(run, proj, order, intr):
    d = run.inspect()
    st = d["stats"]
    n = run.n
    flags = d["flags"].cpu().numpy()
    assert np.array_equal(flags & 7, proj.flags), "in_front/valid/on_screen flags"
    on = proj.on_screen
    assert st.visible == int(on.sum())
    assert st.degenerate == proj.degenerate
    assert np.array_equal(d["bbox"].cpu().numpy().astype(np.int64)[on], proj.bbox[on]), "bbox"
    assert np.array_equal(d["z"].cpu().numpy()[on], proj.z[on]), "float64 z"
    assert np.array_equal(d["order"].cpu().numpy().astype(np.int64), drawn_order(proj.bbox, order)), "depth order"
    drawn = on & (proj.bbox[:, 0] <= proj.bbox[:, 1]) & (proj.bbox[:, 2] <= proj.bbox[:, 3])
    assert np.array_equal((flags >> 3) & 1, drawn.astype(np.uint8)), "drawn flag"
    start, ids = O.tile_lists(proj, order, intr)
    assert st.pairs == len(ids)
    assert np.array_equal(d["pair_ids"].cpu().numpy().astype(np.int64), ids), "tile lists"
    rg = d["ranges"].cpu().numpy()
    cnt = rg[:, 1] - rg[:, 0]
    assert np.array_equal(cnt, np.diff(start)), "per-tile counts"
    assert np.array_equal(rg[:, 0][cnt > 0], start[:-1][cnt > 0]), "tile starts"
    return n


# ------------------------------------------------------------- vs reference goldens

@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_binning_bit_exact_vs_reference(goldens, name):
    g = goldens[name]
    run = Run(g.surfels, g.pose, g.intr, g.cfg)
    d = run.inspect()
    on = g["on_screen"]
    flags = d["flags"].cpu().numpy()
    assert np.array_equal((flags & 4) != 0, on)
    assert np.array_equal((flags & 2) != 0, g["valid"])
    assert np.array_equal((flags & 1) != 0, g["in_front"])
    assert d["stats"].degenerate == int(g["degenerate"])
    assert np.array_equal(d["bbox"].cpu().numpy().astype(np.int64)[on], g["bbox"][on])
    assert np.array_equal(d["z"].cpu().numpy()[on], g["z"][on])
    assert np.array_equal(d["order"].cpu().numpy().astype(np.int64), drawn_order(g["bbox"], g["order"]))
    proj = O.project(g.surfels, g.pose, g.intr, g.cfg)
    check_binning(run, proj, g["order"], g.intr)


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_images_vs_reference(goldens, name):
    g = goldens[name]
    im = Run(g.surfels, g.pose, g.intr, g.cfg).images()
    for key in ("color", "depth", "accumulation", "max_w"):
        ok, mx, l2 = gate(im[key], g[key])
        assert ok, (key, mx, l2)
    # render_with_argmax: the index output is bit-exact (float64 weights/transmittance in the
    # argmax variant of the forward, _raster_kernels.py:52-54, rasterizer.py:327-328)
    assert np.array_equal(im["arg_w"], g["arg_w"]), int((im["arg_w"] != g["arg_w"]).sum())


@pytest.mark.parametrize("name", ["kat_random40", "c1", "c1_posed"])
def test_grad_color_opacity_vs_reference(goldens, name):
    g = goldens[name]
    w = g["loss_weights"]
    gc, go, loss = R.grad_color_opacity(g.surfels, g.pose, g.intr, g["target_rgb"], g["target_depth"],
                                        R.LossWeights(float(w[0]), float(w[1])), g.cfg)
    for a, b, nm in ((gc, g["grad_color"], "color"), (go, g["grad_opacity"], "opacity")):
        ok, mx, l2 = gate(a, b)
        assert ok, (nm, mx, l2)
    assert abs(loss - float(g["loss"])) <= 1e-4 * abs(float(g["loss"]))


@pytest.mark.parametrize("name", ["kat_random40", "c1", "c1_posed"])
def test_per_surfel_max_weight_vs_reference(goldens, name):
    g = goldens[name]
    ma, mm = R.per_surfel_max_weight(g.surfels, g.pose, g.intr, g["mw_mask"], g.cfg)
    for a, b in ((ma, g["max_all"]), (mm, g["max_marked"])):
        ok, mx, l2 = gate(a, b)
        assert ok, (mx, l2)


# ------------------------------------------------------------- vs oracle, configs 1-3

def _config_cases():
    c1, c2, c3 = scenes.config1(0), scenes.config2(0), scenes.config3(0)
    return [("c1", c1, c1.poses[0]), ("c2", c2, c2.poses[0]), ("c3p0", c3, c3.poses[0]),
            ("c3p5", c3, c3.poses[5])]


CASES = _config_cases()


@pytest.mark.parametrize("name,sc,pose", CASES, ids=[c[0] for c in CASES])
def test_config_binning_and_images(name, sc, pose):
    run = Run(sc.surfels, pose, sc.intr)
    proj = O.project(sc.surfels, pose, sc.intr)
    check_binning(run, proj, O.depth_order(proj), sc.intr)
    im = run.images()
    ref = O.render(sc.surfels, pose, sc.intr)
    for key in ("color", "depth", "accumulation", "normal", "max_w"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)


@pytest.mark.parametrize("name,sc,pose", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("kind", ["mse", "l1"])
def test_config_gradients(name, sc, pose, kind):
    """All five parameter groups (geometry included) vs the float64 oracle."""
    run = Run(sc.surfels, pose, sc.intr, normal=True, argmax=False)
    ref = O.render(sc.surfels, pose, sc.intr)
    rng = np.random.default_rng(17)
    trgb, tdep = far_targets(ref.color, ref.depth, rng)
    mask = kind == "mse"
    g, loss = run.backward(kind, trgb, tdep, 1.0, 0.1, mask)
    oloss, og, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


@pytest.mark.parametrize("kind", ["mse", "l1"])
def test_saturated_opacity_gradients(kind):
    """Opacities at 1 (where Adam's clip leaves them) and just around the weight clamp: the
    forward's clamp decisions travel to the backward in the blend stream; all five parameter
    groups vs the float64 oracle."""
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
    run = Run(s, pose, sc.intr, normal=True, argmax=False)
    ref = O.render(s, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(19))
    mask = kind == "mse"
    g, loss = run.backward(kind, trgb, tdep, 1.0, 0.1, mask)
    oloss, og, _ = O.loss_and_grads(s, pose, sc.intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


def test_external_seeds_normal_and_accumulation_grads():
    """Upstream gradients on all four outputs (normal and accumulation included)."""
    sc = scenes.config2(1)
    pose = sc.poses[0]
    rng = np.random.default_rng(3)
    h, w = sc.intr.height, sc.intr.width
    seeds = [rng.normal(size=(h, w, 3)) * 1e-3, rng.normal(size=(h, w)) * 1e-3, rng.normal(size=(h, w, 3)) * 1e-3,
             rng.normal(size=(h, w)) * 1e-3]
    run = Run(sc.surfels, pose, sc.intr, normal=True, argmax=False)
    g, _ = run.backward("external", d_color=seeds[0], d_depth=seeds[1], d_normal=seeds[2], d_acc=seeds[3])
    ref = O.render(sc.surfels, pose, sc.intr)
    og = O.backward(sc.surfels, pose, sc.intr, ref, *seeds)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


# ------------------------------------------------------------- known answers and edge cases

INTR = R.CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
EXACT = RasterConfig(weight_clamp=1.0)
ID = SE3Pose.identity()


def _arr(rows):
    means, quats, scales, ops, cols = zip(*rows)
    return SurfelArrays(np.array(means, float), np.array(quats, float), np.array(scales, float),
                        np.array(ops, float), np.array(cols, float))


def test_two_surfel_compositing(goldens):
    g = goldens["kat_two_exact"]
    b = R.render(g.surfels, ID, INTR, EXACT)
    c1, c2 = np.array([0.9, 0.1, 0.2]), np.array([0.0, 0.8, 0.4])
    assert np.allclose(b.color[24, 32], 0.5 * c1 + 0.25 * c2, atol=2e-7)
    assert abs(b.accumulation[24, 32] - 0.75) <= 1e-7
    assert abs(b.depth[24, 32] - 1.0) <= 2e-7


def test_single_opaque_surfel_and_empty_scene():
    s = _arr([([0, 0, 2.0], [1, 0, 0, 0], [0.05, 0.05], 1.0, [1.0, 0, 0])])
    b = R.render(s, ID, INTR, EXACT)
    assert np.allclose(b.color[24, 32], [1, 0, 0]) and abs(b.depth[24, 32] - 2.0) < 1e-6
    assert b.accumulation[24, 32] == 1.0
    e = R.render(SurfelArrays.empty(), ID, INTR)
    assert not e.color.any() and not e.depth.any() and not e.accumulation.any()
    gc, go, loss = R.grad_color_opacity(SurfelArrays.empty(), ID, INTR, np.zeros((48, 64, 3)), np.zeros((48, 64)))
    assert gc.shape == (0, 3) and go.shape == (0,) and loss == 0.0


def test_opaque_occluder_exact_and_clamp_leakage(goldens):
    g = goldens["kat_occluder_exact"]
    front = g.surfels.select(np.array([0]))
    with_back = R.render(g.surfels, ID, INTR, EXACT)
    without = R.render(front, ID, INTR, EXACT)
    covered = without.accumulation >= 1.0
    assert covered.any()
    assert np.array_equal(with_back.color[covered], without.color[covered])
    assert np.array_equal(with_back.depth[covered], without.depth[covered])
    with_back = R.render(g.surfels, ID, INTR)
    without = R.render(front, ID, INTR)
    sat = without.accumulation >= 0.999 - 1e-6
    assert sat.any()
    assert np.max(np.abs(with_back.color[sat] - without.color[sat])) <= 1.5e-3


def test_degenerate_and_culled():
    s = _arr([([0, 0, 2.0], [0.5, 0.5, 0.5, 0.5], [1e-9, 0.1], 1.0, [1, 1, 1]),  # edge-on: degenerate
              ([0, 0, -1.0], [1, 0, 0, 0], [0.1, 0.1], 1.0, [1, 1, 1]),  # behind the camera
              ([50.0, 0, 1.0], [1, 0, 0, 0], [0.1, 0.1], 1.0, [1, 1, 1])])  # beyond the view angle
    b = R.render(s, ID, INTR)
    assert b.degenerate_skipped == 1
    assert not b.accumulation.any()


def test_image_sizes_not_multiple_of_tile_and_huge_splat():
    rng = np.random.default_rng(2)
    intr = R.CameraIntrinsics(30.0, 30.0, 18.0, 11.0, 37, 23)
    s = scenes.random_surfels(rng, 257)
    big = _arr([([0, 0, 1.5], [1, 0, 0, 0], [2.0, 2.0], 0.3, [0.2, 0.4, 0.6])])
    s = SurfelArrays.concatenate([s, big])
    for pose in (ID, Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0, 0, 1.0], 0.3), np.zeros(3))):
        run = Run(s, pose, intr)
        proj = O.project(s, pose, intr)
        check_binning(run, proj, O.depth_order(proj), intr)
        im = run.images()
        ref = O.render(s, pose, intr)
        for key in ("color", "depth", "accumulation", "normal"):
            ok, mx, l2 = gate(im[key], getattr(ref, key))
            assert ok, (key, mx, l2)


@pytest.mark.parametrize("n", [1, 255, 256, 257, 4095, 4097])
def test_ragged_surfel_counts(n):
    sc = scenes.config2(5)
    s = sc.surfels.select(np.arange(n))
    run = Run(s, sc.poses[0], sc.intr)
    proj = O.project(s, sc.poses[0], sc.intr)
    check_binning(run, proj, O.depth_order(proj), sc.intr)


def test_input_order_independence_and_determinism():
    sc = scenes.config2(0)
    pose = sc.poses[0]
    a = Run(sc.surfels, pose, sc.intr).images()
    b = Run(sc.surfels, pose, sc.intr).images()
    perm = np.random.default_rng(9).permutation(len(sc.surfels))
    c = Run(sc.surfels.select(perm), pose, sc.intr).images()
    for key in ("color", "depth", "accumulation", "normal"):
        assert a[key].tobytes() == b[key].tobytes(), key
        assert a[key].tobytes() == c[key].tobytes(), key


def test_pair_capacity_overflow_regrows():
    """A too-small pair capacity is reported (stats.overflow) and regrown by the caller."""
    import ctypes
    from paper_2604_03092_b200 import _native as N
    from paper_2604_03092_b200.engine import DeviceContext, View, ImageBuffers, camera_struct, config_struct
    c3 = scenes.config3(0)
    v = View(DeviceContext.get())
    v.reserve_pairs(4096)
    run = Run(c3.surfels, c3.poses[0], c3.intr, view=v)   # forward_checked regrows
    assert run.stats.pairs > 4096 and not run.stats.overflow
    ok, mx, l2 = gate(run.images()["color"], O.render(c3.surfels, c3.poses[0], c3.intr).color)
    assert ok, (mx, l2)
    v.reserve_pairs(4096)
    img = ImageBuffers.allocate(c3.intr.height, c3.intr.width, run.dev)
    v.forward(run.params, run.n, c3.poses[0], camera_struct(c3.intr), config_struct(R.DEFAULT_RASTER_CONFIG), img)
    st = v.stats()
    assert st.overflow == 1 and st.pairs == run.stats.pairs and st.pairs_stored == 4096
    assert N.lib().s2d_view_reserve_pairs(v.handle, ctypes.c_int64(1 << 31)) == N.S2D_ERR_INVALID


def test_stationary_point():
    """Targets equal to the model's own render: gradients vanish (test_rasterizer.py:244-250)."""
    sc = scenes.config1(2)
    pose = sc.poses[0]
    run = Run(sc.surfels, pose, sc.intr, normal=False, argmax=False)
    im = run.images()
    g, loss = run.backward("mse", im["color"], im["depth"], 1.0, 0.05, True)
    assert loss == 0.0
    for f in g:
        assert np.abs(g[f]).max() == 0.0, f


@pytest.mark.parametrize("kind", ["mse", "l1"])
def test_tiny_splats_on_pixel_centres(kind):
    """Splats far below a pixel (scales 1e-9 .. 1e-5, and some near 1e-40) whose centres project
    exactly onto pixel centres (x = y = 0 maps to the integer principal point): the reference
    blends each at that one pixel with m = 0.
    Exercises the block-relative offsets at an exact integer centre, near-singular Minv (up to
    ~1e7 per pixel) on the lanes around it, and the branch-free backward's masking of those
    lanes (finite values only), beside a normal scene; images and all gradients vs the oracle."""
    sc = scenes.config2(3)
    rng = np.random.default_rng(23)
    rows = []
    for k in range(40):
        z = 1.0 + 0.11 * k
        # down to 1e-40 (a float32 subnormal): Minv beyond the float32 range, clamped
        sc_ = 10.0 ** (rng.uniform(-9, -5) if k % 8 else -40.0 + 0.1 * k)
        q = rng.normal(size=4)
        rows.append(([0.0, 0.0, z], q / np.linalg.norm(q), [sc_, sc_ * rng.uniform(0.5, 2.0)],
                     rng.uniform(0.3, 0.95), rng.uniform(0, 1, 3)))
    t = _arr(rows)  # float32-representable inputs, as the device sees them
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    t = SurfelArrays(f32(t.means), f32(t.quats), f32(t.scales), f32(t.opacities), f32(t.colors))
    s = SurfelArrays.concatenate([sc.surfels, t])
    pose = SE3Pose.identity()
    intr = R.CameraIntrinsics(250.0, 250.0, 160.0, 120.0, 320, 240)
    run = Run(s, pose, intr, normal=True, argmax=False)
    proj = O.project(s, pose, intr)
    check_binning(run, proj, O.depth_order(proj), intr)
    ref = O.render(s, pose, intr)
    im = run.images()
    for key in ("color", "depth", "accumulation", "normal"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(29))
    mask = kind == "mse"
    g, loss = run.backward(kind, trgb, tdep, 1.0, 0.1, mask)
    for f, v in g.items():
        assert np.isfinite(v).all(), f
    oloss, og, _ = O.loss_and_grads(s, pose, intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


def test_needle_splat_geometry_gradients():
    """config2(4) seen head-on holds a needle-like splat (surfel 273: cov2 eigenvalues 6.2 and
    1.6e-5 px^2, kappa(M) ~ 620).  In float32 its whitened offsets u = A ex + (B ey + lo) would
    cancel ~1e3 down to O(1); as an accurate slot (kappa(M) > ~32) both raster passes evaluate
    them from the float64 Minv, so all five gradient groups meet the 1e-4 gate."""
    sc = scenes.config2(4)
    pose = SE3Pose.identity()
    intr = R.CameraIntrinsics(250.0, 250.0, 160.0, 120.0, 320, 240)
    run = Run(sc.surfels, pose, intr, normal=True, argmax=False)
    ref = O.render(sc.surfels, pose, intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(29))
    for kind in ("mse", "l1"):
        mask = kind == "mse"
        g, loss = run.backward(kind, trgb, tdep, 1.0, 0.1, mask)
        oloss, og, _ = O.loss_and_grads(sc.surfels, pose, intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss)
        for f in ("colors", "opacities", "means", "quats", "scales"):
            ok, mx, l2 = gate(g[f], getattr(og, f))
            assert ok, (kind, f, mx, l2)


@pytest.mark.parametrize("seed", range(32))
def test_config2_seed_sweep_all_groups(seed):
    """BASELINE config 2 scenes, seeds 0-31 (each holds a few ill-conditioned splats): images and
    all five parameter groups within the 1e-4 gate, MSE (reference depth mask) and L1."""
    sc = scenes.config2(seed)
    pose = sc.poses[0]
    run = Run(sc.surfels, pose, sc.intr, normal=True, argmax=True)
    ref = O.render(sc.surfels, pose, sc.intr)
    im = run.images()
    for key in ("color", "depth", "accumulation", "normal", "max_w"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    assert np.array_equal(im["arg_w"], ref.arg_w)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(100 + seed))
    for kind in ("mse", "l1"):
        mask = kind == "mse"
        g, loss = run.backward(kind, trgb, tdep, 1.0, 0.1, mask)
        oloss, og, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss)
        for f in ("colors", "opacities", "means", "quats", "scales"):
            ok, mx, l2 = gate(g[f], getattr(og, f))
            assert ok, (seed, kind, f, mx, l2)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_depth_mask_count_matches_float64(seed):
    """The MSE depth mask `accumulation > 0.5` (rasterizer.py:365-376): after the backward
    (k_mask_fixup re-decides the pixels within the float32 error band in float64) the mask
    count equals the float64 oracle's exactly, on scenes with many half-covered pixels
    (opacities around 0.5)."""
    sc = scenes.config2(seed)
    s = sc.surfels
    rng = np.random.default_rng(40 + seed)
    op = np.asarray(s.opacities, np.float64)
    op = np.float32(0.5) + (rng.random(len(op)) < 0.5) * np.float32(rng.normal(0, 0.02, len(op)))
    s = SurfelArrays(s.means, s.quats, s.scales, np.asarray(op, np.float32).astype(np.float64), s.colors)
    pose = sc.poses[0]
    run = Run(s, pose, sc.intr, normal=False, argmax=False)
    ref = O.render(s, pose, sc.intr)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(7))
    g, loss = run.backward("mse", trgb, tdep, 1.0, 0.1, True)
    st = run.view.stats()
    near = int((np.abs(ref.accumulation - 0.5) < 1e-4).sum())
    assert st.n_mask == int((ref.accumulation > 0.5).sum()), (st.n_mask, near)
    oloss, og, _ = O.loss_and_grads(s, pose, sc.intr, trgb, tdep, "mse", 1.0, 0.1, mask_depth=True)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)
