"""Depth-order edge cases on the GPU (rasterizer.py:318-320: lexsort((index, z))): a whole
keyframe at one exact depth, millimetre-quantised depth, and long runs of distinct depths that
share one sort key (the float64 z differ below the key's resolution).  The order, the tile lists
and the images must equal the oracle's; the exact-tie cases must not cost more than a normal
keyframe's depth sort."""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import Run, drawn_order, gate
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.engine import ImageBuffers, View, DeviceContext, camera_struct, config_struct, forward_checked
from paper_2604_03092_b200.geometry import SE3Pose
from paper_2604_03092_b200.rasterizer import SurfelArrays

pytestmark = pytest.mark.gpu

INTR = R.CameraIntrinsics(400.0, 400.0, 256.0, 192.0, 512, 384)


def _plane(depth, seed=0):
    """Pixel-aligned surfels of one 512x384 keyframe (config 3 recipe) at the given per-pixel
    depth, facing the camera, float32-representable."""
    rng = np.random.default_rng(seed)
    h, w = depth.shape
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
    pts = np.stack([(xs - INTR.cx) / INTR.fx * depth, (ys - INTR.cy) / INTR.fy * depth, depth], -1).reshape(-1, 3)
    n = w * h
    q = np.tile([1.0, 0.0, 0.0, 0.0], (n, 1))
    scales = (depth.reshape(-1, 1) / INTR.fx) * rng.uniform(0.8, 1.5, (n, 2))
    f32 = scenes.f32
    return SurfelArrays(f32(pts), f32(q), f32(scales), f32(rng.uniform(0.5, 1.0, n)), f32(rng.uniform(0, 1, (n, 3))))


def _check(s, pose=None):
    pose = pose or SE3Pose.identity()
    run = Run(s, pose, INTR, normal=True, argmax=False)
    proj = O.project(s, pose, INTR)
    order = O.depth_order(proj)
    d = run.inspect()
    assert np.array_equal(d["order"].cpu().numpy().astype(np.int64), drawn_order(proj.bbox, order)), "depth order"
    start, ids = O.tile_lists(proj, order, INTR)
    assert np.array_equal(d["pair_ids"].cpu().numpy().astype(np.int64), ids), "tile lists"
    ref = O.render(s, pose, INTR)
    im = run.images()
    for key in ("color", "depth", "accumulation"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    return proj


def _depth_sort_ms(s, pose, reps=5):
    v = View(DeviceContext.get())
    run = Run(s, pose, INTR, normal=False, argmax=False, view=v)
    img = ImageBuffers.allocate(INTR.height, INTR.width, run.dev, normal=False)
    v.set_timing(True)
    v.timing(reset=True)
    for _ in range(reps):
        forward_checked(v, run.params, run.n, pose, camera_struct(INTR), config_struct(R.DEFAULT_RASTER_CONFIG), img)
    t = v.timing(reset=True)
    v.set_timing(False)
    return t["depth_sort"] / max(t["n_forward"], 1)


def test_one_exact_depth_keyframe():
    """196,608 surfels at z = 2 exactly (identity pose): one run of equal keys, already in the
    reference order (index order) after the order-preserving compaction."""
    s = _plane(np.full((384, 512), 2.0))
    proj = _check(s)
    assert len(np.unique(proj.z[proj.on_screen])) == 1


def test_millimetre_quantised_depth():
    """Sensor-like depth quantised to 1 mm: long runs of exactly equal z."""
    rng = np.random.default_rng(3)
    d = scenes._depth_field(rng, 512, 384)
    s = _plane(np.round(d * 1000.0) / 1000.0, seed=1)
    proj = _check(s)
    z = proj.z[proj.on_screen]
    assert len(np.unique(z)) < len(z) // 20


def test_exact_ties_cost_like_a_normal_keyframe():
    """The depth-sort phase of the tie cases stays within 2x of config 3's."""
    c3 = scenes.config3(0)
    base = _depth_sort_ms(c3.surfels, c3.poses[0])
    flat = _depth_sort_ms(_plane(np.full((384, 512), 2.0)), SE3Pose.identity())
    rng = np.random.default_rng(3)
    quant = _depth_sort_ms(_plane(np.round(scenes._depth_field(rng, 512, 384) * 1000.0) / 1000.0, 1),
                           SE3Pose.identity())
    print(f"depth sort ms: c3 {base:.4f}  one depth {flat:.4f}  1 mm quantised {quant:.4f}")
    assert flat <= 2.0 * base + 0.01 and quant <= 2.0 * base + 0.01, (base, flat, quant)


@pytest.mark.parametrize("n_rows", [8, 384])
def test_long_runs_of_distinct_depths_in_one_key(n_rows):
    """A wall at z = 2 seen with a 1e-7 rad rotation: camera depths 2 + ~1e-7 (a y - b x),
    mostly distinct in float64 but within the depth key's resolution (2^-20 either side of 2),
    and not in index order: runs of thousands of entries full of inversions, sorted by the
    cooperative long-run path (k_tie_long)."""
    from paper_2604_03092_b200.geometry import Sim3Transform, UnitQuaternion
    d = np.full((384, 512), 4.0)
    d[:n_rows] = 2.0
    s = _plane(d, seed=2)
    pose = Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0.3, 1.0, 0.0], 1e-7), np.zeros(3))
    proj = _check(s, pose)
    z = proj.z[proj.on_screen]
    near = z[z < 3.0]
    assert len(np.unique(near)) > len(near) // 4  # distinct depths
    assert np.all(np.abs(near - 2.0) < 2.0 ** -20)  # two depth keys (either side of 2)


def test_short_runs_mixed_with_exact_ties():
    """Config 3 with every other row pushed to its neighbour's depth: many short runs of equal
    keys, some exactly equal z, some not."""
    c3 = scenes.config3(1)
    m = np.asarray(c3.surfels.means, np.float64).reshape(384, 512, 3).copy()
    m[1::2, :, 2] = m[0::2, :, 2]
    s = SurfelArrays(scenes.f32(m.reshape(-1, 3)), c3.surfels.quats, c3.surfels.scales, c3.surfels.opacities,
                     c3.surfels.colors)
    _check(s, c3.poses[2])
