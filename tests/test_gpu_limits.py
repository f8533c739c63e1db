"""Size limits of the path: an image of 64,000 16x16 tiles (tile ids use the full 16 bits of the
pair key, two tile-sort passes), a 1x1 image, and the rejections just past the limits."""
import ctypes

import numpy as np
import pytest

import oracle as O
from gpu_helpers import Run, far_targets, fused_grads, gate
from paper_2604_03092_b200 import _native as N
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.engine import DeviceContext, ImageBuffers, View, camera_struct, config_struct
from paper_2604_03092_b200.geometry import SE3Pose

pytestmark = pytest.mark.gpu


def test_64000_tiles_binning_and_images():
    """4096x4000 image (256 x 250 = 64,000 tiles), 3,000 config-1 surfels (scales x 0.25) spread over it:
    tile lists bit-exact, images and L1 gradients against the oracle."""
    from test_gpu_parity import check_binning
    rng = np.random.default_rng(5)
    intr = R.CameraIntrinsics(3200.0, 3200.0, 2048.0, 2000.0, 4096, 4000)
    s = scenes.random_surfels(rng, 3000)
    s = type(s)(s.means, s.quats, scenes.f32(np.asarray(s.scales) * 0.25), s.opacities, s.colors)
    pose = SE3Pose.identity()
    run = Run(s, pose, intr, normal=True, argmax=False)
    proj = O.project(s, pose, intr)
    check_binning(run, proj, O.depth_order(proj), intr)
    assert run.inspect()["ranges"].shape[0] == 64000
    ref = O.render(s, pose, intr)
    im = run.images()
    for key in ("color", "depth", "accumulation", "normal"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    trgb, tdep = far_targets(ref.color, ref.depth, np.random.default_rng(6))
    g, loss, _, _ = fused_grads(s, pose, intr, "l1", trgb, tdep)
    oloss, og, _ = O.loss_and_grads(s, pose, intr, trgb, tdep, "l1", 1.0, 0.1, mask_depth=False)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    for f in ("colors", "opacities", "means", "quats", "scales"):
        ok, mx, l2 = gate(g[f], getattr(og, f))
        assert ok, (f, mx, l2)


def test_one_pixel_image():
    rng = np.random.default_rng(8)
    intr = R.CameraIntrinsics(2.0, 2.0, 0.0, 0.0, 1, 1)
    s = scenes.random_surfels(rng, 200)
    pose = SE3Pose.identity()
    run = Run(s, pose, intr, normal=True, argmax=True)
    ref = O.render(s, pose, intr)
    im = run.images()
    for key in ("color", "depth", "accumulation", "normal"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    assert np.array_equal(im["arg_w"], ref.arg_w)


def test_limits_rejected():
    """Past 65,536 tiles, past 32,767 pixels a side, 2^30 surfels: S2D_ERR_INVALID, no launch."""
    v = View(DeviceContext.get())
    img = ImageBuffers.allocate(1, 1, DeviceContext.get().device, normal=False)
    cfg = config_struct(R.DEFAULT_RASTER_CONFIG)
    pose = N.as_doubles([1, 0, 0, 0, 1, 0, 0, 0])
    for w, h in ((4112, 4096), (32768, 16)):  # 257 x 256 tiles; too wide
        cam = N.Camera(100.0, 100.0, 1.0, 1.0, w, h)
        rc = N.lib().s2d_forward(v.handle, None, None, 0, pose, ctypes.byref(cam), ctypes.byref(cfg),
                                 ctypes.byref(img.struct()), None, None, None)
        assert rc == N.S2D_ERR_INVALID, (w, h)
    cam = N.Camera(100.0, 100.0, 1.0, 1.0, 16, 16)
    rc = N.lib().s2d_forward(v.handle, None, None, ctypes.c_int64(1 << 30), pose, ctypes.byref(cam),
                             ctypes.byref(cfg), ctypes.byref(img.struct()), None, None, None)
    assert rc == N.S2D_ERR_INVALID
