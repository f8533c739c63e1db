"""The properties the reference's own rasterizer tests assert (pkg/tests/test_rasterizer.py:
projection, render, render_loss, gradients, max weights), checked through this package's
drop-in API on the GPU.  Written independently; the scenes are seeded config-1 style scenes."""
import numpy as np
import pytest

from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.engine import DeviceContext, ImageBuffers, View, camera_struct, config_struct, \
    forward_checked, pack_params
from paper_2604_03092_b200.geometry import SE3Pose
from paper_2604_03092_b200.rasterizer import LossWeights, RasterConfig, SurfelArrays

pytestmark = pytest.mark.gpu

INTR = R.CameraIntrinsics(100.0, 100.0, 64.0, 48.0, 128, 96)
ID = SE3Pose.identity()


def _surfels(rows):
    f = lambda k: np.array([r[k] for r in rows], dtype=np.float64)  # noqa: E731
    return SurfelArrays(f(0), f(1), f(2), f(3), f(4))


def _records(s, intr=INTR, pose=ID):
    """Device splat records of an on-screen set: Minv (A, C, B, D) per surfel and the flags."""
    ctx = DeviceContext.get()
    v = View(ctx)
    params = pack_params(s, ctx.device)
    img = ImageBuffers.allocate(intr.height, intr.width, ctx.device, normal=False)
    forward_checked(v, params, len(s), pose, camera_struct(intr), config_struct(R.DEFAULT_RASTER_CONFIG), img)
    d = v.inspect()
    return d["records"].double().cpu().numpy(), d["flags"].cpu().numpy()


def _cov2(rec):
    """Screen covariance from a record's whitening matrix: Sigma = M M^T with M = Minv^-1."""
    A, C, B, D = rec[4:8]
    minv = np.array([[A, B], [C, D]])
    m = np.linalg.inv(minv)
    return m @ m.T


def test_projection_isotropic_on_axis():
    """A round surfel facing the camera on the optical axis projects to (f s / z)^2 I."""
    s = _surfels([([0.0, 0.0, 2.0], [1.0, 0, 0, 0], [0.05, 0.05], 0.8, [0.2, 0.3, 0.4])])
    rec, fl = _records(s)
    assert fl[0] & 4
    cov = _cov2(rec[0])
    expect = (100.0 * 0.05 / 2.0) ** 2
    assert np.allclose(cov, np.diag([expect, expect]), rtol=1e-5, atol=1e-6 * expect)


def test_projection_roll_swaps_eigen_axes():
    """An elongated surfel rolled 90 degrees about the view axis swaps its screen axes."""
    q90 = [np.cos(np.pi / 4), 0.0, 0.0, np.sin(np.pi / 4)]
    s = _surfels([([0.0, 0.0, 2.0], [1.0, 0, 0, 0], [0.08, 0.02], 0.8, [0.2, 0.3, 0.4]),
                  ([0.0, 0.0, 2.0], q90, [0.08, 0.02], 0.8, [0.2, 0.3, 0.4])])
    rec, _ = _records(s)
    c0, c1 = _cov2(rec[0]), _cov2(rec[1])
    assert c0[0, 0] > 10 * c0[1, 1] and c1[1, 1] > 10 * c1[0, 0]
    assert np.allclose([c0[0, 0], c0[1, 1]], [c1[1, 1], c1[0, 0]], rtol=1e-4)


def test_projection_behind_camera_culled():
    s = _surfels([([0.0, 0.0, -2.0], [1.0, 0, 0, 0], [0.05, 0.05], 0.8, [0.2, 0.3, 0.4]),
                  ([0.0, 0.0, 2.0], [1.0, 0, 0, 0], [0.05, 0.05], 0.8, [0.2, 0.3, 0.4])])
    _, fl = _records(s)
    assert fl[0] & 7 == 0 and fl[1] & 4


def test_projection_covariance_matches_monte_carlo():
    """Points sampled from the surfel's tangent-plane Gaussian, projected through the pinhole:
    their screen covariance approaches the projected 2D covariance (small surfel, so the
    first-order projection is accurate)."""
    rng = np.random.default_rng(3)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    mu, sc = np.array([0.1, -0.05, 2.5]), np.array([0.02, 0.008])
    s = _surfels([(mu, q, sc, 0.8, [0.2, 0.3, 0.4])])
    rec, _ = _records(s)
    cov = _cov2(rec[0])
    w, x, y, z = q
    Rm = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                   [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                   [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    uv = rng.normal(size=(400000, 2)) * sc
    pts = mu + uv @ Rm[:, :2].T
    px = np.stack([100.0 * pts[:, 0] / pts[:, 2] + 64.0, 100.0 * pts[:, 1] / pts[:, 2] + 48.0], 1)
    emp = np.cov(px.T)
    assert np.allclose(emp, cov, rtol=0.02, atol=0.02 * np.abs(cov).max())


def test_render_bounds_and_empty_pixels():
    """0 <= accumulation <= 1, and depth (expected, un-normalised) is zero where nothing blends."""
    sc = scenes.config1(4)
    buf = R.render(sc.surfels, ID, INTR)
    assert buf.accumulation.min() >= 0.0 and buf.accumulation.max() <= 1.0
    empty = buf.accumulation == 0.0
    assert np.all(buf.depth[empty] == 0.0) and np.all(buf.color[empty] == 0.0)
    s = sc.surfels.select(np.arange(0))
    e = R.render(s, ID, INTR)
    assert not e.color.any() and not e.depth.any() and not e.accumulation.any()


def test_accumulation_monotone_in_surfels():
    """Adding surfels never lowers a pixel's accumulation (transmittance only decreases)."""
    sc = scenes.config1(5)
    n = len(sc.surfels)
    a = R.render(sc.surfels.select(np.arange(n // 2)), ID, INTR).accumulation
    b = R.render(sc.surfels, ID, INTR).accumulation
    assert np.all(b >= a - 1e-6)


def test_render_loss_properties():
    sc = scenes.config1(6)
    buf = R.render(sc.surfels, ID, INTR)
    assert R.render_loss(buf, buf.color, buf.depth) == 0.0
    off = 0.1
    l = R.render_loss(buf, buf.color + off, buf.depth, LossWeights(mse=1.0, depth=0.0))
    assert abs(l - off * off) <= 1e-12
    with pytest.raises(ValueError):
        R.render_loss(buf, buf.color[:-1], buf.depth)


def test_gradients_channel_separable():
    """A target that differs from the render in one colour channel only gives colour gradients
    in that channel only."""
    sc = scenes.config1(7)
    buf = R.render(sc.surfels, ID, INTR)
    tgt = buf.color.copy()
    tgt[..., 1] += 0.1
    gc, go, _ = R.grad_color_opacity(sc.surfels, ID, INTR, tgt, buf.depth, LossWeights(mse=1.0, depth=0.0))
    assert np.abs(gc[:, 1]).max() > 0.0
    assert np.abs(gc[:, 0]).max() == 0.0 and np.abs(gc[:, 2]).max() == 0.0


def test_max_weight_front_surfel_dominates_and_mask():
    """Two coincident-footprint surfels: the front one carries the larger max weight; a mask
    away from both leaves their masked maxima at zero, a mask over them keeps the front one's."""
    s = _surfels([([0.0, 0.0, 2.0], [1.0, 0, 0, 0], [0.1, 0.1], 0.7, [0.9, 0.1, 0.1]),
                  ([0.0, 0.0, 3.0], [1.0, 0, 0, 0], [0.15, 0.15], 0.7, [0.1, 0.9, 0.1])])
    mx, _ = R.per_surfel_max_weight(s, ID, INTR)
    assert mx[0] > mx[1] > 0.0
    far = np.zeros((96, 128), bool)
    far[:4, :4] = True
    _, mm = R.per_surfel_max_weight(s, ID, INTR, mask=far)
    assert np.all(mm == 0.0)
    centre = np.zeros((96, 128), bool)
    centre[40:56, 56:72] = True
    mx2, mm2 = R.per_surfel_max_weight(s, ID, INTR, mask=centre)
    assert np.allclose(mm2[0], mx2[0]) and mm2[0] > 0.0
