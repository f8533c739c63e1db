"""Cross-check the oracle against the live reference (build container only; skipped on the
GPU box, where /root/reference does not exist).  Also validates the NEW geometry
gradients (N2) against central finite differences of the reference's own
render_loss(render(...)) on a smooth (footprint_sigma=7) configuration."""
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")


@pytest.fixture(scope="module")
def R():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_s2d")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    from surfelslam import rasterizer
    return rasterizer


def _scene(rng, n, nonunit=False):
    from paper_2604_03092_b200.rasterizer import SurfelArrays
    means = np.stack([rng.uniform(-.8, .8, n), rng.uniform(-.6, .6, n), rng.uniform(1.5, 3.5, n)], 1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    if nonunit:
        q *= rng.uniform(0.9, 1.1, (n, 1))
    return SurfelArrays(means, q, rng.uniform(0.05, 0.18, (n, 2)), rng.uniform(.3, .8, n),
                        rng.uniform(.1, .9, (n, 3)))


def _ref(R, s):
    n = len(s)
    return R.SurfelArrays(s.means, s.quats, s.scales, s.opacities, s.colors, np.ones(n), np.zeros(n, np.int64),
                          np.zeros(n, np.int64))


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_live_render_and_grads(R, seed):
    import oracle as O
    from surfelslam.geometry import Sim3Transform, UnitQuaternion
    rng = np.random.default_rng(seed)
    s = _scene(rng, 300, nonunit=True)
    intr = R.CameraIntrinsics(80.0, 80.0, 40.0, 30.0, 80, 60)
    pose = Sim3Transform(rng.uniform(0.8, 1.2), UnitQuaternion.from_axis_angle(rng.normal(size=3), 0.2),
                         rng.normal(0, 0.1, 3))
    arr = _ref(R, s)
    st = R._render_state(arr, pose, intr, R.DEFAULT_RASTER_CONFIG)
    b = O.render(s, pose, intr)
    assert np.array_equal(b.order, st.order)
    assert np.array_equal(b.color, st.buffers.color)
    assert np.array_equal(b.accumulation, st.buffers.accumulation)
    trgb = np.clip(st.buffers.color + rng.normal(0, .1, st.buffers.color.shape), 0, 1)
    tdep = np.abs(st.buffers.depth + rng.normal(0, .1, st.buffers.depth.shape))
    gc, go, loss = R.grad_color_opacity(arr, pose, intr, trgb, tdep, R.LossWeights(1.0, 0.2))
    l2, gr, _ = O.loss_and_grads(s, pose, intr, trgb, tdep, "mse", 1.0, 0.2)
    assert np.array_equal(gr.colors, gc) and np.array_equal(gr.opacities, go)
    assert abs(l2 - loss) <= 1e-12 * abs(loss)


def test_geometry_gradients_vs_reference_fd(R):
    """N2 (no reference counterpart): analytic d loss / d(means, quats, scales) of the oracle
    vs central FD of the reference's render_loss(render()) with footprint_sigma=7 (smooth)."""
    import oracle as O
    from surfelslam.geometry import Sim3Transform, UnitQuaternion
    rng = np.random.default_rng(3)
    s = _scene(rng, 12, nonunit=True)
    intr = R.CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)
    pose = Sim3Transform(1.1, UnitQuaternion.from_axis_angle([0.2, 1, 0.3], 0.1), np.array([0.05, -0.02, 0.03]))
    cfg = R.RasterConfig(footprint_sigma=7.0)
    arr = _ref(R, s)
    buf = R.render(arr, pose, intr, cfg)
    assert np.min(np.abs(buf.accumulation - 0.5)) > 1e-6
    trgb = np.clip(buf.color + rng.normal(0, .1, buf.color.shape), 0, 1)
    tdep = np.abs(buf.depth + rng.normal(0, .1, buf.depth.shape))
    w = R.LossWeights(1.0, 0.2)
    _, gr, _ = O.loss_and_grads(s, pose, intr, trgb, tdep, "mse", 1.0, 0.2, cfg=cfg)

    def L(a):
        return R.render_loss(R.render(a, pose, intr, cfg), trgb, tdep, w)

    h = 1e-6
    for field, G in (("means", gr.means), ("quats", gr.quats), ("scales", gr.scales)):
        errs, mags = [], []
        for idx in np.ndindex(getattr(arr, field).shape):
            a = arr.copy()
            getattr(a, field)[idx] += h
            lp = L(a)
            a = arr.copy()
            getattr(a, field)[idx] -= h
            lm = L(a)
            fd = (lp - lm) / (2 * h)
            errs.append(abs(G[idx] - fd))
            mags.append(abs(fd))
        assert max(errs) <= 1e-6 * max(mags), field
