"""The oracle's NEW pieces (no reference counterpart — "parity unpinned by reference tests"):
normal channel (N1), geometry + normal + accumulation gradients (N2) checked by central
finite differences of the oracle's own float64 forward, L1 seeds (N3), Adam (N4)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2604_03092_b200.geometry import Sim3Transform, UnitQuaternion, quat_to_matrix, pk_inverse
from paper_2604_03092_b200.rasterizer import CameraIntrinsics, RasterConfig, SurfelArrays

INTR = CameraIntrinsics(60.0, 60.0, 32.0, 24.0, 64, 48)


def scene(seed, n=12):
    rng = np.random.default_rng(seed)
    means = np.stack([rng.uniform(-.8, .8, n), rng.uniform(-.6, .6, n), rng.uniform(1.5, 3.5, n)], 1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return SurfelArrays(means, q, rng.uniform(0.05, 0.18, (n, 2)), rng.uniform(.3, .8, n),
                        rng.uniform(.1, .9, (n, 3))), rng


def test_normal_channel_definition():
    """Single opaque surfel: rendered normal = R_cw R(q)[:,2], flipped to face the camera."""
    q = UnitQuaternion.from_axis_angle([1.0, 0.5, 0.0], 0.6).array()
    s = SurfelArrays(np.array([[0.0, 0.0, 2.0]]), q[None], np.array([[0.3, 0.3]]), np.array([1.0]),
                     np.array([[1.0, 1.0, 1.0]]))
    pose = Sim3Transform(1.0, UnitQuaternion.from_axis_angle([0, 1.0, 0], 0.1), np.zeros(3))
    b = O.render(s, pose, INTR, RasterConfig(weight_clamp=1.0))
    inv = pk_inverse(pose.packed())
    n = quat_to_matrix(inv[4:8]) @ quat_to_matrix(q)[:, 2]
    p = inv[0] * (quat_to_matrix(inv[4:8]) @ np.array([0.0, 0.0, 2.0])) + inv[1:4]
    if n @ p > 0:
        n = -n
    cov = b.accumulation > 0
    assert cov.sum() > 20
    # one contributor per pixel: normal = acc * n exactly
    assert np.allclose(b.normal[cov] / b.accumulation[cov][:, None], n[None, :], atol=1e-12)


@pytest.mark.parametrize("seed", [1, 2])
def test_full_gradients_vs_oracle_fd(seed):
    """Linear loss L = <g_rgb, C> + <g_d, D> + <g_n, N> + <g_a, A> with random seeds;
    analytic grads w.r.t. every parameter vs central FD (footprint_sigma=7: smooth)."""
    s, rng = scene(seed)
    cfg = O.DEFAULTS.__class__(**{**vars(O.DEFAULTS), "footprint_sigma": 7.0})
    pose = Sim3Transform(0.9, UnitQuaternion.from_axis_angle(rng.normal(size=3), 0.15), rng.normal(0, .05, 3))
    gr = rng.normal(size=(48, 64, 3))
    gd = rng.normal(size=(48, 64))
    gn = rng.normal(size=(48, 64, 3))
    ga = rng.normal(size=(48, 64))

    def L(a):
        b = O.render(a, pose, INTR, cfg)
        return float(np.sum(gr * b.color) + np.sum(gd * b.depth) + np.sum(gn * b.normal) + np.sum(ga * b.accumulation))

    b = O.render(s, pose, INTR, cfg)
    G = O.backward(s, pose, INTR, b, gr, gd, gn, ga, cfg=cfg)
    h = 1e-6
    for field, g in (("colors", G.colors), ("opacities", G.opacities), ("means", G.means), ("quats", G.quats),
                     ("scales", G.scales)):
        errs, mags = [], []
        for idx in np.ndindex(getattr(s, field).shape):
            a = s.copy()
            getattr(a, field)[idx] += h
            lp = L(a)
            a = s.copy()
            getattr(a, field)[idx] -= h
            lm = L(a)
            fd = (lp - lm) / (2 * h)
            errs.append(abs(g[idx] - fd))
            mags.append(abs(fd))
        assert max(errs) <= 2e-6 * max(mags), (field, max(errs), max(mags))


def test_l1_seeds_definition():
    rng = np.random.default_rng(4)
    h, w = 6, 5
    buf = type("B", (), {})()
    buf.color = rng.uniform(size=(h, w, 3))
    buf.depth = rng.uniform(1, 2, size=(h, w))
    buf.accumulation = rng.uniform(size=(h, w))
    trgb = rng.uniform(size=(h, w, 3))
    tdep = rng.uniform(1, 2, size=(h, w))
    loss, g_rgb, g_d = O.loss_seeds(buf, trgb, tdep, "l1", 1.0, 0.1, mask_depth=False)
    ref = np.mean(np.abs(buf.color - trgb)) + 0.1 * np.mean(np.abs(buf.depth - tdep))
    assert abs(loss - ref) <= 1e-12
    assert np.allclose(g_rgb, np.sign(buf.color - trgb) / (3 * h * w))
    assert np.allclose(g_d, 0.1 * np.sign(buf.depth - tdep) / (h * w))
    loss_m, _, g_dm = O.loss_seeds(buf, trgb, tdep, "l1", 1.0, 0.1, mask_depth=True)
    m = buf.accumulation > 0.5
    assert np.allclose(g_dm[~m], 0.0) and np.allclose(g_dm[m], 0.1 * np.sign(buf.depth - tdep)[m] / m.sum())


def test_adam_matches_torch():
    """N4: oracle Adam == torch.optim.Adam (float64) on the packed block before the projection."""
    rng = np.random.default_rng(5)
    n = 50
    p0 = np.concatenate([rng.normal(size=3 * n), np.tile([1.0, 0, 0, 0], n), rng.uniform(0.1, 1, 2 * n),
                         rng.uniform(0.2, 0.8, n), rng.uniform(0.2, 0.8, 3 * n)])
    p = p0.copy()
    m1 = np.zeros_like(p)
    m2 = np.zeros_like(p)
    tp = torch.tensor(p0.copy(), dtype=torch.float64, requires_grad=True)
    means = tp[:3 * n]
    opt = torch.optim.Adam([{"params": [torch.nn.Parameter(tp[:3 * n].detach().clone())], "lr": 1e-3},
                            {"params": [torch.nn.Parameter(tp[3 * n:].detach().clone())], "lr": 5e-3}],
                           betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 4):
        g = rng.normal(size=p.size) * 1e-2
        O.adam_step(p, g, m1, m2, step, scale_min=0.0)
        opt.param_groups[0]["params"][0].grad = torch.tensor(g[:3 * n])
        opt.param_groups[1]["params"][0].grad = torch.tensor(g[3 * n:])
        opt.step()
        # projection of the reference for the rest block: quats normalised, clip opac/colors
        with torch.no_grad():
            rest = opt.param_groups[1]["params"][0]
            q = rest[:4 * n].view(n, 4)
            q /= q.norm(dim=1, keepdim=True)
            rest[6 * n:].clamp_(0, 1)
        tref = torch.cat([opt.param_groups[0]["params"][0], opt.param_groups[1]["params"][0]]).detach().numpy()
        assert np.allclose(p, tref, rtol=0, atol=1e-12)
    assert means is not None
