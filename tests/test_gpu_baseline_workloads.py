"""Parity on the BASELINE.json workloads as written (configs 2-5), not on synthetic far targets:

* config 2: the target is the render of the perturbed copy (means + N(0, .01), rgb + N(0, .05));
  MSE (the reference loss) at the plain 1e-4 gate; L1 + 0.1 L1 depth with the sign-ambiguous
  pixels (float64 residual below the float32 render error) seeded with the GPU's sign and counted;
* config 3: all 8 poses, images and all five parameter groups;
* config 5: L1 gradients against exposure-gained targets (gain U(.7, 1.3) per view);
* config 4: one full step through AdamRefiner(inflight=16, cuda_graph=True) against the sum of
  the oracle's per-view gradients, and a 10-iteration Adam trajectory on a reduced config 4
  checked step by step against the float64 oracle (gradients and the Adam update)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import Run, f32, fused_grads, gate, l1_oracle_grads
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.engine import unpack_params
from paper_2604_03092_b200.mapper import AdamConfig, AdamRefiner, ViewLoss
from paper_2604_03092_b200.rasterizer import SurfelArrays

pytestmark = pytest.mark.gpu

GROUPS = ("colors", "opacities", "means", "quats", "scales")


def _gate_all(g, og, tol=1e-4, tag=""):
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], getattr(og, f), tol)
        assert ok, (tag, f, mx, l2)


def _target(surfels, pose, intr, gain=1.0):
    t = O.render(surfels, pose, intr, with_normal=False)
    return f32(t.color * gain), f32(t.depth)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_config2_perturbed_copy_target(seed):
    sc = scenes.config2(seed)
    pose = sc.poses[0]
    trgb, tdep = _target(sc.extra["target_surfels"], pose, sc.intr)
    run = Run(sc.surfels, pose, sc.intr, normal=False, argmax=False)
    # MSE (rasterizer.py:346-357): plain gate
    g, loss = run.backward("mse", trgb, tdep, 1.0, 0.1, True)
    oloss, og, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, "mse", 1.0, 0.1, mask_depth=True)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    _gate_all(g, og, tag="mse")
    # L1 RGB + 0.1 L1 depth (BASELINE config 2)
    g, loss = run.backward("l1", trgb, tdep, 1.0, 0.1, False)
    im = run.images()
    oloss, og, namb = l1_oracle_grads(sc.surfels, pose, sc.intr, trgb, tdep, 1.0, 0.1, im["color"], im["depth"])
    print(f"config2 seed {seed}: sign-ambiguous L1 pixel channels {namb} of {4 * 320 * 240}")
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    _gate_all(g, og, tag="l1")


@pytest.fixture(scope="module")
def c3():
    return scenes.config3(0)


@pytest.mark.parametrize("k", range(8))
def test_config3_all_poses(c3, k):
    pose = c3.poses[k]
    run = Run(c3.surfels, pose, c3.intr, normal=True, argmax=False)
    ref = O.render(c3.surfels, pose, c3.intr)
    im = run.images()
    for key in ("color", "depth", "accumulation", "normal"):
        ok, mx, l2 = gate(im[key], getattr(ref, key))
        assert ok, (key, mx, l2)
    # target: the keyframe's own map perturbed (means + N(0, .01), rgb + N(0, .05)), rendered
    tgt = scenes.perturbed(c3.surfels, np.random.default_rng(50 + k))
    trgb, tdep = _target(tgt, pose, c3.intr)
    g, loss = run.backward("mse", trgb, tdep, 1.0, 0.1, True)
    oloss, og, _ = O.loss_and_grads(c3.surfels, pose, c3.intr, trgb, tdep, "mse", 1.0, 0.1, mask_depth=True)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    _gate_all(g, og, tag=f"pose {k} mse")
    g, loss = run.backward("l1", trgb, tdep, 1.0, 0.1, False)
    oloss, og, namb = l1_oracle_grads(c3.surfels, pose, c3.intr, trgb, tdep, 1.0, 0.1, im["color"], im["depth"])
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    _gate_all(g, og, tag=f"pose {k} l1")


def test_config5_exposure_gain_gradients():
    """BASELINE config 5 (4M surfels, 1296x968): L1 gradients of the perturbed map against
    targets rendered from the unperturbed map times the view's exposure gain."""
    sc = scenes.config5(0)
    surf = sc.extra["perturbed"]
    for v in (3, 77):
        pose = sc.poses[v]
        trgb, tdep = _target(sc.surfels, pose, sc.intr, float(sc.gains[v]))
        run = Run(surf, pose, sc.intr, normal=False, argmax=False)
        g, loss = run.backward("l1", trgb, tdep, 1.0, 0.1, False)
        im = run.images()
        oloss, og, namb = l1_oracle_grads(surf, pose, sc.intr, trgb, tdep, 1.0, 0.1, im["color"], im["depth"])
        print(f"config5 view {v} gain {sc.gains[v]:.3f}: sign-ambiguous {namb}")
        assert abs(loss - oloss) <= 1e-5 * abs(oloss)
        _gate_all(g, og, tag=f"view {v}")
        del run
        torch.cuda.empty_cache()
        # the one-kernel path the refine step runs (s2d_forward_backward), same oracle
        gf, lossf, imf, _ = fused_grads(surf, pose, sc.intr, "l1", trgb, tdep, 1.0, 0.1, False, image=True)
        assert np.array_equal(imf["color"], im["color"]) and np.array_equal(imf["depth"], im["depth"])
        assert abs(lossf - oloss) <= 1e-5 * abs(oloss)
        _gate_all(gf, og, tag=f"view {v} fused")
        torch.cuda.empty_cache()


def _oracle_step_grads(surf, sc, views, trgbs, tdeps, colors, depths, threads=None):
    """Sum over views of the oracle's L1 gradients (float64), views in parallel host threads."""
    def one(v):
        return l1_oracle_grads(surf, sc.poses[v], sc.intr, trgbs[v], tdeps[v], 1.0, 0.1, colors[v], depths[v])
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, views))
    tot = {f: sum(getattr(r[1], f) for r in res) for f in GROUPS}
    return sum(r[0] for r in res), tot


def _gpu_renders(surf, sc, views):
    colors, depths = {}, {}
    for v in views:
        im = Run(surf, sc.poses[v], sc.intr, normal=False, argmax=False).images()
        colors[v], depths[v] = im["color"], im["depth"]
    return colors, depths


def test_config4_full_step_inflight_graph_vs_oracle_sum():
    """One refine iteration of the bench workload (1M surfels, 32 views 640x480, 16 views in
    flight, CUDA graph): the summed gradient block equals the sum of the oracle's per-view
    gradients, and the Adam step equals the float64 oracle Adam on that gradient."""
    sc = scenes.config4(0)
    surf = sc.extra["perturbed"]
    views = list(range(len(sc.poses)))
    trgbs, tdeps = {}, {}
    for v in views:
        im = Run(sc.surfels, sc.poses[v], sc.intr, normal=False, argmax=False).images()
        trgbs[v], tdeps[v] = im["color"], im["depth"]
    ref = AdamRefiner(surf, sc.intr, sc.poses, [trgbs[v] for v in views], [tdeps[v] for v in views],
                      ViewLoss("l1", 1.0, 0.1, False), AdamConfig(), inflight=16, cuda_graph=True)
    ref.step()  # eager step (sizes the capacities); the graph is captured on the next one
    p1 = ref.params.clone()
    m1, m2 = ref.m1.clone(), ref.m2.clone()
    loss = ref.step()  # graph replay
    g = {k: v.double().cpu().numpy() for k, v in unpack_params(ref.grads, ref.n).items()}
    P1 = {k: v.double().cpu().numpy() for k, v in unpack_params(p1, ref.n).items()}
    s1 = SurfelArrays(P1["means"], P1["quats"], P1["scales"], P1["opacities"], P1["colors"])
    colors, depths = _gpu_renders(s1, sc, views)
    oloss, og = _oracle_step_grads(s1, sc, views, trgbs, tdeps, colors, depths)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss), (loss, oloss)
    for f in GROUPS:
        ok, mx, l2 = gate(g[f], og[f])
        assert ok, (f, mx, l2)
    # the fused Adam step (step 2) vs the float64 oracle Adam on the same gradient
    pn = p1.double().cpu().numpy()
    O.adam_step(pn, ref.grads.double().cpu().numpy(), m1.double().cpu().numpy(), m2.double().cpu().numpy(), 2)
    ok, mx, l2 = gate(ref.params.double().cpu().numpy(), pn, 1e-6)
    assert ok, (mx, l2)


def test_reduced_config4_adam_trajectory_10_steps():
    """10 Adam iterations (lr 1e-3 means, 5e-3 the rest) on a reduced config 4 (2 keyframes x
    50k surfels, 8 views 640x480), checked step by step: each step's summed gradients against the
    oracle's at the same parameters (1e-4), and the fused Adam update against the float64 oracle
    Adam from the same state.  The free-running loss trace of an all-oracle loop is reported."""
    sc = scenes.config4(1, n_keyframes=2, per_keyframe=50_000, n_views=8)
    surf = sc.extra["perturbed"]
    views = list(range(len(sc.poses)))
    trgbs, tdeps = {}, {}
    for v in views:
        im = Run(sc.surfels, sc.poses[v], sc.intr, normal=False, argmax=False).images()
        trgbs[v], tdeps[v] = im["color"], im["depth"]
    ref = AdamRefiner(surf, sc.intr, sc.poses, [trgbs[v] for v in views], [tdeps[v] for v in views],
                      ViewLoss("l1", 1.0, 0.1, False), AdamConfig(), inflight=4, cuda_graph=True)
    losses = []
    for step in range(1, 11):
        pk = ref.params.clone()
        mk, vk = ref.m1.clone(), ref.m2.clone()
        loss = ref.step()
        losses.append(loss)
        Pk = {k: v.double().cpu().numpy() for k, v in unpack_params(pk, ref.n).items()}
        sk = SurfelArrays(Pk["means"], Pk["quats"], Pk["scales"], Pk["opacities"], Pk["colors"])
        colors, depths = _gpu_renders(sk, sc, views)
        oloss, og = _oracle_step_grads(sk, sc, views, trgbs, tdeps, colors, depths)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss), (step, loss, oloss)
        g = {k: v.double().cpu().numpy() for k, v in unpack_params(ref.grads, ref.n).items()}
        for f in GROUPS:
            ok, mx, l2 = gate(g[f], og[f])
            assert ok, (step, f, mx, l2)
        pn = pk.double().cpu().numpy()
        O.adam_step(pn, ref.grads.double().cpu().numpy(), mk.double().cpu().numpy(), vk.double().cpu().numpy(), step)
        ok, mx, l2 = gate(ref.params.double().cpu().numpy(), pn, 1e-6)
        assert ok, (step, mx, l2)
    assert losses[-1] < losses[0]
    print("loss trace", [round(x, 6) for x in losses])
