"""refine (reference semantics, mapper.py:276-349) and the multi-view AdamRefiner on the GPU."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import Run, gate
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.engine import unpack_params
from paper_2604_03092_b200.geometry import Sim3Transform
from paper_2604_03092_b200.mapper import (AdamConfig, AdamRefiner, GlobalSurfelMap, RefinementConfig, ViewLoss,
                                          refine)

pytestmark = pytest.mark.gpu


def small_map(seed=0):
    rng = np.random.default_rng(seed)
    intr = R.CameraIntrinsics(75.0, 75.0, 48.0, 36.0, 96, 72)
    surf, _ = scenes.depth_field_surfels(rng, intr)
    poses = {0: Sim3Transform.identity(), 6: scenes._small_pose(rng, 4.0, 0.1)}
    surf.keyframe_ids = np.array([(0, 6)[i % 2] for i in range(len(surf))], dtype=np.int64)
    m = GlobalSurfelMap(surf, dict(poses))
    return m, intr, rng


def observations(m, intr, frames):
    obs = {}
    for f in frames:
        b = R.render(m.surfels, m.keyframe_poses[f], intr)
        obs[f] = (b.color, b.depth / np.maximum(b.accumulation, 1e-12))
    return obs


def test_refine_recovers_psnr_with_decreasing_loss():
    m, intr, rng = small_map(0)
    obs = observations(m, intr, [0, 6])
    m.surfels.colors = np.clip(m.surfels.colors + rng.uniform(-0.15, 0.15, m.surfels.colors.shape), 0, 1)
    rep = refine(m, [0, 6], obs, intr, RefinementConfig(iterations=10))
    assert rep.psnr_after - rep.psnr_before >= 1.0, (rep.psnr_before, rep.psnr_after)
    assert all(b < a for a, b in zip(rep.losses, rep.losses[1:]))
    assert rep.accepted_steps >= 1


def test_refine_zero_iterations_bitwise_noop():
    m, intr, rng = small_map(1)
    obs = observations(m, intr, [0])
    c0, o0 = m.surfels.colors.tobytes(), m.surfels.opacities.tobytes()
    refine(m, [0], obs, intr, RefinementConfig(iterations=0))
    assert m.surfels.colors.tobytes() == c0 and m.surfels.opacities.tobytes() == o0


def test_refine_untargeted_untouched_and_stationary():
    m, intr, rng = small_map(2)
    m.surfels.colors = np.clip(m.surfels.colors + rng.uniform(-0.2, 0.2, m.surfels.colors.shape), 0, 1)
    outside = m.surfels.keyframe_ids == 6
    before = m.surfels.colors[outside].copy()
    obs = observations(m, intr, [0])
    obs = {0: (np.clip(obs[0][0] + 0.05, 0, 1), obs[0][1])}
    refine(m, [0], obs, intr, RefinementConfig(iterations=3))
    assert np.array_equal(m.surfels.colors[outside], before)
    # targets = the map's own renders: exact stationary point (no accepted step changes the loss)
    m2, intr2, _ = small_map(3)
    own = {}
    for f in (0, 6):
        b = R.render(m2.surfels, m2.keyframe_poses[f], intr2)
        own[f] = (b.color, b.depth)
    rep = refine(m2, [0, 6], own, intr2, RefinementConfig(iterations=3, loss=R.LossWeights(1.0, 0.0)))
    assert len(rep.losses) <= 1 or rep.losses[-1] - rep.losses[0] < 1e-10


def _c4_small(seed=0, views=4):
    sc = scenes.config4(seed, n_keyframes=2, per_keyframe=20_000, n_views=views)
    dev = torch.device("cuda", 0)
    import bench
    rgbs, deps = bench.render_targets(sc, dev)
    return sc, rgbs, deps


def test_adam_refiner_grads_are_sum_of_views_and_step_matches_oracle_adam():
    sc, rgbs, deps = _c4_small(0, 3)
    ref = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss("mse", 1.0, 0.1, True),
                      AdamConfig())
    ref.compute_grads()
    torch.cuda.synchronize()
    total = ref.grads.double().cpu().numpy().copy()
    acc = np.zeros_like(total)
    for v, pose in enumerate(sc.poses):
        run = Run(sc.extra["perturbed"], pose, sc.intr, normal=False, argmax=False)
        g, _ = run.backward("mse", rgbs[v].cpu().numpy(), deps[v].cpu().numpy(), 1.0, 0.1, True)
        acc += np.concatenate([g[k].ravel() for k in ("means", "quats", "scales", "opacities", "colors")])
    ok, mx, l2 = gate(total, acc, tol=1e-5)
    assert ok, (mx, l2)
    # one fused Adam step vs the float64 oracle Adam on the same gradients
    p0 = ref.params.double().cpu().numpy().copy()
    ref.step()
    p = p0.copy()
    g = ref.grads.double().cpu().numpy()
    m1 = np.zeros_like(p)
    m2 = np.zeros_like(p)
    O.adam_step(p, g, m1, m2, 1, 1e-3, 5e-3, 0.9, 0.999, 1e-8, 1e-7)
    got = ref.params.double().cpu().numpy()
    assert np.max(np.abs(got - p)) <= 2e-6, np.max(np.abs(got - p))


def test_adam_refiner_loss_decreases_and_mask_freezes():
    sc, rgbs, deps = _c4_small(1, 4)
    n = len(sc.surfels)
    mask = np.zeros(n, bool)
    mask[: n // 2] = True
    ref = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(), mask=mask)
    frozen0 = ref.params.view(13, -1) if False else None
    P0 = {k: v.clone() for k, v in unpack_params(ref.params, n).items()}
    losses = [ref.step() for _ in range(8)]
    assert losses[-1] < losses[0]
    P1 = unpack_params(ref.params, n)
    for k in P0:
        assert torch.equal(P0[k][n // 2:], P1[k][n // 2:]), k
        assert not torch.equal(P0[k][: n // 2], P1[k][: n // 2]), k
    q = P1["quats"][: n // 2]
    assert torch.allclose(q.norm(dim=1), torch.ones_like(q[:, 0]), atol=1e-5)
    assert float(P1["opacities"].min()) >= 0 and float(P1["opacities"].max()) <= 1
    assert frozen0 is None


def test_host_target_path_matches_device_path():
    sc, rgbs, deps = _c4_small(2, 3)
    a = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps)
    b = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, [r.cpu() for r in rgbs], [d.cpu() for d in deps],
                    host_targets=True)
    assert b.h2d_bytes_per_step == sum(r.numel() + d.numel() for r, d in zip(rgbs, deps)) * 4
    for _ in range(3):
        la, lb = a.step(), b.step()
        assert abs(la - lb) <= 1e-6 * abs(la)
    # float atomics reorder sums; Adam maps a near-zero gradient's sign to a full lr step, so
    # compare statistically: almost all parameters agree to 1e-6, none by more than 3 steps
    d = (a.params - b.params).abs()
    assert float((d > 1e-6).float().mean()) < 1e-3
    assert float(d.max()) <= 3 * 2 * 5e-3


def test_host_target_path_with_cuda_graph():
    """The bench's end-to-end configuration: host targets uploaded on the copy stream inside a
    captured step, each view's fused raster kernel waiting on its own upload event, queued
    steps; the losses follow the device-target run."""
    sc, rgbs, deps = _c4_small(2, 4)
    a = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, inflight=2)
    b = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, [r.cpu() for r in rgbs], [d.cpu() for d in deps],
                    host_targets=True, inflight=2, cuda_graph=True)
    assert b.fused
    la = [a.step() for _ in range(4)]
    for _ in range(4):
        b.step(sync=False)
    lb = b.losses()
    assert np.allclose(la, lb, rtol=1e-5), (la, lb)


def test_sharded_optimizer_path_on_nccl_world_of_one():
    """The N > 1 optimizer path (reduce-scatter -> fused Adam on the shard -> all-gather) run
    through NCCL on a one-rank group equals the replicated path (up to the order of the
    float32 gradient atomics)."""
    import os
    import socket
    import torch.distributed as dist
    sc, rgbs, deps = _c4_small(2, 3)
    n = len(sc.surfels)
    mask = np.arange(n) % 5 != 0
    plain = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(), mask=mask)
    l_plain = [plain.step() for _ in range(3)]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        sh = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(), mask=mask,
                         shard_optimizer=True)
        assert sh.sharded
        l_sh = [sh.step() for _ in range(3)]
        torch.cuda.synchronize()
        assert np.allclose(l_sh, l_plain, rtol=1e-6)
        # (gradient atomics sum in a run-dependent order; compare in norm, see the graph test)
        assert float(torch.linalg.norm(sh.params - plain.params) / torch.linalg.norm(plain.params)) < 1e-4
    finally:
        dist.destroy_process_group()


def test_cuda_graph_step_matches_eager_and_regrows():
    """AdamRefiner(cuda_graph=True): one graph replay per step gives the eager steps' results;
    a pair-capacity overflow inside a replay is detected, the capacity regrown and the graph
    captured again."""
    sc, rgbs, deps = _c4_small(3, 4)
    eager = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig())
    l_e = [eager.step() for _ in range(4)]
    graph = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(),
                        cuda_graph=True)
    l_g = [graph.step() for _ in range(2)]
    graph._reserve(2048)  # too small: the next replay overflows and must be re-run
    graph._graph = None
    l_g += [graph.step() for _ in range(2)]
    assert graph._graph is not None and graph.kernel_launches > 0
    assert np.allclose(l_g, l_e, rtol=1e-5)
    # gradient atomics sum in a run-dependent order, and Adam turns a sign flip of a ~0
    # gradient into a full lr step: compare the parameter blocks in norm
    assert float(torch.linalg.norm(graph.params - eager.params) / torch.linalg.norm(eager.params)) < 1e-4


def test_shard_major_layout_forward_backward():
    """s2d_view_set_layout: a view rendered from the shard-major packed block (3 shards of
    c < n surfels, the N > 1 optimizer layout) gives the plain block's images bit for bit, and
    its gradient block is the plain one in shard-major order."""
    import ctypes
    from paper_2604_03092_b200 import _native as N
    from paper_2604_03092_b200.distributed import from_shard_major, to_shard_major
    from paper_2604_03092_b200.engine import (DeviceContext, ImageBuffers, View, camera_struct, config_struct,
                                              forward_checked, pack_params)
    from paper_2604_03092_b200.rasterizer import DEFAULT_RASTER_CONFIG, loss_struct
    sc, rgbs, deps = _c4_small(4, 1)
    surf = sc.extra["perturbed"]
    n = len(surf)
    c = (n + 2) // 3
    ctx = DeviceContext.get()
    plain = pack_params(surf, ctx.device)
    sm = to_shard_major(plain, n, c)
    assert sm.numel() == 13 * 3 * c
    out = []
    for params, layout in ((plain, 0), (sm, c)):
        v = View(ctx)
        N.check(N.lib().s2d_view_set_layout(v.handle, layout), "s2d_view_set_layout")
        img = ImageBuffers.allocate(sc.intr.height, sc.intr.width, ctx.device, normal=True)
        forward_checked(v, params, n, sc.poses[0], camera_struct(sc.intr), config_struct(DEFAULT_RASTER_CONFIG), img)
        g = torch.zeros_like(params)
        v.backward(params, n, img, loss_struct(N.LOSS_L1, 1.0, 0.1, False, rgbs[0], deps[0]), g)
        torch.cuda.synchronize()
        out.append((img, g))
    for k in ("color", "depth", "accumulation", "normal"):
        assert torch.equal(getattr(out[0][0], k), getattr(out[1][0], k)), k
    g_plain, g_sm = out[0][1], from_shard_major(out[1][1], n, c)
    ok, mx, l2 = gate(g_sm.double().cpu().numpy(), g_plain.double().cpu().numpy(), 1e-6)
    assert ok, (mx, l2)
    # the padding of the last shard receives no gradient
    assert torch.equal(to_shard_major(g_sm, n, c), out[1][1])


def test_async_steps_match_synchronous_steps():
    """step(sync=False) queues iterations without a host round trip; losses() returns the same
    values as synchronous steps, including across an overflow that the device skipped and the
    host re-ran one iteration later."""
    sc, rgbs, deps = _c4_small(5, 3)
    a = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, cuda_graph=True)
    la = [a.step() for _ in range(5)]
    b = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, cuda_graph=True)
    for k in range(5):
        if k == 2:
            b._reserve(2048)  # too small: the device skips this iteration's Adam step
            b._graph = None
        b.step(sync=False)
    lb = b.losses()
    assert b.regrows >= 1 and b.step_count == 5 and len(lb) == 5
    assert np.allclose(la, lb, rtol=1e-5), (la, lb)
