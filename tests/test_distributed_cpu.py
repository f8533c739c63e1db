"""N>1 host path on CPU: world_size-2 gloo processes shard the views, compute per-view
gradients (CPU oracle stands in for the device kernels), all-reduce them with the same
distributed.allreduce_grads the GPU path uses, and take identical Adam steps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views():
    from paper_2604_03092_b200 import scenes
    from paper_2604_03092_b200.geometry import Sim3Transform, UnitQuaternion
    sc = scenes.config1(0)
    rng = np.random.default_rng(9)
    poses = [Sim3Transform(1.0, UnitQuaternion.from_axis_angle(rng.normal(size=3), rng.uniform(0, 0.05)),
                           rng.normal(0, 0.05, 3)) for _ in range(5)]
    return sc, poses


def _packed_grads(sc, pose, seed):
    import oracle as O
    buf = O.render(sc.surfels, pose, sc.intr)
    rng = np.random.default_rng(seed)
    trgb = np.clip(buf.color + rng.normal(0, .05, buf.color.shape), 0, 1)
    tdep = buf.depth + rng.normal(0, .05, buf.depth.shape)
    loss, g, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, "l1", 1.0, 0.1, mask_depth=False)
    flat = np.concatenate([g.means.ravel(), g.quats.ravel(), g.scales.ravel(), g.opacities.ravel(),
                           g.colors.ravel()])
    return flat, loss


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_03092_b200.distributed import allreduce_grads, shard_views
    import oracle as O
    sc, poses = _views()
    n = len(sc.surfels)
    grads = torch.zeros(13 * n, dtype=torch.float64)
    loss = torch.zeros(1, dtype=torch.float64)
    for v in shard_views(len(poses), rank, world):
        g, l = _packed_grads(sc, poses[v], v)
        grads += torch.from_numpy(g)
        loss += l
    allreduce_grads(grads, loss)
    s = sc.surfels
    p = np.concatenate([s.means.ravel(), s.quats.ravel(), s.scales.ravel(), s.opacities.ravel(), s.colors.ravel()])
    m1 = np.zeros_like(p)
    m2 = np.zeros_like(p)
    O.adam_step(p, grads.numpy().copy(), m1, m2, 1)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), grads=grads.numpy(), loss=loss.numpy(), params=p)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_process(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    sc, poses = _views()
    ref = None
    ref_loss = 0.0
    for v in range(len(poses)):
        g, l = _packed_grads(sc, poses[v], v)
        ref = g if ref is None else ref + g
        ref_loss += l
    r0 = np.load(tmp_path / "r0.npz")
    r1 = np.load(tmp_path / "r1.npz")
    assert np.array_equal(r0["grads"], r1["grads"])
    assert np.array_equal(r0["params"], r1["params"])
    assert np.allclose(r0["grads"], ref, rtol=1e-12, atol=1e-15)
    assert abs(float(r0["loss"][0]) - ref_loss) <= 1e-12 * ref_loss


def _sharded_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_03092_b200.distributed import (ShardedOptimizerState, allreduce_grads, from_shard_major,
                                                   shard_views, sharded_step, to_shard_major)
    import oracle as O
    sc, poses = _views()
    n = len(sc.surfels)
    grads = torch.zeros(13 * n, dtype=torch.float64)
    loss = torch.zeros(1, dtype=torch.float64)
    for v in shard_views(len(poses), rank, world):
        g, l = _packed_grads(sc, poses[v], v)
        grads += torch.from_numpy(g)
        loss += l
    allreduce_grads(loss)
    s = sc.surfels
    params = torch.from_numpy(np.concatenate([s.means.ravel(), s.quats.ravel(), s.scales.ravel(),
                                              s.opacities.ravel(), s.colors.ravel()]))
    mask = torch.from_numpy((np.arange(n) % 7 != 0).astype(np.uint8))
    state = ShardedOptimizerState(n, dtype=torch.float64, mask=mask)
    assert state.m1.numel() == 13 * state.c < 13 * n
    # the shard-major layout (s2d_view_set_layout): one contiguous slice per rank
    params = to_shard_major(params, n, state.c)
    grads = to_shard_major(grads, n, state.c)
    assert params.numel() == 13 * world * state.c

    def adam_fn(p, g, m1, m2, c, smask):
        O.adam_step(p.numpy(), g.numpy(), m1.numpy(), m2.numpy(), step[0],
                    mask=None if smask is None else smask.numpy().astype(bool))

    for k in range(3):
        step = [k + 1]
        sharded_step(params, grads.clone(), state, adam_fn)
    params = from_shard_major(params, n, state.c)
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), params=params.numpy(), loss=loss.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_optimizer_matches_replicated_adam(tmp_path, world):
    """One reduce-scatter -> Adam on each rank's contiguous surfel shard -> one all-gather, on the
    shard-major packed blocks, == the replicated step (bit-exact in float64), with a surfel mask
    and an uneven (zero-padded) last shard."""
    mp.start_processes(_sharded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    import oracle as O
    sc, poses = _views()
    n = len(sc.surfels)
    ref = None
    for v in range(len(poses)):
        g, _ = _packed_grads(sc, poses[v], v)
        ref = g if ref is None else ref + g
    s = sc.surfels
    p = np.concatenate([s.means.ravel(), s.quats.ravel(), s.scales.ravel(), s.opacities.ravel(), s.colors.ravel()])
    m1 = np.zeros_like(p)
    m2 = np.zeros_like(p)
    mask = np.arange(n) % 7 != 0
    for k in range(3):
        O.adam_step(p, ref.copy(), m1, m2, k + 1, mask=mask)
    outs = [np.load(tmp_path / f"s{r}.npz")["params"] for r in range(world)]
    for o in outs:
        assert np.array_equal(o, outs[0])
    assert np.allclose(outs[0], p, rtol=1e-13, atol=1e-15)


def test_shard_major_round_trip():
    from paper_2604_03092_b200.distributed import from_shard_major, to_shard_major
    for n, c in ((10, 4), (7, 7), (9, 3), (5, 100)):
        flat = torch.arange(13 * n, dtype=torch.float64)
        sm = to_shard_major(flat, n, c)
        w = (n + c - 1) // c
        assert sm.numel() == 13 * w * c
        assert torch.equal(from_shard_major(sm, n, c), flat)
        # surfel i of shard s: means at 13 c s + 3 j, colours at 13 c s + 10 c + 3 j
        blk = sm.view(w, 13 * c)
        for i in range(n):
            s_, j = divmod(i, c)
            assert blk[s_, 3 * j + 1] == flat[3 * i + 1]
            assert blk[s_, 10 * c + 3 * j + 2] == flat[10 * n + 3 * i + 2]
            assert blk[s_, 9 * c + j] == flat[9 * n + i]
