"""N > 1 NCCL ranks on one node (skipped with fewer than 2 GPUs): view-sharded AdamRefiner with
the sharded optimizer (shard-major blocks, one reduce-scatter + one in-place all-gather per
iteration) against the single-process run of all views."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from paper_2604_03092_b200 import scenes
    return scenes.config4(3, n_keyframes=2, per_keyframe=30_000, n_views=6)


def _targets(sc, dev):
    import bench
    return bench.render_targets(sc, dev)


def _worker(rank, port, out):
    import torch.distributed as dist
    from paper_2604_03092_b200.mapper import AdamConfig, AdamRefiner, ViewLoss
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD)
    dev = torch.device("cuda", rank)
    sc = _scene()
    rgbs, deps = _targets(sc, dev)
    ref = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(), device=dev,
                      inflight=3, cuda_graph=True)
    assert ref.sharded and ref.shard < ref.n
    for _ in range(3):
        ref.step(sync=False)
    losses = ref.losses()
    if rank == 0:
        np.savez(out, losses=np.array(losses), params=ref.plain_params().double().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < WORLD, reason="needs 2 GPUs")
def test_two_nccl_ranks_match_one_process(tmp_path):
    out = str(tmp_path / "r0.npz")
    mp.start_processes(_worker, args=(_port(), out), nprocs=WORLD, start_method="spawn")
    from paper_2604_03092_b200.mapper import AdamConfig, AdamRefiner, ViewLoss
    dev = torch.device("cuda", 0)
    sc = _scene()
    rgbs, deps = _targets(sc, dev)
    one = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(), device=dev)
    l1 = [one.step() for _ in range(3)]
    r = np.load(out)
    assert np.allclose(r["losses"], l1, rtol=1e-5)
    p1 = one.plain_params().double().cpu().numpy()
    assert np.linalg.norm(r["params"] - p1) / np.linalg.norm(p1) < 1e-4
