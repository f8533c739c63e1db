"""Host-side logic and the C ABI surface (no GPU needed)."""
import ctypes

import numpy as np
import pytest
import torch

from conftest import REFERENCE_SRC, reference_available
from paper_2604_03092_b200 import _native as N
from paper_2604_03092_b200 import geometry as Gm
from paper_2604_03092_b200 import rasterizer as R
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.distributed import shard_views


def test_library_exports_every_header_symbol():
    L = N.lib()
    names = N.header_functions()
    assert len(names) >= 15
    missing = [f for f in names if not hasattr(L, f)]
    assert not missing, missing
    assert L.s2d_version() >= 100


def _random_poses(k, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(k):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        out.append(np.concatenate([[rng.uniform(0.3, 3.0)], rng.normal(0, 2, 3), q]))
    return out


def test_pose_inverse_c_abi_bit_exact():
    """s2d_pose_inverse (host float64, -ffp-contract=off) == pk_inverse (numpy order, geometry.py:188-195)."""
    L = N.lib()
    for a in _random_poses(200):
        out = (ctypes.c_double * 8)()
        N.check(L.s2d_pose_inverse(N.as_doubles(a), out))
        assert np.array_equal(np.array(out[:]), Gm.pk_inverse(a))


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_geometry_matches_reference():
    import sys
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    from surfelslam import geometry as RG
    for a in _random_poses(100, 1):
        assert np.array_equal(Gm.pk_inverse(a), RG.pk_inverse(a))
        v = np.random.default_rng(2).normal(size=(7, 3))
        assert np.array_equal(Gm.quat_rotate(np.broadcast_to(a[4:8], (7, 4)), v),
                              RG.quat_rotate(np.broadcast_to(a[4:8], (7, 4)), v))
        assert np.array_equal(Gm.quat_to_matrix(a[4:8] * 1.3), RG.quat_to_matrix(a[4:8] * 1.3))
        b = _random_poses(1, int(a[0] * 1000))[0]
        assert np.array_equal(Gm.quat_mul(a[4:8], b[4:8]), RG.quat_mul(a[4:8], b[4:8]))


def test_c_abi_rejects_bad_arguments_without_gpu():
    L = N.lib()
    cam = N.Camera(-1.0, 10.0, 1.0, 1.0, 4, 4)
    cfg = N.RasterCfg(0.999, 1e-4, 3.0, 1e-3, 1e8, 80.0, 0.5)
    img = N.Image()
    rc = L.s2d_forward(None, None, None, 0, N.as_doubles([1, 0, 0, 0, 1, 0, 0, 0]), ctypes.byref(cam),
                       ctypes.byref(cfg), ctypes.byref(img), None, None, None)
    assert rc == N.S2D_ERR_INVALID
    assert b"NULL" in L.s2d_last_error()
    cfgA = N.AdamCfg(1e-3, 5e-3, 0.9, 0.999, 1e-8, 1e-7)
    assert L.s2d_adam_step(None, None, None, None, None, 10, 0, ctypes.byref(cfgA), None) == N.S2D_ERR_INVALID
    # s2d_forward_backward: no view / no loss / no gradient block
    loss = N.Loss(N.LOSS_L1, 0, 1.0, 0.1, None, None, None, None, None, None)
    pose = N.as_doubles([1, 0, 0, 0, 1, 0, 0, 0])
    assert L.s2d_forward_backward(None, None, None, 0, pose, ctypes.byref(cam), ctypes.byref(cfg), None,
                                  ctypes.byref(loss), None, None, None) == N.S2D_ERR_INVALID
    assert b"NULL" in L.s2d_last_error()


def test_intrinsics_and_surfel_validation():
    """Same ValueErrors as the reference (rasterizer.py:36-40, 66-68)."""
    with pytest.raises(ValueError):
        R.CameraIntrinsics(0.0, 1.0, 1.0, 1.0, 4, 4)
    with pytest.raises(ValueError):
        R.CameraIntrinsics(1.0, 1.0, 4.0, 1.0, 4, 4)
    with pytest.raises(ValueError):
        R.Surfel(np.zeros(3), Gm.UnitQuaternion.identity(), np.array([0.1, 0.0]), 0.5, np.zeros(3))
    s = R.Surfel(np.zeros(3), Gm.UnitQuaternion.identity(), np.array([0.1, 0.1]), 1.7, np.zeros(3))
    assert s.opacity == 1.0
    arr = R.SurfelArrays.from_surfels([s, s])
    assert len(arr) == 2 and arr.quats.shape == (2, 4)


def test_render_loss_host(goldens):
    g = goldens["c1"]
    buf = R.RenderBuffers(g["color"], g["depth"], g["accumulation"])
    w = g["loss_weights"]
    val = R.render_loss(buf, g["target_rgb"], g["target_depth"], R.LossWeights(float(w[0]), float(w[1])))
    assert val == float(g["render_loss"])
    with pytest.raises(ValueError):
        R.render_loss(buf, np.zeros((2, 2, 3)), np.zeros((2, 2)))


def test_product_fails_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = scenes.config1(0)
    with pytest.raises(N.NativeLibraryError):
        R.render(g.surfels, g.poses[0], g.intr)


@pytest.mark.parametrize("nv,ws", [(32, 1), (32, 2), (32, 8), (128, 8), (7, 3), (3, 4)])
def test_shard_views_partition(nv, ws):
    parts = [shard_views(nv, r, ws) for r in range(ws)]
    flat = [v for p in parts for v in p]
    assert flat == list(range(nv))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def test_scene_generators_seeded_and_float32():
    a = scenes.config1(3).surfels
    b = scenes.config1(3).surfels
    assert np.array_equal(a.means, b.means) and np.array_equal(a.quats, b.quats)
    assert np.array_equal(a.means, a.means.astype(np.float32).astype(np.float64))
    c3 = scenes.config3(0)
    assert len(c3.surfels) == 512 * 384 and len(c3.poses) == 8
    assert np.all(np.asarray(c3.surfels.scales) > 0)


def test_bench_spawns_n_ranks_outside_torchrun(monkeypatch):
    """`python bench.py --gpus N` outside torchrun re-launches itself under torch.distributed.run
    with N ranks on one node and a 127.0.0.1 rendezvous (the driver's launch line)."""
    import subprocess
    import sys
    import bench
    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--warmup", "3"])
    monkeypatch.delenv("RANK", raising=False)
    args = bench.parse()
    assert bench.spawn_ranks(args) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]
