"""Map maintenance on the CPU: the float64 oracle restatements of
transform_surfels / fuse / prune pinned against the reference's own outputs
(tests/golden/map_ops.npz, made by tests/golden/make_golden.py), and the surfel PLY writer /
reader (host code) against bytes the reference wrote."""
import os
from types import SimpleNamespace

import numpy as np
import pytest

import oracle as O
from paper_2604_03092_b200 import io as PIO
from paper_2604_03092_b200.rasterizer import SurfelArrays

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(HERE, "golden", "map_ops.npz")))


def _intr(v):
    return SimpleNamespace(fx=v[0], fy=v[1], cx=v[2], cy=v[3], width=int(v[4]), height=int(v[5]))


def _arrays(g, p):
    return SimpleNamespace(means=g[p + "means"], quats=g[p + "quats"], scales=g[p + "scales"],
                           opacities=g[p + "opacities"], colors=g[p + "colors"])


def test_oracle_transform_surfels_bit_exact(g):
    m, q, s = O.transform_surfels(g["tr_means"], g["tr_quats"], g["tr_scales"], g["tr_pose"])
    assert np.array_equal(m, g["tr_out_means"])
    assert np.array_equal(q, g["tr_out_quats"])
    assert np.array_equal(s, g["tr_out_scales"])
    assert not np.signbit(q[:, 0]).any()


def test_oracle_quat_canonicalize_ties():
    q = np.array([[0.0, -0.0, -1.0, 0.0], [-0.0, 0.0, 0.0, -1.0], [-1.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0]])
    c = O.quat_canonicalize(q)
    assert np.array_equal(c, [[0, 0, 1, 0], [0, 0, 0, 1], [1, 0, 0, 0], [0, 0, 0, 0]])
    assert not np.signbit(c).any()
    assert np.array_equal(O.quat_canonicalize(-q), c)


def test_oracle_fuse_vs_reference(g):
    intr = _intr(g["fu_intr"])
    keep, m, q, s = O.fuse(_arrays(g, "fu_map_"), _arrays(g, "fu_cand_"), g["fu_p1"], intr)
    assert int(keep.sum()) == int(g["fu_inserted"])
    assert np.array_equal(m, g["fu_new_means"])
    assert np.array_equal(q, g["fu_new_quats"])
    assert np.array_equal(s, g["fu_new_scales"])
    # the gate alone, on the reference's own accumulation
    assert np.array_equal(O.fuse_gate(g["fu_acc"], g["fu_cand_means"], intr), keep)


def test_oracle_prune_vs_reference(g):
    intr = _intr(g["fu_intr"])
    victims, marked = O.prune(_arrays(g, "pr_map_"), g["pr_p0"], intr, g["pr_obs_rgb"], g["pr_obs_depth"])
    assert np.array_equal(marked, g["pr_marked"])
    assert np.array_equal(victims, g["pr_victims"])
    assert len(victims) > 0 and marked.sum() > 0


def _ply_arrays(g):
    return SurfelArrays(g["ply_means"], g["ply_quats"], g["ply_scales"], g["ply_opacities"], g["ply_colors"],
                        g["ply_conf"], g["ply_kf"], g["ply_submap"])


def test_ply_writer_bytes_equal_reference(g, tmp_path):
    path = tmp_path / "s.ply"
    PIO.write_surfel_ply(path, _ply_arrays(g))
    assert np.array_equal(np.frombuffer(path.read_bytes(), np.uint8), g["ply_bytes"])


def test_ply_reader_reads_reference_file_exactly(g, tmp_path):
    path = tmp_path / "ref.ply"
    path.write_bytes(g["ply_bytes"].tobytes())
    s = PIO.read_surfel_ply(path)
    ref = _ply_arrays(g)
    for f in ("means", "quats", "scales", "opacities", "colors", "confidences", "keyframe_ids", "submap_ids"):
        assert np.array_equal(getattr(s, f), getattr(ref, f)), f
    assert s.keyframe_ids.dtype == np.int64


def test_ply_round_trip_empty_and_errors(tmp_path):
    p = tmp_path / "e.ply"
    PIO.write_surfel_ply(p, SurfelArrays.empty())
    assert len(PIO.read_surfel_ply(p)) == 0
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"not a ply\n")
    with pytest.raises(ValueError):
        PIO.read_surfel_ply(bad)
    trunc = tmp_path / "t.ply"
    trunc.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 0\n")
    with pytest.raises(ValueError):
        PIO.read_surfel_ply(trunc)
    missing = tmp_path / "m.ply"
    missing.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 0\nproperty double x\nend_header\n")
    with pytest.raises(ValueError):
        PIO.read_surfel_ply(missing)
