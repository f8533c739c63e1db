"""Pin the CPU oracle to the reference: golden vectors were produced by running the
reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN_NAMES, max_rel


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_projection_bit_exact(goldens, name):
    g = goldens[name]
    p = O.project(g.surfels, g.pose, g.intr, g.cfg)
    valid = g["valid"]
    # rasterizer.py:201-249 — z for all surfels, the rest where the reference marks valid
    assert np.array_equal(p.z, g["z"])
    assert np.array_equal(p.in_front, g["in_front"])
    assert np.array_equal(p.valid, valid)
    assert p.degenerate == int(g["degenerate"])
    assert np.array_equal(p.centers[valid], g["centers"][valid])
    assert np.array_equal(p.cov2[valid], g["cov2"][valid])
    assert np.array_equal(p.inv_abc[valid], g["inv_abc"][valid])
    # _footprint_boxes (rasterizer.py:262-281)
    on = g["on_screen"]
    assert np.array_equal(p.on_screen, on)
    assert np.array_equal(p.bbox[on], g["bbox"][on])


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_depth_order_exact(goldens, name):
    g = goldens[name]
    p = O.project(g.surfels, g.pose, g.intr, g.cfg)
    assert np.array_equal(O.depth_order(p), g["order"])


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_tile_lists_match_definition(goldens, name):
    """tiles(i) from the reference bbox, each tile's list = the reference order restricted to it."""
    g = goldens[name]
    p = O.project(g.surfels, g.pose, g.intr, g.cfg)
    start, ids = O.tile_lists(p, g["order"], g.intr)
    T = 16
    ntx = (g.intr.width + T - 1) // T
    nty = (g.intr.height + T - 1) // T
    lists = [[] for _ in range(ntx * nty)]
    for i in g["order"]:
        x0, x1, y0, y1 = g["bbox"][i]
        if x0 > x1 or y0 > y1:
            continue
        for ty in range(y0 // T, y1 // T + 1):
            for tx in range(x0 // T, x1 // T + 1):
                lists[ty * ntx + tx].append(i)
    flat = np.array([i for l in lists for i in l], dtype=np.int64)
    assert np.array_equal(ids, flat)
    assert np.array_equal(np.diff(start), [len(l) for l in lists])


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_forward_images(goldens, name):
    g = goldens[name]
    b = O.render(g.surfels, g.pose, g.intr, g.cfg)
    f64 = g["color"].dtype == np.float64
    for key in ("color", "depth", "accumulation", "max_w"):
        ref = getattr(b, key)
        if f64:
            assert np.array_equal(ref, g[key]), key
        else:
            assert max_rel(ref.astype(np.float32), g[key]) <= 1e-6, key
    assert np.array_equal(b.arg_w, g["arg_w"])
    assert b.degenerate_skipped == int(g["degenerate_skipped"])


GRAD_NAMES = [n for n in GOLDEN_NAMES if n in ("kat_random40", "c1", "c1_posed")]


@pytest.mark.parametrize("name", GRAD_NAMES)
def test_color_opacity_gradients(goldens, name):
    g = goldens[name]
    w = g["loss_weights"]
    loss, gr, _ = O.loss_and_grads(g.surfels, g.pose, g.intr, g["target_rgb"], g["target_depth"], "mse",
                                   float(w[0]), float(w[1]), cfg=g.cfg)
    assert np.array_equal(gr.colors, g["grad_color"])
    assert np.array_equal(gr.opacities, g["grad_opacity"])
    assert abs(loss - float(g["loss"])) <= 1e-12 * abs(float(g["loss"]))


@pytest.mark.parametrize("name", GRAD_NAMES)
def test_max_blend_weights(goldens, name):
    g = goldens[name]
    ma, mm = O.max_blend_weights(g.surfels, g.pose, g.intr, g["mw_mask"], g.cfg)
    assert np.array_equal(ma, g["max_all"])
    assert np.array_equal(mm, g["max_marked"])


def test_known_answers(goldens):
    """Analytic known answers the reference's tests assert (test_rasterizer.py:105-186)."""
    g = goldens["kat_two_exact"]
    b = O.render(g.surfels, g.pose, g.intr, g.cfg)
    c1, c2 = np.array([0.9, 0.1, 0.2]), np.array([0.0, 0.8, 0.4])
    assert np.allclose(b.color[24, 32], 0.5 * c1 + 0.25 * c2, atol=1e-12)
    assert abs(b.accumulation[24, 32] - 0.75) <= 1e-12
    assert abs(b.depth[24, 32] - (0.5 * 1.0 + 0.25 * 2.0)) <= 1e-12
    e = goldens["kat_edge"]
    be = O.render(e.surfels, e.pose, e.intr, e.cfg)
    assert be.degenerate_skipped == 1 and not be.accumulation.any()
