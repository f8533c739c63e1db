"""INTEGRATION.md §2 run verbatim: the reference-side ctypes stub over s2d_render_host (float64
host arrays in and out) against the reference's golden vectors.  The stub imports
``surfelslam.rasterizer``; on the GPU box (no reference sources) that module is provided by
the drop-in's own types (the same names: RenderBuffers, SurfelArrays, _as_camera_packed)."""
import os
import re
import sys
import types

import numpy as np
import pytest

from conftest import GOLDEN_NAMES, ROOT
from gpu_helpers import gate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stub():
    from paper_2604_03092_b200 import _native
    from paper_2604_03092_b200 import rasterizer as R
    from paper_2604_03092_b200.geometry import as_packed_pose
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# pkg/src/surfelslam/_raster_b200\.py\n.*?)```", text, re.S).group(1)
    fake_pkg = types.ModuleType("surfelslam")
    fake = types.ModuleType("surfelslam.rasterizer")
    fake.RenderBuffers = R.RenderBuffers
    fake.SurfelArrays = R.SurfelArrays
    fake._as_camera_packed = as_packed_pose
    saved = {k: sys.modules.get(k) for k in ("surfelslam", "surfelslam.rasterizer")}
    sys.modules["surfelslam"], sys.modules["surfelslam.rasterizer"] = fake_pkg, fake
    os.environ["S2D_LIB"] = _native.LIB_PATH
    ns = {"__name__": "surfelslam._raster_b200"}
    try:
        exec(compile(block, "INTEGRATION.md:_raster_b200.py", "exec"), ns)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return ns


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_stub_render_vs_reference_goldens(stub, goldens, name):
    g = goldens[name]
    buf = stub["render"](g.surfels, g.pose, g.intr, g.cfg)
    assert buf.degenerate_skipped == int(g["degenerate"])
    for key in ("color", "depth", "accumulation"):
        ok, mx, l2 = gate(getattr(buf, key), g[key])
        assert ok, (key, mx, l2)


def test_stub_errors_and_empty(stub, goldens):
    from paper_2604_03092_b200.rasterizer import SurfelArrays
    g = goldens["c1"]
    bad = types.SimpleNamespace(fx=-1.0, fy=100.0, cx=64.0, cy=48.0, width=128, height=96)
    with pytest.raises(ValueError):
        stub["render"](g.surfels, g.pose, bad, g.cfg)
    e = stub["render"](SurfelArrays.empty(), g.pose, g.intr, g.cfg)
    assert not e.color.any() and not e.accumulation.any() and e.degenerate_skipped == 0
