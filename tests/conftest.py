"""Shared fixtures.  `-m "not gpu"` runs the CPU suite (oracle vs golden vectors, host logic,
C-ABI symbol checks, gloo multi-process); `-m gpu` runs the parity tests through the C ABI."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity through the C ABI")
    config.addinivalue_line("markers", "slow: longer-running test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


GOLDEN_NAMES = ["kat_two_exact", "kat_edge", "kat_occluder_exact", "kat_occluder_clamp", "kat_random40", "c1",
                "c1_posed", "c2"]


class G:
    """Golden record adapter: surfels / pose / intrinsics / config objects from the npz."""

    def __init__(self, name):
        from paper_2604_03092_b200.rasterizer import CameraIntrinsics, RasterConfig, SurfelArrays
        self.name = name
        self.d = load_golden(name)
        d = self.d
        self.surfels = SurfelArrays(d["means"], d["quats"], d["scales"], d["opacities"], d["colors"])
        self.pose = d["pose"]
        fx, fy, cx, cy, w, h = d["intr"]
        self.intr = CameraIntrinsics(fx, fy, cx, cy, int(w), int(h))
        c = d["cfg"]
        self.cfg = RasterConfig(*[float(x) for x in c])

    def __getitem__(self, k):
        return self.d[k]

    def __contains__(self, k):
        return k in self.d


@pytest.fixture(scope="session")
def goldens():
    return {n: G(n) for n in GOLDEN_NAMES}


def reference_available():
    return os.path.isdir(os.path.join(REFERENCE_SRC, "surfelslam"))


def max_rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if b.size else 0.0


def l2_rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)) if b.size else 0.0
