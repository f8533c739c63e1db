"""Backward step statistics of one config-4 view (diagnostic build only: -DS2D_DIAG): guard_hits =
steps of the column-half split, degenerate = steps of a row-quarter split, n_mask = steps of a row-half
split, pairs_stored = entries (the counters are repurposed in that build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.mapper import AdamRefiner, ViewLoss, AdamConfig
import bench

sc = scenes.config4(0)
sc.poses = sc.poses[12:13]
rgbs, deps = bench.render_targets(sc, torch.device("cuda", 0))
ref = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig())
ref.cuda_graph = False
ref.step()
torch.cuda.synchronize()
st = ref.view.stats()
print({k: getattr(st, k) for k, _ in st._fields_})
