"""Short config-4 refine workload for ncu (profiled region = one refine iteration over 4 views)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_03092_b200 import scenes
from paper_2604_03092_b200.mapper import AdamRefiner, ViewLoss, AdamConfig
import bench

nviews = int(os.environ.get("PROFILE_VIEWS", "4"))
sc = scenes.config5(0) if os.environ.get("PROFILE_CONFIG", "4") == "5" else scenes.config4(0)
first = int(os.environ.get("PROFILE_FIRST", "12"))
sc.poses = sc.poses[first:first + nviews]
rgbs, deps = bench.render_targets(sc, torch.device("cuda", 0))
ref = AdamRefiner(sc.extra["perturbed"], sc.intr, sc.poses, rgbs, deps, ViewLoss(), AdamConfig(),
                  fused=os.environ.get("PROFILE_FUSED", "1") == "1")
for _ in range(2):
    ref.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ref.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profile_view done")
