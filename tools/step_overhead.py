"""Per-step fixed cost of the config-4 refine step: time steps over 16, 32 and 64 views (the
32 views repeated); a linear fit gives the per-view slope and the per-step intercept."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2604_03092_b200.mapper import AdamConfig, AdamRefiner, ViewLoss

dev = torch.device("cuda", 0)
sc = bench.make_workload(0, False, 4)
rgbs, deps = bench.render_targets(sc, dev)
res = []
for nv in (8, 16, 32, 64):
    idx = [i % len(sc.poses) for i in range(nv)]
    ref = AdamRefiner(sc.extra["perturbed"], sc.intr, [sc.poses[i] for i in idx], [rgbs[i] for i in idx],
                      [deps[i] for i in idx], ViewLoss("l1", 1.0, 0.1, False), AdamConfig(), device=dev,
                      inflight=16, cuda_graph=True)
    for _ in range(4):
        ref.step(sync=False)
    ref.losses()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ref.step(sync=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res.append((nv, ms))
    print(f"views {nv}: {ms:.3f} ms/step, {ms / nv:.4f} ms/view", flush=True)
    del ref
    torch.cuda.empty_cache()
x = np.array([r[0] for r in res], float); y = np.array([r[1] for r in res])
a, b = np.polyfit(x, y, 1)
print(f"fit: {a:.4f} ms/view + {b:.3f} ms/step")
