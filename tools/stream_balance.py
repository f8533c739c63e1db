"""Work balance of the backward's column halves: per (tile, warp block) the two half streams are
walked in step, so a warp takes max(n0, n1) steps for n0 + n1 entries.  Prints the half-entry
slot utilisation sum(n0 + n1) / (2 sum max(n0, n1)) for config-4 views (two-kernel forward)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2604_03092_b200.engine import (DeviceContext, ImageBuffers, View, camera_struct, config_struct,
                                          forward_checked, pack_params)
from paper_2604_03092_b200.rasterizer import DEFAULT_RASTER_CONFIG

dev = torch.device("cuda", 0)
sc = bench.make_workload(0, False, 4)
ctx = DeviceContext.get(dev)
view = View(ctx)
params = pack_params(sc.extra["perturbed"], dev)
img = ImageBuffers.allocate(sc.intr.height, sc.intr.width, dev, normal=False)
for v in (0, 12, 31):
    forward_checked(view, params, len(sc.surfels), sc.poses[v], camera_struct(sc.intr),
                    config_struct(DEFAULT_RASTER_CONFIG), img)
    d = view.inspect()
    sl = d["stream_lengths"].long()
    n0, n1 = sl[..., 0], sl[..., 1]
    e = int((n0 + n1).sum()); steps = int(torch.maximum(n0, n1).sum())
    both = int(((n0 > 0) & (n1 > 0)).sum()); blocks = int(((n0 + n1) > 0).sum())
    nb = int((d["pixel_state"][:, 0] & ((1 << 29) - 1)).long().sum())
    print(f"view {v}: blended (pixel, surfel) pairs {nb}, lanes used per half-entry {nb / e:.2f} of 16")
    print(f"view {v}: entries {e}, warp steps {steps}, slot use {e / (2 * steps):.3f}, "
          f"blocks with work {blocks}, both halves {both}, mean |n0-n1| {float((n0 - n1).abs().float().mean()):.1f}")
