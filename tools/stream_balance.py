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

# quarter streams (4x2 pixel groups: column half x row pair) instead of column halves: entries
# per quarter and the warp steps if the four quarters walked their own streams in step
print("quarter-stream estimate:")
for v in (0, 12, 31):
    forward_checked(view, params, len(sc.surfels), sc.poses[v], camera_struct(sc.intr),
                    config_struct(DEFAULT_RASTER_CONFIG), img)
    d = view.inspect()
    sl = d["stream_lengths"].long().reshape(-1)            # (ntiles*16,)
    rg = d["ranges"].long()                                # (ntiles, 2)
    ln = (rg[:, 1] - rg[:, 0]).clamp(min=0)
    t = torch.arange(rg.shape[0], device=dev).repeat_interleave(16)
    wh = torch.arange(16, device=dev).repeat(rg.shape[0])
    start = 16 * rg[t, 0] + wh * ln[t]
    seg = torch.arange(sl.numel(), device=dev).repeat_interleave(sl)
    first = torch.cumsum(sl, 0) - sl
    idx = start[seg] + (torch.arange(seg.numel(), device=dev) - first[seg])
    mask = d["streams"][idx, 1].long() & 0xffffffff
    rp0 = (mask & 0xffff) != 0
    rp1 = (mask >> 16) != 0
    f = float((rp0.long() + rp1.long()).float().mean())
    # per (tile, warp, half, rowpair) counts -> per warp max over the 4 quarters
    q = torch.zeros(sl.numel() * 2, dtype=torch.long, device=dev)
    q.index_add_(0, seg * 2, rp0.long())
    q.index_add_(0, seg * 2 + 1, rp1.long())
    q = q.reshape(-1, 8, 4)   # (tile, warp, half*2 + rowpair)
    steps_q = int(q.max(-1).values.sum())
    h = sl.reshape(-1, 8, 2)
    steps_h = int(h.max(-1).values.sum())
    print(f"view {v}: quarter-entries per half-entry {f:.2f}, warp steps halves {steps_h} quarters {steps_q} "
          f"({steps_h / max(steps_q, 1):.2f}x fewer), quarter slot use {int(q.sum()) / (4 * steps_q):.3f}")
