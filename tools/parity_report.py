"""Print GPU-vs-oracle parity numbers for configs 1-3 (diagnostic; needs a GPU)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2604_03092_b200 import rasterizer as R, scenes
from paper_2604_03092_b200.engine import DeviceContext, pack_params, ImageBuffers, camera_struct, config_struct, forward_checked


def rel(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    m = max(np.abs(b).max(), 1e-30)
    return np.abs(a - b).max() / m, np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def binning_check(sc, pose):
    ctx = DeviceContext.get()
    v = ctx.thread_view()
    params = pack_params(sc.surfels)
    n = len(sc.surfels)
    img = ImageBuffers.allocate(sc.intr.height, sc.intr.width, ctx.device)
    st = forward_checked(v, params, n, pose, camera_struct(sc.intr), config_struct(R.DEFAULT_RASTER_CONFIG), img)
    d = v.inspect()
    P = O.project(sc.surfels, pose, sc.intr)
    order = O.depth_order(P)
    start, ids = O.tile_lists(P, order, sc.intr)
    on = P.on_screen
    flags = d["flags"].cpu().numpy()
    bbox = d["bbox"].cpu().numpy().astype(np.int64)
    z = d["z"].cpu().numpy()
    res = {
        "V": (st.visible, int(on.sum())),
        "degenerate": (st.degenerate, P.degenerate),
        "flags_eq": bool(np.array_equal(flags, P.flags)),
        "bbox_eq": bool(np.array_equal(bbox[on], P.bbox[on])),
        "z_eq": bool(np.array_equal(z[on], P.z[on])),
        "order_eq": bool(np.array_equal(d["order"].cpu().numpy().astype(np.int64), order)),
        "pairs": (st.pairs, len(ids)),
        "pairs_eq": bool(np.array_equal(d["pair_ids"].cpu().numpy().astype(np.int64), ids)),
        "guard_hits": st.guard_hits,
    }
    rg = d["ranges"].cpu().numpy()
    res["ranges_eq"] = bool(np.array_equal(rg[:, 0][rg[:, 1] > rg[:, 0]], start[:-1][start[1:] > start[:-1]]))
    return res


def main():
    for name, sc in [("c1", scenes.config1(0)), ("c2", scenes.config2(0)), ("c3", scenes.config3(0))]:
        pose = sc.poses[-1]
        t0 = time.time()
        print(name, "binning", binning_check(sc, pose))
        buf = R.render(sc.surfels, pose, sc.intr)
        ref = O.render(sc.surfels, pose, sc.intr)
        for f in ("color", "depth", "accumulation", "normal"):
            print(f"  {name} {f:13s} max-rel {rel(getattr(buf, f), getattr(ref, f))[0]:.3e}  l2-rel {rel(getattr(buf, f), getattr(ref, f))[1]:.3e}")
        rng = np.random.default_rng(5)
        trgb = np.clip(ref.color + rng.normal(0, 0.05, ref.color.shape), 0, 1)
        tdep = ref.depth + rng.normal(0, 0.05, ref.depth.shape)
        for kind, mask in (("mse", True), ("l1", False)):
            g, loss = R.grad_all(sc.surfels, pose, sc.intr, trgb, tdep, kind=kind, w_rgb=1.0, w_depth=0.1, depth_mask=mask)
            ol, og, _ = O.loss_and_grads(sc.surfels, pose, sc.intr, trgb, tdep, kind, 1.0, 0.1, mask_depth=mask)
            print(f"  {name} {kind} loss {loss:.8e} oracle {ol:.8e} rel {abs(loss-ol)/abs(ol):.2e}")
            for f in ("colors", "opacities", "means", "quats", "scales"):
                a, b = rel(g[f], getattr(og, f))
                print(f"    grad {f:10s} max-rel {a:.3e} l2-rel {b:.3e}")
        print(f"  {name} took {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
