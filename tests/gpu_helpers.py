"""Helpers shared by the GPU tests (call the product through the C ABI)."""
import numpy as np
import torch

from paper_2604_03092_b200 import _native as N
from paper_2604_03092_b200.engine import (DeviceContext, ImageBuffers, View, camera_struct, config_struct,
                                          forward_checked, pack_params, unpack_params)
from paper_2604_03092_b200.rasterizer import DEFAULT_RASTER_CONFIG


class Run:
    """One forward (and optionally backward) of a scene on the GPU, with introspection."""

    def __init__(self, surfels, pose, intr, cfg=DEFAULT_RASTER_CONFIG, normal=True, argmax=True, view=None):
        self.ctx = DeviceContext.get()
        self.dev = self.ctx.device
        self.view = view or View(self.ctx)
        self.n = len(surfels)
        self.params = pack_params(surfels, self.dev) if self.n else torch.zeros(13, device=self.dev)
        self.intr = intr
        self.img = ImageBuffers.allocate(intr.height, intr.width, self.dev, normal=normal, argmax=argmax)
        self.stats = forward_checked(self.view, self.params, self.n, pose, camera_struct(intr), config_struct(cfg),
                                     self.img)

    def images(self):
        out = {k: getattr(self.img, k).double().cpu().numpy() for k in ("color", "depth", "accumulation")}
        if self.img.normal is not None:
            out["normal"] = self.img.normal.double().cpu().numpy()
        if self.img.arg_w is not None:
            out["arg_w"] = self.img.arg_w.cpu().numpy().astype(np.int64)
            out["max_w"] = self.img.max_w.double().cpu().numpy()
        return out

    def inspect(self):
        return self.view.inspect()

    def backward(self, kind="mse", trgb=None, tdep=None, w_rgb=1.0, w_depth=0.05, depth_mask=True,
                 d_color=None, d_depth=None, d_normal=None, d_acc=None):
        grads = torch.zeros_like(self.params)
        loss = torch.zeros(1, dtype=torch.float64, device=self.dev)
        t = lambda a: None if a is None else torch.as_tensor(np.asarray(a, dtype=np.float32)).to(self.dev)  # noqa: E731
        keep = [t(trgb), t(tdep), t(d_color), t(d_depth), t(d_normal), t(d_acc)]
        code = {"mse": N.LOSS_MSE, "l1": N.LOSS_L1, "external": N.LOSS_EXTERNAL}[kind]
        ls = N.Loss(code, int(depth_mask), float(w_rgb), float(w_depth), *[N.dptr(k) for k in keep])
        self.view.backward(self.params, self.n, self.img, ls, grads, loss)
        torch.cuda.synchronize()
        g = {k: v.double().cpu().numpy() for k, v in unpack_params(grads, self.n).items()}
        return g, float(loss.item())


def fused_grads(surfels, pose, intr, kind, trgb, tdep, w_rgb=1.0, w_depth=0.1, depth_mask=False,
                cfg=DEFAULT_RASTER_CONFIG, image=False, view=None):
    """Loss and gradients through s2d_forward_backward (one raster kernel for the losses
    without the depth mask).  Returns (grads dict, loss, images dict or None, stats)."""
    ctx = DeviceContext.get()
    dev = ctx.device
    view = view or View(ctx)
    n = len(surfels)
    params = pack_params(surfels, dev) if n else torch.zeros(13, device=dev)
    grads = torch.zeros_like(params)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32)).to(dev)  # noqa: E731
    keep = [t(trgb), t(tdep)]
    code = {"mse": N.LOSS_MSE, "l1": N.LOSS_L1}[kind]
    ls = N.Loss(code, int(depth_mask), float(w_rgb), float(w_depth), N.dptr(keep[0]), N.dptr(keep[1]),
                None, None, None, None)
    img = ImageBuffers.allocate(intr.height, intr.width, dev, normal=False) if image else None
    view.reserve_pairs(max(65536, 64 * n))
    view.forward_backward(params, n, pose, camera_struct(intr), config_struct(cfg), img, ls, grads, loss)
    torch.cuda.synchronize()
    st = view.stats()
    assert st.overflow == 0
    g = {k: v.double().cpu().numpy() for k, v in unpack_params(grads, n).items()}
    im = None if img is None else {k: getattr(img, k).double().cpu().numpy()
                                   for k in ("color", "depth", "accumulation")}
    return g, float(loss.item()), im, st


def far_targets(ref_color, ref_depth, rng, gap=0.05):
    """Targets bounded away from the render (|C - C*| >= gap): L1 seeds have no sign ambiguity."""
    s = rng.choice([-1.0, 1.0], size=ref_color.shape)
    trgb = ref_color + s * (gap + np.abs(rng.normal(0, 0.02, ref_color.shape)))
    sd = rng.choice([-1.0, 1.0], size=ref_depth.shape)
    tdep = ref_depth + sd * (gap + np.abs(rng.normal(0, 0.02, ref_depth.shape)))
    return trgb, tdep


def gate(a, b, tol=1e-4):
    """Parity gate: max|d| <= tol*max|ref| and ||d||/||ref|| <= tol."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if b.size == 0:
        return True, 0.0, 0.0
    mx = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
    l2 = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    return (mx <= tol and l2 <= tol), mx, l2


def drawn_order(bbox, order):
    """The reference depth order restricted to the surfels whose integer bbox is non-empty
    (the only ones that touch a pixel, _raster_kernels.py:32-34): the set the device sorts."""
    order = np.asarray(order, dtype=np.int64)
    b = np.asarray(bbox)[order]
    return order[(b[:, 0] <= b[:, 1]) & (b[:, 2] <= b[:, 3])]


def l1_oracle_grads(surfels, pose, intr, trgb, tdep, w_rgb, w_depth, gpu_color, gpu_depth, band=1e-5):
    """Float64 oracle gradients of the L1 loss (no depth mask) for a GPU comparison.

    sign(C - C*) is not determined at float32 precision where the float64 residual is within
    the float32 render error; there (|C64 - C*| <= band, |D64 - D*| <= band |D*|) the seed takes
    the GPU render's sign, everywhere else the oracle's own.  Returns (loss, grads, number of
    such sign-ambiguous pixel channels)."""
    import oracle as O
    buf = O.render(surfels, pose, intr)
    loss, g_rgb, g_d = O.loss_seeds(buf, trgb, tdep, "l1", w_rgb, w_depth, mask_depth=False)
    h, w = buf.depth.shape
    npx = h * w
    amb = np.abs(buf.color - trgb) <= band
    g_rgb[amb] = (w_rgb / (3.0 * npx)) * np.sign(np.asarray(gpu_color, float) - trgb)[amb]
    ambd = np.abs(buf.depth - tdep) <= band * np.maximum(np.abs(tdep), 1e-30)
    g_d[ambd] = (w_depth / npx) * np.sign(np.asarray(gpu_depth, float) - tdep)[ambd]
    grads = O.backward(surfels, pose, intr, buf, g_rgb, g_d)
    return loss, grads, int(amb.sum() + ambd.sum())


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)
