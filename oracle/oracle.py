"""ctypes front end of the float64 CPU oracle (s2d_oracle.c).

TEST INFRASTRUCTURE ONLY (see package docstring).  Inputs are duck-typed:
surfels expose ``means, quats, scales, opacities, colors`` arrays; the pose is
anything with ``as_sim3()``/``packed()`` or a packed (8,) array; intrinsics
expose ``fx, fy, cx, cy, width, height``; the raster config exposes the
reference ``RasterConfig`` fields (rasterizer.py:150-171).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

__all__ = [
    "build_oracle", "load", "pose_inverse", "project", "depth_order", "tile_lists",
    "render", "loss_seeds", "backward", "loss_and_grads", "max_blend_weights",
    "adam_step", "DEFAULTS", "quat_mul", "quat_canonicalize", "transform_surfels", "fuse_gate", "fuse",
    "prune_mark", "prune", "refine",
]

DEFAULTS = SimpleNamespace(weight_clamp=0.999, termination_transmittance=1e-4, footprint_sigma=3.0,
                           near_plane=1e-3, max_condition=1e8, max_view_angle_deg=80.0,
                           center_margin_frac=0.5)


class _Cam(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int64), ("height", ctypes.c_int64)]


class _Cfg(ctypes.Structure):
    _fields_ = [("weight_clamp", ctypes.c_double), ("term_t", ctypes.c_double),
                ("sigma", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("max_cond", ctypes.c_double), ("tan_max", ctypes.c_double),
                ("margin_frac", ctypes.c_double)]


def build_oracle(force: bool = False) -> str:
    src = os.path.join(_HERE, "s2d_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "_build/liboracle.so"], check=True)
    return _LIB_PATH


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_oracle()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.o_project.restype = ctypes.c_int64
        _lib.o_depth_order.restype = ctypes.c_int64
        _lib.o_tile_lists.restype = ctypes.c_int64
        _lib.o_loss_seeds.restype = ctypes.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


# --- host-side pose math (restates geometry.py:59-64, 132-142, 188-195 in float64) ---

def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def _qrot(q, v):
    u = q[..., 1:]
    w = q[..., 0:1]
    uv = _cross(u, v)
    return v + 2.0 * (w * uv + _cross(u, uv))


def _qmat(q):
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def _packed(pose):
    if hasattr(pose, "as_sim3"):
        pose = pose.as_sim3()
    if hasattr(pose, "packed"):
        return np.asarray(pose.packed(), dtype=float)
    return np.asarray(pose, dtype=float).reshape(8)


def pose_inverse(pose):
    """(inv[8], m_cw[3,3], r_cw[3,3]) exactly as rasterizer.py:204,214."""
    a = _packed(pose)
    s_inv = 1.0 / a[0]
    qc = a[4:8].copy()
    qc[1:] = -qc[1:]
    inv = np.empty(8)
    inv[0] = s_inv
    inv[1:4] = -s_inv * _qrot(qc, a[1:4])
    inv[4:8] = qc
    r_cw = _qmat(inv[4:8])
    m_cw = inv[0] * r_cw
    return inv, np.ascontiguousarray(m_cw), np.ascontiguousarray(r_cw)


def _cam(intr):
    return _Cam(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                int(intr.width), int(intr.height))


def _cfg(cfg):
    cfg = cfg or DEFAULTS
    return _Cfg(float(cfg.weight_clamp), float(cfg.termination_transmittance),
                float(cfg.footprint_sigma), float(cfg.near_plane), float(cfg.max_condition),
                float(np.tan(np.radians(cfg.max_view_angle_deg))), float(cfg.center_margin_frac))


def _arrays(s):
    n = len(np.asarray(s.means).reshape(-1, 3))
    return (n, _f64(s.means, (n, 3)), _f64(s.quats, (n, 4)), _f64(s.scales, (n, 2)),
            _f64(s.opacities, (n,)), _f64(s.colors, (n, 3)))


def project(surfels, pose, intr, cfg=None):
    """_project_batch + _footprint_boxes (rasterizer.py:201-281) + camera normals."""
    L = load()
    n, means, quats, scales, _, _ = _arrays(surfels)
    inv, m_cw, r_cw = pose_inverse(pose)
    out = SimpleNamespace(
        centers=np.zeros((n, 2)), cov2=np.zeros((n, 3)), inv_abc=np.zeros((n, 3)), z=np.zeros(n),
        flags=np.zeros(n, np.uint8), bbox=np.zeros((n, 4), np.int64), normals=np.zeros((n, 3)))
    cam, c = _cam(intr), _cfg(cfg)
    out.degenerate = int(L.o_project(
        ctypes.c_int64(n), _p(means), _p(quats), _p(scales), _p(inv), _p(m_cw), _p(r_cw),
        ctypes.byref(cam), ctypes.byref(c), _p(out.centers), _p(out.cov2), _p(out.inv_abc),
        _p(out.z), _p(out.flags), _p(out.bbox), _p(out.normals)))
    out.in_front = (out.flags & 1) != 0
    out.valid = (out.flags & 2) != 0
    out.on_screen = (out.flags & 4) != 0
    return out


def depth_order(proj):
    L = load()
    n = len(proj.z)
    order = np.zeros(n, np.int64)
    v = L.o_depth_order(ctypes.c_int64(n), _p(proj.z), _p(proj.flags), _p(order))
    return order[:v].copy()


def tile_lists(proj, order, intr, tile=16):
    """(tile_start[ntiles+1], tile_ids[P]) — per-tile surfel indices in global depth order."""
    L = load()
    ntx = (intr.width + tile - 1) // tile
    nty = (intr.height + tile - 1) // tile
    start = np.zeros(ntx * nty + 1, np.int64)
    order = np.ascontiguousarray(order, dtype=np.int64)
    total = L.o_tile_lists(ctypes.c_int64(len(order)), _p(order), _p(proj.bbox),
                           ctypes.c_int64(intr.width), ctypes.c_int64(intr.height),
                           ctypes.c_int64(tile), _p(start), None, ctypes.c_int64(0))
    ids = np.zeros(max(total, 1), np.int64)
    L.o_tile_lists(ctypes.c_int64(len(order)), _p(order), _p(proj.bbox), ctypes.c_int64(intr.width),
                   ctypes.c_int64(intr.height), ctypes.c_int64(tile), _p(start), _p(ids),
                   ctypes.c_int64(total))
    return start, ids[:total]


def render(surfels, pose, intr, cfg=None, with_normal=True):
    """Forward render: color (H,W,3), depth, accumulation, normal, max_w, arg_w, degenerate.

    blend_forward (_raster_kernels.py:22-55) via _render_state (rasterizer.py:301-331).
    """
    L = load()
    cfg = cfg or DEFAULTS
    n, _, _, _, opac, colors = _arrays(surfels)
    h, w = int(intr.height), int(intr.width)
    color = np.zeros((h, w, 3))
    depth = np.zeros((h, w))
    trans = np.ones((h, w))
    normal = np.zeros((h, w, 3))
    max_w = np.zeros((h, w))
    arg_w = np.full((h, w), -1, np.int64)
    proj = project(surfels, pose, intr, cfg) if n else None
    order = depth_order(proj) if n else np.zeros(0, np.int64)
    if len(order):
        L.o_blend_forward(
            ctypes.c_int64(len(order)), _p(order), _p(proj.centers), _p(proj.inv_abc), _p(proj.z),
            _p(opac), _p(colors), _p(proj.normals), _p(proj.bbox),
            ctypes.c_double(cfg.weight_clamp), ctypes.c_double(cfg.termination_transmittance),
            ctypes.c_double(cfg.footprint_sigma ** 2), ctypes.c_int64(w), _p(color), _p(depth),
            _p(trans), _p(normal) if with_normal else None, _p(max_w), _p(arg_w))
    return SimpleNamespace(color=color, depth=depth, accumulation=1.0 - trans, trans=trans,
                           normal=normal, max_w=max_w, arg_w=arg_w,
                           degenerate_skipped=proj.degenerate if proj is not None else 0,
                           proj=proj, order=order)


def loss_seeds(buf, target_rgb, target_depth, kind="mse", w_rgb=1.0, w_depth=0.05, mask_depth=None):
    """Per-pixel dL/dC, dL/dD and the loss.  kind "mse" = reference render_loss
    (rasterizer.py:346-357, seeds :375-380); kind "l1" = L1 RGB + w_depth L1 depth."""
    L = load()
    h, w = buf.depth.shape
    npx = h * w
    g_rgb = np.zeros((h, w, 3))
    g_depth = np.zeros((h, w))
    kid = 0 if kind == "mse" else 1
    md = 1 if (mask_depth if mask_depth is not None else kid == 0) else 0
    loss = L.o_loss_seeds(ctypes.c_int(kid), ctypes.c_int64(npx), _p(_f64(buf.color)),
                          _p(_f64(buf.depth)), _p(_f64(buf.accumulation)), _p(_f64(target_rgb)),
                          _p(_f64(target_depth)), ctypes.c_double(w_rgb), ctypes.c_double(w_depth),
                          ctypes.c_int(md), _p(g_rgb), _p(g_depth))
    return float(loss), g_rgb, g_depth


def backward(surfels, pose, intr, buf, g_rgb, g_depth, g_normal=None, g_acc=None, cfg=None):
    """Gradients of a loss with per-pixel seeds, w.r.t. all surfel parameters.

    Returns SimpleNamespace(colors, opacities, means, quats, scales, g2, gn) (input order).
    colors/opacities: blend_gradients (_raster_kernels.py:58-113) generalised;
    means/quats/scales: N2 geometry chain (o_geometry_backward).
    """
    L = load()
    cfg = cfg or DEFAULTS
    n, means, quats, scales, opac, colors = _arrays(surfels)
    h, w = int(intr.height), int(intr.width)
    gc = np.zeros((n, 3))
    go = np.zeros(n)
    g2 = np.zeros((n, 8))
    gn = np.zeros((n, 3))
    gm = np.zeros((n, 3))
    gq = np.zeros((n, 4))
    gs = np.zeros((n, 2))
    proj, order = buf.proj, buf.order
    if n and len(order):
        gnorm = _f64(g_normal) if g_normal is not None else None
        gacc = _f64(g_acc) if g_acc is not None else None
        L.o_blend_backward(
            ctypes.c_int64(len(order)), _p(order), _p(proj.centers), _p(proj.inv_abc), _p(proj.z),
            _p(opac), _p(colors), _p(proj.normals), _p(proj.bbox),
            ctypes.c_double(cfg.weight_clamp), ctypes.c_double(cfg.termination_transmittance),
            ctypes.c_double(cfg.footprint_sigma ** 2), ctypes.c_int64(h), ctypes.c_int64(w),
            _p(_f64(buf.color)), _p(_f64(buf.depth)), _p(_f64(buf.normal)), _p(_f64(buf.trans)),
            _p(_f64(g_rgb)), _p(_f64(g_depth)), _p(gnorm), _p(gacc), _p(gc), _p(go), _p(g2), _p(gn))
        inv, m_cw, r_cw = pose_inverse(pose)
        cam = _cam(intr)
        L.o_geometry_backward(ctypes.c_int64(n), _p(means), _p(quats), _p(scales), _p(inv),
                              _p(m_cw), _p(r_cw), ctypes.byref(cam), _p(proj.flags),
                              _p(proj.inv_abc), _p(g2), _p(gn), _p(gm), _p(gq), _p(gs))
    return SimpleNamespace(colors=gc, opacities=go, means=gm, quats=gq, scales=gs, g2=g2, gn=gn)


def loss_and_grads(surfels, pose, intr, target_rgb, target_depth, kind="mse", w_rgb=1.0,
                   w_depth=0.05, mask_depth=None, cfg=None):
    buf = render(surfels, pose, intr, cfg)
    loss, g_rgb, g_depth = loss_seeds(buf, target_rgb, target_depth, kind, w_rgb, w_depth, mask_depth)
    grads = backward(surfels, pose, intr, buf, g_rgb, g_depth, cfg=cfg)
    return loss, grads, buf


def max_blend_weights(surfels, pose, intr, mask=None, cfg=None):
    """per_surfel_max_weight (rasterizer.py:402-428) -> (max_all, max_marked)."""
    L = load()
    cfg = cfg or DEFAULTS
    n, _, _, _, opac, _ = _arrays(surfels)
    max_all = np.zeros(n)
    max_marked = np.zeros(n)
    if n == 0:
        return max_all, max_marked
    proj = project(surfels, pose, intr, cfg)
    order = depth_order(proj)
    m = np.zeros((intr.height, intr.width), np.uint8) if mask is None else \
        np.ascontiguousarray(np.asarray(mask).astype(np.uint8))
    if len(order):
        L.o_max_blend_weights(ctypes.c_int64(len(order)), _p(order), _p(proj.centers),
                              _p(proj.inv_abc), _p(opac), _p(proj.bbox),
                              ctypes.c_double(cfg.weight_clamp),
                              ctypes.c_double(cfg.termination_transmittance),
                              ctypes.c_double(cfg.footprint_sigma ** 2), _p(m),
                              ctypes.c_int64(intr.height), ctypes.c_int64(intr.width),
                              _p(max_all), _p(max_marked))
    return max_all, max_marked


def adam_step(params, grads, m1, m2, step, lr_means=1e-3, lr_rest=5e-3, b1=0.9, b2=0.999,
              eps=1e-8, scale_min=1e-7, mask=None):
    """In-place float64 Adam + projection on packed (13N,) arrays."""
    L = load()
    n = params.size // 13
    for a in (params, grads, m1, m2):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    mk = None if mask is None else np.ascontiguousarray(mask.astype(np.uint8))
    L.o_adam_step(ctypes.c_int64(n), _p(params), _p(grads), _p(m1), _p(m2), ctypes.c_int64(step),
                  ctypes.c_double(lr_means), ctypes.c_double(lr_rest), ctypes.c_double(b1),
                  ctypes.c_double(b2), ctypes.c_double(eps), ctypes.c_double(scale_min), _p(mk))


# ---------------------------------------------------------------- map maintenance (§8(f) 2-3)
# numpy float64 restatements; each elementwise expression keeps the reference's association.

def quat_mul(q1, q2):
    """geometry.py:39-50"""
    w1, x1, y1, z1 = q1[..., 0], q1[..., 1], q1[..., 2], q1[..., 3]
    w2, x2, y2, z2 = q2[..., 0], q2[..., 1], q2[..., 2], q2[..., 3]
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=-1)


def quat_canonicalize(q):
    """geometry.py:71-84: w >= 0, ties on the first non-zero vector component, no -0.0."""
    q = np.asarray(q, dtype=float)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    flip = (w < 0) | ((w == 0) & ((x < 0) | ((x == 0) & ((y < 0) | ((y == 0) & (z < 0))))))
    return np.where(flip[..., None], -q, q) + 0.0


def transform_surfels(means, quats, scales, pose):
    """mapper.py:184-197 on the geometric fields -> (means, quats, scales); pose packed Sim(3)."""
    a = _packed(pose)
    m = a[0] * _qrot(np.broadcast_to(a[4:8], (len(means), 4)), np.asarray(means, float)) + a[1:4]
    q = quat_canonicalize(quat_mul(a[4:8][None, :], np.asarray(quats, float)))
    return m, q, a[0] * np.asarray(scales, float)


def fuse_gate(accumulation, cand_means, intr, accum_threshold=0.5):
    """mapper.py:215-224: keep flags of camera-frame candidates (map non-empty)."""
    cm = np.asarray(cand_means, float)
    z = cm[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        px = np.round(intr.fx * cm[:, 0] / z + intr.cx).astype(int)
        py = np.round(intr.fy * cm[:, 1] / z + intr.cy).astype(int)
    inside = (px >= 0) & (px < intr.width) & (py >= 0) & (py < intr.height) & (z > 0)
    acc = np.zeros(len(cm))
    acc[inside] = np.asarray(accumulation)[py[inside], px[inside]]
    return acc < accum_threshold


def fuse(map_surfels, cand, pose, intr, accum_threshold=0.5, cfg=None):
    """mapper.py:200-230 -> (keep flags, world means, quats, scales of the kept candidates)."""
    n_map = len(np.asarray(map_surfels.means).reshape(-1, 3))
    if n_map == 0:
        keep = np.ones(len(cand.means), bool)
    else:
        buf = render(map_surfels, pose, intr, cfg, with_normal=False)
        keep = fuse_gate(buf.accumulation, cand.means, intr, accum_threshold)
    m, q, s = transform_surfels(np.asarray(cand.means)[keep], np.asarray(cand.quats)[keep],
                                np.asarray(cand.scales)[keep], pose)
    return keep, m, q, s


def prune_mark(color, depth, accumulation, observed_rgb, observed_depth, rgb_error=0.2, depth_error_frac=0.10):
    """mapper.py:246-253"""
    covered = accumulation > 0.5
    rgb_err = np.max(np.abs(color - observed_rgb), axis=2) > rgb_error
    depth_norm = depth / np.maximum(accumulation, 1e-12)
    obs = np.asarray(observed_depth, dtype=float)
    depth_err = (obs > 0) & (np.abs(depth_norm - obs) > depth_error_frac * obs)
    return covered & (rgb_err | depth_err)


def prune(map_surfels, pose, intr, observed_rgb, observed_depth, rgb_error=0.2, depth_error_frac=0.10,
          contribution_floor=0.1, cfg=None):
    """mapper.py:238-260 -> (victim indices, marked pixel mask)."""
    buf = render(map_surfels, pose, intr, cfg, with_normal=False)
    marked = prune_mark(buf.color, buf.depth, buf.accumulation, observed_rgb, observed_depth, rgb_error,
                        depth_error_frac)
    if not marked.any():
        return np.zeros(0, np.int64), marked
    _, max_marked = max_blend_weights(map_surfels, pose, intr, marked, cfg)
    return np.flatnonzero(max_marked > contribution_floor), marked


# ---------------------------------------------------------------- refine (mapper.py:276-349)

def _psnr(rendered, target):
    """evaluation.psnr (evaluation.py:63-72)."""
    mse = float(np.mean((np.asarray(rendered, float) - np.asarray(target, float)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)


def refine(surfels, keyframe_ids, target_mask, poses, observations, intr, iterations=20, initial_step=0.1,
           min_step=1e-6, w_mse=1.0, w_depth=0.05, cfg=None):
    """Float64 restatement of mapper.refine (mapper.py:276-349) on SurfelArrays-like inputs:
    summed per-view render_loss and colour/opacity gradients (rasterizer.py:346-399 via this
    oracle's render / loss_seeds / backward), target-masked L-inf-normalised backtracking steps
    with halving, np.clip to [0, 1] of every surfel, warm-started step scale, restore on failure.
    Returns (losses, psnr_before, psnr_after, accepted, colors, opacities); inputs untouched."""
    colors = np.array(surfels.colors, dtype=float, copy=True)
    opac = np.array(surfels.opacities, dtype=float, copy=True)
    cur = SimpleNamespace(means=surfels.means, quats=surfels.quats, scales=surfels.scales, opacities=opac,
                          colors=colors)
    views = [(poses[k], *observations[k]) for k in keyframe_ids]
    mask = np.asarray(target_mask, bool)

    def psnrs():
        vals = [_psnr(render(cur, p, intr, cfg, with_normal=False).color, rgb) for p, rgb, _ in views]
        finite = [v for v in vals if np.isfinite(v)]
        return float(np.mean(finite)) if finite else float("inf")

    def loss_grads():
        tot, gc, go = 0.0, np.zeros_like(cur.colors), np.zeros_like(cur.opacities)
        for p, rgb, dep in views:
            buf = render(cur, p, intr, cfg, with_normal=False)
            loss, g_rgb, g_d = loss_seeds(buf, rgb, dep, "mse", w_mse, w_depth, True)
            g = backward(cur, p, intr, buf, g_rgb, g_d, cfg=cfg)
            tot += loss
            gc += g.colors
            go += g.opacities
        return tot, gc, go

    before = psnrs()
    if iterations == 0 or not views or not mask.any():
        return [], before, before, 0, cur.colors, cur.opacities
    loss, gc, go = loss_grads()
    losses, accepted, scale = [loss], 0, initial_step
    for _ in range(iterations):
        gc[~mask] = 0.0
        go[~mask] = 0.0
        gnorm = max(float(np.max(np.abs(gc))), float(np.max(np.abs(go))))
        if gnorm < 1e-14:
            break
        step = scale / gnorm
        c0, o0 = cur.colors.copy(), cur.opacities.copy()
        improved = False
        while step >= min_step / gnorm:
            cur.colors = np.clip(c0 - step * gc, 0.0, 1.0)
            cur.opacities = np.clip(o0 - step * go, 0.0, 1.0)
            new_loss, ngc, ngo = loss_grads()
            if new_loss < loss:
                loss, gc, go = new_loss, ngc, ngo
                losses.append(loss)
                accepted += 1
                improved = True
                scale = min(2.0 * step * gnorm, initial_step)
                break
            step *= 0.5
        if not improved:
            cur.colors, cur.opacities = c0, o0
            break
    return losses, before, psnrs(), accepted, cur.colors, cur.opacities
