"""float64 oracle of the ray-splat footprint mode (S2D_SPLAT_RAY) — TEST INFRASTRUCTURE ONLY.

The mode has no reference counterpart (the reference projects the
tangent-plane covariance affinely).  This restates the GPU mode in PyTorch float64 so
gradients come from autograd, independently of the hand-derived chain in k_raster_bwd /
k_project_bwd:

* visibility gates, depth order: the reference's (float64 projection of oracle/, ties by
  index), so the surfel set and order are those of the affine mode;
* footprint: tangent axes a = Bc[:,0], b = Bc[:,1], centre p (camera frame); H = K [a b p];
  (U, V, S) = H^-1 (x, y, 1), (u, v) = (U, V) / S, intersection depth z = 1 / S;
* bbox: the pixel AABB of the projected sigma-square of the tangent plane (all four
  corners must be in front of the camera);
* blending: blend_forward's rules (termination before blending, cut u^2 + v^2 > sigma^2,
  weight clamp, w <= 0 skips), blending the intersection depth.

`intersect_uv` restates the same intersection from first principles (ray / plane
intersection and projection onto the tangent axes) for pinning the homography form.
"""

from __future__ import annotations

import numpy as np
import torch

from .oracle import DEFAULTS, _packed, depth_order, pose_inverse, project

__all__ = ["render_ray", "intersect_uv"]


def _quat_to_matrix(q):
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    return torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def intersect_uv(a, b, p, intr, x, y):
    """Tangent-plane coordinates (u, v) and depth of the intersection of pixel (x, y)'s ray
    with the plane p + u a + v b (camera frame), by ray / plane intersection."""
    r = np.array([(x - intr.cx) / intr.fx, (y - intr.cy) / intr.fy, 1.0])
    n = np.cross(a, b)
    lam = n.dot(p) / n.dot(r)
    q = lam * r - p
    G = np.array([[a.dot(a), a.dot(b)], [a.dot(b), b.dot(b)]])
    u, v = np.linalg.solve(G, [q.dot(a), q.dot(b)])
    return u, v, lam


def render_ray(params: dict, pose, intr, cfg=None):
    """Ray-mode render of float64 torch parameters (means (n,3), quats (n,4), scales (n,2),
    opacities (n,), colors (n,3); may require grad).  Returns color, depth, accumulation,
    normal (torch, differentiable) and the per-surfel visibility / bbox used."""
    cfg = cfg or DEFAULTS
    sig2 = cfg.footprint_sigma ** 2
    means, quats, scales = params["means"], params["quats"], params["scales"]
    opac, colors = params["opacities"], params["colors"]
    n = means.shape[0]
    arrays = type("S", (), {})()
    arrays.means, arrays.quats, arrays.scales = (means.detach().numpy(), quats.detach().numpy(),
                                                 scales.detach().numpy())
    arrays.opacities, arrays.colors = opac.detach().numpy(), colors.detach().numpy()
    proj = project(arrays, pose, intr, cfg)
    valid = (proj.flags & 2) != 0
    inv, m_cw, r_cw = pose_inverse(pose)
    mcw = torch.tensor(m_cw, dtype=torch.float64)
    rcw = torch.tensor(r_cw, dtype=torch.float64)
    t = torch.tensor(inv[1:4], dtype=torch.float64)
    p = means @ mcw.T + t
    R = _quat_to_matrix(quats)
    Bc = (mcw @ R[:, :, :2]) * scales[:, None, :]
    nrm = (rcw @ R[:, :, 2:3])[:, :, 0]
    sg = torch.where((nrm * p).sum(-1).detach() > 0, -1.0, 1.0).to(torch.float64)
    nrm = nrm * sg[:, None]
    K = torch.tensor([[intr.fx, 0.0, intr.cx], [0.0, intr.fy, intr.cy], [0.0, 0.0, 1.0]], dtype=torch.float64)
    A = torch.stack([Bc[:, :, 0], Bc[:, :, 1], p], -1)  # (n, 3, 3) columns a, b, p
    H = K @ A
    # visibility and bbox (no gradient)
    Ad = A.detach().numpy()
    W, Hh = intr.width, intr.height
    on = np.zeros(n, bool)
    bbox = np.zeros((n, 4), np.int64)
    k = cfg.footprint_sigma
    for i in np.flatnonzero(valid):
        a, b, c = Ad[i, :, 0], Ad[i, :, 1], Ad[i, :, 2]
        xs, ys, ok = [], [], True
        for su in (-k, k):
            for sv in (-k, k):
                X = c + su * a + sv * b
                if not X[2] > cfg.near_plane:
                    ok = False
                xs.append(intr.fx * X[0] / X[2] + intr.cx)
                ys.append(intr.fy * X[1] / X[2] + intr.cy)
        if not ok or not (max(xs) >= 0 and min(xs) <= W - 1 and max(ys) >= 0 and min(ys) <= Hh - 1):
            continue
        if not abs(np.linalg.det(H[i].detach().numpy())) > 1e-300:
            continue
        on[i] = True
        bbox[i] = [min(max(int(np.ceil(max(min(xs), -1.0))), 0), W - 1),
                   min(max(int(np.floor(min(max(xs), W))), 0), W - 1),
                   min(max(int(np.ceil(max(min(ys), -1.0))), 0), Hh - 1),
                   min(max(int(np.floor(min(max(ys), Hh))), 0), Hh - 1)]
    # depth order of the visible surfels: the reference's (float64 z, ties by index)
    proj.flags = ((proj.flags & 3) | (on.astype(np.uint8) << 2)).astype(np.uint8)
    order = depth_order(proj)
    Hi = torch.linalg.inv(H)
    npx = W * Hh
    C = torch.zeros(npx, 3, dtype=torch.float64)
    D = torch.zeros(npx, dtype=torch.float64)
    Nn = torch.zeros(npx, 3, dtype=torch.float64)
    T = torch.ones(npx, dtype=torch.float64)
    for i in order:
        x0, x1, y0, y1 = bbox[i]
        if x0 > x1 or y0 > y1:
            continue
        ys, xs = np.mgrid[y0:y1 + 1, x0:x1 + 1]
        idx = torch.as_tensor((ys * W + xs).reshape(-1))
        X = torch.stack([torch.as_tensor(xs.reshape(-1), dtype=torch.float64),
                         torch.as_tensor(ys.reshape(-1), dtype=torch.float64),
                         torch.ones(idx.numel(), dtype=torch.float64)], 0)
        UVS = Hi[i] @ X
        S = UVS[2]
        live = (S.detach() > 0) & (T[idx].detach() >= cfg.termination_transmittance)
        Ssafe = torch.where(live, S, torch.ones_like(S))
        u, v = UVS[0] / Ssafe, UVS[1] / Ssafe
        m = u * u + v * v
        live = live & (m.detach() <= sig2)
        w = opac[i] * torch.exp(-0.5 * m)
        w = torch.where(w.detach() > cfg.weight_clamp, torch.full_like(w, cfg.weight_clamp), w)
        live = live & (w.detach() > 0)
        if not bool(live.any()):
            continue
        sel = idx[live]
        wl, zl, Tl = w[live], 1.0 / Ssafe[live], T[sel]
        contrib = wl * Tl
        C = C.index_add(0, sel, contrib[:, None] * colors[i][None, :])
        D = D.index_add(0, sel, contrib * zl)
        Nn = Nn.index_add(0, sel, contrib[:, None] * nrm[i][None, :])
        T = T.index_put((sel,), Tl * (1.0 - wl))
    return {"color": C.reshape(Hh, W, 3), "depth": D.reshape(Hh, W), "accumulation": (1.0 - T).reshape(Hh, W),
            "normal": Nn.reshape(Hh, W, 3), "on": on, "bbox": bbox, "order": order}


def params_from_arrays(s, requires_grad=True) -> dict:
    f = lambda a: torch.tensor(np.asarray(a, dtype=np.float64), dtype=torch.float64,  # noqa: E731
                               requires_grad=requires_grad)
    return {"means": f(s.means), "quats": f(s.quats), "scales": f(s.scales), "opacities": f(s.opacities),
            "colors": f(s.colors)}
