/*
 * s2d_oracle.c — CPU float64 restatement of the reference's surfel render path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference arm use it, always as the checker or the
 * timed CPU baseline, never as the thing shipped.
 *
 * Parity pin: the tests/golden npz files were produced by running the reference
 * itself (tests/golden/make_golden.py, PYTHONPATH=/root/reference/pkg/src);
 * tests/test_oracle_golden.py checks this restatement against them
 * (projection/bbox/order/tile lists bit-exact, images and colour/opacity
 * gradients to 1e-12).
 *
 * Each function names the reference lines it restates.  Arithmetic follows
 * the reference's float64 operation order: numpy elementwise ufuncs and
 * numba (no fastmath) never fuse multiply-adds, so this file is compiled with
 * -ffp-contract=off; the three stacked matmuls of rasterizer.py:216,224
 * run through OpenBLAS, which accumulates a dot product as
 * acc = a0*b0; acc = fma(a1,b1,acc); ... — restated with explicit fma().
 *
 * New pieces with no reference counterpart ("parity unpinned by reference
 * tests") are restated here from their definitions in
 * the camera-frame normal channel, the geometry backward (derived
 * through the conic/covariance chain, deliberately NOT the device's M^-1
 * chain, so the two are independent), L1 loss seeds and Adam.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double fx, fy, cx, cy;
    int64_t width, height;
} o_cam;

typedef struct {
    double weight_clamp;   /* rasterizer.py:162 */
    double term_t;         /* :163 */
    double sigma;          /* :164  footprint_sigma */
    double near_plane;     /* :165 */
    double max_cond;       /* :166 */
    double tan_max;        /* np.tan(np.radians(max_view_angle_deg)), :207 (host) */
    double margin_frac;    /* :168 */
} o_cfg;

/* ---------------------------------------------------------------- helpers */

/* quat_rotate, geometry.py:59-64 (np.cross association: a1*b2 - a2*b1 ...) */
static void o_quat_rotate(const double q[4], const double v[3], double out[3]) {
    const double w = q[0], u0 = q[1], u1 = q[2], u2 = q[3];
    const double uv0 = u1 * v[2] - u2 * v[1];
    const double uv1 = u2 * v[0] - u0 * v[2];
    const double uv2 = u0 * v[1] - u1 * v[0];
    const double uuv0 = u1 * uv2 - u2 * uv1;
    const double uuv1 = u2 * uv0 - u0 * uv2;
    const double uuv2 = u0 * uv1 - u1 * uv0;
    out[0] = v[0] + 2.0 * (w * uv0 + uuv0);
    out[1] = v[1] + 2.0 * (w * uv1 + uuv1);
    out[2] = v[2] + 2.0 * (w * uv2 + uuv2);
}

/* quat_to_matrix, geometry.py:132-142 (raw, un-normalised q) */
static void o_quat_to_matrix(const double q[4], double r[9]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* numpy float64 -> int64 cast on x86-64 (cvttsd2si): out of range or NaN gives INT64_MIN */
static int64_t o_f2i(double v) {
    if (!(v > -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
    return (int64_t)v;
}

static int64_t o_clip(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* -------------------------------------------------------------- projection */

/*
 * _project_batch (rasterizer.py:201-249) followed by _footprint_boxes
 * (rasterizer.py:262-281).  inv = pk_inverse(pose) and m_cw = inv[0]*R(inv_q)
 * are computed on the host (same as the reference, :204, :214).
 * Outputs per surfel: centers (2), cov2 (a,b,c), inv_abc (3), z, flags
 * (bit0 in_front incl. margin gate, bit1 valid, bit2 on_screen), bbox int64 (4),
 * normal (3, camera frame, oriented toward the camera; N1).
 * Returns the degenerate count (:244).
 */
int64_t o_project(int64_t n, const double *means, const double *quats, const double *scales,
                  const double inv[8], const double m_cw[9], const double r_cw[9],
                  const o_cam *cam, const o_cfg *cfg,
                  double *centers, double *cov2, double *inv_abc, double *zs,
                  uint8_t *flags, int64_t *bbox, double *normals) {
    int64_t degenerate = 0;
    const double mx = cfg->margin_frac * (double)cam->width;
    const double my = cfg->margin_frac * (double)cam->height;
    const double wmax = (double)(cam->width - 1) + mx;
    const double hmax = (double)(cam->height - 1) + my;
    for (int64_t i = 0; i < n; ++i) {
        double r[3];
        o_quat_rotate(inv + 4, means + 3 * i, r);
        double p[3];
        p[0] = inv[0] * r[0] + inv[1];
        p[1] = inv[0] * r[1] + inv[2];
        p[2] = inv[0] * r[2] + inv[3];
        const double z = p[2];
        int in_front = (z > cfg->near_plane) && (hypot(p[0], p[1]) <= cfg->tan_max * z);

        double R[9];
        o_quat_to_matrix(quats + 4 * i, R);
        double B[3][2];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 2; ++k) B[a][k] = R[3 * a + k] * scales[2 * i + k];
        /* einsum("ij,njk->nik"): plain sequential sum (rasterizer.py:215) */
        double Bc[3][2];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 2; ++k)
                Bc[a][k] = m_cw[3 * a + 0] * B[0][k] + m_cw[3 * a + 1] * B[1][k] + m_cw[3 * a + 2] * B[2][k];
        /* basis_cam @ basis_cam^T (:216) */
        double C[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) C[a][b] = fma(Bc[a][1], Bc[b][1], Bc[a][0] * Bc[b][0]);
        const double zsafe = in_front ? z : 1.0;
        double J[2][3];
        J[0][0] = cam->fx / zsafe;
        J[0][1] = 0.0;
        J[0][2] = -cam->fx * p[0] / (zsafe * zsafe);
        J[1][0] = 0.0;
        J[1][1] = cam->fy / zsafe;
        J[1][2] = -cam->fy * p[1] / (zsafe * zsafe);
        /* (jac @ cov_cam) @ jac^T (:224) */
        double T1[2][3], X[2][2];
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 3; ++c)
                T1[a][c] = fma(J[a][2], C[2][c], fma(J[a][1], C[1][c], J[a][0] * C[0][c]));
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c)
                X[a][c] = fma(T1[a][2], J[c][2], fma(T1[a][1], J[c][1], T1[a][0] * J[c][0]));
        const double ca = 0.5 * (X[0][0] + X[0][0]);
        const double cb = 0.5 * (X[0][1] + X[1][0]);
        const double cc = 0.5 * (X[1][1] + X[1][1]);
        const double cx = cam->fx * p[0] / zsafe + cam->cx;
        const double cy = cam->fy * p[1] / zsafe + cam->cy;
        in_front = in_front && (cx >= -mx) && (cx <= wmax) && (cy >= -my) && (cy <= hmax);

        const double half_tr = 0.5 * (ca + cc);
        double d2 = 0.25 * ((ca - cc) * (ca - cc)) + cb * cb;
        if (!(d2 >= 0.0) && !isnan(d2)) d2 = 0.0;   /* np.maximum(x, 0) keeps NaN */
        const double dev = sqrt(d2);
        const double lmin = half_tr - dev, lmax = half_tr + dev;
        const int well = (lmin > 0.0) && (lmax <= cfg->max_cond * lmin);
        if (in_front && !well) degenerate++;
        const int valid = in_front && well;
        const double det = valid ? (ca * cc - cb * cb) : 1.0;
        const double ia = cc / det, ib = -cb / det, ic = ca / det;

        /* _footprint_boxes (:262-281) */
        double dinv = ia * ic - ib * ib;
        if (!(dinv > 0.0)) dinv = 1.0;
        double qx = ic / dinv, qy = ia / dinv;
        if (qx < 0.0) qx = 0.0;
        if (qy < 0.0) qy = 0.0;
        const double rx = cfg->sigma * sqrt(qx);
        const double ry = cfg->sigma * sqrt(qy);
        int64_t x0 = o_clip(o_f2i(ceil(cx - rx)), 0, cam->width - 1);
        int64_t x1 = o_clip(o_f2i(floor(cx + rx)), 0, cam->width - 1);
        int64_t y0 = o_clip(o_f2i(ceil(cy - ry)), 0, cam->height - 1);
        int64_t y1 = o_clip(o_f2i(floor(cy + ry)), 0, cam->height - 1);
        const int on_screen = valid && (cx + rx >= 0.0) && (cx - rx <= (double)(cam->width - 1)) &&
                              (cy + ry >= 0.0) && (cy - ry <= (double)(cam->height - 1));

        centers[2 * i] = cx;
        centers[2 * i + 1] = cy;
        cov2[3 * i] = ca;
        cov2[3 * i + 1] = cb;
        cov2[3 * i + 2] = cc;
        inv_abc[3 * i] = ia;
        inv_abc[3 * i + 1] = ib;
        inv_abc[3 * i + 2] = ic;
        zs[i] = z;
        flags[i] = (uint8_t)((in_front ? 1 : 0) | (valid ? 2 : 0) | (on_screen ? 4 : 0));
        bbox[4 * i] = x0;
        bbox[4 * i + 1] = x1;
        bbox[4 * i + 2] = y0;
        bbox[4 * i + 3] = y1;
        if (normals) {
            /* N1: camera-frame normal R_cw R(q)[:,2], flipped to face the camera */
            double nn[3];
            for (int a = 0; a < 3; ++a)
                nn[a] = r_cw[3 * a] * R[2] + r_cw[3 * a + 1] * R[5] + r_cw[3 * a + 2] * R[8];
            const double dp = nn[0] * p[0] + nn[1] * p[1] + nn[2] * p[2];
            const double sg = dp > 0.0 ? -1.0 : 1.0;
            normals[3 * i] = sg * nn[0];
            normals[3 * i + 1] = sg * nn[1];
            normals[3 * i + 2] = sg * nn[2];
        }
    }
    return degenerate;
}

/* ------------------------------------------------------------ depth order */

/* thread-local: the oracle is called from several host threads at once (view-parallel CPU
 * baseline, summed multi-view gradients in the tests) */
static _Thread_local const double *g_sort_z;
static int cmp_z_idx(const void *a, const void *b) {
    const int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
    const double za = g_sort_z[ia], zb = g_sort_z[ib];
    if (za < zb) return -1;
    if (za > zb) return 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

/* order = keep[lexsort((keep, z[keep]))]  (rasterizer.py:318-320): ascending z, ties by index */
int64_t o_depth_order(int64_t n, const double *zs, const uint8_t *flags, int64_t *order) {
    int64_t v = 0;
    for (int64_t i = 0; i < n; ++i)
        if (flags[i] & 4) order[v++] = i;
    g_sort_z = zs;
    qsort(order, (size_t)v, sizeof(int64_t), cmp_z_idx);
    return v;
}

/*
 * Tile-intersection lists derived from the reference bbox:
 * tiles(i) = {(tx,ty): x0/T <= tx <= x1/T, y0/T <= ty <= y1/T}, empty when
 * x0 > x1 or y0 > y1; each tile's list is the global order restricted to it.
 * tile_start has ntiles+1 entries; tile_ids (capacity cap) receives surfel
 * indices.  Returns the pair count (may exceed cap: then only counts).
 */
int64_t o_tile_lists(int64_t v, const int64_t *order, const int64_t *bbox, int64_t width,
                     int64_t height, int64_t tile, int64_t *tile_start, int64_t *tile_ids,
                     int64_t cap) {
    const int64_t ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
    const int64_t nt = ntx * nty;
    int64_t *cnt = (int64_t *)calloc((size_t)nt + 1, sizeof(int64_t));
    for (int64_t r = 0; r < v; ++r) {
        const int64_t *bb = bbox + 4 * order[r];
        if (bb[0] > bb[1] || bb[2] > bb[3]) continue;
        for (int64_t ty = bb[2] / tile; ty <= bb[3] / tile; ++ty)
            for (int64_t tx = bb[0] / tile; tx <= bb[1] / tile; ++tx) cnt[ty * ntx + tx]++;
    }
    tile_start[0] = 0;
    for (int64_t t = 0; t < nt; ++t) tile_start[t + 1] = tile_start[t] + cnt[t];
    const int64_t total = tile_start[nt];
    if (total <= cap) {
        memset(cnt, 0, sizeof(int64_t) * (size_t)nt);
        for (int64_t r = 0; r < v; ++r) {
            const int64_t i = order[r];
            const int64_t *bb = bbox + 4 * i;
            if (bb[0] > bb[1] || bb[2] > bb[3]) continue;
            for (int64_t ty = bb[2] / tile; ty <= bb[3] / tile; ++ty)
                for (int64_t tx = bb[0] / tile; tx <= bb[1] / tile; ++tx) {
                    const int64_t t = ty * ntx + tx;
                    tile_ids[tile_start[t] + cnt[t]++] = i;
                }
        }
    }
    free(cnt);
    return total;
}

/* ------------------------------------------------------------ blend forward */

/*
 * blend_forward (_raster_kernels.py:22-55) over the sorted order, plus the
 * normal channel (N1).  Buffers are caller-initialised like rasterizer.py:304-308
 * (color/depth/normal 0, trans 1, max_w 0, arg_w -1).  arg_w receives the
 * input index (the reference remaps sorted->input at rasterizer.py:327-328).
 */
void o_blend_forward(int64_t v, const int64_t *order, const double *centers, const double *inv_abc,
                     const double *zs, const double *opac, const double *colors,
                     const double *normals, const int64_t *bbox, double w_clamp, double term_t,
                     double maha_cut, int64_t width, double *color, double *depth, double *trans,
                     double *normal_out, double *max_w, int64_t *arg_w) {
    for (int64_t r = 0; r < v; ++r) {
        const int64_t i = order[r];
        const double cx = centers[2 * i], cy = centers[2 * i + 1];
        const double ia = inv_abc[3 * i], ib = inv_abc[3 * i + 1], ic = inv_abc[3 * i + 2];
        const int64_t *bb = bbox + 4 * i;
        for (int64_t y = bb[2]; y <= bb[3]; ++y) {
            const double dy = (double)y - cy;
            for (int64_t x = bb[0]; x <= bb[1]; ++x) {
                const int64_t p = y * width + x;
                const double t = trans[p];
                if (t < term_t) continue;
                const double dx = (double)x - cx;
                const double m = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                if (m > maha_cut) continue;
                double w = opac[i] * exp(-0.5 * m);
                if (w > w_clamp) w = w_clamp;
                if (w <= 0.0) continue;
                const double contrib = w * t;
                color[3 * p] += contrib * colors[3 * i];
                color[3 * p + 1] += contrib * colors[3 * i + 1];
                color[3 * p + 2] += contrib * colors[3 * i + 2];
                depth[p] += contrib * zs[i];
                if (normal_out) {
                    normal_out[3 * p] += contrib * normals[3 * i];
                    normal_out[3 * p + 1] += contrib * normals[3 * i + 1];
                    normal_out[3 * p + 2] += contrib * normals[3 * i + 2];
                }
                if (contrib > max_w[p]) {
                    max_w[p] = contrib;
                    arg_w[p] = i;
                }
                trans[p] = t * (1.0 - w);
            }
        }
    }
}

/* max_blend_weights (_raster_kernels.py:116-147); outputs indexed by input index */
void o_max_blend_weights(int64_t v, const int64_t *order, const double *centers,
                         const double *inv_abc, const double *opac, const int64_t *bbox,
                         double w_clamp, double term_t, double maha_cut, const uint8_t *mask,
                         int64_t height, int64_t width, double *max_all, double *max_marked) {
    double *trans = (double *)malloc(sizeof(double) * (size_t)(height * width));
    for (int64_t p = 0; p < height * width; ++p) trans[p] = 1.0;
    for (int64_t r = 0; r < v; ++r) {
        const int64_t i = order[r];
        const double cx = centers[2 * i], cy = centers[2 * i + 1];
        const double ia = inv_abc[3 * i], ib = inv_abc[3 * i + 1], ic = inv_abc[3 * i + 2];
        const int64_t *bb = bbox + 4 * i;
        for (int64_t y = bb[2]; y <= bb[3]; ++y) {
            const double dy = (double)y - cy;
            for (int64_t x = bb[0]; x <= bb[1]; ++x) {
                const int64_t p = y * width + x;
                const double t = trans[p];
                if (t < term_t) continue;
                const double dx = (double)x - cx;
                const double m = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                if (m > maha_cut) continue;
                double w = opac[i] * exp(-0.5 * m);
                if (w > w_clamp) w = w_clamp;
                if (w <= 0.0) continue;
                const double alpha = w * t;
                if (alpha > max_all[i]) max_all[i] = alpha;
                if (mask[p] != 0 && alpha > max_marked[i]) max_marked[i] = alpha;
                trans[p] = t * (1.0 - w);
            }
        }
    }
    free(trans);
}

/* --------------------------------------------------------------- loss seeds */

/*
 * kind 0: render_loss / grad seeds of the reference (rasterizer.py:346-357, 375-380):
 *   mse*mean((C-C*)^2) + depth*mean_{acc>0.5}((D-D*)^2)
 * kind 1: L1 (BASELINE configs 2,4,5; N3): w_rgb*mean|C-C*| + w_depth*mean|D-D*|,
 *   depth term over all pixels (mask_depth=0) or over acc>0.5 (mask_depth=1).
 * Writes g_rgb (X,3), g_depth (X); returns the loss.
 */
double o_loss_seeds(int kind, int64_t npx, const double *color, const double *depth,
                    const double *acc, const double *t_rgb, const double *t_depth, double w_rgb,
                    double w_depth, int mask_depth, double *g_rgb, double *g_depth) {
    int64_t n_mask = 0;
    const int use_mask = (kind == 0) ? 1 : mask_depth;
    for (int64_t p = 0; p < npx; ++p)
        if (!use_mask || acc[p] > 0.5) n_mask++;
    double srgb = 0.0, sd = 0.0;
    if (kind == 0) {
        const double k = w_rgb * (2.0 / (double)(npx * 3));
        for (int64_t p = 0; p < 3 * npx; ++p) {
            const double d = color[p] - t_rgb[p];
            srgb += d * d;
            g_rgb[p] = k * d;
        }
        for (int64_t p = 0; p < npx; ++p) {
            g_depth[p] = 0.0;
            if (w_depth != 0.0 && n_mask && acc[p] > 0.5) {
                const double d = depth[p] - t_depth[p];
                sd += d * d;
                g_depth[p] = w_depth * (2.0 / (double)n_mask) * d;
            }
        }
        double loss = w_rgb * (srgb / (double)(npx * 3));
        if (w_depth != 0.0 && n_mask) loss += w_depth * (sd / (double)n_mask);
        return loss;
    }
    const double k = w_rgb / (double)(npx * 3);
    for (int64_t p = 0; p < 3 * npx; ++p) {
        const double d = color[p] - t_rgb[p];
        srgb += fabs(d);
        g_rgb[p] = d > 0.0 ? k : (d < 0.0 ? -k : 0.0);
    }
    const double kd = n_mask ? w_depth / (double)n_mask : 0.0;
    for (int64_t p = 0; p < npx; ++p) {
        g_depth[p] = 0.0;
        if (use_mask && !(acc[p] > 0.5)) continue;
        const double d = depth[p] - t_depth[p];
        sd += fabs(d);
        g_depth[p] = d > 0.0 ? kd : (d < 0.0 ? -kd : 0.0);
    }
    double loss = w_rgb * srgb / (double)(npx * 3);
    if (n_mask) loss += w_depth * sd / (double)n_mask;
    return loss;
}

/* ------------------------------------------------------------ blend backward */

/*
 * blend_gradients (_raster_kernels.py:58-113) generalised: same forward-order
 * recomputation with prefix sums; colour/opacity gradients are exactly the
 * reference's.  Extra outputs (N2 inputs), all indexed by INPUT surfel index:
 *   g2[i*8 + 0..7] = dL/d(ia, ib, ic, cx, cy, z, -, -)
 *   gn[i*3 + 0..2] = dL/d(normal)
 * g_normal / g_acc seeds may be NULL.
 */
void o_blend_backward(int64_t v, const int64_t *order, const double *centers,
                      const double *inv_abc, const double *zs, const double *opac,
                      const double *colors, const double *normals, const int64_t *bbox,
                      double w_clamp, double term_t, double maha_cut, int64_t height,
                      int64_t width, const double *final_color, const double *final_depth,
                      const double *final_normal, const double *final_trans, const double *g_rgb,
                      const double *g_depth, const double *g_normal, const double *g_acc,
                      double *grad_color, double *grad_opac, double *g2, double *gn) {
    const int64_t X = height * width;
    double *trans = (double *)malloc(sizeof(double) * (size_t)X);
    double *pc = (double *)calloc((size_t)(3 * X), sizeof(double));
    double *pd = (double *)calloc((size_t)X, sizeof(double));
    double *pn = (double *)calloc((size_t)(3 * X), sizeof(double));
    for (int64_t p = 0; p < X; ++p) trans[p] = 1.0;
    for (int64_t r = 0; r < v; ++r) {
        const int64_t i = order[r];
        const double cx = centers[2 * i], cy = centers[2 * i + 1];
        const double ia = inv_abc[3 * i], ib = inv_abc[3 * i + 1], ic = inv_abc[3 * i + 2];
        const double *ci = colors + 3 * i;
        const double *ni = normals ? normals + 3 * i : NULL;
        const int64_t *bb = bbox + 4 * i;
        for (int64_t y = bb[2]; y <= bb[3]; ++y) {
            const double dy = (double)y - cy;
            for (int64_t x = bb[0]; x <= bb[1]; ++x) {
                const int64_t p = y * width + x;
                const double t = trans[p];
                if (t < term_t) continue;
                const double dx = (double)x - cx;
                const double m = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                if (m > maha_cut) continue;
                const double g = exp(-0.5 * m);
                const double w_raw = opac[i] * g;
                const int clamped = w_raw > w_clamp;
                const double w = clamped ? w_clamp : w_raw;
                if (w <= 0.0) continue;
                const double alpha = w * t;
                for (int ch = 0; ch < 3; ++ch) grad_color[3 * i + ch] += g_rgb[3 * p + ch] * alpha;
                g2[8 * i + 5] += g_depth[p] * alpha;
                if (g_normal && ni)
                    for (int ch = 0; ch < 3; ++ch) gn[3 * i + ch] += g_normal[3 * p + ch] * alpha;
                if (!clamped) {
                    double acc = 0.0;
                    if (w < 1.0) {
                        const double inv_rest = 1.0 / (1.0 - w);
                        for (int ch = 0; ch < 3; ++ch) {
                            const double suffix = final_color[3 * p + ch] - pc[3 * p + ch] - alpha * ci[ch];
                            acc += g_rgb[3 * p + ch] * (t * ci[ch] - suffix * inv_rest);
                        }
                        const double sfx_d = final_depth[p] - pd[p] - alpha * zs[i];
                        acc += g_depth[p] * (t * zs[i] - sfx_d * inv_rest);
                        if (g_normal && ni)
                            for (int ch = 0; ch < 3; ++ch) {
                                const double s = final_normal[3 * p + ch] - pn[3 * p + ch] - alpha * ni[ch];
                                acc += g_normal[3 * p + ch] * (t * ni[ch] - s * inv_rest);
                            }
                        if (g_acc) acc += g_acc[p] * final_trans[p] * inv_rest;
                    } else {
                        for (int ch = 0; ch < 3; ++ch) acc += g_rgb[3 * p + ch] * t * ci[ch];
                        acc += g_depth[p] * t * zs[i];
                        if (g_normal && ni)
                            for (int ch = 0; ch < 3; ++ch) acc += g_normal[3 * p + ch] * t * ni[ch];
                        if (g_acc) acc += g_acc[p] * t;
                    }
                    grad_opac[i] += g * acc;
                    /* dL/dm = dL/dw * dw/dm = acc * (-0.5 * w) */
                    const double gm = -0.5 * w * acc;
                    g2[8 * i + 0] += gm * dx * dx;
                    g2[8 * i + 1] += gm * 2.0 * dx * dy;
                    g2[8 * i + 2] += gm * dy * dy;
                    g2[8 * i + 3] += gm * (-2.0 * (ia * dx + ib * dy));
                    g2[8 * i + 4] += gm * (-2.0 * (ib * dx + ic * dy));
                }
                for (int ch = 0; ch < 3; ++ch) pc[3 * p + ch] += alpha * ci[ch];
                pd[p] += alpha * zs[i];
                if (ni)
                    for (int ch = 0; ch < 3; ++ch) pn[3 * p + ch] += alpha * ni[ch];
                trans[p] = t * (1.0 - w);
            }
        }
    }
    free(trans);
    free(pc);
    free(pd);
    free(pn);
}

/* ---------------------------------------------------- geometry backward (N2) */

/* d R(q) / d q contracted with G (3x3, row-major): returns dL/dq (4) for raw q */
static void o_dR_dq(const double q[4], const double G[9], double out[4]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    /* R entries as in o_quat_to_matrix */
    /* dR/dw */
    const double dw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
    const double dx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
    const double dy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
    const double dz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
    double a = 0, b = 0, c = 0, d = 0;
    for (int k = 0; k < 9; ++k) {
        a += G[k] * dw[k];
        b += G[k] * dx[k];
        c += G[k] * dy[k];
        d += G[k] * dz[k];
    }
    out[0] = a;
    out[1] = b;
    out[2] = c;
    out[3] = d;
}

/*
 * Chain dL/d(ia,ib,ic,cx,cy,z,normal) of each on-screen surfel back to its
 * parameters through the reference's own forward map (rasterizer.py:204-248):
 * inv_abc <- cov2 = J C J^T <- (J(p), C = Bc Bc^T), Bc = m_cw R(q)[:, :2] diag(s),
 * p = s_inv R(q_inv) mu + t_inv.  Accumulates (+=) into grad_means (N,3),
 * grad_quats (N,4), grad_scales (N,2).  Normal flip sign recomputed.
 */
void o_geometry_backward(int64_t n, const double *means, const double *quats,
                         const double *scales, const double inv[8], const double m_cw[9],
                         const double r_cw[9], const o_cam *cam, const uint8_t *flags,
                         const double *inv_abc, const double *g2, const double *gn,
                         double *grad_means, double *grad_quats, double *grad_scales) {
    double Rinv[9];
    o_quat_to_matrix(inv + 4, Rinv);
    for (int64_t i = 0; i < n; ++i) {
        if (!(flags[i] & 4)) continue;
        double r[3], p[3];
        o_quat_rotate(inv + 4, means + 3 * i, r);
        for (int a = 0; a < 3; ++a) p[a] = inv[0] * r[a] + inv[1 + a];
        const double z = p[2], x = p[0], y = p[1];
        double R[9];
        o_quat_to_matrix(quats + 4 * i, R);
        const double s0 = scales[2 * i], s1 = scales[2 * i + 1];
        double Bc[3][2];
        for (int a = 0; a < 3; ++a) {
            Bc[a][0] = (m_cw[3 * a] * R[0] + m_cw[3 * a + 1] * R[3] + m_cw[3 * a + 2] * R[6]) * s0;
            Bc[a][1] = (m_cw[3 * a] * R[1] + m_cw[3 * a + 1] * R[4] + m_cw[3 * a + 2] * R[7]) * s1;
        }
        double C[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) C[a][b] = Bc[a][0] * Bc[b][0] + Bc[a][1] * Bc[b][1];
        double J[2][3] = {{cam->fx / z, 0.0, -cam->fx * x / (z * z)}, {0.0, cam->fy / z, -cam->fy * y / (z * z)}};
        /* dL/dSigma^-1 (symmetric): G = [[gia, gib/2],[gib/2, gic]] */
        const double ia = inv_abc[3 * i], ib = inv_abc[3 * i + 1], ic = inv_abc[3 * i + 2];
        const double *gg = g2 + 8 * i;
        const double G00 = gg[0], G01 = 0.5 * gg[1], G11 = gg[2];
        const double S[2][2] = {{ia, ib}, {ib, ic}};
        const double Gm[2][2] = {{G00, G01}, {G01, G11}};
        double SG[2][2], H[2][2];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) SG[a][b] = S[a][0] * Gm[0][b] + S[a][1] * Gm[1][b];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) H[a][b] = -(SG[a][0] * S[0][b] + SG[a][1] * S[1][b]);
        /* X = J C J^T : dL/dJ = 2 H J C ; dL/dC = J^T H J */
        double HJ[2][3];
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 3; ++c) HJ[a][c] = H[a][0] * J[0][c] + H[a][1] * J[1][c];
        double gJ[2][3];
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 3; ++c) gJ[a][c] = 2.0 * (HJ[a][0] * C[0][c] + HJ[a][1] * C[1][c] + HJ[a][2] * C[2][c]);
        double gC[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) gC[a][b] = J[0][a] * HJ[0][b] + J[1][a] * HJ[1][b];
        /* C = Bc Bc^T : dL/dBc = (gC + gC^T) Bc */
        double gBc[3][2];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 2; ++k) {
                double s = 0.0;
                for (int b = 0; b < 3; ++b) s += (gC[a][b] + gC[b][a]) * Bc[b][k];
                gBc[a][k] = s;
            }
        /* Bc[:,k] = m_cw R[:,k] s_k */
        double gR[9] = {0};
        double gs0 = 0.0, gs1 = 0.0;
        for (int b = 0; b < 3; ++b) {
            double t0 = 0.0, t1 = 0.0;
            for (int a = 0; a < 3; ++a) {
                t0 += m_cw[3 * a + b] * gBc[a][0];
                t1 += m_cw[3 * a + b] * gBc[a][1];
            }
            gR[3 * b + 0] += t0 * s0;
            gR[3 * b + 1] += t1 * s1;
            gs0 += t0 * R[3 * b + 0];
            gs1 += t1 * R[3 * b + 1];
        }
        /* normal n = sg * R_cw R[:,2] */
        if (gn) {
            double nn[3];
            for (int a = 0; a < 3; ++a) nn[a] = r_cw[3 * a] * R[2] + r_cw[3 * a + 1] * R[5] + r_cw[3 * a + 2] * R[8];
            const double sg = (nn[0] * x + nn[1] * y + nn[2] * z) > 0.0 ? -1.0 : 1.0;
            for (int b = 0; b < 3; ++b) {
                double t = 0.0;
                for (int a = 0; a < 3; ++a) t += r_cw[3 * a + b] * gn[3 * i + a];
                gR[3 * b + 2] += sg * t;
            }
        }
        double gq[4];
        o_dR_dq(quats + 4 * i, gR, gq);
        for (int k = 0; k < 4; ++k) grad_quats[4 * i + k] += gq[k];
        grad_scales[2 * i] += gs0;
        grad_scales[2 * i + 1] += gs1;
        /* p: J(p), centers(p), z */
        double gp[3] = {0.0, 0.0, gg[5]};
        const double fx = cam->fx, fy = cam->fy;
        gp[0] += gJ[0][2] * (-fx / (z * z));
        gp[2] += gJ[0][0] * (-fx / (z * z)) + gJ[0][2] * (2.0 * fx * x / (z * z * z));
        gp[1] += gJ[1][2] * (-fy / (z * z));
        gp[2] += gJ[1][1] * (-fy / (z * z)) + gJ[1][2] * (2.0 * fy * y / (z * z * z));
        gp[0] += gg[3] * (fx / z);
        gp[2] += gg[3] * (-fx * x / (z * z));
        gp[1] += gg[4] * (fy / z);
        gp[2] += gg[4] * (-fy * y / (z * z));
        /* p = s_inv * Rot(q_inv) mu + t  (quat_rotate is linear in mu; unit q_inv -> R(q_inv)) */
        for (int b = 0; b < 3; ++b) {
            double t = 0.0;
            for (int a = 0; a < 3; ++a) t += Rinv[3 * a + b] * gp[a];
            grad_means[3 * i + b] += inv[0] * t;
        }
    }
}

/* ------------------------------------------------------------------ Adam (N4) */

/*
 * torch.optim.Adam update (bias-corrected, eps outside the sqrt) on the packed
 * parameter block [means 3N | quats 4N | scales 2N | opac N | colors 3N], then the
 * post-step projection of DESIGN.md: quats renormalised, scales >= scale_min,
 * opacity and colours clipped to [0,1] (mapper.py:334-335).  mask (N) may be NULL.
 */
void o_adam_step(int64_t n, double *params, const double *grads, double *m1, double *m2,
                 int64_t step, double lr_means, double lr_rest, double b1, double b2, double eps,
                 double scale_min, const uint8_t *mask) {
    const double bc1 = 1.0 - pow(b1, (double)step);
    const double bc2 = 1.0 - pow(b2, (double)step);
    const int64_t seg[6] = {0, 3 * n, 7 * n, 9 * n, 10 * n, 13 * n};
    const int per[5] = {3, 4, 2, 1, 3};
    for (int s = 0; s < 5; ++s) {
        const double lr = s == 0 ? lr_means : lr_rest;
        for (int64_t e = seg[s]; e < seg[s + 1]; ++e) {
            const int64_t i = (e - seg[s]) / per[s];
            if (mask && !mask[i]) continue;
            const double g = grads[e];
            m1[e] = b1 * m1[e] + (1.0 - b1) * g;
            m2[e] = b2 * m2[e] + (1.0 - b2) * g * g;
            const double denom = sqrt(m2[e]) / sqrt(bc2) + eps;
            params[e] -= (lr / bc1) * m1[e] / denom;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        if (mask && !mask[i]) continue;
        double *q = params + 3 * n + 4 * i;
        const double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (nq > 0.0)
            for (int k = 0; k < 4; ++k) q[k] /= nq;
        for (int k = 0; k < 2; ++k) {
            double *s = params + 7 * n + 2 * i + k;
            if (*s < scale_min) *s = scale_min;
        }
        double *o = params + 9 * n + i;
        *o = *o < 0.0 ? 0.0 : (*o > 1.0 ? 1.0 : *o);
        for (int k = 0; k < 3; ++k) {
            double *c = params + 10 * n + 3 * i + k;
            *c = *c < 0.0 ? 0.0 : (*c > 1.0 ? 1.0 : *c);
        }
    }
}
