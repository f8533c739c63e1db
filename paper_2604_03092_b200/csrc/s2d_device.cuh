// s2d_device.cuh — device-side data layout and the exact float64 projection.
//
// Every per-surfel geometry quantity that decides WHICH pixels a surfel
// touches and in WHICH order (z, centre, inverse covariance, integer bbox,
// validity) is evaluated in float64 with the reference's operation order,
// using round-to-nearest intrinsics (__dmul_rn/__dadd_rn/...) that the
// compiler never contracts.  This makes z, centres, bbox, on-screen flags and
// hence the depth order and tile lists bit-identical to the reference
// (rasterizer.py:201-281, 318-320).  Per-pixel blending then runs in float32
// with float64 re-checks inside guard bands (see raster.cu).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace s2d {

constexpr int kTile = 16;          // 16x16 pixel tiles, one CTA each
constexpr int kRasterThreads = 256;

// Per-view constants, passed by value as a kernel parameter.
struct ViewParams {
    double inv[8];   // pk_inverse(pose) = [s_inv, t_inv(3), q_inv(4)]  (geometry.py:188-195)
    double m_cw[9];  // inv[0] * quat_to_matrix(q_inv)                  (rasterizer.py:214)
    double r_cw[9];  // quat_to_matrix(q_inv) (rotation only; normals)
    double fx, fy, cx, cy;
    double near_plane, tan_max, max_cond, sigma;
    double mx, my, wmax, hmax;  // centre-margin gate (rasterizer.py:231-236)
    double wm1, hm1;            // W-1, H-1 (rasterizer.py:278-279)
    double w_clamp, maha_cut;   // 0.999, sigma^2
    double term_t;              // termination_transmittance (float64: the argmax variant)
    float w_clamp_f, term_t_f, maha_cut_f;
    int W, H, ntx, nty;
    int64_t n;
    int64_t shard;  // surfels per shard of the packed block (n: the plain layout)
    int mode;  // S2D_SPLAT_AFFINE / S2D_SPLAT_RAY
};

// 64-byte splat record, one per on-screen surfel, indexed by input index.
//   q0: cx_hi, cy_hi, half2(cx_lo, cy_lo) bits, opacity
//   q1: Minv columns (A, C, B, D): (u, v) = (A dx + B dy, C dx + D dy), m = u^2 + v^2 (column
//       order, so (A, C) and (B, D) are register pairs for the packed f32x2 evaluation)
//   q2: r, g, b, z
//   q3: nx, ny, nz, guard band of m around the 3-sigma cut
struct __align__(16) SplatRecord {
    float4 q0, q1, q2, q3;
};

// ---------------------------------------------------------------- exact ops
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// numpy float64 -> int64 cast on x86-64 (cvttsd2si): NaN / out of range -> INT64_MIN
__device__ __forceinline__ int64_t f2i_x86(double v) {
    if (!(v > -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
    return (int64_t)v;
}
__device__ __forceinline__ int64_t clip64(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}
// clip64(f2i_x86(v), 0, hi) for an integral double v without 64-bit integer arithmetic:
// NaN / out of int64 range -> INT64_MIN -> 0; otherwise v clipped to [0, hi]
__device__ __forceinline__ int64_t clip_coord(double v, int64_t hi) {
    if (!(v > -9223372036854775808.0 && v < 9223372036854775808.0) || !(v > 0.0)) return 0;
    return v >= (double)hi ? hi : (int64_t)(int)v;
}

// quat_rotate (geometry.py:59-64), numpy.cross association
__device__ __forceinline__ void quat_rotate_exact(const double q[4], const double v[3], double o[3]) {
    const double w = q[0], u0 = q[1], u1 = q[2], u2 = q[3];
    const double uv0 = dsub(dmul(u1, v[2]), dmul(u2, v[1]));
    const double uv1 = dsub(dmul(u2, v[0]), dmul(u0, v[2]));
    const double uv2 = dsub(dmul(u0, v[1]), dmul(u1, v[0]));
    const double uu0 = dsub(dmul(u1, uv2), dmul(u2, uv1));
    const double uu1 = dsub(dmul(u2, uv0), dmul(u0, uv2));
    const double uu2 = dsub(dmul(u0, uv1), dmul(u1, uv0));
    o[0] = dadd(v[0], dmul(2.0, dadd(dmul(w, uv0), uu0)));
    o[1] = dadd(v[1], dmul(2.0, dadd(dmul(w, uv1), uu1)));
    o[2] = dadd(v[2], dmul(2.0, dadd(dmul(w, uv2), uu2)));
}

// quat_to_matrix (geometry.py:132-142), raw quaternion
__device__ __forceinline__ void quat_to_matrix_exact(const double q[4], double r[9]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
    r[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
    r[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
    r[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
    r[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
    r[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
    r[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
    r[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
    r[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
}

// Packed parameter block: W shards of c surfels each, shard s = [means 3c | quats 4c | scales 2c |
// opac c | colors 3c] for surfels [s c, (s + 1) c).  c = n (one shard) is the plain layout
// [means 3n | quats 4n | scales 2n | opac n | colors 3n]; with W ranks sharding the optimizer,
// c = ceil(n / W) makes each rank's slice of the parameter and gradient blocks contiguous (one
// reduce-scatter and one in-place all-gather, distributed.py).
template <class T>
struct SurfelPtrs {
    T *means, *quats, *scales, *opac, *colors;
};
template <class T>
__host__ __device__ __forceinline__ SurfelPtrs<T> surfel_ptrs(T *base, int64_t n, int64_t c, int64_t i) {
    const int64_t s = c >= n ? 0 : (int64_t)((uint32_t)i / (uint32_t)c);
    const int64_t j = i - s * c;
    T *b = base + s * 13 * c;
    return {b + 3 * j, b + 3 * c + 4 * j, b + 7 * c + 2 * j, b + 9 * c + j, b + 10 * c + 3 * j};
}
using ParamPtrs = SurfelPtrs<const float>;

struct ExactProj {
    double p[3];        // camera-frame mean
    double R[9];        // quat_to_matrix(q)
    double Bc[3][2];    // basis_cam
    double J[2][3];     // projection Jacobian at p
    double a, b, c;     // cov2
    double cx, cy;      // pixel centre
    double ia, ib, ic;  // inv_abc
    double lmin, lmax;
    double rx, ry;
    int64_t x0, x1, y0, y1;
    bool in_front, valid, on_screen;
};

// _project_batch (rasterizer.py:201-249) + _footprint_boxes (rasterizer.py:262-281)
// for one surfel, bit-exact with the reference (see header comment).
__device__ __forceinline__ void project_exact(const ViewParams &P, const ParamPtrs &pv, ExactProj &o) {
    const double mu[3] = {(double)pv.means[0], (double)pv.means[1],
                          (double)pv.means[2]};
    double r[3];
    quat_rotate_exact(P.inv + 4, mu, r);
    o.p[0] = dadd(dmul(P.inv[0], r[0]), P.inv[1]);
    o.p[1] = dadd(dmul(P.inv[0], r[1]), P.inv[2]);
    o.p[2] = dadd(dmul(P.inv[0], r[2]), P.inv[3]);
    const double z = o.p[2];
    bool in_front = z > P.near_plane;
    if (in_front) {
        // hypot(x, y) <= tan_max z (rasterizer.py:206-210): decided on x^2 + y^2 against t^2 when
        // they differ by more than 1e-12 relative (far beyond the few ulps separating
        // sqrt(x^2 + y^2) from hypot), else by hypot itself; overflow / NaN fall through to hypot
        const double t = dmul(P.tan_max, z), t2 = dmul(t, t);
        const double s2 = dfma(o.p[0], o.p[0], dmul(o.p[1], o.p[1]));
        if (s2 < t2 * (1.0 - 1e-12)) in_front = true;
        else if (s2 > t2 * (1.0 + 1e-12)) in_front = false;
        else in_front = hypot(o.p[0], o.p[1]) <= t;
    }
    const double zs = in_front ? z : 1.0;
    o.cx = dadd(ddiv(dmul(P.fx, o.p[0]), zs), P.cx);
    o.cy = dadd(ddiv(dmul(P.fy, o.p[1]), zs), P.cy);
    in_front = in_front && (o.cx >= -P.mx) && (o.cx <= P.wmax) && (o.cy >= -P.my) && (o.cy <= P.hmax);
    o.in_front = in_front;
    if (!in_front) {  // not in front: valid = on_screen = false, nothing else is used
        o.valid = o.on_screen = false;
        return;
    }

    const double q[4] = {(double)pv.quats[0], (double)pv.quats[1],
                         (double)pv.quats[2], (double)pv.quats[3]};
    quat_to_matrix_exact(q, o.R);
    const double s0 = (double)pv.scales[0], s1 = (double)pv.scales[1];
    double B[3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        B[a][0] = dmul(o.R[3 * a], s0);
        B[a][1] = dmul(o.R[3 * a + 1], s1);
    }
    // einsum("ij,njk->nik") : plain sequential sum (rasterizer.py:215)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < 2; ++k)
            o.Bc[a][k] = dadd(dadd(dmul(P.m_cw[3 * a], B[0][k]), dmul(P.m_cw[3 * a + 1], B[1][k])),
                              dmul(P.m_cw[3 * a + 2], B[2][k]));
    // basis_cam @ basis_cam^T (rasterizer.py:216): BLAS dot = a0*b0, then fma
    double C[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) C[a][b] = dfma(o.Bc[a][1], o.Bc[b][1], dmul(o.Bc[a][0], o.Bc[b][0]));
    const double zz = dmul(zs, zs);
    o.J[0][0] = ddiv(P.fx, zs);
    o.J[0][1] = 0.0;
    o.J[0][2] = ddiv(dmul(-P.fx, o.p[0]), zz);
    o.J[1][0] = 0.0;
    o.J[1][1] = ddiv(P.fy, zs);
    o.J[1][2] = ddiv(dmul(-P.fy, o.p[1]), zz);
    // (jac @ cov_cam) @ jac^T (rasterizer.py:224)
    double T1[2][3], X[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            T1[a][c] = dfma(o.J[a][2], C[2][c], dfma(o.J[a][1], C[1][c], dmul(o.J[a][0], C[0][c])));
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c)
            X[a][c] = dfma(T1[a][2], o.J[c][2], dfma(T1[a][1], o.J[c][1], dmul(T1[a][0], o.J[c][0])));
    o.a = dmul(0.5, dadd(X[0][0], X[0][0]));
    o.b = dmul(0.5, dadd(X[0][1], X[1][0]));
    o.c = dmul(0.5, dadd(X[1][1], X[1][1]));

    const double half_tr = dmul(0.5, dadd(o.a, o.c));
    const double amc = dsub(o.a, o.c);
    double d2 = dadd(dmul(0.25, dmul(amc, amc)), dmul(o.b, o.b));
    if (d2 < 0.0) d2 = 0.0;  // np.maximum(x, 0.0); NaN propagates
    const double dev = __dsqrt_rn(d2);
    o.lmin = dsub(half_tr, dev);
    o.lmax = dadd(half_tr, dev);
    const bool well = (o.lmin > 0.0) && (o.lmax <= dmul(P.max_cond, o.lmin));
    o.valid = well;  // in_front holds here
    if (!well) {  // no bbox, no inverse: nothing downstream reads them (on_screen = false)
        o.on_screen = false;
        return;
    }
    // inv_abc (rasterizer.py:247-248): the raster's guard path re-checks m with it
    const double det = dsub(dmul(o.a, o.c), dmul(o.b, o.b));
    o.ia = ddiv(o.c, det);
    o.ib = ddiv(-o.b, det);
    o.ic = ddiv(o.a, det);
    // Footprint radii.  The reference takes rx = sigma sqrt(inv_c / det(inv_abc)) through
    // inv_abc (rasterizer.py:247-248, 264-267), which is sigma sqrt(a) up to rounding amplified
    // by the conditioning: |rx_ref - sigma sqrt(a)| <= 8 eps (kappa + 2) rx, kappa = lmax / lmin
    // (the cancellations in det and det(inv_abc) are bounded by kappa).  When every bbox and
    // on-screen decision below is farther than that (plus the rounding of the sum) from its
    // threshold, it is taken on sigma sqrt(a), else on the reference's own chain (rare: a bbox
    // edge within ~1e-14 px of an integer).
    {
        const double rxf = dmul(P.sigma, __dsqrt_rn(o.a)), ryf = dmul(P.sigma, __dsqrt_rn(o.c));
        const double kap = (double)((float)o.lmax * __frcp_rn((float)o.lmin));  // inf if lmin underflows
        const double vx0 = dsub(o.cx, rxf), vx1 = dadd(o.cx, rxf), vy0 = dsub(o.cy, ryf), vy1 = dadd(o.cy, ryf);
        const double tx = rxf * (4e-15 * (kap + 2.0)), ty = ryf * (4e-15 * (kap + 2.0));
        auto far_int = [](double v, double t) { return fabs(v - rint(v)) > t + 4.5e-16 * fabs(v) + 1e-300; };
        auto far_val = [](double v, double c, double t) {
            return fabs(v - c) > t + 4.5e-16 * (fabs(v) + fabs(c)) + 1e-300;
        };
        if (far_int(vx0, tx) && far_int(vx1, tx) && far_int(vy0, ty) && far_int(vy1, ty) && far_val(vx1, 0.0, tx) &&
            far_val(vx0, P.wm1, tx) && far_val(vy1, 0.0, ty) && far_val(vy0, P.hm1, ty)) {
            o.rx = rxf;
            o.ry = ryf;
            o.x0 = clip_coord(ceil(vx0), P.W - 1);
            o.x1 = clip_coord(floor(vx1), P.W - 1);
            o.y0 = clip_coord(ceil(vy0), P.H - 1);
            o.y1 = clip_coord(floor(vy1), P.H - 1);
            o.on_screen = vx1 >= 0.0 && vx0 <= P.wm1 && vy1 >= 0.0 && vy0 <= P.hm1;
            return;
        }
    }
    double dinv = dsub(dmul(o.ia, o.ic), dmul(o.ib, o.ib));
    if (!(dinv > 0.0)) dinv = 1.0;
    double qx = ddiv(o.ic, dinv), qy = ddiv(o.ia, dinv);
    if (qx < 0.0) qx = 0.0;
    if (qy < 0.0) qy = 0.0;
    o.rx = dmul(P.sigma, __dsqrt_rn(qx));
    o.ry = dmul(P.sigma, __dsqrt_rn(qy));
    o.x0 = clip_coord(ceil(dsub(o.cx, o.rx)), P.W - 1);
    o.x1 = clip_coord(floor(dadd(o.cx, o.rx)), P.W - 1);
    o.y0 = clip_coord(ceil(dsub(o.cy, o.ry)), P.H - 1);
    o.y1 = clip_coord(floor(dadd(o.cy, o.ry)), P.H - 1);
    o.on_screen = o.valid && (dadd(o.cx, o.rx) >= 0.0) && (dsub(o.cx, o.rx) <= P.wm1) &&
                  (dadd(o.cy, o.ry) >= 0.0) && (dsub(o.cy, o.ry) <= P.hm1);
}

// The float64 quantities the per-pixel decisions depend on (reference centre and inv_abc),
// written per on-screen surfel by k_project for the raster guard-band re-checks.  For an
// ill-conditioned splat (accurate_slot below) k_project also writes Minv = M^-1 in float64
// (rows (a, b), (c, d)), which the raster kernels use to evaluate its whitened offset without
// the float32 cancellation.
struct ExactRec {
    double cx, cy, ia, ib, ic;
};

// An ill-conditioned splat (accurate slot, below) also gets its float64 centre and Minv = M^-1
// (rows (ma, mb), (mc, md)) in a separate array, written only for such splats, which the raster
// kernels use to evaluate its whitened offset without the float32 cancellation.
struct AccurateRec {
    double cx, cy, ma, mb, mc, md;
};

// Prefetch an AccurateRec (48 B: at most two 128-B lines) into L1 when an accurate slot is
// staged, so that the later uniform slow branch finds it in L1 instead of waiting on L2.
__device__ __forceinline__ void prefetch_accurate(const AccurateRec *e) {
    const char *p = reinterpret_cast<const char *>(e);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 47));
}

// A splat whose float32 guard band exceeds this (kappa(M) above ~64, or a sub-pixel sigma_min)
// is an "accurate" slot: the float32 whitened offset u = A ex + (B ey + lo) cancels by
// ~kappa(M), which leaves ~5e-7 kappa relative error in its weights and ~3 eps kappa in (u, v),
// i.e. beyond the 1e-4 gradient gate for kappa ~ 100+ (the threshold keeps a 1.5x margin; the
// config-2 seed sweep passes at kappa > 32 and > 64 alike, and > 64 is 7% faster on the
// forward).  Its per-pixel offsets are evaluated in
// float64 from its AccurateRec in both raster passes (same code, so both see the same weights).
#ifndef S2D_ACCURATE_GB
#define S2D_ACCURATE_GB 2.6e-3f
#endif
constexpr float kAccurateGb = S2D_ACCURATE_GB;

// Whitened offset (u, v) = Minv (p - c) and m = |(u, v)|^2 of pixel (px, py) in float64 (the
// accurate-slot path of k_raster_fwd / k_raster_bwd).  Returns m rounded to float32.
__device__ __forceinline__ float accurate_uvm(const AccurateRec &e, int px, int py, float &u, float &v, double &m64) {
    const double dx = dsub((double)px, e.cx), dy = dsub((double)py, e.cy);
    const double U = dfma(e.mb, dy, dmul(e.ma, dx));
    const double V = dfma(e.md, dy, dmul(e.mc, dx));
    m64 = dfma(U, U, dmul(V, V));
    u = (float)U;
    v = (float)V;
    return (float)m64;
}

// Band around the cut inside which the accurate path defers to the reference's own formula
// (exact_maha): the reference's conic m carries ~few eps64 kappa(Sigma) relative error, kappa
// estimated from the guard band (gb ~ 4e-5 kappa(M)); generous by orders of magnitude.
__device__ __forceinline__ double accurate_band(float gb, double cut) {
    const double q = (double)gb * 2.5e4;
    return 4e-14 * (1.0 + q * q) * cut + 1e-12;
}

// Ray-splat footprint (S2D_SPLAT_RAY).  With the camera-frame tangent axes
// a = Bc[:,0], b = Bc[:,1] and centre p, H = K [a b p] maps tangent-plane (u, v, 1) to
// z (x, y, 1), so Hi = H^-1 gives (U, V, S) = Hi (x, y, 1) with (u, v) = (U, V) / S and
// z = 1 / S; the record holds Hi T(x0, y0), acting on pixel offsets from the bbox corner.  The bbox is the pixel AABB of the projected sigma-square [-s, s]^2 of the
// tangent plane, which contains the projected sigma-disk when all four corners are in front
// of the camera (the surfel is dropped otherwise).  Plain float64 (no parity claim).
__device__ __forceinline__ bool ray_setup(const ViewParams &P, const ExactProj &e, double Hi[9], int64_t bb[4]) {
    const double a[3] = {e.Bc[0][0], e.Bc[1][0], e.Bc[2][0]}, b[3] = {e.Bc[0][1], e.Bc[1][1], e.Bc[2][1]};
    const double *c = e.p;
    const double k = P.sigma;
    double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double su = (q & 1) ? k : -k, sv = (q & 2) ? k : -k;
        const double X = c[0] + su * a[0] + sv * b[0], Y = c[1] + su * a[1] + sv * b[1];
        const double Z = c[2] + su * a[2] + sv * b[2];
        if (!(Z > P.near_plane)) return false;
        const double x = P.fx * X / Z + P.cx, y = P.fy * Y / Z + P.cy;
        xmin = fmin(xmin, x);
        xmax = fmax(xmax, x);
        ymin = fmin(ymin, y);
        ymax = fmax(ymax, y);
    }
    if (!(xmax >= 0.0 && xmin <= P.wm1 && ymax >= 0.0 && ymin <= P.hm1)) return false;
    bb[0] = clip64((int64_t)ceil(fmax(xmin, -1.0)), 0, P.W - 1);
    bb[1] = clip64((int64_t)floor(fmin(xmax, P.wm1 + 1.0)), 0, P.W - 1);
    bb[2] = clip64((int64_t)ceil(fmax(ymin, -1.0)), 0, P.H - 1);
    bb[3] = clip64((int64_t)floor(fmin(ymax, P.hm1 + 1.0)), 0, P.H - 1);
    const double H[9] = {P.fx * a[0] + P.cx * a[2], P.fx * b[0] + P.cx * b[2], P.fx * c[0] + P.cx * c[2],
                         P.fy * a[1] + P.cy * a[2], P.fy * b[1] + P.cy * b[2], P.fy * c[1] + P.cy * c[2],
                         a[2], b[2], c[2]};
    const double A0 = H[4] * H[8] - H[5] * H[7], A1 = H[5] * H[6] - H[3] * H[8], A2 = H[3] * H[7] - H[4] * H[6];
    const double det = H[0] * A0 + H[1] * A1 + H[2] * A2;
    if (!(fabs(det) > 1e-300) || !isfinite(det)) return false;  // the plane contains the camera centre
    const double id = 1.0 / det;
    Hi[0] = A0 * id;
    Hi[1] = (H[2] * H[7] - H[1] * H[8]) * id;
    Hi[2] = (H[1] * H[5] - H[2] * H[4]) * id;
    Hi[3] = A1 * id;
    Hi[4] = (H[0] * H[8] - H[2] * H[6]) * id;
    Hi[5] = (H[2] * H[3] - H[0] * H[5]) * id;
    Hi[6] = A2 * id;
    Hi[7] = (H[1] * H[6] - H[0] * H[7]) * id;
    Hi[8] = (H[0] * H[4] - H[1] * H[3]) * id;
    // relative to the bbox corner: Hi T(x0, y0) acts on (x - x0, y - y0, 1), so the float32
    // per-pixel evaluation has no cancellation between large pixel coordinates
    const double x0 = (double)bb[0], y0 = (double)bb[2];
#pragma unroll
    for (int r = 0; r < 3; ++r) Hi[3 * r + 2] += Hi[3 * r] * x0 + Hi[3 * r + 1] * y0;
    return true;
}

// Reference Mahalanobis distance at integer pixel (x, y), float64 with the
// reference's association (_raster_kernels.py:38-39), for guard-band re-checks.
__device__ __forceinline__ double exact_maha(double cx, double cy, double ia, double ib, double ic, int x, int y) {
    const double dx = dsub((double)x, cx);
    const double dy = dsub((double)y, cy);
    return dadd(dadd(dmul(dmul(ia, dx), dx), dmul(dmul(dmul(2.0, ib), dx), dy)), dmul(dmul(ic, dy), dy));
}

// Conservative minimum over the continuous rectangle [x0,x1]x[y0,y1] (pixel coordinates,
// relative to the splat centre) of m(d) = |Minv d|^2: 0 if the centre is inside, else the
// smaller of the minima over the (at most two) edges visible from the centre (the closest
// point of a convex polygon to an outside point, in the whitened metric, lies on a visible
// edge; affine maps keep visibility).  Each edge minimum is a 1-D convex quadratic with the
// minimiser clamped to the edge.
__device__ __forceinline__ float rect_min_maha(float dx0, float dx1, float dy0, float dy1, float A, float B,
                                              float C, float D) {
    const bool vx = dx0 > 0.f || dx1 < 0.f, vy = dy0 > 0.f || dy1 < 0.f;
    if (!vx && !vy) return 0.f;
    const float ac = A * A + C * C, bd = B * B + D * D, x = A * B + C * D;
    // approximate reciprocals are fine: the edge minimiser only needs to be close (the value
    // at a nearby t exceeds the minimum by O(dt^2), far inside the 1e-3 culling slack)
    float iac, ibd;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(iac) : "f"(ac));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ibd) : "f"(bd));
    float best = 3.0e38f;
    if (vy) {  // horizontal edge y = dy0 (centre below) or dy1 (above): minimise over d.x
        const float y = dy0 > 0.f ? dy0 : dy1;
        const float t = fminf(fmaxf(-x * y * iac, dx0), dx1);
        const float u = A * t + B * y, v = C * t + D * y;
        best = u * u + v * v;
    }
    if (vx) {  // vertical edge x = dx0 (centre left) or dx1 (right): minimise over d.y
        const float xx = dx0 > 0.f ? dx0 : dx1;
        const float t = fminf(fmaxf(-x * xx * ibd, dy0), dy1);
        const float u = A * xx + B * t, v = C * xx + D * t;
        best = fminf(best, u * u + v * v);
    }
    return best;
}

// Whether the splat's 3-sigma ellipse can reach the 8x4 warp block with top-left pixel
// (bx0, by0): the continuous minimum of m over the block's pixel-centre rectangle against the
// cut padded by twice the guard band (+1e-3), so the cull is conservative with respect to the
// reference's float64 decision (the pixel test itself re-checks m exactly).
__device__ __forceinline__ bool block_reach(int bx0, int by0, const SplatRecord &r, float cut) {
    const uint32_t lob = __float_as_uint(r.q0.z);
    const __half2 lo = *reinterpret_cast<const __half2 *>(&lob);
    const float cx = r.q0.x + __low2float(lo), cy = r.q0.y + __high2float(lo);
    const float thr = cut + 2.f * fabsf(r.q3.w) + 1e-3f;
    return rect_min_maha((float)bx0 - cx, (float)(bx0 + 7) - cx, (float)by0 - cy, (float)(by0 + 3) - cy, r.q1.x,
                         r.q1.z, r.q1.y, r.q1.w) <= thr;
}

// ---------------------------------------------------------- small utilities
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void st_relaxed_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Release/acquire ticket for "last CTA to finish" patterns: the CTA's earlier global writes
// (ordered before this by __syncthreads) are released with the increment, and the CTA that
// draws the last ticket acquires everyone's.  Much cheaper than __threadfence() (fence.sc).
__device__ __forceinline__ uint32_t atomic_add_acq_rel(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Decoupled look-back status word: [flag:2 | value:30]
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

// Decoupled look-back (chained scan).  Tile order is the dynamic ticket order, so every
// predecessor is already running and will publish (no deadlock).

// Warp-cooperative look-back of ONE value: all 32 lanes of one warp call it; each round
// reads 32 predecessors at once, so the walk costs ~1 round trip per 32 predecessors.
// Returns the exclusive prefix (to every lane).
__device__ __forceinline__ uint32_t lookback_warp(uint32_t *status, int tile, uint32_t agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed_u32(status, kFlagInc | agg);
        return 0;
    }
    if (lane == 0) st_relaxed_u32(status + tile, kFlagAgg | agg);
    uint32_t prefix = 0;
    int base = tile - 1;
    while (true) {
        const int j = base - lane;
        const uint32_t s = j >= 0 ? ld_relaxed_u32(status + j) : kFlagInc;
        const uint32_t f = s & ~kValMask;
        const uint32_t inc = __ballot_sync(0xffffffffu, f == kFlagInc);
        const uint32_t pend = __ballot_sync(0xffffffffu, f == 0);
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const uint32_t range = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
        if (pend & range) continue;  // a predecessor in the window has not published yet
        uint32_t v = lane <= first_inc ? (s & kValMask) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (first_inc < 32) break;
        base -= 32;
    }
    if (lane == 0) st_relaxed_u32(status + tile, kFlagInc | (prefix + agg));
    return prefix;
}

// Per-thread look-back of one column of a [tile][stride] status table (one thread per
// digit): predecessors are read 16 at a time (independent loads in flight).
__device__ __forceinline__ uint32_t lookback_batched(uint32_t *status, int stride, int tile, uint32_t agg) {
    if (tile == 0) {
        st_relaxed_u32(status, kFlagInc | agg);
        return 0;
    }
    st_relaxed_u32(status + (size_t)tile * stride, kFlagAgg | agg);
    uint32_t prefix = 0;
    int j = tile - 1;
    while (true) {
        uint32_t s[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) s[k] = (j - k >= 0) ? ld_relaxed_u32(status + (size_t)(j - k) * stride) : kFlagInc;
        int consumed = 0;
        bool done = false;
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // stop at the first unpublished or inclusive word
            const uint32_t f = s[k] & ~kValMask;
            if (f == 0) break;
            prefix += s[k] & kValMask;
            ++consumed;
            if (f == kFlagInc) {
                done = true;
                break;
            }
        }
        if (done) break;
        j -= consumed;
    }
    st_relaxed_u32(status + (size_t)tile * stride, kFlagInc | (prefix + agg));
    return prefix;
}

}  // namespace s2d
