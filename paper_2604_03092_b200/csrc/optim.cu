// optim.cu — projection backward (N2) and the fused Adam step (N4).
//
// k_project_bwd: per on-screen surfel, chains the per-view 2D gradients
//   affine: [dL/d opacity, dL/d rgb(3), dL/dz, K = sum dL/dm w w^T (3), e = sum dL/dm w (2), dL/d normal(3)]
//   ray:    [dL/d opacity, dL/d rgb(3), dL/dHi (9), dL/d normal(3)]
// through Minv = (J(p) Bc)^-1, centre(p), z (affine) or the ray-splat homography
// Hi = (K [Bc p])^-1 (ray), and normal = R_cw R(q)[:,2], back to the parameters (means, raw
// quats, scales, opacity, colours), in float64, and ACCUMULATES into the packed gradient block
// with atomic reductions (views sum with no extra pass, mapper.py:300-307, and views in flight
// on several streams may share it).  It zeroes the consumed 2D gradients so the per-view
// buffer is clean for the next view without a memset.
// k_adam: torch.optim.Adam arithmetic on the packed block, one thread per
// surfel (so the per-surfel mask and the quaternion renormalisation are
// local), followed by the post-step projection of DESIGN.md.
#include "s2d_kernels.h"

#ifndef S2D_PBWD_THREADS
#define S2D_PBWD_THREADS 64
#endif
#ifdef S2D_PBWD_MINB
#define S2D_PBWD_BOUNDS __launch_bounds__(S2D_PBWD_THREADS, S2D_PBWD_MINB)
#else
#define S2D_PBWD_BOUNDS __launch_bounds__(S2D_PBWD_THREADS)
#endif

namespace s2d {

namespace {

__device__ __forceinline__ void dR_dq(const double q[4], const double G[9], double out[4]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double dw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
    const double dx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
    const double dy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
    const double dz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
    double a = 0, b = 0, c = 0, d = 0;
#pragma unroll
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

template <bool kRay>
__global__ void S2D_PBWD_BOUNDS k_project_bwd(const ProjectBwdArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const ViewParams &P = a.P;
    if (i >= P.n) return;
    const uint8_t fl = __ldg(a.flags + i);
    if (!(fl & 8)) return;  // not drawn: no pixel, no 2D gradient
    // all independent loads are issued up front (one exposed memory latency); stores at the end
    const int64_t n = P.n;
    // the raster backward's row of this surfel: 12 floats (affine, no normal seeds) or 16
    const bool wide = a.g2_stride == 16;
    const float4 *__restrict__ g4 = reinterpret_cast<const float4 *>(a.grad2d + (size_t)i * a.g2_stride);
    const float4 G0 = g4[0], G1 = g4[1], G2 = g4[2];
    const float4 G3 = wide ? g4[3] : make_float4(0.f, 0.f, 0.f, 0.f);

    // Geometry for the chain rule: plain float64 (contractions allowed) — only the forward's
    // decisions need the reference's exact arithmetic.
    const ParamPtrs pv = surfel_ptrs(a.params, n, P.shard, i);
    double p[3], R[9], Bc[3][2];
    {
        const double mu[3] = {(double)pv.means[0], (double)pv.means[1], (double)pv.means[2]};
#pragma unroll
        for (int r = 0; r < 3; ++r)
            p[r] = P.m_cw[3 * r] * mu[0] + P.m_cw[3 * r + 1] * mu[1] + P.m_cw[3 * r + 2] * mu[2] + P.inv[1 + r];
        const double w = pv.quats[0], x = pv.quats[1], y = pv.quats[2], z = pv.quats[3];
        R[0] = 1.0 - 2.0 * (y * y + z * z);
        R[1] = 2.0 * (x * y - w * z);
        R[2] = 2.0 * (x * z + w * y);
        R[3] = 2.0 * (x * y + w * z);
        R[4] = 1.0 - 2.0 * (x * x + z * z);
        R[5] = 2.0 * (y * z - w * x);
        R[6] = 2.0 * (x * z - w * y);
        R[7] = 2.0 * (y * z + w * x);
        R[8] = 1.0 - 2.0 * (x * x + y * y);
        const double s0 = pv.scales[0], s1 = pv.scales[1];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            Bc[r][0] = (P.m_cw[3 * r] * R[0] + P.m_cw[3 * r + 1] * R[3] + P.m_cw[3 * r + 2] * R[6]) * s0;
            Bc[r][1] = (P.m_cw[3 * r] * R[1] + P.m_cw[3 * r + 1] * R[4] + P.m_cw[3 * r + 2] * R[7]) * s1;
        }
    }
    const double fx = P.fx, fy = P.fy;
    // -> dL/dBc (camera-frame tangent axes), dL/dp (camera-frame centre), dL/d normal
    double gBc[3][2], gp[3], gn[3];
    if (kRay) {
        // record (k_raster_bwd, ray): [opacity, rgb(3), dL/dHi' (3x3 row-major), normal(3)] with
        // Hi' = Hi T(x0, y0) for the bbox corner (x0, y0), and
        // Hi = H^-1, H = K [a b p]:  dL/dH = -Hi^T dL/dHi Hi^T,  dL/d[a b p] = K^T dL/dH
        const double H[9] = {fx * Bc[0][0] + P.cx * Bc[2][0], fx * Bc[0][1] + P.cx * Bc[2][1], fx * p[0] + P.cx * p[2],
                             fy * Bc[1][0] + P.cy * Bc[2][0], fy * Bc[1][1] + P.cy * Bc[2][1], fy * p[1] + P.cy * p[2],
                             Bc[2][0], Bc[2][1], p[2]};
        const double A0 = H[4] * H[8] - H[5] * H[7], A1 = H[5] * H[6] - H[3] * H[8], A2 = H[3] * H[7] - H[4] * H[6];
        const double id = 1.0 / (H[0] * A0 + H[1] * A1 + H[2] * A2);
        const double Hi[9] = {A0 * id, (H[2] * H[7] - H[1] * H[8]) * id, (H[1] * H[5] - H[2] * H[4]) * id,
                              A1 * id, (H[0] * H[8] - H[2] * H[6]) * id, (H[2] * H[3] - H[0] * H[5]) * id,
                              A2 * id, (H[1] * H[6] - H[0] * H[7]) * id, (H[0] * H[4] - H[1] * H[3]) * id};
        // the raster kernel summed g (x - x0, y - y0, 1), the gradient w.r.t. Hi' = Hi T(x0, y0):
        // dL/dHi = dL/dHi' T^T
        const short4 bb = a.rect[i];
        const double x0 = bb.x, y0 = bb.z;
        const double GHi[9] = {G1.x + G1.z * x0, G1.y + G1.z * y0, G1.z,
                               G1.w + G2.y * x0, G2.x + G2.y * y0, G2.y,
                               G2.z + G3.x * x0, G2.w + G3.x * y0, G3.x};
        double T[9], GH[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                T[3 * r + c] = Hi[r] * GHi[c] + Hi[3 + r] * GHi[3 + c] + Hi[6 + r] * GHi[6 + c];  // Hi^T GHi
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                GH[3 * r + c] = -(T[3 * r] * Hi[3 * c] + T[3 * r + 1] * Hi[3 * c + 1] + T[3 * r + 2] * Hi[3 * c + 2]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double g0 = fx * GH[j], g1 = fy * GH[3 + j], g2 = P.cx * GH[j] + P.cy * GH[3 + j] + GH[6 + j];
            if (j < 2) {
                gBc[0][j] = g0;
                gBc[1][j] = g1;
                gBc[2][j] = g2;
            } else {
                gp[0] = g0;
                gp[1] = g1;
                gp[2] = g2;
            }
        }
        gn[0] = G3.y;
        gn[1] = G3.z;
        gn[2] = G3.w;
    } else {
        const double iz = 1.0 / p[2], iz2 = iz * iz, iz3 = iz2 * iz;
        const double J[2][3] = {{fx * iz, 0.0, -fx * p[0] * iz2}, {0.0, fy * iz, -fy * p[1] * iz2}};
        const double M00 = J[0][0] * Bc[0][0] + J[0][2] * Bc[2][0];
        const double M01 = J[0][0] * Bc[0][1] + J[0][2] * Bc[2][1];
        const double M10 = J[1][1] * Bc[1][0] + J[1][2] * Bc[2][0];
        const double M11 = J[1][1] * Bc[1][1] + J[1][2] * Bc[2][1];
        const double id = 1.0 / (M00 * M11 - M01 * M10);
        const double N[2][2] = {{M11 * id, -M01 * id}, {-M10 * id, M00 * id}};
        // record (k_raster_bwd, affine): [opacity, rgb(3), z, K(uu, uv, vv), e(u, v), normal(3)]
        // with K = sum dL/dm w w^T and e = sum dL/dm w over the pixels, w = N d the whitened
        // offset (d = pixel - centre, m = |w|^2):   dL/dN = 2 K M^T,   dL/dcentre = -2 N^T e
        const double K[2][2] = {{G1.y, G1.z}, {G1.z, G1.w}};
        const double Mm[2][2] = {{M00, M01}, {M10, M11}};
        double GN[2][2];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) GN[r][c] = 2.0 * (K[r][0] * Mm[c][0] + K[r][1] * Mm[c][1]);
        const double gcx = -2.0 * (N[0][0] * G2.x + N[1][0] * G2.y);
        const double gcy = -2.0 * (N[0][1] * G2.x + N[1][1] * G2.y);
        // dL/dM = -N^T GN N^T
        double T[2][2], GM[2][2];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) T[r][c] = N[0][r] * GN[0][c] + N[1][r] * GN[1][c];  // N^T GN
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) GM[r][c] = -(T[r][0] * N[c][0] + T[r][1] * N[c][1]);  // (N^T GN) N^T
        // M = J Bc
        double gJ[2][3];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) gJ[r][c] = GM[r][0] * Bc[c][0] + GM[r][1] * Bc[c][1];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int k = 0; k < 2; ++k) gBc[c][k] = J[0][c] * GM[0][k] + J[1][c] * GM[1][k];
        // camera-frame mean: J(p), centre(p), z
        const double x = p[0], y = p[1];
        gp[0] = gJ[0][2] * (-fx * iz2) + gcx * (fx * iz);
        gp[1] = gJ[1][2] * (-fy * iz2) + gcy * (fy * iz);
        gp[2] = (double)G1.x + gJ[0][0] * (-fx * iz2) + gJ[0][2] * (2.0 * fx * x * iz3) + gJ[1][1] * (-fy * iz2) +
                gJ[1][2] * (2.0 * fy * y * iz3) + gcx * (-fx * x * iz2) + gcy * (-fy * y * iz2);
        gn[0] = G2.z;
        gn[1] = G2.w;
        gn[2] = G3.x;
    }
    // Bc[:,k] = m_cw R[:,k] s_k
    const double s0 = (double)pv.scales[0], s1 = (double)pv.scales[1];
    double gR[9];
    double gs0 = 0.0, gs1 = 0.0;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            t0 += P.m_cw[3 * r + b] * gBc[r][0];
            t1 += P.m_cw[3 * r + b] * gBc[r][1];
        }
        gR[3 * b + 0] = t0 * s0;
        gR[3 * b + 1] = t1 * s1;
        gs0 += t0 * R[3 * b + 0];
        gs1 += t1 * R[3 * b + 1];
    }
    // normal = sg * R_cw R[:,2]
    {
        double nn[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) nn[k] = P.r_cw[3 * k] * R[2] + P.r_cw[3 * k + 1] * R[5] + P.r_cw[3 * k + 2] * R[8];
        const double sg = (nn[0] * p[0] + nn[1] * p[1] + nn[2] * p[2]) > 0.0 ? -1.0 : 1.0;
#pragma unroll
        for (int b = 0; b < 3; ++b)
            gR[3 * b + 2] = sg * (P.r_cw[b] * gn[0] + P.r_cw[3 + b] * gn[1] + P.r_cw[6 + b] * gn[2]);
    }
    const double q[4] = {(double)pv.quats[0], (double)pv.quats[1], (double)pv.quats[2],
                         (double)pv.quats[3]};
    double gq[4];
    dR_dq(q, gR, gq);
    const SurfelPtrs<float> gout = surfel_ptrs(a.grads, n, P.shard, i);  // same layout as the parameters
    // p = s_inv R(q_inv) mu + t_inv.  Accumulation is atomic (fire-and-forget reductions), so
    // views running concurrently on different streams may share one gradient block.
#pragma unroll
    for (int b = 0; b < 3; ++b)
        atomicAdd(gout.means + b,
                  (float)(P.inv[0] * (P.r_cw[b] * gp[0] + P.r_cw[3 + b] * gp[1] + P.r_cw[6 + b] * gp[2])));
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(gout.quats + k, (float)gq[k]);
    atomicAdd(gout.scales, (float)gs0);
    atomicAdd(gout.scales + 1, (float)gs1);
    atomicAdd(gout.opac, G0.x);
    atomicAdd(gout.colors, G0.y);
    atomicAdd(gout.colors + 1, G0.z);
    atomicAdd(gout.colors + 2, G0.w);
    // leave the per-view 2D gradient buffer zeroed for the next view
    float4 *zero = reinterpret_cast<float4 *>(a.grad2d + (size_t)i * a.g2_stride);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    zero[0] = z4;
    zero[1] = z4;
    zero[2] = z4;
    if (wide) zero[3] = z4;
}

struct AdamK {
    float lr_means, lr_rest, b1, b2, eps, scale_min;
    float step_means, step_rest;  // lr / bias_correction1
    float inv_sqrt_bc2;           // 1 / sqrt(bias_correction2)
};

__device__ __forceinline__ float adam_one(float p, float g, float &m, float &v, float step_size,
                                          const AdamK &k) {
    m = k.b1 * m + (1.f - k.b1) * g;
    v = k.b2 * v + (1.f - k.b2) * g * g;
    // approximate sqrt / reciprocal (~1e-7 relative on a step of ~lr): the IEEE forms cost
    // ~3x the instructions in this instruction-bound kernel, which runs alone at the step's end
    float sv, r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sv) : "f"(v));
    const float denom = sv * k.inv_sqrt_bc2 + k.eps;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(denom));
    return p - step_size * (m * r);
}

__global__ void __launch_bounds__(256) k_adam(float *__restrict__ params, const float *__restrict__ grads,
                                              float *__restrict__ m1, float *__restrict__ m2, int64_t n,
                                              const AdamK k, const uint8_t *__restrict__ mask,
                                              const int32_t *__restrict__ skip) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (skip && *skip)) return;
    if (mask && !mask[i]) return;
    // means
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t e = 3 * i + c;
        float mm = m1[e], vv = m2[e];
        params[e] = adam_one(params[e], grads[e], mm, vv, k.step_means, k);
        m1[e] = mm;
        m2[e] = vv;
    }
    // quats (renormalised after the step)
    float q[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t e = 3 * n + 4 * i + c;
        float mm = m1[e], vv = m2[e];
        q[c] = adam_one(params[e], grads[e], mm, vv, k.step_rest, k);
        m1[e] = mm;
        m2[e] = vv;
    }
    const float nq = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const float inq = nq > 0.f ? 1.f / nq : 1.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) params[3 * n + 4 * i + c] = q[c] * inq;
    // scales
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int64_t e = 7 * n + 2 * i + c;
        float mm = m1[e], vv = m2[e];
        params[e] = fmaxf(adam_one(params[e], grads[e], mm, vv, k.step_rest, k), k.scale_min);
        m1[e] = mm;
        m2[e] = vv;
    }
    // opacity, colours: clip to [0, 1] (mapper.py:334-335)
    {
        const int64_t e = 9 * n + i;
        float mm = m1[e], vv = m2[e];
        params[e] = fminf(fmaxf(adam_one(params[e], grads[e], mm, vv, k.step_rest, k), 0.f), 1.f);
        m1[e] = mm;
        m2[e] = vv;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t e = 10 * n + 3 * i + c;
        float mm = m1[e], vv = m2[e];
        params[e] = fminf(fmaxf(adam_one(params[e], grads[e], mm, vv, k.step_rest, k), 0.f), 1.f);
        m1[e] = mm;
        m2[e] = vv;
    }
}

// mapper.refine's backtracking step (mapper.py:319-335) on the contiguous opacity + colour part
// of the packed block (elements [9n, 13n)): x = clip(x0 - step * g, 0, 1), with g zeroed for
// surfels outside the target mask (mapper.py:320-321); every surfel is clipped, as the
// reference's np.clip over the whole arrays does.
__global__ void __launch_bounds__(256) k_refine_gd(float *__restrict__ x, const float *__restrict__ x0,
                                                   const float *__restrict__ g, int64_t n, double step,
                                                   const uint8_t *__restrict__ mask) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 4 * n) return;
    const int64_t surf = e < n ? e : (e - n) / 3;
    const double gi = (mask && !mask[surf]) ? 0.0 : (double)g[e];
    const double v = (double)x0[e] - step * gi;
    x[e] = (float)fmin(fmax(v, 0.0), 1.0);
}

// max |g| over the targeted surfels' opacity + colour gradients (the L-inf norm of
// mapper.py:322); non-negative floats order like their bit patterns.
__global__ void __launch_bounds__(256) k_refine_gnorm(const float *__restrict__ g, int64_t n,
                                                      const uint8_t *__restrict__ mask, float *out) {
    float mx = 0.f;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < 4 * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t surf = e < n ? e : (e - n) / 3;
        if (!mask || mask[surf]) mx = fmaxf(mx, fabsf(g[e]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.f) atomicMax(reinterpret_cast<int *>(out), __float_as_int(mx));
}

}  // namespace

void launch_refine_gd(float *x, const float *x0, const float *g, int64_t n, double step, const uint8_t *mask,
                      cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    k_refine_gd<<<(unsigned)((4 * n + 255) / 256), 256, 0, s>>>(x, x0, g, n, step, mask);
}

void launch_refine_gnorm(const float *g, int64_t n, const uint8_t *mask, float *out, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    int blocks = (int)((4 * n + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    k_refine_gnorm<<<blocks, 256, 0, s>>>(g, n, mask, out);
}

void launch_project_backward(const ProjectBwdArgs &a, cudaStream_t s) {
    const int64_t blocks = (a.P.n + S2D_PBWD_THREADS - 1) / S2D_PBWD_THREADS;
    if (blocks > 0) {
        count_launch();
        if (a.P.mode == S2D_SPLAT_RAY) k_project_bwd<true><<<(unsigned)blocks, S2D_PBWD_THREADS, 0, s>>>(a);
        else k_project_bwd<false><<<(unsigned)blocks, S2D_PBWD_THREADS, 0, s>>>(a);
    }
}

// The same update over float4 chunks of the packed block (n % 4 == 0, so no chunk straddles a
// segment and every quaternion is one aligned chunk): coalesced 16-B accesses to the four
// arrays instead of one thread per surfel walking strided elements.  Chunk c covers elements
// 4c .. 4c + 3 of segment means [0, 3n) | quats [3n, 7n) | scales [7n, 9n) | opacity [9n, 10n) |
// colours [10n, 13n); an element of a segment with d values per surfel belongs to surfel
// (e - start) / d (the mask).
__global__ void __launch_bounds__(256) k_adam_vec(float4 *__restrict__ params, const float4 *__restrict__ grads,
                                                  float4 *__restrict__ m1, float4 *__restrict__ m2, int64_t n,
                                                  const AdamK k, const uint8_t *__restrict__ mask,
                                                  const int32_t *__restrict__ skip) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 13 * n / 4 || (skip && *skip)) return;
    const int64_t e0 = 4 * c;
    int seg;
    int64_t start;
    int dim;
    if (e0 < 3 * n) { seg = 0; start = 0; dim = 3; }
    else if (e0 < 7 * n) { seg = 1; start = 3 * n; dim = 4; }
    else if (e0 < 9 * n) { seg = 2; start = 7 * n; dim = 2; }
    else if (e0 < 10 * n) { seg = 3; start = 9 * n; dim = 1; }
    else { seg = 4; start = 10 * n; dim = 3; }
    float4 pp = params[c], mm = m1[c], vv = m2[c];
    const float4 g = grads[c];
    float *pv = &pp.x, *mv = &mm.x, *vvv = &vv.x;
    const float *gv = &g.x;
    const float step = seg == 0 ? k.step_means : k.step_rest;
    bool on[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        on[j] = !mask || mask[(e0 + j - start) / dim];
        if (on[j]) pv[j] = adam_one(pv[j], gv[j], mv[j], vvv[j], step, k);
    }
    if (seg == 1) {  // quaternion: renormalised after the step (all four share the surfel's mask)
        if (on[0]) {
            const float nq = sqrtf(pp.x * pp.x + pp.y * pp.y + pp.z * pp.z + pp.w * pp.w);
            const float inq = nq > 0.f ? 1.f / nq : 1.f;
            pp.x *= inq;
            pp.y *= inq;
            pp.z *= inq;
            pp.w *= inq;
        }
    } else if (seg == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) pv[j] = on[j] ? fmaxf(pv[j], k.scale_min) : pv[j];
    } else if (seg >= 3) {  // opacity, colours: clip to [0, 1] (mapper.py:334-335)
#pragma unroll
        for (int j = 0; j < 4; ++j) pv[j] = on[j] ? fminf(fmaxf(pv[j], 0.f), 1.f) : pv[j];
    }
    params[c] = pp;
    m1[c] = mm;
    m2[c] = vv;
}

void launch_adam(float *params, const float *grads, float *m1, float *m2, int64_t n, int64_t step,
                 const s2d_adam_config &cfg, const uint8_t *mask, const int32_t *skip, cudaStream_t s) {
    AdamK k;
    k.lr_means = (float)cfg.lr_means;
    k.lr_rest = (float)cfg.lr_rest;
    k.b1 = (float)cfg.beta1;
    k.b2 = (float)cfg.beta2;
    k.eps = (float)cfg.eps;
    k.scale_min = (float)cfg.scale_min;
    const double bc1 = 1.0 - pow(cfg.beta1, (double)step);
    const double bc2 = 1.0 - pow(cfg.beta2, (double)step);
    k.step_means = (float)(cfg.lr_means / bc1);
    k.step_rest = (float)(cfg.lr_rest / bc1);
    k.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
    if (n > 0 && n % 4 == 0 && ((uintptr_t)params | (uintptr_t)grads | (uintptr_t)m1 | (uintptr_t)m2) % 16 == 0) {
        count_launch();
        const int64_t chunks = 13 * n / 4;
        k_adam_vec<<<(unsigned)((chunks + 255) / 256), 256, 0, s>>>(
            reinterpret_cast<float4 *>(params), reinterpret_cast<const float4 *>(grads), reinterpret_cast<float4 *>(m1),
            reinterpret_cast<float4 *>(m2), n, k, mask, skip);
        return;
    }
    const int64_t blocks = (n + 255) / 256;
    if (blocks > 0) {
        count_launch();
        k_adam<<<(unsigned)blocks, 256, 0, s>>>(params, grads, m1, m2, n, k, mask, skip);
    }
}

}  // namespace s2d
