// optim.cu — projection backward (N2) and the fused Adam step (N4).
//
// k_project_bwd: per on-screen surfel, chains the per-view 2D gradients
//   [dL/d opacity, dL/d rgb(3), dL/dz, K = sum dL/dm w w^T (3), e = sum dL/dm w (2), dL/d normal(3)]
// through Minv = (J(p) Bc)^-1, centre(p), z, normal = R_cw R(q)[:,2] back to
// the parameters (means, raw quats, scales, opacity, colours), in float64, and
// ACCUMULATES into the packed gradient block with atomic reductions (views sum with no
// extra pass, mapper.py:300-307, and views in flight on several streams may share it).  It zeroes the consumed 2D gradients so the per-view
// buffer is clean for the next view without a memset.
// k_adam: torch.optim.Adam arithmetic on the packed block, one thread per
// surfel (so the per-surfel mask and the quaternion renormalisation are
// local), followed by the post-step projection of DESIGN.md.
#include "s2d_kernels.h"

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

__global__ void __launch_bounds__(128) k_project_bwd(const ProjectBwdArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const ViewParams &P = a.P;
    if (i >= P.n) return;
    const uint8_t fl = __ldg(a.flags + i);
    if (!(fl & 4)) return;
    // all independent loads are issued up front (one exposed memory latency); stores at the end
    const int64_t n = P.n;
    const float4 *__restrict__ g4 = reinterpret_cast<const float4 *>(a.grad2d + (size_t)i * 16);
    const float4 G0 = g4[0], G1 = g4[1], G2 = g4[2];
    const float G3 = a.grad2d[(size_t)i * 16 + 12];
    float *gmeans = a.grads, *gquats = a.grads + 3 * n;
    float *gscales = a.grads + 7 * n, *gopac = a.grads + 9 * n;
    float *gcol = a.grads + 10 * n;

    // Geometry for the chain rule: plain float64 (contractions allowed, one division for 1/z and
    // one for 1/det M) — only the forward's decisions need the reference's exact arithmetic.
    const ParamView pv(a.params, n);
    struct {
        double p[3], R[9], Bc[3][2], J[2][3];
    } e;
    {
        const double mu[3] = {(double)pv.means[3 * i], (double)pv.means[3 * i + 1], (double)pv.means[3 * i + 2]};
#pragma unroll
        for (int r = 0; r < 3; ++r)
            e.p[r] = P.m_cw[3 * r] * mu[0] + P.m_cw[3 * r + 1] * mu[1] + P.m_cw[3 * r + 2] * mu[2] + P.inv[1 + r];
        const double w = pv.quats[4 * i], x = pv.quats[4 * i + 1], y = pv.quats[4 * i + 2], z = pv.quats[4 * i + 3];
        e.R[0] = 1.0 - 2.0 * (y * y + z * z);
        e.R[1] = 2.0 * (x * y - w * z);
        e.R[2] = 2.0 * (x * z + w * y);
        e.R[3] = 2.0 * (x * y + w * z);
        e.R[4] = 1.0 - 2.0 * (x * x + z * z);
        e.R[5] = 2.0 * (y * z - w * x);
        e.R[6] = 2.0 * (x * z - w * y);
        e.R[7] = 2.0 * (y * z + w * x);
        e.R[8] = 1.0 - 2.0 * (x * x + y * y);
        const double s0 = pv.scales[2 * i], s1 = pv.scales[2 * i + 1];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            e.Bc[r][0] = (P.m_cw[3 * r] * e.R[0] + P.m_cw[3 * r + 1] * e.R[3] + P.m_cw[3 * r + 2] * e.R[6]) * s0;
            e.Bc[r][1] = (P.m_cw[3 * r] * e.R[1] + P.m_cw[3 * r + 1] * e.R[4] + P.m_cw[3 * r + 2] * e.R[7]) * s1;
        }
        const double iz = 1.0 / e.p[2];
        e.J[0][0] = P.fx * iz;
        e.J[0][1] = 0.0;
        e.J[0][2] = -P.fx * e.p[0] * iz * iz;
        e.J[1][0] = 0.0;
        e.J[1][1] = P.fy * iz;
        e.J[1][2] = -P.fy * e.p[1] * iz * iz;
    }
    const double M00 = e.J[0][0] * e.Bc[0][0] + e.J[0][2] * e.Bc[2][0];
    const double M01 = e.J[0][0] * e.Bc[0][1] + e.J[0][2] * e.Bc[2][1];
    const double M10 = e.J[1][1] * e.Bc[1][0] + e.J[1][2] * e.Bc[2][0];
    const double M11 = e.J[1][1] * e.Bc[1][1] + e.J[1][2] * e.Bc[2][1];
    const double id = 1.0 / (M00 * M11 - M01 * M10);
    const double N[2][2] = {{M11 * id, -M01 * id}, {-M10 * id, M00 * id}};
    // 2D gradient record (k_raster_bwd): [opacity, rgb(3), z, K(uu, uv, vv), e(u, v), normal(3)]
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
    double gJ[2][3], gBc[3][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) gJ[r][c] = GM[r][0] * e.Bc[c][0] + GM[r][1] * e.Bc[c][1];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 2; ++k) gBc[c][k] = e.J[0][c] * GM[0][k] + e.J[1][c] * GM[1][k];
    // Bc[:,k] = m_cw R[:,k] s_k
    const double s0 = (double)pv.scales[2 * i], s1 = (double)pv.scales[2 * i + 1];
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
        gs0 += t0 * e.R[3 * b + 0];
        gs1 += t1 * e.R[3 * b + 1];
    }
    // normal = sg * R_cw R[:,2]
    {
        double nn[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            nn[k] = P.r_cw[3 * k] * e.R[2] + P.r_cw[3 * k + 1] * e.R[5] + P.r_cw[3 * k + 2] * e.R[8];
        const double sg = (nn[0] * e.p[0] + nn[1] * e.p[1] + nn[2] * e.p[2]) > 0.0 ? -1.0 : 1.0;
        const double gn[3] = {G2.z, G2.w, G3};
#pragma unroll
        for (int b = 0; b < 3; ++b)
            gR[3 * b + 2] = sg * (P.r_cw[b] * gn[0] + P.r_cw[3 + b] * gn[1] + P.r_cw[6 + b] * gn[2]);
    }
    const double q[4] = {(double)pv.quats[4 * i], (double)pv.quats[4 * i + 1], (double)pv.quats[4 * i + 2],
                         (double)pv.quats[4 * i + 3]};
    double gq[4];
    dR_dq(q, gR, gq);
    // camera-frame mean: J(p), centre(p), z
    const double x = e.p[0], y = e.p[1], z = e.p[2];
    const double fx = P.fx, fy = P.fy;
    const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    double gp0 = 0.0, gp1 = 0.0, gp2 = (double)G1.x;
    gp0 += gJ[0][2] * (-fx * iz2);
    gp2 += gJ[0][0] * (-fx * iz2) + gJ[0][2] * (2.0 * fx * x * iz3);
    gp1 += gJ[1][2] * (-fy * iz2);
    gp2 += gJ[1][1] * (-fy * iz2) + gJ[1][2] * (2.0 * fy * y * iz3);
    gp0 += gcx * (fx * iz);
    gp2 += gcx * (-fx * x * iz2);
    gp1 += gcy * (fy * iz);
    gp2 += gcy * (-fy * y * iz2);
    // p = s_inv R(q_inv) mu + t_inv.  Accumulation is atomic (fire-and-forget reductions), so
    // views running concurrently on different streams may share one gradient block.
#pragma unroll
    for (int b = 0; b < 3; ++b)
        atomicAdd(gmeans + 3 * i + b, (float)(P.inv[0] * (P.r_cw[b] * gp0 + P.r_cw[3 + b] * gp1 + P.r_cw[6 + b] * gp2)));
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(gquats + 4 * i + k, (float)gq[k]);
    atomicAdd(gscales + 2 * i, (float)gs0);
    atomicAdd(gscales + 2 * i + 1, (float)gs1);
    atomicAdd(gopac + i, G0.x);
    atomicAdd(gcol + 3 * i, G0.y);
    atomicAdd(gcol + 3 * i + 1, G0.z);
    atomicAdd(gcol + 3 * i + 2, G0.w);
    // leave the per-view 2D gradient buffer zeroed for the next view
    float4 *zero = reinterpret_cast<float4 *>(a.grad2d + (size_t)i * 16);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    zero[0] = z4;
    zero[1] = z4;
    zero[2] = z4;
    zero[3] = z4;
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
    const float denom = sqrtf(v) * k.inv_sqrt_bc2 + k.eps;
    return p - step_size * (m / denom);
}

__global__ void __launch_bounds__(256) k_adam(float *__restrict__ params, const float *__restrict__ grads,
                                              float *__restrict__ m1, float *__restrict__ m2, int64_t n,
                                              const AdamK k, const uint8_t *__restrict__ mask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
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

}  // namespace

void launch_project_backward(const ProjectBwdArgs &a, cudaStream_t s) {
    const int64_t blocks = (a.P.n + 127) / 128;
    if (blocks > 0) {
        count_launch();
        k_project_bwd<<<(unsigned)blocks, 128, 0, s>>>(a);
    }
}

void launch_adam(float *params, const float *grads, float *m1, float *m2, int64_t n, int64_t step,
                 const s2d_adam_config &cfg, const uint8_t *mask, cudaStream_t s) {
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
    const int64_t blocks = (n + 255) / 256;
    if (blocks > 0) {
        count_launch();
        k_adam<<<(unsigned)blocks, 256, 0, s>>>(params, grads, m1, m2, n, k, mask);
    }
}

}  // namespace s2d
