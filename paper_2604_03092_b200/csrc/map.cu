// map.cu — map maintenance around the render path:
//
//   k_transform   transform_surfels (mapper.py:184-197): Sim(3) warp of packed surfels --
//                 means by pk_act (geometry.py:198-199), rotations left-composed with
//                 quat_mul (geometry.py:39-50) and canonicalised (geometry.py:71-84), tangent
//                 scales times the pose scale; opacity and colour copied.
//   k_fuse_gate   fuse's accumulation gate (mapper.py:212-224): each candidate's own pixel
//                 round(f x / z + c), looked up in the map's rendered accumulation.
//   k_prune_mark  prune's error mask (mapper.py:246-253): covered pixels whose colour or
//                 normalised depth disagrees with the observation.
//   k_prune_keep  prune's victim test (mapper.py:255-256): surfels whose max blending weight
//                 over the marked pixels exceeds the contribution floor are removed.
//
// One thread per surfel / pixel.  The arithmetic is float64 in the reference's operation
// order (round-to-nearest intrinsics, nothing contracted), on float32 inputs; transformed
// parameters are rounded to float32 once at the end.
#include "s2d_kernels.h"

namespace s2d {

namespace {

__device__ __forceinline__ void quat_mul_exact(const double a[4], const double b[4], double o[4]) {
    o[0] = dsub(dsub(dsub(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2])), dmul(a[3], b[3]));
    o[1] = dsub(dadd(dadd(dmul(a[0], b[1]), dmul(a[1], b[0])), dmul(a[2], b[3])), dmul(a[3], b[2]));
    o[2] = dadd(dadd(dsub(dmul(a[0], b[2]), dmul(a[1], b[3])), dmul(a[2], b[0])), dmul(a[3], b[1]));
    o[3] = dadd(dsub(dadd(dmul(a[0], b[3]), dmul(a[1], b[2])), dmul(a[2], b[1])), dmul(a[3], b[0]));
}

// quat_canonicalize: hemisphere w >= 0, ties broken on the first non-zero vector component,
// then + 0.0 so negative zeros become positive.
__device__ __forceinline__ void quat_canonicalize_exact(double q[4]) {
    const bool flip = (q[0] < 0.0) ||
                      (q[0] == 0.0 && ((q[1] < 0.0) || (q[1] == 0.0 && ((q[2] < 0.0) || (q[2] == 0.0 && q[3] < 0.0)))));
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = dadd(flip ? -q[k] : q[k], 0.0);
}

__global__ void __launch_bounds__(256) k_transform(const float *__restrict__ in, float *__restrict__ out, int64_t n,
                                                   const double4 pa, const double4 pq) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ParamPtrs pv = surfel_ptrs(in, n, n, i);
    const double s = pa.x;
    const double q[4] = {pq.x, pq.y, pq.z, pq.w};
    const double t[3] = {pa.y, pa.z, pa.w};
    // means: pk_act = s * quat_rotate(q, p) + t
    const double mu[3] = {(double)pv.means[0], (double)pv.means[1], (double)pv.means[2]};
    double r[3];
    quat_rotate_exact(q, mu, r);
    float *om = out, *oq = out + 3 * n, *os = out + 7 * n, *oo = out + 9 * n, *oc = out + 10 * n;
#pragma unroll
    for (int k = 0; k < 3; ++k) om[3 * i + k] = __double2float_rn(dadd(dmul(s, r[k]), t[k]));
    // rotations: canonicalize(quat_mul(q, q_i))
    const double qi[4] = {(double)pv.quats[0], (double)pv.quats[1], (double)pv.quats[2],
                          (double)pv.quats[3]};
    double qo[4];
    quat_mul_exact(q, qi, qo);
    quat_canonicalize_exact(qo);
#pragma unroll
    for (int k = 0; k < 4; ++k) oq[4 * i + k] = __double2float_rn(qo[k]);
    os[2 * i] = __double2float_rn(dmul(s, (double)pv.scales[0]));
    os[2 * i + 1] = __double2float_rn(dmul(s, (double)pv.scales[1]));
    oo[i] = pv.opac[0];
#pragma unroll
    for (int k = 0; k < 3; ++k) oc[3 * i + k] = pv.colors[k];
}

__global__ void __launch_bounds__(256) k_fuse_gate(const float *__restrict__ acc, const float *__restrict__ params,
                                                   int64_t n, double fx, double fy, double cx, double cy, int W,
                                                   int H, double thr, uint8_t *__restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = params[3 * i], y = params[3 * i + 1], z = params[3 * i + 2];
    // np.round(intr.fx * x / z + intr.cx).astype(int): round half to even, x86 cast
    const int64_t px = f2i_x86(rint(dadd(ddiv(dmul(fx, x), z), cx)));
    const int64_t py = f2i_x86(rint(dadd(ddiv(dmul(fy, y), z), cy)));
    const bool inside = px >= 0 && px < W && py >= 0 && py < H && z > 0.0;
    const double a = inside ? (double)acc[py * W + px] : 0.0;
    keep[i] = a < thr ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_prune_mark(const float *__restrict__ color, const float *__restrict__ depth,
                                                    const float *__restrict__ acc, const float *__restrict__ orgb,
                                                    const float *__restrict__ odep, int64_t npx, double rgb_err,
                                                    double depth_frac, uint8_t *__restrict__ marked) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const double a = acc[p];
    const bool covered = a > 0.5;
    double e = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) e = fmax(e, fabs(dsub((double)color[3 * p + c], (double)orgb[3 * p + c])));
    const bool re = e > rgb_err;
    const double dn = ddiv((double)depth[p], fmax(a, 1e-12));
    const double ob = odep[p];
    const bool de = ob > 0.0 && fabs(dsub(dn, ob)) > dmul(depth_frac, ob);
    marked[p] = (covered && (re || de)) ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_prune_keep(const float *__restrict__ max_marked, int64_t n, double floor_,
                                                    uint8_t *__restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = (double)max_marked[i] > floor_ ? 0 : 1;
}

unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void launch_transform(const float *in, float *out, int64_t n, const double pose[8], cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    k_transform<<<blocks_for(n), 256, 0, s>>>(in, out, n, make_double4(pose[0], pose[1], pose[2], pose[3]),
                                              make_double4(pose[4], pose[5], pose[6], pose[7]));
}

void launch_fuse_gate(const float *acc, const s2d_camera &cam, const float *params, int64_t n, double thr,
                      uint8_t *keep, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    k_fuse_gate<<<blocks_for(n), 256, 0, s>>>(acc, params, n, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                                              thr, keep);
}

void launch_prune_mark(const float *color, const float *depth, const float *acc, const float *orgb,
                       const float *odep, int64_t npx, double rgb_err, double depth_frac, uint8_t *marked,
                       cudaStream_t s) {
    if (npx <= 0) return;
    count_launch();
    k_prune_mark<<<blocks_for(npx), 256, 0, s>>>(color, depth, acc, orgb, odep, npx, rgb_err, depth_frac, marked);
}

void launch_prune_keep(const float *max_marked, int64_t n, double floor_, uint8_t *keep, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    k_prune_keep<<<blocks_for(n), 256, 0, s>>>(max_marked, n, floor_, keep);
}

}  // namespace s2d
