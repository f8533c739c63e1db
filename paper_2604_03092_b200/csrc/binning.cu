// binning.cu — projection, depth order and tile binning.
//
//   k_project     per-surfel float64 projection (bit-exact with rasterizer.py:201-281),
//                 64-B splat record, bbox; the drawn surfels' (depth key, index) pairs,
//                 compacted within each tile; min/max key; per-tile and per-chunk counts.
//   k_compact_hist concatenates the tiles' pairs in index order, rebases
//                 the keys to 24 bits (key - min, shifted right only if the depth range
//                 spans more than 2^24 key steps) and builds the digit histograms of all
//                 3 passes in the same read.
//   k_onesweep    one stable LSD radix pass (8-bit digits) with decoupled look-back; each
//                 tile is regrouped by digit in shared memory, then written out as
//                 contiguous per-digit runs.
//   k_tie_fix     the depth key is the (rebased) upper 32 bits of the float64 z; runs of
//                 equal keys whose z differ in the low bits are re-sorted by (z64, index),
//                 giving exactly the reference order lexsort((index, z))
//                 (rasterizer.py:318-320).
//   k_scan_emit   chained scan of per-surfel tile counts in depth order, fused with
//                 pair emission: (tile id, surfel index) pairs come out in depth order,
//                 so a stable sort on tile id alone yields per-tile depth-ordered lists.
//   k_tile_ranges [start, end) of each tile in the sorted pair list.
#include <cuda_fp16.h>

#include "s2d_kernels.h"

#ifndef S2D_PROJ_MINB
#define S2D_PROJ_MINB 3
#endif
// 3 CTAs of 256 threads per SM (<= 85 registers): without the bound the compiler takes 98
// registers for k_onesweep and only 2 CTAs fit, which makes every radix pass ~30% slower
#ifndef S2D_SORT_MINB
#define S2D_SORT_MINB 3
#endif
#define S2D_SORT_BOUNDS __launch_bounds__(kSortThreads, S2D_SORT_MINB)
#ifdef S2D_EMIT_MINB
#define S2D_EMIT_BOUNDS __launch_bounds__(256, S2D_EMIT_MINB)
#else
#define S2D_EMIT_BOUNDS __launch_bounds__(256)
#endif

namespace s2d {

namespace {

constexpr uint32_t kFull = 0xffffffffu;

// block-wide exclusive scan of one uint32 per thread (256 threads); returns exclusive
// value, writes block total to *total.
__device__ __forceinline__ uint32_t block_exclusive_scan_256(uint32_t v, uint32_t *smem8,
                                                             uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem8[warp] = x;
    __syncthreads();
    uint32_t wsum = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t t = smem8[w];
        if (w < warp) wsum += t;
        tot += t;
    }
    *total = tot;
    return wsum + x - v;
}

// ------------------------------------------------------------------ projection

// Conservative early rejection: true only when the surfel certainly fails the reference's
// in-front gates (rasterizer.py:206-210, 231-236), judged in float32 with a wide margin.
// Such surfels have in_front = valid = on_screen = false exactly, so the float64 projection
// (divisions, square roots) is skipped for them; everything near a gate boundary takes the
// exact path.
__device__ __forceinline__ bool clearly_out(const ViewParams &P, const ParamPtrs &pv) {
    const float mx = pv.means[0], my = pv.means[1], mz = pv.means[2];
    float p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
        p[r] = (float)P.m_cw[3 * r] * mx + (float)P.m_cw[3 * r + 1] * my + (float)P.m_cw[3 * r + 2] * mz +
               (float)P.inv[1 + r];
    // float32 p carries an absolute error of about 1e-6 |m_cw||mu| + |t|; keep a generous slack
    const float slack = 1e-4f * (fabsf(mx) + fabsf(my) + fabsf(mz) + fabsf((float)P.inv[1]) +
                                 fabsf((float)P.inv[2]) + fabsf((float)P.inv[3]) + 1.f);
    const float z = p[2];
    if (z + slack <= (float)P.near_plane) return true;  // certainly z <= near
    if (z - slack <= 0.f) return false;                 // too close to call: exact path
    const float zl = z - slack, zh = z + slack;
    // centre x range over the z / x uncertainty (fx > 0)
    const float xl = p[0] - slack, xh = p[0] + slack, yl = p[1] - slack, yh = p[1] + slack;
    const float fx = (float)P.fx, fy = (float)P.fy;
    // approximate quotients (2 ulp) are far inside the 1e-3 relative tolerance below
    const float izl = __frcp_rn(zl), izh = __frcp_rn(zh);
    const float cxl = fx * fminf(xl * izl, xl * izh) + (float)P.cx, cxh = fx * fmaxf(xh * izl, xh * izh) + (float)P.cx;
    const float cyl = fy * fminf(yl * izl, yl * izh) + (float)P.cy, cyh = fy * fmaxf(yh * izl, yh * izh) + (float)P.cy;
    const float tol = 1e-3f * (fabsf(cxl) + fabsf(cxh) + fabsf(cyl) + fabsf(cyh) + 1.f);
    return cxh + tol < -(float)P.mx || cxl - tol > (float)P.wmax || cyh + tol < -(float)P.my ||
           cyl - tol > (float)P.hmax;
}

template <bool kRay>
__global__ void __launch_bounds__(kProjThreads, S2D_PROJ_MINB * 256 / kProjThreads) k_project(const ProjectArgs a) {
    __shared__ uint32_t s_wcnt[kProjThreads / 32];
    const int tile = blockIdx.x;
    const int64_t i = (int64_t)tile * kProjThreads + threadIdx.x;
    const ViewParams &P = a.P;
    bool on = false, degen = false;
    uint32_t key = 0xffffffffu;
    const ParamPtrs pv = surfel_ptrs(a.params, P.n, P.shard, i < P.n ? i : 0);
    if (i < P.n && clearly_out(P, pv)) {
        a.flags[i] = 0;
    } else if (i < P.n) {
        ExactProj e;
        project_exact(P, pv, e);
        degen = e.in_front && !e.valid;
        double Hi[9];
        int64_t bb[4] = {e.x0, e.x1, e.y0, e.y1};
        on = kRay ? (e.valid && ray_setup(P, e, Hi, bb)) : e.on_screen;
        // drawn: on screen with a non-empty integer bbox (the sorted, binned set; flag bit 3)
        const bool drawn_b = on && bb[0] <= bb[1] && bb[2] <= bb[3];
        a.flags[i] = (uint8_t)((e.in_front ? 1 : 0) | (e.valid ? 2 : 0) | (on ? 4 : 0) | (drawn_b ? 8 : 0));
        if (on) {
            // camera-frame normal R_cw R(q)[:,2], oriented toward the camera (N1)
            double nn[3];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                nn[k] = P.r_cw[3 * k] * e.R[2] + P.r_cw[3 * k + 1] * e.R[5] + P.r_cw[3 * k + 2] * e.R[8];
            const double sg = (nn[0] * e.p[0] + nn[1] * e.p[1] + nn[2] * e.p[2]) > 0.0 ? -1.0 : 1.0;
            SplatRecord r;
            if (kRay) {
                // q0 = (Hi00, Hi01, Hi02, opacity), q1 = (Hi10, Hi11, Hi12, Hi20),
                // q2 = (r, g, b, Hi21), q3 = (normal, Hi22)
                r.q0 = make_float4((float)Hi[0], (float)Hi[1], (float)Hi[2], pv.opac[0]);
                r.q1 = make_float4((float)Hi[3], (float)Hi[4], (float)Hi[5], (float)Hi[6]);
                r.q2 = make_float4(pv.colors[0], pv.colors[1], pv.colors[2], (float)Hi[7]);
                r.q3 = make_float4((float)(sg * nn[0]), (float)(sg * nn[1]), (float)(sg * nn[2]), (float)Hi[8]);
            } else {
                // M = J Bc (2x2), Minv = M^-1; Sigma = M M^T equals the reference cov2.
                const double M00 = e.J[0][0] * e.Bc[0][0] + e.J[0][2] * e.Bc[2][0];
                const double M01 = e.J[0][0] * e.Bc[0][1] + e.J[0][2] * e.Bc[2][1];
                const double M10 = e.J[1][1] * e.Bc[1][0] + e.J[1][2] * e.Bc[2][0];
                const double M11 = e.J[1][1] * e.Bc[1][1] + e.J[1][2] * e.Bc[2][1];
                const double det = M00 * M11 - M01 * M10;
                const double id = __drcp_rn(det);
                const float cxh = (float)e.cx, cyh = (float)e.cy;
                const __half2 lo = __floats2half2_rn((float)(e.cx - (double)cxh), (float)(e.cy - (double)cyh));
                r.q0 = make_float4(cxh, cyh, __uint_as_float(*reinterpret_cast<const uint32_t *>(&lo)), pv.opac[0]);
                // Minv = (A B; C D) stored by columns: (A, C, B, D), clamped to the float32 range
                // (a splat below ~1e-38 px would overflow to inf, and inf * 0 at its centre pixel
                // would give NaN where the reference has m = 0; FLT_MAX * 0 = 0)
                auto f32c = [](double x) { return (float)fmin(fmax(x, -3.4028234663852886e38), 3.4028234663852886e38); };
                r.q1 = make_float4(f32c(M11 * id), f32c(-M10 * id), f32c(-M01 * id), f32c(M00 * id));
                r.q2 = make_float4(pv.colors[0], pv.colors[1], pv.colors[2], (float)e.p[2]);
                // guard band of the float32 Mahalanobis distance (covers float32 rounding of Minv,
                // of the pixel offset and of u, v, m)
                // (float32 with 1% headroom: it is a bound, not a decision)
                const float lmin_f = (float)e.lmin, lmax_f = (float)e.lmax;
                // (approximate sqrt / rsqrt: ~1e-7 relative, far inside the 1% headroom; a NaN or
                // overflowing band becomes infinite, i.e. every pixel of the splat is re-checked)
                const float rl = rsqrtf(lmin_f);
                float gb = 1.01f * (4e-5f * (lmax_f * rsqrtf(lmax_f)) * rl + 1e-5f * rl + 4e-6f);
                if (!(gb <= 3.0e38f)) gb = __int_as_float(0x7f800000);
                // the guard band is stored negated when the opacity is within 8e-6 of the weight
                // clamp, so the raster kernels test both with one load
                const bool nearclamp = pv.opac[0] > P.w_clamp_f - 8e-6f;
                r.q3 = make_float4((float)(sg * nn[0]), (float)(sg * nn[1]), (float)(sg * nn[2]),
                                   nearclamp ? -gb : gb);
                ExactRec x;
                x.cx = e.cx;
                x.cy = e.cy;
                x.ia = e.ia;
                x.ib = e.ib;
                x.ic = e.ic;
                a.exact[i] = x;
                if (!(gb <= kAccurateGb)) {  // accurate slot (s2d_device.cuh): float64 centre, Minv
                    AccurateRec ar;
                    ar.cx = e.cx;
                    ar.cy = e.cy;
                    ar.ma = M11 * id;
                    ar.mb = -M01 * id;
                    ar.mc = -M10 * id;
                    ar.md = M00 * id;
                    a.acc[i] = ar;
                }
            }
            a.rec[i] = r;
            a.rect[i] = make_short4((short)bb[0], (short)bb[1], (short)bb[2], (short)bb[3]);
            a.z64[i] = e.p[2];
            if (drawn_b) key = (uint32_t)((uint64_t)__double_as_longlong(e.p[2]) >> 32);  // z > 0: monotone
        }
    }
    // per-view counters: visible, drawn, degenerate (rasterizer.py:244), key range
    const bool drawn = key != 0xffffffffu;
    const uint32_t vm = __ballot_sync(kFull, on), dm = __ballot_sync(kFull, degen);
    const uint32_t wm = __ballot_sync(kFull, drawn);
    uint32_t kmin = drawn ? key : 0xffffffffu, kmax = drawn ? key : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(kFull, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        if (vm) atomicAdd(&a.stats->visible, __popc(vm));
        if (wm) {
            atomicMax(a.key_range, ~kmin);  // the sync region starts zeroed: store ~min
            atomicMax(a.key_range + 1, kmax);
        }
        if (dm) atomicAdd(&a.stats->degenerate, __popc(dm));
        s_wcnt[warp] = __popc(wm);
    }
    __syncthreads();
    // The drawn surfels' (depth key, index) pairs, compacted within the tile in index order into
    // the tile's own segment [tile kProjThreads, + count); k_compact_hist concatenates the segments
    // in tile order, so the keys enter the stable radix passes in index order and runs of exactly
    // equal z need no re-sorting (k_tie_fix).  No inter-tile dependency here.
    if (drawn) {
        uint32_t o = (uint32_t)tile * kProjThreads + __popc(wm & lanemask_lt());
        for (int w = 0; w < warp; ++w) o += s_wcnt[w];
        a.keys[o] = key;
        a.vals[o] = (uint32_t)i;
    }
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kProjThreads / 32; ++w) tot += s_wcnt[w];
        a.tcount[tile] = tot;
        // per chunk of kCompactTiles tiles: k_compact_hist derives every chunk's offset from
        // these totals (a few coalesced loads per CTA, no chained scan) and the drawn total
        // (one atomic per tile on a per-chunk word: no single contended counter)
        if (tot) atomicAdd(a.ccount + tile / kCompactTiles, tot);
    }
}

// --------------------------------------------------------------- radix sorting

// Order-preserving compaction + depth-key rebase + digit histograms: CTA c copies the pairs of
// projection tiles [32 c, 32 c + 32) from their segments (k_project) to their place in tile
// order (= index order): the chunk's offset is the sum of the earlier chunks' totals (one
// coalesced warp pass over them), the tiles' offsets within the chunk a warp scan.  Each key is
// rebased to [0, 2^24) (key - min, shifted right only if the depth range spans more than 2^24
// key steps; ties are resolved by k_tie_fix) and its three 8-bit digits histogrammed.
__global__ void __launch_bounds__(256) k_compact_hist(const uint32_t *__restrict__ skeys,
                                                      const uint32_t *__restrict__ svals,
                                                      const uint32_t *__restrict__ tcount,
                                                      const uint32_t *__restrict__ ccount, int ntp,
                                                      const uint32_t *__restrict__ key_range, uint32_t *keys,
                                                      uint32_t *vals, uint32_t *hist, int *n_drawn) {
    __shared__ uint32_t sh[3 * kRadix];
    __shared__ uint32_t s_cnt[kCompactTiles], s_off[kCompactTiles];
    const int tid = threadIdx.x, c = blockIdx.x;
    for (int k = tid; k < 3 * kRadix; k += blockDim.x) sh[k] = 0;
    if (tid < 32) {
        uint32_t base = 0;
        for (int j = tid; j < c; j += 32) base += ccount[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
        const int t = kCompactTiles * c + tid;
        const uint32_t cnt = t < ntp ? tcount[t] : 0u;
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (tid >= o) x += y;
        }
        s_cnt[tid] = cnt;
        s_off[tid] = base + x - cnt;
        if (tid == 31 && c == (int)gridDim.x - 1) *n_drawn = (int)(base + x);  // the drawn total
    }
    __syncthreads();
    const uint32_t kmin = ~key_range[0], kmax = key_range[1];
    const uint32_t span = kmax >= kmin ? kmax - kmin : 0u;
    const int shift = span >= (1u << 24) ? (32 - __clz(span)) - 24 : 0;
    for (int s = tid; s < kCompactTiles * kProjThreads; s += blockDim.x) {
        const int t = s / kProjThreads, j = s % kProjThreads;
        if ((uint32_t)j >= s_cnt[t]) continue;
        const size_t src = (size_t)(kCompactTiles * c + t) * kProjThreads + j;
        const uint32_t k = (skeys[src] - kmin) >> shift;
        const uint32_t o = s_off[t] + j;
        keys[o] = k;
        vals[o] = svals[src];
#pragma unroll
        for (int p = 0; p < 3; ++p) atomicAdd(&sh[p * kRadix + ((k >> (kRadixBits * p)) & (kRadix - 1))], 1u);
    }
    __syncthreads();
    for (int k = tid; k < 3 * kRadix; k += blockDim.x)
        if (sh[k]) atomicAdd(&hist[k], sh[k]);
}

// static shared memory of k_onesweep: the regrouped tile (2 kSortTile words) + per-warp digit
// counts and scans (~10.3 KB); S2D_SORT_ITEMS (keys per thread) is bounded by the 48 KB static limit
static_assert(2 * kSortTile * 4 + (8 * kRadix + 2 * kRadix + 16 + 1) * 4 <= 48 * 1024,
              "k_onesweep: S2D_SORT_ITEMS too large for 48 KB of static shared memory");

__global__ void S2D_SORT_BOUNDS k_onesweep(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, const int *__restrict__ d_n, int n_host, int shift,
    const uint32_t *__restrict__ hist, uint32_t *status, int *ticket) {
    __shared__ uint32_t s_wh[8][kRadix];
    __shared__ uint32_t s_base[kRadix], s_lstart[kRadix];
    __shared__ uint32_t s_w[8], s_w2[8];
    __shared__ uint32_t s_key[kSortTile], s_val[kSortTile];  // the tile regrouped by digit
    __shared__ int s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // n_host >= 0: a pass over n_host entries that skips sentinel keys (0xffffffff); every call
    // passes -1 (the *d_n entries).  The branch is kept on purpose: with it ptxas allocates 80
    // registers and no spills at 3 CTAs/SM; without it, 98 registers (2 CTAs/SM) or 16 B of
    // spills under the same bound, and every radix pass was 20-25% slower.
    const bool drop = n_host >= 0;
    const int n = drop ? n_host : *d_n;
    // the grid is sized for the capacity: CTAs past the entries leave before taking a ticket
    if ((int)blockIdx.x * kSortTile >= n) return;
    if (tid == 0) s_tile = atomicAdd(ticket, 1);
#pragma unroll
    for (int w = 0; w < 8; ++w) s_wh[w][tid] = 0;
    __syncthreads();
    const int tile = s_tile;
    const int start = tile * kSortTile;
    if (start >= n) return;
    const int wbase = start + warp * 32 * kSortItems;
    uint32_t key[kSortItems];
    uint32_t pos[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int idx = wbase + r * 32 + lane;
        key[r] = idx < n ? kin[idx] : 0u;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int idx = wbase + r * 32 + lane;
        const bool valid = idx < n && !(drop && key[r] == 0xffffffffu);
        const uint32_t d = (key[r] >> shift) & (kRadix - 1);
        const uint32_t peers = __match_any_sync(kFull, valid ? d : (kRadix + lane));
        const uint32_t rank = __popc(peers & lt);
        const uint32_t b = valid ? s_wh[warp][d] : 0u;
        __syncwarp();
        if (valid && rank == 0) s_wh[warp][d] = b + __popc(peers);
        __syncwarp();
        pos[r] = b + rank;
    }
    __syncthreads();
    // per digit: exclusive over warps (warp-major = input order), block total
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t c = s_wh[w][tid];
        s_wh[w][tid] = run;
        run += c;
    }
    // global start of each digit (exclusive scan of the pass histogram)
    uint32_t htot;
    const uint32_t dstart = block_exclusive_scan_256(hist[tid], s_w, &htot);
    // block-local start of each digit: the tile is regrouped by digit in shared memory, so the
    // global writes go out as contiguous runs per digit instead of a 256-way scatter
    uint32_t btot;
    const uint32_t lstart = block_exclusive_scan_256(run, s_w2, &btot);
    s_lstart[tid] = lstart;
    const uint32_t prefix = lookback_batched(status + tid, kRadix, tile, run);
    s_base[tid] = dstart + prefix - lstart;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int idx = wbase + r * 32 + lane;
        if (idx < n && !(drop && key[r] == 0xffffffffu)) {
            const uint32_t d = (key[r] >> shift) & (kRadix - 1);
            const uint32_t l = s_lstart[d] + s_wh[warp][d] + pos[r];
            s_key[l] = key[r];
            s_val[l] = vin[idx];
        }
    }
    __syncthreads();
    for (uint32_t l = tid; l < btot; l += kSortThreads) {
        const uint32_t k = s_key[l];
        const uint32_t o = s_base[(k >> shift) & (kRadix - 1)] + l;
        kout[o] = k;
        vout[o] = s_val[l];
    }
}

// Runs of equal (rebased upper-32-bit) depth keys: restore (z64, index) order.
//
// The compaction is order-preserving and the radix passes are stable, so a run of equal keys
// arrives in index order: runs of exactly equal z (a fronto-parallel plane, quantised depth) are
// already in the reference order and cost one comparison per position.  Only keys whose float64
// z differ below the key resolution can be inverted.  Per position:
//   - the head of a run of <= kTieShort entries checks it and, if needed, insertion-sorts it
//     (bounded work, one thread per run, so no claims are needed);
//   - the head of a longer run lists it and checks its first kTieShort entries; an inversion
//     further in is seen by the inverted entry itself (its predecessor kTieShort back shares
//     the key); either sets a flag, and the last CTA of k_tie_fix then sorts the listed runs
//     cooperatively (tie_long).
constexpr int kTieShort = 64;

__device__ __forceinline__ bool zi_less(const double *z64, uint32_t a, uint32_t b) {
    const double za = z64[a], zb = z64[b];
    return za < zb || (za == zb && a < b);
}

__device__ __forceinline__ void tie_fix_at(const uint32_t *__restrict__ keys, uint32_t *vals,
                                           const double *__restrict__ z64, int n, uint32_t *ctl, uint32_t *list,
                                           int r) {
    if (r >= n) return;
    const uint32_t k = keys[r];
    if (r > 0 && keys[r - 1] == k) {
        // not a head: an inversion kTieShort or more entries into a run belongs to a long run
        // (positions r - kTieShort .. r share the key); nearer ones are the head's to check
        if (r >= kTieShort && keys[r - kTieShort] == k && !zi_less(z64, vals[r - 1], vals[r]))
            atomicExch(ctl + 1, 1u);
        return;
    }
    if (r + 1 >= n || keys[r + 1] != k) return;  // run of one (the common case)
    // run head: check the first kTieShort entries; a longer run is listed for tie_long
    const bool longrun = r + kTieShort < n && keys[r + kTieShort] == k;
    int e = r + 1;
    bool sorted = true;
    while (e < n && e - r < kTieShort && keys[e] == k) {
        sorted = sorted && zi_less(z64, vals[e - 1], vals[e]);
        ++e;
    }
    if (longrun) {
        list[atomicAdd(ctl, 1u)] = (uint32_t)r;
        if (!sorted) atomicExch(ctl + 1, 1u);
        return;
    }
    if (sorted) return;
    for (int j = r + 1; j < e; ++j) {  // insertion sort of <= kTieShort entries, by the head only
        const uint32_t v = vals[j];
        const double zv = z64[v];
        int t = j - 1;
        while (t >= r) {
            const uint32_t u = vals[t];
            const double zu = z64[u];
            if (zu > zv || (zu == zv && u > v)) {
                vals[t + 1] = u;
                --t;
            } else {
                break;
            }
        }
        vals[t + 1] = v;
    }
}

// Cooperative sort of the long runs (only when one of them holds an inversion), by one CTA:
// each run's end is found 256 entries at a time; chunks of kTieChunk entries are bitonic-
// sorted in shared memory, then merged pairwise (merge path, 256 threads) through `scratch`.
constexpr int kTieChunk = 512;

__device__ void tie_bitonic_chunk(uint32_t *v, int len, const double *z64, double *sz, uint32_t *si) {
    const int tid = threadIdx.x;
    for (int j = tid; j < kTieChunk; j += blockDim.x) {
        si[j] = j < len ? v[j] : 0xffffffffu;
        sz[j] = j < len ? z64[si[j]] : __longlong_as_double(0x7ff0000000000000ll);  // +inf pads last
    }
    __syncthreads();
    for (int size = 2; size <= kTieChunk; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < kTieChunk / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double za = sz[lo], zb = sz[hi];
                const uint32_t ia = si[lo], ib = si[hi];
                const bool gt = za > zb || (za == zb && ia > ib);
                if (gt == up) {
                    sz[lo] = zb;
                    sz[hi] = za;
                    si[lo] = ib;
                    si[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < len; j += blockDim.x) v[j] = si[j];
    __syncthreads();
}

__device__ void tie_long(const uint32_t *__restrict__ keys, uint32_t *vals, const double *__restrict__ z64, int n,
                         const uint32_t *ctl, const uint32_t *list, uint32_t *scratch) {
    __shared__ double sz[kTieChunk];
    __shared__ uint32_t si[kTieChunk];
    __shared__ int s_end;
    const int tid = threadIdx.x;
    const int nruns = (int)ctl[0];
    for (int q = 0; q < nruns; ++q) {
        const int r0 = (int)list[q];
        const uint32_t k = keys[r0];
        if (tid == 0) s_end = n;
        __syncthreads();
        for (int base = r0 + kTieShort;; base += blockDim.x) {
            const int pos = base + tid;
            if (pos < n && keys[pos] != k) atomicMin(&s_end, pos);
            __syncthreads();
            const int e = s_end;
            __syncthreads();
            if (e < n || base + (int)blockDim.x >= n) break;
        }
        const int len = s_end - r0;
        for (int c = 0; c < len; c += kTieChunk) tie_bitonic_chunk(vals + r0 + c, min(kTieChunk, len - c), z64, sz, si);
        // pairwise merges: src -> dst, widths kTieChunk, 2 kTieChunk, ...
        uint32_t *src = vals + r0, *dst = scratch + r0;
        for (int w = kTieChunk; w < len; w <<= 1) {
            for (int s0 = 0; s0 < len; s0 += 2 * w) {
                const int na = min(w, len - s0), nb = min(w, max(len - s0 - w, 0));
                const uint32_t *A = src + s0, *B = src + s0 + na;
                const int tot = na + nb;
                const int per = (tot + blockDim.x - 1) / blockDim.x;
                const int d0 = min(tid * per, tot), d1 = min(d0 + per, tot);
                // merge path: the split (i, d0 - i) of the first d0 outputs
                int lo = max(0, d0 - nb), hi = min(d0, na);
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (zi_less(z64, B[d0 - mid - 1], A[mid])) hi = mid;  // A[mid] comes after
                    else lo = mid + 1;
                }
                int ia = lo, ib = d0 - lo;
                for (int d = d0; d < d1; ++d) {
                    const bool takeA = ib >= nb || (ia < na && !zi_less(z64, B[ib], A[ia]));
                    dst[s0 + d] = takeA ? A[ia++] : B[ib++];
                }
            }
            __syncthreads();
            uint32_t *t = src;
            src = dst;
            dst = t;
        }
        if (src != vals + r0)
            for (int j = tid; j < len; j += blockDim.x) vals[r0 + j] = src[j];
        __syncthreads();
    }
}

// One thread per position (tie_fix_at); the last CTA to finish (ticket) sorts the long runs when
// one of them holds an inversion (tie_long), so no second launch is needed.
__global__ void __launch_bounds__(256) k_tie_fix(const uint32_t *__restrict__ keys, uint32_t *vals,
                                                 const double *__restrict__ z64, const int *__restrict__ d_n,
                                                 uint32_t *ctl, uint32_t *list, uint32_t *scratch) {
    __shared__ bool s_last;
    const int n = *d_n;
    // the grid is sized for the capacity: CTAs past the drawn count leave at once (they take
    // no ticket, so the last of the active ones runs tie_long)
    const int active = (n + (int)blockDim.x - 1) / (int)blockDim.x;
    if ((int)blockIdx.x >= active) return;
    tie_fix_at(keys, vals, z64, n, ctl, list, blockIdx.x * blockDim.x + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomic_add_acq_rel(ctl + 2, 1u) == (uint32_t)active - 1;
    __syncthreads();
    if (!s_last) return;
    if (*reinterpret_cast<volatile uint32_t *>(ctl + 1) == 0u) return;  // no inversion in any long run
    tie_long(keys, vals, z64, n, ctl, list, scratch);
}

// ----------------------------------------------------------- scan + emission

// The pairs of surfel j of this thread (bbox rc): calls f(tile key, k) for its k-th pair, k
// counting from 0, in the reference's order (rows of tiles, then columns).
template <typename F>
__device__ __forceinline__ void for_each_pair(const short4 rc, int ntx, F &&f) {
    if (!(rc.x <= rc.y && rc.z <= rc.w)) return;
    const int tx0 = rc.x >> 4, tx1 = rc.y >> 4, ty0 = rc.z >> 4, ty1 = rc.w >> 4;
    int k = 0;
    for (int ty = ty0; ty <= ty1; ++ty) {
        // rows of 4-pixel warp blocks the integer bbox overlaps (4 bits -> pairs of mask bits)
        const int by = ty * kTile;
        uint32_t rows = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (rc.z <= by + 4 * q + 3 && rc.w >= by + 4 * q) rows |= 3u << (2 * q);
        for (int tx = tx0; tx <= tx1; ++tx) {
            const int bx = tx * kTile;
            const uint32_t cols = (rc.x <= bx + 7 && rc.y >= bx ? 0x55u : 0u) |
                                  (rc.x <= bx + 15 && rc.y >= bx + 8 ? 0xAAu : 0u);
            // key: tile | bbox-vs-warp-block mask << 16; the forward ORs the ellipse mask into
            // bits 24-31 (raster.cu)
            f((uint32_t)(ty * ntx + tx) | ((rows & cols) << 16), k++);
        }
    }
}

// Per-surfel tile counts scanned in depth order (decoupled look-back across CTAs) and the
// pairs emitted at the scanned offsets.  While warp 0 looks back, the CTA builds its pairs in
// shared memory at their CTA-local offsets (and counts the tile-id digit histograms); after the
// barrier they are written out contiguously from the CTA's base (coalesced).  A CTA whose pairs
// exceed the staging buffer (huge splats) writes them directly after the look-back.
__global__ void S2D_EMIT_BOUNDS k_scan_emit(const EmitArgs a) {
    __shared__ int s_tile;
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_base;
    __shared__ uint32_t s_hist[2 * kRadix];
    __shared__ uint2 s_pairs[kEmitStage > 0 ? kEmitStage : 1];
    const int tid = threadIdx.x;
    const int nv = *a.d_v;
    // the grid is sized for the capacity: CTAs past the drawn surfels leave before the ticket
    if ((int)blockIdx.x * kEmitTile >= nv) return;
    if (tid == 0) s_tile = atomicAdd(a.ticket, 1);
    for (int k = tid; k < 2 * kRadix; k += 256) s_hist[k] = 0;
    __syncthreads();
    const int tile = s_tile;
    const int start = tile * kEmitTile;
    if (start >= nv) return;
    const int r0 = start + tid * kEmitItems;
    uint32_t ids[kEmitItems];
    short4 rc[kEmitItems];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kEmitItems; ++j) {
        const int r = r0 + j;
        ids[j] = r < nv ? a.order[r] : 0u;
        rc[j] = r < nv ? a.rect[ids[j]] : make_short4(1, 0, 1, 0);
        const int tx0 = rc[j].x >> 4, tx1 = rc[j].y >> 4, ty0 = rc[j].z >> 4, ty1 = rc[j].w >> 4;
        if (rc[j].x <= rc[j].y && rc[j].z <= rc[j].w) cnt += (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan_256(cnt, s_w, &tot);
    const bool staged = kEmitStage > 0 && tot <= (uint32_t)kEmitStage;  // CTA-uniform
    const bool two = a.pair_passes > 1;
    if (tid < 32) {
        const uint32_t pre = lookback_warp(a.status, tile, tot);
        const int ntiles = (nv + kEmitTile - 1) / kEmitTile;
        if (tid == 0) s_base = pre;
        if (tid == 0 && tile == ntiles - 1) {
            const uint32_t total = pre + tot;
            a.stats->pairs = (int)total;
            a.stats->pairs_stored = (int)(total < a.pcap ? total : a.pcap);
            if (total > a.pcap) a.stats->overflow = 1;
        }
    }
    if (staged) {
        uint32_t lo = ex;
#pragma unroll
        for (int j = 0; j < kEmitItems; ++j) {
            const uint32_t id = ids[j];
            for_each_pair(rc[j], a.ntx, [&](uint32_t key, int k) {
                s_pairs[lo + k] = make_uint2(key, id);
                const uint32_t t = key & 0xffffu;
                atomicAdd(&s_hist[t & (kRadix - 1)], 1u);
                if (two) atomicAdd(&s_hist[kRadix + ((t >> kRadixBits) & (kRadix - 1))], 1u);
            });
            lo += (rc[j].x <= rc[j].y && rc[j].z <= rc[j].w)
                      ? (uint32_t)(((rc[j].y >> 4) - (rc[j].x >> 4) + 1) * ((rc[j].w >> 4) - (rc[j].z >> 4) + 1))
                      : 0u;
        }
    }
    __syncthreads();
    const uint32_t base = s_base;
    if (staged) {
        for (uint32_t k = tid; k < tot; k += 256) {
            const uint32_t off = base + k;
            const uint2 pr = s_pairs[k];
            if (off < a.pcap) {
                a.pkeys[off] = pr.x;
                a.pvals[off] = pr.y;
            } else {
                // the tile-id passes sort the stored pairs only (pairs_stored entries): their
                // digit histograms must count exactly those, or an overflowing view's passes
                // would place entries past the capacity
                const uint32_t t = pr.x & 0xffffu;
                atomicSub(&s_hist[t & (kRadix - 1)], 1u);
                if (two) atomicSub(&s_hist[kRadix + ((t >> kRadixBits) & (kRadix - 1))], 1u);
            }
        }
    } else {
        uint32_t off = base + ex;
#pragma unroll
        for (int j = 0; j < kEmitItems; ++j) {
            const uint32_t id = ids[j];
            for_each_pair(rc[j], a.ntx, [&](uint32_t key, int) {
                if (off < a.pcap) {
                    a.pkeys[off] = key;
                    a.pvals[off] = id;
                    const uint32_t t = key & 0xffffu;
                    atomicAdd(&s_hist[t & (kRadix - 1)], 1u);
                    if (two) atomicAdd(&s_hist[kRadix + ((t >> kRadixBits) & (kRadix - 1))], 1u);
                }
                ++off;
            });
        }
    }
    __syncthreads();
    for (int k = tid; k < a.pair_passes * kRadix; k += 256)
        if (s_hist[k]) atomicAdd(&a.pair_hist[k], s_hist[k]);
}

__global__ void __launch_bounds__(256) k_tile_ranges(const uint32_t *__restrict__ pkeys,
                                                     const int *__restrict__ d_p, uint32_t pcap,
                                                     int2 *ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int np = *d_p;
    if ((uint32_t)np > pcap) return;  // overflow: leave all tiles empty
    if (i >= np) return;
    const uint32_t k = pkeys[i] & 0xffffu;
    if (i == 0 || (pkeys[i - 1] & 0xffffu) != k) ranges[k].x = i;
    if (i == np - 1 || (pkeys[i + 1] & 0xffffu) != k) ranges[k].y = i + 1;
}

}  // namespace

void launch_project(const ProjectArgs &a, cudaStream_t s) {
    const int blocks = (int)((a.P.n + kProjThreads - 1) / kProjThreads);  // one surfel per thread
    if (blocks > 0) {
        count_launch();
        if (a.P.mode == S2D_SPLAT_RAY) k_project<true><<<blocks, kProjThreads, 0, s>>>(a);
        else k_project<false><<<blocks, kProjThreads, 0, s>>>(a);
    }
}

void launch_compact_hist(const uint32_t *skeys, const uint32_t *svals, const uint32_t *tcount,
                         const uint32_t *ccount, int64_t n, const uint32_t *key_range, uint32_t *keys,
                         uint32_t *vals, uint32_t *hist, int *n_drawn, cudaStream_t s) {
    const int ntp = (int)((n + kProjThreads - 1) / kProjThreads);
    const int blocks = (ntp + kCompactTiles - 1) / kCompactTiles;
    if (blocks > 0) {
        count_launch();
        k_compact_hist<<<blocks, 256, 0, s>>>(skeys, svals, tcount, ccount, ntp, key_range, keys, vals, hist,
                                               n_drawn);
    }
}

void launch_onesweep(const uint32_t *kin, const uint32_t *vin, uint32_t *kout, uint32_t *vout,
                     const int *d_n, int cap, int shift, const uint32_t *hist_pass,
                     uint32_t *status, int *ticket, cudaStream_t s) {
    const int blocks = (cap + kSortTile - 1) / kSortTile;
    if (blocks > 0) {
        count_launch();
        k_onesweep<<<blocks, kSortThreads, 0, s>>>(kin, vin, kout, vout, d_n, -1, shift, hist_pass, status,
                                                   ticket);
    }
}

void launch_tie_fix(const uint32_t *keys, uint32_t *vals, const double *z64, const int *d_n, int cap,
                    uint32_t *ctl, uint32_t *list, uint32_t *scratch, cudaStream_t s) {
    const int blocks = (cap + 255) / 256;
    if (blocks > 0) {
        count_launch();
        k_tie_fix<<<blocks, 256, 0, s>>>(keys, vals, z64, d_n, ctl, list, scratch);
    }
}

void launch_scan_emit(const EmitArgs &a, cudaStream_t s) {
    const int blocks = (a.cap_v + kEmitTile - 1) / kEmitTile;
    if (blocks > 0) {
        count_launch();
        k_scan_emit<<<blocks, 256, 0, s>>>(a);
    }
}

void launch_tile_ranges(const uint32_t *pkeys, const int *d_p, uint32_t pcap, int2 *ranges,
                        cudaStream_t s) {
    const int blocks = (int)((pcap + 255) / 256);
    if (blocks > 0) {
        count_launch();
        k_tile_ranges<<<blocks, 256, 0, s>>>(pkeys, d_p, pcap, ranges);
    }
}

}  // namespace s2d
