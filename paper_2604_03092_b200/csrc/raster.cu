// raster.cu — per-tile front-to-back compositing and its reverse-order backward
// (SURVEY.md §8(a) A7-A9, N1-N3).
//
// A 16x16 tile is split into 8 warp blocks of 8x4 pixels (2 columns x 4 rows); a CTA holds
// kFwdWarps / kBwdWarps of them (4: half a tile).  Lane l owns pixel (l & 7, l >> 3) of its
// warp's block.
//
// Forward (k_raster_fwd): each warp streams its own candidates from the tile's depth-ordered
// list (entries whose bbox bit for its block is set, k_scan_emit) into a warp-private
// double-buffered ring of 80-B slots (cp.async).  A lane-parallel prep phase (one slot per
// lane) culls them against the block with the exact ellipse test and rewrites each kept slot
// to block-relative form (block_centre: exact per-lane pixel offsets, the two cut thresholds,
// a slow-path flag), so the per-candidate work of a lane is 8 FMA-class ops for m, one
// compare, and, on the fast path (m below the guard band, no clamp possible), the blend.  A
// lane whose transmittance fell below the termination threshold carries a NaN x offset, so
// its m fails the cut test with no extra check; the warp stops when every lane has.  For
// every slot its pixels blended the warp appends (surfel, lane mask of the pixels that blended
// it, lane mask of those whose weight clamped) to its blend stream.
//
// Backward (k_raster_bwd): each warp walks its blend streams newest first — one per column
// half of its block, the halves in step, one entry each per step — and runs the reverse
// recurrence (transmittance recovered by division, normalised suffix S <- w c + (1 - w) S) on
// exactly the forward's blended set.  Every lane of a half runs the half's entry (branch-free:
// lanes outside the entry's mask take w = 0, which leaves their state unchanged and zeroes
// their values); each half reduces its entry's 2D gradients over its 16 lanes (transposed
// butterfly) and adds them with one atomic per value.
//
// Fused (k_raster_fused, the refine step's losses without the depth mask): both, per warp
// block — the forward, the loss seeds from the lanes' registers, then the backward traversal
// of the streams just written (still in L2), in one kernel.
//
// Semantics follow blend_forward (_raster_kernels.py:22-55) exactly: the termination test
// precedes blending, pixel (row y, col x) samples (x, y), the Mahalanobis cut is
// `m > sigma^2` on the integer bbox, weights clamp at weight_clamp, `w <= 0` skips.  m and
// the weight clamp are evaluated in float32; inside a per-surfel guard band around the cut
// and around the clamp the decision is re-taken in float64 with the reference's formula, so
// the set of blended pairs equals the reference's.
#include <cuda_fp16.h>

#include <type_traits>

#include "s2d_kernels.h"

#ifndef S2D_FWD_WARPS  // warp blocks (8x4 pixels) per raster CTA: 8 = the whole 16x16 tile
#define S2D_FWD_WARPS 4
#endif
#ifndef S2D_BWD_WARPS
#define S2D_BWD_WARPS 4
#endif
#ifndef S2D_FWD_MINB
#define S2D_FWD_MINB 5
#endif
#ifndef S2D_BWD_MINB
#define S2D_BWD_MINB 4
#endif

namespace s2d {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
// |(1 - T) - 0.5| band of the float32 transmittance inside which the depth mask is re-decided
// in float64 (the float32 T of a pixel is within ~1e-5 of the reference's; 10x margin)
constexpr float kMaskBand = 1e-4f;
constexpr int kFwdWarps = S2D_FWD_WARPS, kBwdWarps = S2D_BWD_WARPS;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Guard-band resolution (rare path): re-takes the reference's decisions for pixel (x, y) and
// surfel `id` in float64 from the projection's exact record.  bit0: the pair blends (pixel
// inside the reference bbox and m <= sigma^2, _raster_kernels.py:32-41); bit1: the weight
// clamps (w > weight_clamp, :43-44).
__device__ __forceinline__ int guard_resolve(const ViewParams &P, const RasterArgs &a, uint32_t id, float op, int x,
                                             int y) {
    const short4 b = a.rect[id];
    if (x < b.x || x > b.y || y < b.z || y > b.w) return 0;
    const ExactRec &e = a.exact[id];
    const double m64 = exact_maha(e.cx, e.cy, e.ia, e.ib, e.ic, x, y);
    if (m64 > P.maha_cut) return 0;
    const double w64 = (double)op * exp(-0.5 * m64);
    return 1 | (w64 > P.w_clamp ? 2 : 0);
}

// Predicated global float add without a branch (one RED instruction under a predicate), so
// a loop step containing it stays one basic block.
__device__ __forceinline__ void red_add_if(float *p, float v, bool c) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.relaxed.gpu.global.add.f32 [%0], %1;\n\t}" ::"l"(p),
        "f"(v), "r"((int)c)
        : "memory");
}

// bits |= bit where w > 0: one predicated OR (the select + OR the compiler emits otherwise)
__device__ __forceinline__ void or_if_positive(uint32_t &bits, uint32_t bit, float w) {
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %2, 0f00000000;\n\t@p or.b32 %0, %0, %1;\n\t}"
        : "+r"(bits)
        : "r"(bit), "f"(w));
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Forward decision for a slow lane: a pair whose float32 m fell at or above the slot's lower
// threshold cut - gb, or any passing lane of a flagged slot (near-clamp opacity, opacity not
// above 1e-30, or an accurate slot).  Returns 0 if the pair does not blend, else the weight the
// reference blends with; `act` false returns w unchanged (lanes of the warp that are not slow).
//  - Accurate slot (|gb| > kAccurateGb, s2d_device.cuh): m is re-evaluated from the float64
//    Minv and centre; within accurate_band of the cut the reference's own formula decides
//    (guard_resolve); the weight is op 2^(-0.72 m) on that m, which k_raster_bwd recomputes
//    with the same code.
//  - Otherwise: below cut - gb the reference's float64 m is below the cut, so the pixel lies
//    inside the reference bbox (the bbox is the ellipse's exact extent) and the pair blends with
//    the float32 weight, which for a non-flagged slot is positive and below the clamp (the fast
//    path in k_raster_fwd).  Inside the band [cut - gb, cut + gb], or when the weight is within
//    4e-6 of the clamp, guard_resolve decides in float64.
// The backward recomputes w with the same float32 operations and takes the clamp decision from
// the forward's blend stream, so both passes see bit-identical weights.
__device__ __forceinline__ float slow_weight(const ViewParams &P, const RasterArgs &a, uint32_t id, float op, float m,
                                          float w, float gbs, bool act, int px, int py, bool &clamped,
                                          int &guard_hits) {
    clamped = false;
    if (!act) return w;
    const float gb = fabsf(gbs);
    const bool nearclamp = gbs < 0.f;
    bool resolve = false;
    if (gb > kAccurateGb) {
        float u, v;
        double m64;
        const float m32 = accurate_uvm(a.acc[id], px, py, u, v, m64);
        if (fabs(m64 - P.maha_cut) <= accurate_band(gb, P.maha_cut)) resolve = true;
        else if (!(m64 <= P.maha_cut)) return 0.f;
        w = __fmul_rn(op, fast_exp2(__fmul_rn(m32, -0.72134752044448170368f)));
        resolve = resolve || (nearclamp && fabsf(w - P.w_clamp_f) <= 4e-6f);
    } else {
        resolve = m >= __fsub_rn(P.maha_cut_f, gb) || (nearclamp && fabsf(w - P.w_clamp_f) <= 4e-6f);
    }
    if (resolve) {
        ++guard_hits;
        const int rr = guard_resolve(P, a, id, op, px, py);
        if (!(rr & 1)) return 0.f;
        clamped = (rr & 2) != 0;
    } else {
        clamped = nearclamp && w > P.w_clamp_f;
    }
    return clamped ? P.w_clamp_f : fmaxf(w, 0.f);
}

// Ray-splat mode (S2D_SPLAT_RAY): (U, V, S) = Hi' (x - x0, y - y0, 1) with Hi' the record's
// homography relative to the bbox corner (x0, y0), (u, v) = (U, V) / S, z = 1 / S;
// blends when S > 0 and u^2 + v^2 <= sigma^2 (float32 decisions, no reference counterpart).
// Shared by forward and backward (identical operations, so both see the same weights).
struct RayEval {
    float U, V, iS, u, v, m, g;
};

__device__ __forceinline__ bool ray_eval(const ViewParams &P, const SplatRecord &r, float pxf, float pyf,
                                         RayEval &e) {
    const float S = __fmaf_rn(r.q2.w, pyf, __fmaf_rn(r.q1.w, pxf, r.q3.w));
    if (!(S > 0.f)) return false;
    e.U = __fmaf_rn(r.q0.y, pyf, __fmaf_rn(r.q0.x, pxf, r.q0.z));
    e.V = __fmaf_rn(r.q1.y, pyf, __fmaf_rn(r.q1.x, pxf, r.q1.z));
    e.iS = __frcp_rn(S);
    e.u = __fmul_rn(e.U, e.iS);
    e.v = __fmul_rn(e.V, e.iS);
    e.m = __fmaf_rn(e.u, e.u, __fmul_rn(e.v, e.v));
    if (!(e.m <= P.maha_cut_f)) return false;
    e.g = fast_exp2(__fmul_rn(e.m, -0.72134752044448170368f));
    return true;
}

// 32x32 bit-matrix transpose across the warp: bit j of lane i's x becomes bit i of lane j's
// result (recursive off-diagonal block swaps, 5 shuffles).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    constexpr uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int s = 16 >> t;
        const uint32_t p = __shfl_xor_sync(kFull, x, s);
        x = (lane & s) ? ((x & ~M[t]) | ((p & ~M[t]) >> s)) : ((x & M[t]) | ((p & M[t]) << s));
    }
    return x;
}

// Warp-private candidate ring.  Each warp streams ITS OWN candidates from the tile's list:
// list entries are read 32 at a time (key + surfel id), the warp keeps those whose bbox bit
// for its 8x4 block is set, and copies their 64-B records into a 2-deep ring of 32 slots with
// cp.async.  Warps never wait on each other, so a warp with a short candidate list (or whose
// pixels all terminated) does not hold the others back at per-batch barriers.
//
// A slot is 80 B (record + meta): the 20-word stride keeps the lane-parallel 16-B accesses of
// the fill and prep phases free of bank conflicts, and a slot's meta is one immediate offset
// from its record.  The prep phase (lane-parallel, one slot per lane) rewrites an affine slot
// so that the per-pixel offset needs no centre arithmetic (see block_centre).
struct __align__(16) Slot {
    SplatRecord r;
    uint4 meta;  // (surfel id, blend lane mask, clamp lane mask, -) as loaded; see the kernels
};
struct WarpRing {
    Slot s[2][32];
};

// Centre of the splat relative to the warp block's origin pixel (x0, y0), split so the
// per-lane offsets are exact.  With the record centre c = c_hi + c_lo (float32 + half):
//   f = c_hi - x0 is exact when |f| <= |c_hi| (both are multiples of ulp(c_hi)), i.e. except
//   for splats centred within a footprint radius of the image's left / top edge, where it is
//   off by at most ulp(f) / 2 (< 1e-6 px, inside the guard band's 1e-5 / sigma_min term),
//   (lx - f) = x - c_hi then exactly (the value the per-pixel form x - c_hi rounds to),
//   Minv (x - c) = Minv (lx - f, ly - g) - Minv c_lo, with lo = -Minv c_lo taken once per slot.
// So u = A ex + (B ey + lo.x), v = C ex + (D ey + lo.y) with ex = lx - f, ey = ly - g carries the
// rounding of the per-pixel form (no error shared by the whole block), and the forward and the
// backward, calling the same code, evaluate bit-identical weights.
struct BlockCentre {
    float f, g;    // c_hi - (x0, y0)
    float2 lo;     // -Minv (cx_lo, cy_lo)
};
__device__ __forceinline__ BlockCentre block_centre(const float4 &q0, const float4 &q1, float x0f, float y0f) {
    const uint32_t lob = __float_as_uint(q0.z);
    const __half2 h = *reinterpret_cast<const __half2 *>(&lob);
    const float lx = __low2float(h), ly = __high2float(h);
    BlockCentre b;
    b.f = __fsub_rn(q0.x, x0f);
    b.g = __fsub_rn(q0.y, y0f);
    // lo = -((A, C) lx + (B, D) ly), per component fma(A, lx, B ly)
    const float2 t = __ffma2_rn(make_float2(q1.x, q1.y), make_float2(lx, lx),
                                __fmul2_rn(make_float2(q1.z, q1.w), make_float2(ly, ly)));
    b.lo = make_float2(-t.x, -t.y);
    return b;
}

// m = |Minv (p - c)|^2 at lane offset (lx, ly) from the block origin (block_centre), with the
// whitened offset (u, v).
// Packed f32x2 (FFMA2): (ex, ey) = (lx, ly) - (f, g), (u, v) = (A, C) ex + ((B, D) ey + lo); each
// component is the scalar fma chain u = fma(A, ex, fma(B, ey, lo.x)).
__device__ __forceinline__ float slot_maha(float2 fg, float2 lo, const float4 &q1, float2 lxy, float &u,
                                           float &v) {
    const float2 e = __ffma2_rn(fg, make_float2(-1.f, -1.f), lxy);
    const float2 t = __ffma2_rn(make_float2(q1.z, q1.w), make_float2(e.y, e.y), lo);
    const float2 uv = __ffma2_rn(make_float2(q1.x, q1.y), make_float2(e.x, e.x), t);
    u = uv.x;
    v = uv.y;
    return __fmaf_rn(u, u, __fmul_rn(v, v));
}

// Cursor over list positions [lo, hi).  The current 32-wide chunk starts at `cb` (lane l holds
// position cb + l); `pend` = the chunk's hits not yet handed out, `nxt` = the prefetched next
// chunk (key, id).
struct ListCursor {
    int lo, hi, cb;
    uint32_t pend;
    uint32_t kid;
    uint2 nxt;
};

__device__ __forceinline__ uint2 load_chunk(const RasterArgs &a, int cb, const ListCursor &c, int lane) {
    const int pos = cb + lane;
    return pos >= c.lo && pos < c.hi ? make_uint2(__ldcg(a.pair_keys + pos), __ldcg(a.pair_ids + pos))
                                     : make_uint2(0u, 0u);
}

__device__ __forceinline__ void cursor_init(ListCursor &c, const RasterArgs &a, int lo, int hi, int lane) {
    c.lo = lo;
    c.hi = hi;
    c.cb = lo - 32;  // virtual chunk before the range; the first advance lands on lo
    c.pend = 0;
    c.kid = 0;
    c.nxt = load_chunk(a, lo, c, lane);
}

// Fill ring half `buf` with up to 32 candidates in list order (records by cp.async): the
// entries whose bbox bit for this warp's block is set.  Returns how many.
__device__ __forceinline__ int ring_fill(WarpRing &rg, int buf, ListCursor &c, const RasterArgs &a, int warp,
                                         int lane) {
    const uint32_t lt = lanemask_lt();
    int n = 0;
    // 1. walk the list: each hit's surfel id goes to its slot's meta.x (list position j at ring
    //    index 31 - j)
    while (n < 32) {
        if (c.pend == 0) {
            if (c.cb + 32 >= c.hi) break;  // no chunk beyond the current one
            const uint2 cur = c.nxt;
            c.cb += 32;
            c.nxt = load_chunk(a, c.cb + 32, c, lane);
            c.kid = cur.y;
            const int pos = c.cb + lane;
            c.pend = __ballot_sync(kFull, pos < c.hi && ((cur.x >> (16 + warp)) & 1u));
            continue;
        }
        const int take = min(__popc(c.pend), 32 - n);
        const int rank = __popc(c.pend & lt);
        const bool mine = ((c.pend >> lane) & 1u) && rank < take;
        if (mine) rg.s[buf][31 - (n + rank)].meta.x = c.kid;
        c.pend &= ~__ballot_sync(kFull, mine);
        n += take;
    }
    // 2. stage the records, one slot per lane (one cp.async round for the whole fill)
    __syncwarp();
    if (lane < n) {
        Slot &sl = rg.s[buf][31 - lane];
        const float4 *g = reinterpret_cast<const float4 *>(a.rec + sl.meta.x);
        float4 *d = reinterpret_cast<float4 *>(&sl.r);
        cp_async16(d + 0, g + 0);
        cp_async16(d + 1, g + 1);
        cp_async16(d + 2, g + 2);
        cp_async16(d + 3, g + 3);
    }
    return n;
}

// Backward ring fill, per column half: the newest up to 16 of the entries [0, e1) of the
// half's blend stream; the j-th newest (entry e1 - 1 - j) at ring index 2 j + half (the two
// halves' slots of a step interleave, so their 16-B reads hit disjoint banks), loaded by the
// half's lane j (coalesced 16-B loads).  Returns how many.
__device__ __forceinline__ int stream_fill(WarpRing &rg, int buf, const uint4 *ws, int e1,
                                           const SplatRecord *rec, const AccurateRec *acc, int half, int jh) {
    const int n = min(16, e1);
    if (jh < n) {
        const uint4 en = __ldcg(ws + (e1 - 1 - jh));
        Slot &sl = rg.s[buf][2 * jh + half];
        if (en.w) prefetch_accurate(acc + en.x);  // accurate slot (k_raster_fwd)
        const float4 *g = reinterpret_cast<const float4 *>(rec + en.x);
        float4 *d = reinterpret_cast<float4 *>(&sl.r);
        cp_async16(d + 0, g + 0);
        cp_async16(d + 1, g + 1);
        cp_async16(d + 2, g + 2);
        cp_async16(d + 3, g + 3);
        sl.meta = en;
    }
    return n;
}

__device__ __forceinline__ float sgnf(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

// Per-pixel loss seeds dL/d(rgb, depth) and the pixel's loss term for the MSE
// (rasterizer.py:375-380) and L1 losses, from the residuals e = rendered - target; `masked` /
// `nm`: the pixel's depth-mask decision and the image's mask count (unused by the losses
// without a depth mask), npx = W H.
__device__ __forceinline__ void loss_seeds(const RasterArgs &a, float e0, float e1, float e2, float ed, bool masked,
                                           int nm, double npx, float &gc0, float &gc1, float &gc2, float &gd,
                                           float &lpx) {
    if (a.loss_kind == S2D_LOSS_MSE) {
        const float k = (float)(a.w_rgb * (2.0 / (3.0 * npx)));
        gc0 = k * e0;
        gc1 = k * e1;
        gc2 = k * e2;
        lpx = (float)(a.w_rgb / (3.0 * npx)) * (e0 * e0 + e1 * e1 + e2 * e2);
        if (a.w_depth != 0.0 && nm > 0 && masked) {
            gd = (float)(a.w_depth * (2.0 / nm)) * ed;
            lpx += (float)(a.w_depth / nm) * ed * ed;
        }
    } else {  // L1
        const float k = (float)(a.w_rgb / (3.0 * npx));
        gc0 = k * sgnf(e0);
        gc1 = k * sgnf(e1);
        gc2 = k * sgnf(e2);
        lpx = k * (fabsf(e0) + fabsf(e1) + fabsf(e2));
        const bool use = a.depth_mask ? masked : true;
        const double nd = a.depth_mask ? (double)nm : npx;
        if (use && nd > 0.0) {
            const float kd = (float)(a.w_depth / nd);
            gd = kd * sgnf(ed);
            lpx += kd * fabsf(ed);
        }
    }
}

// The reverse traversal of one warp block (k_raster_bwd below; also run by the fused
// forward + backward right after its forward)
template <bool kExt, bool kRay>
__device__ __forceinline__ void bwd_traverse(const RasterArgs &a, WarpRing &ring, int tile, int warp, int lane,
                                             int wx0, int wy0, float gc0, float gc1, float gc2, float gd, float gn0,
                                             float gn1, float gn2, float ga, float Tn, int cnt0, int cnt1);

#ifndef S2D_BWD_CTAS_PER_SM
#define S2D_BWD_CTAS_PER_SM (S2D_BWD_MINB * 8 / kBwdWarps)
#endif

// Forward compositing of one warp block (k_raster_fwd).  kFused (k_raster_fused,
// s2d_forward_backward, losses without the whole-image depth mask): each warp then seeds the
// loss from its pixels' final state and runs the backward's reverse traversal over the blend
// streams it just wrote (bwd_traverse).
template <bool kArg, bool kMaxW, bool kNormal, bool kRay, bool kFused>
__device__ __forceinline__ void raster_fwd_body(const RasterArgs &a) {
    static_assert(!kFused || !(kArg || kMaxW || kNormal), "the fused variant renders colour and depth only");
    __shared__ WarpRing s_ring[kFwdWarps];
    const ViewParams &P = a.P;
    const int tile = blockIdx.x / (8 / kFwdWarps);
    const int tx = tile % P.ntx, ty = tile / P.ntx;
    // a CTA holds kFwdWarps of the tile's 8 warp blocks; warp = the block's index in the tile
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = (blockIdx.x % (8 / kFwdWarps)) * kFwdWarps + (tid >> 5);
    const int wx0 = tx * kTile + (warp & 1) * 8, wy0 = ty * kTile + (warp >> 1) * 4;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const bool inside = px < P.W && py < P.H;
    const float pxf = (float)px, pyf = (float)py;
    const float kNaN = __int_as_float(0x7fffffff);
    // affine mode: a terminated (or outside) lane carries lxy.x = NaN, so its m is NaN and fails
    // the cut test; no per-candidate `done` test is needed
    float2 lxy = make_float2(inside ? (float)(lane & 7) : kNaN, (float)(lane >> 3));
    const int2 rg = a.ranges[tile];

    float T = 1.0f;
    // accumulated (r, g), (b, depth), (nx, ny), nz: register pairs for the packed FFMA2
    float2 c01 = make_float2(0.f, 0.f), c2d = make_float2(0.f, 0.f), n01 = make_float2(0.f, 0.f);
    float n2 = 0.f;
    float maxw = 0.f;
    double T64 = 1.0, maxw64 = 0.0;  // argmax variant (affine): the reference's float64 state
    int argw = -1, nblend = 0, guard = 0;
    bool done = !inside;  // ray mode
    const float term_t = P.term_t_f;
    WarpRing &ring = s_ring[tid >> 5];

    // this warp's blend stream: one (surfel, lane mask) entry per pair its pixels blended, in
    // list order (the backward's work list)
    // Two streams per warp, one per column half of its block (lane bit 2 clear / set): an entry
    // goes to each half whose pixels blended it, so the backward's halves walk them apart.
    // Segment of (warp w, half h) of tile t: 16 ranges[t].x + (2 w + h) len(t), len = list length.
    const size_t seg = (size_t)max(rg.y - rg.x, 0);
    uint4 *wp0 = a.bstream + 16 * (size_t)rg.x + (size_t)(2 * warp) * seg, *wp1 = wp0 + seg;
    int wc0 = 0, wc1 = 0;
    if (rg.y > rg.x && !__all_sync(kFull, done)) {
        ListCursor cur;
        cursor_init(cur, a, rg.x, rg.y, lane);
        int buf = 0;
        int n = ring_fill(ring, 0, cur, a, warp, lane);  // bbox bit (k_scan_emit)
        cp_commit();
        while (n > 0) {
            const int nn = ring_fill(ring, buf ^ 1, cur, a, warp, lane);
            cp_commit();
            cp_wait<1>();
            __syncwarp();
            // prep phase, lane-parallel over the staged candidates (lane = slot): the exact
            // ellipse cull against the block (ray mode: the bbox bits only) and, for the kept
            // affine slots, the block-origin offset and cut thresholds (slot_prep comment above)
            bool keep = false;
            if (lane < n) {
                Slot &sl = ring.s[buf][31 - lane];
                if (kRay) {
                    keep = true;
                } else {
                    const float4 q0 = sl.r.q0, q1 = sl.r.q1;
                    const float gbs = sl.r.q3.w, gb = fabsf(gbs), op = q0.w;
                    // a non-positive (or NaN) opacity never blends: w = op g <= 0 (or NaN) is
                    // skipped by the reference and by guard_resolve's caller alike
                    keep = op > 0.f && block_reach(wx0, wy0, sl.r, P.maha_cut_f);
                    if (keep) {
                        const BlockCentre bc = block_centre(q0, q1, (float)wx0, (float)wy0);
                        const float thi = __fadd_rn(P.maha_cut_f, gb), tlo = __fsub_rn(P.maha_cut_f, gb);
                        // flagged slots send every passing lane to slow_weight
                        const bool slow = gbs < 0.f || !(op > 1e-30f) || gb > kAccurateGb;
                        if (gb > kAccurateGb) prefetch_accurate(a.acc + sl.meta.x);
                        // forward slot: q0 = (f, g, cut + gb, opacity),
                        // meta = (id, cut - gb or -3e38 (flagged), lo.x, lo.y)
                        sl.r.q0 = make_float4(bc.f, bc.g, thi, op);
                        sl.meta.y = __float_as_uint(slow ? -3.0e38f : tlo);
                        sl.meta.z = __float_as_uint(bc.lo.x);
                        sl.meta.w = __float_as_uint(bc.lo.y);
                    }
                }
            }
            // bit p of rm = ring index p = list position 31 - p, so the highest set bit is the
            // next candidate in list order
            uint32_t rm = __brev(__ballot_sync(kFull, keep));
            __syncwarp();
            // per lane, bit 31 - j of bl_bits / cl_bits: this pixel blended list position j / with a
            // clamped weight; transposed into per-slot lane masks once per chunk
            uint32_t bl_bits = 0u, cl_bits = 0u;
            while (rm) {
                uint32_t kb, bit;  // ring index k = highest set bit of rm
                asm("bfind.u32 %0, %1;" : "=r"(kb) : "r"(rm));
                asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(kb));
                const int k = (int)kb;
                rm ^= bit;
                const Slot &sl = ring.s[buf][k];
                float contrib = 0.f;
                // blend (blend_forward, _raster_kernels.py:47-55)
                auto blend = [&](float w, float zpix) {
                    bl_bits |= bit;
                    contrib = w * T;
                    const float4 q2 = sl.r.q2;
                    const float2 cc = make_float2(contrib, contrib);
                    c01 = __ffma2_rn(cc, make_float2(q2.x, q2.y), c01);
                    c2d = __ffma2_rn(cc, make_float2(q2.z, kRay ? zpix : q2.w), c2d);
                    if (kNormal) {
                        const float4 q3 = sl.r.q3;
                        n01 = __ffma2_rn(cc, make_float2(q3.x, q3.y), n01);
                        n2 = fmaf(contrib, q3.z, n2);
                    }
                    if (kArg && contrib > maxw) {
                        maxw = contrib;
                        argw = (int)sl.meta.x;
                    }
                    T = fmaf(-w, T, T);  // T (1 - w), one rounding (T - w T loses bits for w near 1)
                    if (kRay) done = T < term_t;
                    else lxy.x = T < term_t ? kNaN : lxy.x;
                };
                if (kRay) {
                    if (!done) {
                        RayEval e;
                        const short4 bb = a.rect[sl.meta.x];
                        if (ray_eval(P, sl.r, pxf - (float)bb.x, pyf - (float)bb.z, e)) {
                            float w = __fmul_rn(sl.r.q0.w, e.g);
                            const bool clamped = w > P.w_clamp_f;
                            w = clamped ? P.w_clamp_f : fmaxf(w, 0.f);
                            if (clamped) cl_bits |= bit;
                            if (w > 0.f) blend(w, e.iS);
                        }
                    }
                } else {
                    const float4 q0 = sl.r.q0, q1 = sl.r.q1;
                    float u, v;
                    const uint4 mt = sl.meta;
                    const float m = slot_maha(make_float2(q0.x, q0.y),
                                              make_float2(__uint_as_float(mt.z), __uint_as_float(mt.w)), q1, lxy, u, v);
                    // Branch-free: every lane runs the blend with w = 0 where the pair does not
                    // blend (m above cut + gb, or NaN for a terminated lane), which leaves its
                    // state unchanged; only a warp with a lane inside a guard band (or a flagged
                    // slot) takes the uniform slow-path branch.
                    const bool pass = m <= q0.z;
                    float w = __fmul_rn(q0.w, fast_exp2(__fmul_rn(m, -0.72134752044448170368f)));
                    w = pass ? w : 0.f;
                    const float tlo = __uint_as_float(mt.y);
                    const bool slow = pass && m >= tlo;
                    if (__any_sync(kFull, slow)) {
                        // a warp-uniform branch; lanes that are not slow keep their w
                        bool clamped = false;
                        w = slow_weight(P, a, mt.x, q0.w, m, w, sl.r.q3.w, slow, px, py, clamped, guard);
                        if (clamped) cl_bits |= bit;
                    }
                    {  // blend (blend_forward, _raster_kernels.py:47-55), a no-op where w = 0
                        or_if_positive(bl_bits, bit, w);
                        contrib = w * T;
                        const float4 q2 = sl.r.q2;
                        const float2 cc = make_float2(contrib, contrib);
                        c01 = __ffma2_rn(cc, make_float2(q2.x, q2.y), c01);
                        c2d = __ffma2_rn(cc, make_float2(q2.z, q2.w), c2d);
                        if (kNormal) {
                            const float4 q3 = sl.r.q3;
                            n01 = __ffma2_rn(cc, make_float2(q3.x, q3.y), n01);
                            n2 = fmaf(contrib, q3.z, n2);
                        }
                        T = fmaf(-w, T, T);  // T (1 - w), one rounding (T - w T loses bits for w near 1)
                        if (kArg) {
                            // render_with_argmax: the reference's float64 weight, transmittance and
                            // strict `contrib > max_w` (_raster_kernels.py:42-55) for the pairs that
                            // blend, so the argmax index and the termination are the reference's
                            if (w > 0.f) {
                                const ExactRec &e = a.exact[mt.x];
                                const double m64 = exact_maha(e.cx, e.cy, e.ia, e.ib, e.ic, px, py);
                                double w64 = dmul((double)q0.w, exp(dmul(-0.5, m64)));
                                if (w64 > P.w_clamp) w64 = P.w_clamp;
                                const double c64 = dmul(w64, T64);
                                if (c64 > maxw64) {
                                    maxw64 = c64;
                                    argw = (int)mt.x;
                                }
                                T64 = dmul(T64, dsub(1.0, w64));
                            }
                            lxy.x = T64 < P.term_t ? kNaN : lxy.x;
                        } else {
                            lxy.x = T < term_t ? kNaN : lxy.x;
                        }
                    }
                }
                if (kMaxW) {
                    const uint32_t id = sl.meta.x;
                    float mx = contrib;
                    float mm = (a.mask != nullptr && inside && a.mask[py * P.W + px]) ? contrib : 0.f;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
                        mm = fmaxf(mm, __shfl_xor_sync(kFull, mm, o));
                    }
                    if (lane == 0) {
                        if (mx > 0.f) atomicMax(reinterpret_cast<int *>(a.max_all + id), __float_as_int(mx));
                        if (mm > 0.f && a.max_marked)
                            atomicMax(reinterpret_cast<int *>(a.max_marked + id), __float_as_int(mm));
                    }
                }
            }
            nblend += __popc(bl_bits);
            // blend stream: lane j now holds list position j's masks; the slots some pixel blended are
            // appended in slot (= list) order with one coalesced store
            {
                const uint32_t bm = transpose32(__brev(bl_bits), lane);
                const uint32_t cm = __any_sync(kFull, cl_bits != 0u) ? transpose32(__brev(cl_bits), lane) : 0u;
                const bool h0 = (bm & 0x0F0F0F0Fu) != 0u, h1 = (bm & 0xF0F0F0F0u) != 0u;
                const uint32_t b0 = __ballot_sync(kFull, h0), b1 = __ballot_sync(kFull, h1);
                // w: 1 for an accurate slot (k_raster_bwd prefetches its float64 data when staging)
                const Slot &me = ring.s[buf][31 - lane];
                const uint4 en = make_uint4(me.meta.x, bm, cm, !kRay && fabsf(me.r.q3.w) > kAccurateGb ? 1u : 0u);
                const uint32_t lt = lanemask_lt();
                if (h0) wp0[__popc(b0 & lt)] = en;
                if (h1) wp1[__popc(b1 & lt)] = en;
                wp0 += __popc(b0);
                wp1 += __popc(b1);
                wc0 += __popc(b0);
                wc1 += __popc(b1);
            }
            if (__all_sync(kFull, kRay ? done : lxy.x != lxy.x)) break;
            __syncwarp();  // slot `buf` is refilled by the next ring_fill
            buf ^= 1;
            n = nn;
        }
        cp_wait<0>();
    }
    if constexpr (kFused) {
        if (lane == 0 && wc0 + wc1) atomicAdd(&a.stats->blended, wc0 + wc1);
        float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f, lpx = 0.f;
        if (inside) {
            const int p = py * P.W + px;
            if (a.color) {  // the image outputs are optional here
                a.color[3 * p] = c01.x;
                a.color[3 * p + 1] = c01.y;
                a.color[3 * p + 2] = c2d.x;
            }
            if (a.depth) a.depth[p] = c2d.y;
            if (a.accum) a.accum[p] = 1.0f - T;
            const float e0 = c01.x - a.target_rgb[3 * p];
            const float e1 = c01.y - a.target_rgb[3 * p + 1];
            const float e2 = c2d.x - a.target_rgb[3 * p + 2];
            const float ed = c2d.y - a.target_depth[p];
            loss_seeds(a, e0, e1, e2, ed, false, 0, (double)P.W * (double)P.H, gc0, gc1, gc2, gd, lpx);
        }
        const int nm = __popc(__ballot_sync(kFull, inside && (1.0f - T) > 0.5f));
        int gsum = guard;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            gsum += __shfl_xor_sync(kFull, gsum, o);
            lpx += __shfl_xor_sync(kFull, lpx, o);
        }
        if (lane == 0) {
            if (gsum) atomicAdd(&a.stats->guard_hits, gsum);
            if (nm) atomicAdd(&a.stats->n_mask, nm);
            if (lpx != 0.f && a.loss_accum) atomicAdd(a.loss_accum, (double)lpx);
        }
        if (wc0 + wc1 == 0) return;  // warp-uniform
        // the blend streams were written by this warp's lanes and are staged (cp.async, L2)
        // by other lanes of it: release them at GPU scope before the warp barrier
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncwarp();
        bwd_traverse<false, kRay>(a, ring, tile, warp, lane, wx0, wy0, gc0, gc1, gc2, gd, 0.f, 0.f, 0.f, 0.f, T, wc0,
                                  wc1);
        return;
    }
    if (lane == 0) {
        a.bcount[16 * tile + 2 * warp] = wc0;
        a.bcount[16 * tile + 2 * warp + 1] = wc1;
        if (wc0 + wc1) atomicAdd(&a.stats->blended, wc0 + wc1);
    }
    if (inside) {
        const int p = py * P.W + px;
        if (a.color) {
            a.color[3 * p] = c01.x;
            a.color[3 * p + 1] = c01.y;
            a.color[3 * p + 2] = c2d.x;
        }
        if (a.depth) a.depth[p] = c2d.y;
        if (a.accum) a.accum[p] = 1.0f - T;
        if (kNormal) {
            a.normal[3 * p] = n01.x;
            a.normal[3 * p + 1] = n01.y;
            a.normal[3 * p + 2] = n2;
        }
        if (kArg) {
            if (a.max_w) a.max_w[p] = kRay ? maxw : (float)maxw64;
            if (a.arg_w) a.arg_w[p] = argw;
        }
        a.aux[p] = make_int2(nblend, __float_as_int(T));
        // `accumulation > 0.5` (the reference's depth mask, rasterizer.py:365-376) within the
        // float32 error band of 0.5: re-decided in float64 by k_mask_fixup when a loss needs it
        if (!kRay && fabsf(0.5f - T) <= kMaskBand) {
            const int slot = atomicAdd(a.amb_count, 1);
            a.amb_list[slot] = p;
        }
    }
    const int nm = __popc(__ballot_sync(kFull, inside && (1.0f - T) > 0.5f));
    int gsum = guard;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gsum += __shfl_xor_sync(kFull, gsum, o);
    if (lane == 0 && gsum) atomicAdd(&a.stats->guard_hits, gsum);
    if (lane == 0 && nm) atomicAdd(&a.stats->n_mask, nm);
}

// The plain variant (the refine path) fits 48 registers, 5 CTAs/SM: besides its own latency
// hiding, a smaller footprint lets it share SMs with the other views' kernels in flight.
template <bool kArg, bool kMaxW, bool kNormal, bool kRay>
__global__ void __launch_bounds__(kFwdWarps * 32, ((kArg || kMaxW || kNormal) ? 4 : S2D_FWD_MINB) * 8 / kFwdWarps)
    k_raster_fwd(const RasterArgs a) {
    raster_fwd_body<kArg, kMaxW, kNormal, kRay, false>(a);
}

// The fused variant runs with the backward's register budget (64, 8 CTAs/SM)
template <bool kRay>
__global__ void __launch_bounds__(kFwdWarps * 32, S2D_BWD_CTAS_PER_SM) k_raster_fused(const RasterArgs a) {
    raster_fwd_body<false, false, false, kRay, true>(a);
}

// Transposed warp reduction of C per-lane values (C <= 32): at each butterfly stage the
// lanes exchange half of their values, so the whole reduction costs about C shuffles
// instead of 5 C.  kMode picks the lane groups reduced separately and the butterfly offsets:
//   0: the whole warp (16, 8, 4, 2, 1);
//   1: the two column halves of the 8x4 block, lane bit 2 clear / set (16, 8, 2, 1);
//   2: the four rows of the block, lanes 8r .. 8r + 7 (4, 2, 1).
// Afterwards each lane holds red_final(C, kMode) sums v[0 ..]; red_map (run once per kernel)
// says which value each is (vi) and whether this lane owns it (each value of each group is
// owned by exactly one lane of the group).
__host__ __device__ constexpr int red_next(int O, int mode) { return (mode == 1 && O == 8) ? 2 : O / 2; }
__host__ __device__ constexpr int red_first(int mode) { return mode == 2 ? 4 : 16; }
__host__ __device__ constexpr int red_final(int C, int mode) {
    int O = red_first(mode);
    while (O >= 1) {
        C = (C + 1) / 2;
        O = red_next(O, mode);
    }
    return C;
}

template <int C, int O, int kMode, int NA>
__device__ __forceinline__ void red_stage(float (&v)[NA], int lane) {
    constexpr int H = (C + 1) / 2, F = C / 2;
    const bool up = lane & O;
#pragma unroll
    for (int j = 0; j + 1 < F; j += 2) {  // two sums per packed FADD2
        const float s0 = up ? v[j] : v[j + H], s1 = up ? v[j + 1] : v[j + 1 + H];
        const float2 keep = make_float2(up ? v[j + H] : v[j], up ? v[j + 1 + H] : v[j + 1]);
        const float2 r = __fadd2_rn(keep, make_float2(__shfl_xor_sync(kFull, s0, O), __shfl_xor_sync(kFull, s1, O)));
        v[j] = r.x;
        v[j + 1] = r.y;
    }
    if constexpr (F % 2) {
        constexpr int j = F - 1;
        const float send = up ? v[j] : v[j + H];
        const float keep = up ? v[j + H] : v[j];
        v[j] = keep + __shfl_xor_sync(kFull, send, O);
    }
    if constexpr (H > F) v[F] += __shfl_xor_sync(kFull, v[F], O);
    if constexpr (O > 1) red_stage<H, red_next(O, kMode), kMode, NA>(v, lane);
}

template <int C, int O, int kMode>
__device__ __forceinline__ void map_stage(int (&ix)[32], bool (&own)[32], int lane) {
    constexpr int H = (C + 1) / 2, F = C / 2;
    const bool up = lane & O;
#pragma unroll
    for (int j = 0; j < F; ++j) {
        const bool send = up ? own[j] : own[j + H];
        const bool psend = __shfl_xor_sync(kFull, (int)send, O) != 0;
        ix[j] = up ? ix[j + H] : ix[j];
        own[j] = (up ? own[j + H] : own[j]) && psend;
    }
    if constexpr (H > F) {
        const bool pown = __shfl_xor_sync(kFull, (int)own[F], O) != 0;  // every lane shuffles
        own[F] = own[F] && pown && !up;
    }
    if constexpr (O > 1) map_stage<H, red_next(O, kMode), kMode>(ix, own, lane);
}

template <int C, int kMode, int RF>
__device__ __forceinline__ void red_map(int lane, int (&vi)[RF], bool (&own)[RF]) {
    int ix[32];
    bool ow[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        ix[j] = j;
        ow[j] = true;
    }
    map_stage<C, red_first(kMode), kMode>(ix, ow, lane);
#pragma unroll
    for (int t = 0; t < RF; ++t) {
        vi[t] = ix[t];
        own[t] = ow[t];
    }
}

template <bool kExt, bool kRay>  // kExt: normal / accumulation seeds present (external loss)
__global__ void __launch_bounds__(kBwdWarps * 32, S2D_BWD_CTAS_PER_SM) k_raster_bwd(const RasterArgs a) {
    __shared__ WarpRing s_ring[kBwdWarps];
    __shared__ float s_loss[kBwdWarps];
    const ViewParams &P = a.P;
    const int tile = blockIdx.x / (8 / kBwdWarps);
    const int tx = tile % P.ntx, ty = tile / P.ntx;
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = (blockIdx.x % (8 / kBwdWarps)) * kBwdWarps + (tid >> 5);  // block index in the tile
    const int wx0 = tx * kTile + (warp & 1) * 8, wy0 = ty * kTile + (warp >> 1) * 4;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const bool inside = px < P.W && py < P.H;
    const int p = py * P.W + px;

    // ---- loss seeds (rasterizer.py:375-380 for MSE; L1; external) ----
    float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f, gn0 = 0.f, gn1 = 0.f, gn2 = 0.f, ga = 0.f;
    float lpx = 0.f;
    float Tn = 1.f;  // transmittance after the contributors processed so far (forward: final T)
    if (inside) {
        const int2 ax = a.aux[p];
        Tn = __int_as_float(ax.y);
        const double npx = (double)P.W * (double)P.H;
        if (a.loss_kind == S2D_LOSS_EXTERNAL) {
            if (a.d_color) {
                gc0 = a.d_color[3 * p];
                gc1 = a.d_color[3 * p + 1];
                gc2 = a.d_color[3 * p + 2];
            }
            if (a.d_depth) gd = a.d_depth[p];
            if (a.d_normal) {
                gn0 = a.d_normal[3 * p];
                gn1 = a.d_normal[3 * p + 1];
                gn2 = a.d_normal[3 * p + 2];
            }
            if (a.d_accum) ga = a.d_accum[p];
        } else {
            const float e0 = a.color[3 * p] - a.target_rgb[3 * p];
            const float e1 = a.color[3 * p + 1] - a.target_rgb[3 * p + 1];
            const float e2 = a.color[3 * p + 2] - a.target_rgb[3 * p + 2];
            const float ed = a.depth[p] - a.target_depth[p];
            const int nm = a.stats->n_mask;
            // aux.x bit 30: the mask was re-decided in float64 (k_mask_fixup), value in bit 29
            const bool masked = (ax.x & (1 << 30)) ? ((ax.x >> 29) & 1) != 0 : a.accum[p] > 0.5f;
            loss_seeds(a, e0, e1, e2, ed, masked, nm, npx, gc0, gc1, gc2, gd, lpx);
        }
    }
    // loss: block reduction (the kernel's only barrier)
    {
        float l = lpx;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
        if (lane == 0) s_loss[tid >> 5] = l;
    }
    __syncthreads();
    if (tid == 0 && a.loss_accum) {
        float l = 0.f;
        for (int w = 0; w < kBwdWarps; ++w) l += s_loss[w];
        if (l != 0.f) atomicAdd(a.loss_accum, (double)l);
    }
    const int cnt0 = a.bcount[16 * tile + 2 * warp], cnt1 = a.bcount[16 * tile + 2 * warp + 1];
    if (cnt0 + cnt1 == 0) return;  // no pixel of this warp's block blended anything (warp-uniform)
    bwd_traverse<kExt, kRay>(a, s_ring[tid >> 5], tile, warp, lane, wx0, wy0, gc0, gc1, gc2, gd, gn0, gn1, gn2, ga,
                             Tn, cnt0, cnt1);
}

template <bool kExt, bool kRay>
__device__ __forceinline__ void bwd_traverse(const RasterArgs &a, WarpRing &ring, int tile, int warp, int lane,
                                             int wx0, int wy0, float gc0, float gc1, float gc2, float gd, float gn0,
                                             float gn1, float gn2, float ga, float Tn, int cnt0, int cnt1) {
    const ViewParams &P = a.P;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const float pxf = (float)px, pyf = (float)py;
    const float2 lxy = make_float2((float)(lane & 7), (float)(lane >> 3));
    const int2 rg = a.ranges[tile];
    const int half = (lane >> 2) & 1;  // column half of the block (lane bit 2)

    // ---- reverse traversal of the pairs this warp's pixels blended ----
    // Per pair, only the lanes in the forward's lane mask work (no cut / guard-band tests);
    // their 2D gradients are warp-reduced (NV values) and added with one atomic per value:
    //   [0] dL/d opacity, [1..3] dL/d rgb, [4] dL/dz,
    //   [5..7] K = sum dL/dm w w^T (uu, uv, vv), [8..9] e = sum dL/dm w, [10..12] dL/d normal
    // with w = (u, v) = Minv d the whitened pixel offset (dL/dMinv = 2 K M^T and
    // dL/dcentre = -2 Minv^T e are formed in k_project_bwd).
    constexpr int NV = kRay ? (kExt ? 16 : 13) : (kExt ? 13 : 10);
    // The two column halves of the block (lane bit 2 clear / set) walk their own blend streams
    // (the entries that touch them, written apart by the forward) in step, one entry per half
    // per step; each half reduces its NV values over its 16 lanes (transposed, offsets 16, 8,
    // 2, 1); lane ownership of the sums is fixed per kernel.
    constexpr int kMode = 1, RF = red_final(NV, kMode);  // sums held per lane after the reduction
    int vi[RF];
    bool own[RF];
    red_map<NV, kMode>(lane, vi, own);
    float *gcol[RF];  // this lane's gradient columns (where it owns a sum)
#pragma unroll
    for (int t = 0; t < RF; ++t) gcol[t] = a.grad2d + vi[t];
    constexpr int kG2 = g2_stride(kRay, kExt);  // floats per surfel row of grad2d
    float R = 1.f;     // prod_{j later} (1 - w_j)
    // suffixes (S_r, S_g), (S_b, S_depth) as register pairs for the packed FFMA2
    float2 S01 = make_float2(0.f, 0.f), S2d = make_float2(0.f, 0.f);
    float Sn0 = 0.f, Sn1 = 0.f, Sn2 = 0.f;
    const float2 gc01 = make_float2(gc0, gc1), gc2d = make_float2(gc2, gd);
    // this lane's half stream; each half stages up to 16 entries per ring buffer, at ring
    // indices 2 j + half (j-th newest), lane position j in the half = jh
    const uint4 *ws = a.bstream + 16 * (size_t)rg.x + (size_t)(2 * warp + half) * (size_t)(rg.y - rg.x);
    const int jh = (lane & 3) | ((lane >> 3) << 2);
    int e1 = half ? cnt1 : cnt0;
    int buf = 0;
    int n = stream_fill(ring, 0, ws, e1, a.rec, a.acc, half, jh);
    e1 -= n;
    cp_commit();
    float v[NV];
    // one entry of the reverse traversal for this lane: updates the pixel state, writes the
    // entry's NV gradient values at v[off ...]
    auto entry = [&](int k, bool act, int off, auto acc_t) -> uint32_t {
        constexpr bool kAcc = decltype(acc_t)::value;  // the chunk holds an accurate slot
        const Slot &sl = ring.s[buf][k];
        const uint4 meta = sl.meta;  // (surfel id, blend / clamp lane masks, lo.y)
        const uint2 mk = make_uint2(meta.y, meta.z);
        // every lane runs the entry; lanes outside the blend mask (or without an entry this
        // step, !act) take w = 0, which leaves their state unchanged and makes their values 0
        const bool inl = act && ((mk.x >> lane) & 1u);
        // the forward's arithmetic (k_raster_fwd / ray_eval), minus the decisions it took
        const SplatRecord &r = sl.r;
        const bool clamped = (mk.y >> lane) & 1u;
        const float4 q2 = r.q2;
        float w, g, z;
        float u = 0.f, vv = 0.f;  // affine: whitened offset
        RayEval re;
        const short4 bb = kRay ? a.rect[sl.meta.x] : make_short4(0, 0, 0, 0);
        const float rx = pxf - (float)bb.x, ry = pyf - (float)bb.z;  // ray: offset from the bbox corner
        if (kRay) {
            // blended in the forward: S > 0, m <= cut; the other lanes get finite zeros
            const bool ok = ray_eval(P, r, rx, ry, re) && inl;
            re.u = ok ? re.u : 0.f;
            re.v = ok ? re.v : 0.f;
            re.m = ok ? re.m : 0.f;
            re.iS = ok ? re.iS : 0.f;
            g = ok ? re.g : 0.f;
            z = re.iS;
            w = clamped ? P.w_clamp_f : __fmul_rn(r.q0.w, g);
        } else {
            // backward slot: q0 = (f, g, lo.x, lo.y), meta.w = opacity (negative: accurate slot)
            const float4 q0 = r.q0, q1 = r.q1;
            const float m = slot_maha(make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), q1, lxy, u, vv);
            // lanes outside the mask: keep (u, v) finite (a near-singular Minv could overflow
            // them far from the splat), so their zero gradient values stay zeros
            u = inl ? u : 0.f;
            vv = inl ? vv : 0.f;
            g = fast_exp2(__fmul_rn(m, -0.72134752044448170368f));
            const float opm = __uint_as_float(meta.w);
            const bool accurate = kAcc && inl && opm < 0.f;
            if (kAcc && __any_sync(kFull, accurate)) {  // warp-uniform: the forward's slow_weight evaluation
                // every lane evaluates (no divergent region in the step; the lanes of a
                // non-accurate slot read an unused record and discard the result)
                double m64;
                float ua, va;
                const float m32 = accurate_uvm(a.acc[meta.x], px, py, ua, va, m64);
                const float ga = fast_exp2(__fmul_rn(m32, -0.72134752044448170368f));
                u = accurate ? ua : u;
                vv = accurate ? va : vv;
                g = accurate ? ga : g;
            }
            z = q2.w;
            w = clamped ? P.w_clamp_f : __fmul_rn(fabsf(opm), g);
        }
        w = inl ? w : 0.f;
        const float Ti = inl ? Tn * fast_rcp(1.0f - w) : Tn;
        Tn = Ti;
        const float alpha = w * Ti;
        const float2 aa = make_float2(alpha, alpha), ww = make_float2(w, w);
        {
            const float2 g01 = __fmul2_rn(gc01, aa), g23 = __fmul2_rn(gc2d, aa);  // (rgb, z) gradients
            v[off + 1] = g01.x;
            v[off + 2] = g01.y;
            v[off + 3] = g23.x;
            if (!kRay) v[off + 4] = g23.y;
        }
        // dL/dw = T_i [ G.(c - S) + gd (z - Sd) + Gn.(n - Sn) ] + ga T_i R; the differences
        // (c - S) also update the suffix: S <- w c + (1 - w) S = S + w (c - S)
        const float2 d01 = __ffma2_rn(S01, make_float2(-1.f, -1.f), make_float2(q2.x, q2.y));
        const float2 d2d = __ffma2_rn(S2d, make_float2(-1.f, -1.f), make_float2(q2.z, z));
        const float2 pd = __ffma2_rn(gc2d, d2d, __fmul2_rn(gc01, d01));
        float dLdw = pd.x + pd.y;
        if (kExt) {
            const float4 q3 = r.q3;
            v[off + (kRay ? 13 : 10)] = gn0 * alpha;
            v[off + (kRay ? 14 : 11)] = gn1 * alpha;
            v[off + (kRay ? 15 : 12)] = gn2 * alpha;
            const float e0 = q3.x - Sn0, e1 = q3.y - Sn1, e2 = q3.z - Sn2;
            dLdw += gn0 * e0 + gn1 * e1 + gn2 * e2 + ga * R;
            Sn0 = fmaf(w, e0, Sn0);
            Sn1 = fmaf(w, e1, Sn1);
            Sn2 = fmaf(w, e2, Sn2);
            R *= 1.0f - w;
        }
        dLdw *= Ti;
        // clamped weights (and lanes outside the mask) carry no opacity / geometry gradient
        const float dg = (clamped || !inl) ? 0.f : dLdw;
        if (kRay) {
            const float gm2 = -w * dg * re.iS;  // 2 dL/dm / S
            const float gU = gm2 * re.u, gV = gm2 * re.v;
            const float gS = -gd * alpha * z * z - gm2 * re.m;
            v[off + 0] = dg * g;
            v[off + 4] = gU * rx;
            v[off + 5] = gU * ry;
            v[off + 6] = gU;
            v[off + 7] = gV * rx;
            v[off + 8] = gV * ry;
            v[off + 9] = gV;
            v[off + 10] = gS * rx;
            v[off + 11] = gS * ry;
            v[off + 12] = gS;
        } else {
            v[off + 0] = dg * g;
            const float gm = -0.5f * w * dg;  // dL/dm
            const float2 uv = make_float2(u, vv);
            const float2 e = __fmul2_rn(make_float2(gm, gm), uv);     // e = dL/dm (u, v)
            const float2 k01 = __fmul2_rn(make_float2(e.x, e.x), uv);  // K = dL/dm (uu, uv)
            v[off + 8] = e.x;
            v[off + 9] = e.y;
            v[off + 5] = k01.x;
            v[off + 6] = k01.y;
            v[off + 7] = e.y * vv;  // dL/dm vv
        }
        S01 = __ffma2_rn(ww, d01, S01);
        S2d = __ffma2_rn(ww, d2d, S2d);
        return meta.x;
    };
    while (true) {
        const int n0 = __shfl_sync(kFull, n, 0), n1 = __shfl_sync(kFull, n, 4);  // per half
        if (n0 + n1 == 0) break;
        const int nn = stream_fill(ring, buf ^ 1, ws, e1, a.rec, a.acc, half, jh);
        e1 -= nn;
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        bool acc_here = false;
        if (!kRay && jh < n) {  // prep: block-relative centre, as the forward computed it
            Slot &sl = ring.s[buf][2 * jh + half];
            const BlockCentre bc = block_centre(sl.r.q0, sl.r.q1, (float)wx0, (float)wy0);
            sl.r.q0.x = bc.f;
            sl.r.q0.y = bc.g;
            // opacity, negated for an accurate slot (s2d_device.cuh kAccurateGb)
            acc_here = fabsf(sl.r.q3.w) > kAccurateGb;
            sl.meta.w = __float_as_uint(acc_here ? -sl.r.q0.w : sl.r.q0.w);
            sl.r.q0.z = bc.lo.x;
            sl.r.q0.w = bc.lo.y;
        }
        // chunks without an accurate slot (most) run the step loop without its per-step check
        const bool chunk_acc = __any_sync(kFull, acc_here);
        __syncwarp();
        const int steps = max(n0, n1);
        const int kidle = n > 0 ? half : 1 - half;  // a staged slot, for idle steps
        auto run_steps = [&](auto acc_t) {
#pragma unroll 2  // lets one step's reduction overlap the next step's entry
            for (int st = 0; st < steps; ++st) {
                const bool act = st < n;  // this half still has an entry in this chunk
                const uint32_t id = entry(act ? 2 * st + half : kidle, act, 0, acc_t);
                red_stage<NV, red_first(kMode), kMode>(v, lane);
#pragma unroll
                for (int t = 0; t < RF; ++t) red_add_if(gcol[t] + (size_t)id * kG2, v[t], own[t] && act);
            }
        };
        if (!kRay && chunk_acc) run_steps(std::integral_constant<bool, !kRay>{});
        else run_steps(std::false_type{});
        __syncwarp();  // slot `buf` is refilled by the next stream_fill
        buf ^= 1;
        n = nn;
    }
    cp_wait<0>();
}

// Float64 re-decision of the depth mask `accumulation > 0.5` (rasterizer.py:365-376) for the
// pixels the forward listed (float32 1 - T within kMaskBand of 0.5): the pixel's transmittance is
// recomputed with the reference's arithmetic (blend_forward, _raster_kernels.py:32-55) over its
// tile's depth-ordered list, one warp per pixel (lanes decide 32 pairs at a time, the product
// runs in list order).  Corrects stats.n_mask, stores the decision in aux.x bits 30/29, and
// clears the list so a second backward of the same forward is a no-op.  One CTA.
__global__ void __launch_bounds__(256) k_mask_fixup(const RasterArgs a) {
    const ViewParams &P = a.P;
    const int cnt = *a.amb_count;
    if (cnt == 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = warp; q < cnt; q += 8) {
        const int p = a.amb_list[q];
        const int px = p % P.W, py = p / P.W;
        const int tile = (py / kTile) * P.ntx + px / kTile;
        const int2 rg = a.ranges[tile];
        double T64 = 1.0;
        bool done = false;
        for (int cb = rg.x; cb < rg.y && !done; cb += 32) {
            const int j = cb + lane;
            double f = 1.0;  // factor (1 - w) of this pair, 1 if it does not blend
            if (j < rg.y) {
                const uint32_t id = a.pair_ids[j];
                const short4 b = a.rect[id];
                if (px >= b.x && px <= b.y && py >= b.z && py <= b.w) {
                    const ExactRec &e = a.exact[id];
                    const double m64 = exact_maha(e.cx, e.cy, e.ia, e.ib, e.ic, px, py);
                    if (m64 <= P.maha_cut) {
                        double w64 = dmul((double)a.rec[id].q0.w, exp(dmul(-0.5, m64)));
                        if (w64 > P.w_clamp) w64 = P.w_clamp;
                        if (w64 > 0.0) f = dsub(1.0, w64);
                    }
                }
            }
            for (int k = 0; k < 32; ++k) {
                const double fk = __shfl_sync(kFull, f, k);
                if (!done) {
                    if (T64 < P.term_t) done = true;
                    else T64 = dmul(T64, fk);
                }
            }
        }
        if (lane == 0) {
            const bool m64 = dsub(1.0, T64) > 0.5;
            const int2 ax = a.aux[p];
            const bool m32 = 1.0f - __int_as_float(ax.y) > 0.5f;
            if (m64 != m32) atomicAdd(&a.stats->n_mask, m64 ? 1 : -1);
            a.aux[p].x = (ax.x & ((1 << 29) - 1)) | (1 << 30) | (m64 ? (1 << 29) : 0);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.amb_count = 0;
}

}  // namespace

void launch_mask_fixup(const RasterArgs &a, cudaStream_t s) {
    if (a.P.mode != S2D_SPLAT_AFFINE) return;
    count_launch();
    k_mask_fixup<<<1, 256, 0, s>>>(a);
}

template <auto Kernel>
static void ensure_smem(int bytes) {
    static int done = 0;  // one flag per kernel (templated on the kernel itself)
    if (done < bytes) {
        cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        done = bytes;
    }
}

template <bool kArg, bool kMaxW, bool kRay>
static void fwd_dispatch(const RasterArgs &a, int tiles, cudaStream_t s) {
    const int grid = tiles * (8 / kFwdWarps);
    if (a.normal) k_raster_fwd<kArg, kMaxW, true, kRay><<<grid, kFwdWarps * 32, 0, s>>>(a);
    else k_raster_fwd<kArg, kMaxW, false, kRay><<<grid, kFwdWarps * 32, 0, s>>>(a);
}

template <bool kRay>
static void fwd_dispatch_mode(const RasterArgs &a, int tiles, cudaStream_t s) {
    const bool arg = a.max_w != nullptr || a.arg_w != nullptr;
    const bool mw = a.max_all != nullptr;
    if (arg && mw) fwd_dispatch<true, true, kRay>(a, tiles, s);
    else if (arg) fwd_dispatch<true, false, kRay>(a, tiles, s);
    else if (mw) fwd_dispatch<false, true, kRay>(a, tiles, s);
    else fwd_dispatch<false, false, kRay>(a, tiles, s);
}

void launch_raster_forward(const RasterArgs &a, cudaStream_t s) {
    const int tiles = a.P.ntx * a.P.nty;
    count_launch();
    if (a.P.mode == S2D_SPLAT_RAY) fwd_dispatch_mode<true>(a, tiles, s);
    else fwd_dispatch_mode<false>(a, tiles, s);
}

template <bool kExt, bool kRay>
static void bwd_launch(const RasterArgs &a, int tiles, cudaStream_t s) {
    k_raster_bwd<kExt, kRay><<<tiles * (8 / kBwdWarps), kBwdWarps * 32, 0, s>>>(a);
}

void launch_raster_fused(const RasterArgs &a, cudaStream_t s) {
    const int grid = a.P.ntx * a.P.nty * (8 / kFwdWarps);
    count_launch();
    if (a.P.mode == S2D_SPLAT_RAY) k_raster_fused<true><<<grid, kFwdWarps * 32, 0, s>>>(a);
    else k_raster_fused<false><<<grid, kFwdWarps * 32, 0, s>>>(a);
}

void launch_raster_backward(const RasterArgs &a, cudaStream_t s) {
    const int tiles = a.P.ntx * a.P.nty;
    const bool full = a.loss_kind == S2D_LOSS_EXTERNAL && (a.d_normal != nullptr || a.d_accum != nullptr);
    count_launch();
    const bool ray = a.P.mode == S2D_SPLAT_RAY;
    if (full && ray) bwd_launch<true, true>(a, tiles, s);
    else if (full) bwd_launch<true, false>(a, tiles, s);
    else if (ray) bwd_launch<false, true>(a, tiles, s);
    else bwd_launch<false, false>(a, tiles, s);
}

}  // namespace s2d
