// capi.cu — extern "C" boundary (include/surfel2d.h): per-view workspace arena,
// host-side float64 pose math, and the launch sequence of one view:
//
//   memset(sync region) -> k_project -> k_compact_hist -> 3 x k_onesweep (depth)
//   -> k_tie_fix -> k_scan_emit -> 1..2 x k_onesweep (tile id) -> k_tile_ranges
//   -> k_raster_fwd                       [s2d_forward]
//   -> k_raster_bwd -> k_project_bwd      [s2d_backward]
//   or, after the tile ranges, k_raster_fused -> k_project_bwd   [s2d_forward_backward]
//
// Every count (visible surfels V, pairs P) stays on the device; kernels read it
// there, so a view is a fixed launch sequence with no host round trip (CUDA-graph
// capturable).  Pair capacity overflow is reported in s2d_view_stats.overflow.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <vector>
#include <cstdio>
#include <cstring>
#include <string>

#include "s2d_kernels.h"

using namespace s2d;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define S2D_CUDA(call)                                                                           \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(e_ == cudaErrorMemoryAllocation ? S2D_ERR_OOM : S2D_ERR_CUDA,            \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                      \
    } while (0)

#define S2D_CHECK_LAUNCH()                                                                       \
    do {                                                                                         \
        cudaError_t e_ = cudaGetLastError();                                                     \
        if (e_ != cudaSuccess) return fail(S2D_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

// ---- float64 host pose math, same operation order as the reference ----
// (built with -ffp-contract=off so nothing is fused)
void h_quat_rotate(const double q[4], const double v[3], double o[3]) {
    const double w = q[0], u0 = q[1], u1 = q[2], u2 = q[3];
    const double uv0 = u1 * v[2] - u2 * v[1];
    const double uv1 = u2 * v[0] - u0 * v[2];
    const double uv2 = u0 * v[1] - u1 * v[0];
    const double uu0 = u1 * uv2 - u2 * uv1;
    const double uu1 = u2 * uv0 - u0 * uv2;
    const double uu2 = u0 * uv1 - u1 * uv0;
    o[0] = v[0] + 2.0 * (w * uv0 + uu0);
    o[1] = v[1] + 2.0 * (w * uv1 + uu1);
    o[2] = v[2] + 2.0 * (w * uv2 + uu2);
}

void h_quat_to_matrix(const double q[4], double r[9]) {
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

// pk_inverse (geometry.py:188-195)
void h_pk_inverse(const double a[8], double out[8]) {
    const double s_inv = 1.0 / a[0];
    const double qc[4] = {a[4], -a[5], -a[6], -a[7]};
    double r[3];
    h_quat_rotate(qc, a + 1, r);
    out[0] = s_inv;
    for (int k = 0; k < 3; ++k) out[1 + k] = -s_inv * r[k];
    for (int k = 0; k < 4; ++k) out[4 + k] = qc[k];
}

int validate_camera(const s2d_camera *cam) {
    if (!cam) return fail(S2D_ERR_INVALID, "camera is NULL");
    // CameraIntrinsics.__post_init__ (rasterizer.py:36-40)
    if (!(cam->fx > 0) || !(cam->fy > 0)) return fail(S2D_ERR_INVALID, "focal lengths must be positive");
    if (cam->width <= 0 || cam->height <= 0) return fail(S2D_ERR_INVALID, "image size must be positive");
    if (!(0 <= cam->cx && cam->cx < cam->width && 0 <= cam->cy && cam->cy < cam->height))
        return fail(S2D_ERR_INVALID, "principal point must lie inside the image");
    if (cam->width > 32767 || cam->height > 32767) return fail(S2D_ERR_INVALID, "image too large (max 32767)");
    const int64_t nt = (int64_t)((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile);
    if (nt > 65536) return fail(S2D_ERR_INVALID, "too many tiles (max 65536)");
    return S2D_OK;
}

void make_view_params(const double pose[8], const s2d_camera &cam, const s2d_raster_config &cfg,
                      int64_t n, ViewParams &P) {
    memset(&P, 0, sizeof(P));
    h_pk_inverse(pose, P.inv);
    h_quat_to_matrix(P.inv + 4, P.r_cw);
    for (int k = 0; k < 9; ++k) P.m_cw[k] = P.inv[0] * P.r_cw[k];
    P.fx = cam.fx;
    P.fy = cam.fy;
    P.cx = cam.cx;
    P.cy = cam.cy;
    P.near_plane = cfg.near_plane;
    P.tan_max = std::tan(cfg.max_view_angle_deg * (M_PI / 180.0));  // np.tan(np.radians(.))
    P.max_cond = cfg.max_condition;
    P.sigma = cfg.footprint_sigma;
    P.mx = cfg.center_margin_frac * (double)cam.width;
    P.my = cfg.center_margin_frac * (double)cam.height;
    P.wmax = (double)(cam.width - 1) + P.mx;
    P.hmax = (double)(cam.height - 1) + P.my;
    P.wm1 = (double)(cam.width - 1);
    P.hm1 = (double)(cam.height - 1);
    P.w_clamp = cfg.weight_clamp;
    P.maha_cut = cfg.footprint_sigma * cfg.footprint_sigma;
    P.w_clamp_f = (float)cfg.weight_clamp;
    P.term_t_f = (float)cfg.termination_transmittance;
    P.term_t = cfg.termination_transmittance;
    P.maha_cut_f = (float)P.maha_cut;
    P.W = cam.width;
    P.H = cam.height;
    P.ntx = (cam.width + kTile - 1) / kTile;
    P.nty = (cam.height + kTile - 1) / kTile;
    P.n = n;
    P.shard = n;
    P.mode = cfg.splat_mode;
}

int bits_for(int64_t v) {  // bits needed to represent values in [0, v)
    int b = 0;
    while (((int64_t)1 << b) < v) ++b;
    return b;
}

template <class T>
int grow(T *&p, int64_t &cap_elems, int64_t need, bool zero = false) {
    if (need <= cap_elems && p) return S2D_OK;
    if (p) cudaFree(p);
    p = nullptr;
    int64_t c = need < 1 ? 1 : need;
    cudaError_t e = cudaMalloc(&p, (size_t)c * sizeof(T));
    if (e != cudaSuccess) {
        cap_elems = 0;
        return fail(S2D_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    if (zero) {
        e = cudaMemset(p, 0, (size_t)c * sizeof(T));
        if (e != cudaSuccess) return fail(S2D_ERR_CUDA, cudaGetErrorString(e));
    }
    cap_elems = c;
    return S2D_OK;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

__global__ void k_stats_accumulate(const s2d_view_stats *s, s2d_view_stats *acc) {
    // atomic: views on concurrent streams may share one accumulator
    atomicMax(&acc->visible, s->visible);
    atomicMax(&acc->pairs, s->pairs);
    atomicMax(&acc->pairs_stored, s->pairs_stored);
    atomicAdd(&acc->degenerate, s->degenerate);
    atomicAdd(&acc->n_mask, s->n_mask);
    atomicAdd(&acc->guard_hits, s->guard_hits);
    atomicOr(&acc->overflow, s->overflow);
    atomicMax(&acc->blended, s->blended);
}

}  // namespace

struct s2d_ctx {
    int device;
};

namespace s2d {
std::atomic<int64_t> g_launches{0};
}

struct s2d_view {
    s2d_ctx *ctx = nullptr;
    // capacities (elements)
    int64_t cap_rec = 0, cap_rect = 0, cap_z = 0, cap_flags = 0, cap_keys[2] = {0, 0},
            cap_vals[2] = {0, 0}, cap_grad = 0, cap_aux = 0, cap_pk[2] = {0, 0}, cap_pv[2] = {0, 0},
            cap_bs = 0, cap_bc = 0, cap_ex = 0, cap_sync = 0, cap_amb = 0, cap_tc = 0, cap_to = 0, cap_acc = 0;
    SplatRecord *rec = nullptr;
    ExactRec *exact = nullptr;  // float64 centre + inv_abc per on-screen surfel (guard-band path)
    AccurateRec *acc = nullptr;  // float64 centre + Minv per accurate (ill-conditioned) surfel
    short4 *rect = nullptr;
    double *z64 = nullptr;
    uint8_t *flags = nullptr;
    uint32_t *keys[2] = {nullptr, nullptr}, *vals[2] = {nullptr, nullptr};
    uint32_t *tcount = nullptr;  // drawn surfels per projection tile
    uint32_t *pkeys[2] = {nullptr, nullptr}, *pvals[2] = {nullptr, nullptr};
    uint4 *bstream = nullptr;  // [16 pcap] per-(warp, column half) (surfel, blend mask, clamp mask) streams
    int *bcount = nullptr;     // [ntiles * 16] stream lengths
    float *grad2d = nullptr;
    int2 *aux = nullptr;
    int *amb = nullptr;  // [npx] ambiguous depth-mask pixels (k_mask_fixup)
    uint8_t *sync = nullptr;
    SyncRegion sr{};
    int64_t pcap = 0;  // pair capacity in use
    int64_t shard = 0;  // surfels per shard of the packed parameter/gradient blocks (0: plain layout)
    // state of the last forward
    bool has_fwd = false;
    ViewParams P{};
    int64_t n = 0;
    int pair_buf = 0;   // which pkeys/pvals buffer holds the sorted pairs
    int order_buf = 0;  // which vals buffer holds the depth order
    cudaStream_t last_stream = nullptr;
    // phase timing (events recorded between kernels, resolved in s2d_view_timing)
    struct TimedCall {
        cudaEvent_t e[6];
        int n;
        int kind;  // 0 forward, 1 backward, 2 fused forward + backward
    };
    bool timing = false;
    std::vector<TimedCall> timed;
    std::vector<cudaEvent_t> free_events;
    double phase_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t n_fwd_timed = 0, n_bwd_timed = 0;
    cudaEvent_t take_event() {
        if (free_events.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = free_events.back();
        free_events.pop_back();
        return e;
    }
    // scratch for the host-buffer entry point
    int64_t cap_hp = 0, cap_himg = 0;
    float *h_params_dev = nullptr, *h_img_dev = nullptr;
    size_t cap_pin = 0;
    float *h_pin = nullptr;  // pinned host staging (grow-only)
};

namespace {

int layout_sync(s2d_view *v, int64_t n, int64_t pcap, int ntiles) {
    const int64_t sort_tiles = (n + kSortTile - 1) / kSortTile + 1;
    const int64_t emit_tiles = (n + kEmitTile - 1) / kEmitTile + 1;
    const int64_t psort_tiles = (pcap + kSortTile - 1) / kSortTile + 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t o_stats = take(sizeof(s2d_view_stats));
    const size_t o_tickets = take(16 * sizeof(int));
    const size_t o_drawn = take(sizeof(int));
    const size_t o_krange = take(2 * 4);
    const size_t o_dhist = take(3 * kRadix * 4);
    const size_t o_dstat = take((size_t)3 * sort_tiles * kRadix * 4);
    const size_t o_emit = take((size_t)emit_tiles * 4);
    const size_t o_phist = take(2 * kRadix * 4);
    const size_t o_pstat = take((size_t)2 * psort_tiles * kRadix * 4);
    const size_t o_tie = take(4 * 4);
    const size_t o_amb = take(4);
    const size_t o_cc = take((size_t)((n + kProjThreads - 1) / kProjThreads / kCompactTiles + 1) * 4);
    const size_t o_ranges = take((size_t)ntiles * sizeof(int2));
    int64_t need = (int64_t)off;
    int rc = grow(v->sync, v->cap_sync, need);
    if (rc) return rc;
    uint8_t *b = v->sync;
    v->sr.stats = reinterpret_cast<s2d_view_stats *>(b + o_stats);
    v->sr.tickets = reinterpret_cast<int *>(b + o_tickets);
    v->sr.n_drawn = reinterpret_cast<int *>(b + o_drawn);
    v->sr.key_range = reinterpret_cast<uint32_t *>(b + o_krange);
    v->sr.depth_hist = reinterpret_cast<uint32_t *>(b + o_dhist);
    v->sr.depth_status = reinterpret_cast<uint32_t *>(b + o_dstat);
    v->sr.emit_status = reinterpret_cast<uint32_t *>(b + o_emit);
    v->sr.pair_hist = reinterpret_cast<uint32_t *>(b + o_phist);
    v->sr.pair_status = reinterpret_cast<uint32_t *>(b + o_pstat);
    v->sr.tie_ctl = reinterpret_cast<uint32_t *>(b + o_tie);
    v->sr.amb_count = reinterpret_cast<int *>(b + o_amb);
    v->sr.ccount = reinterpret_cast<uint32_t *>(b + o_cc);
    v->sr.ranges = reinterpret_cast<int2 *>(b + o_ranges);
    v->sr.bytes = off;
    return S2D_OK;
}

int ensure_capacity(s2d_view *v, int64_t n, int64_t npx, int ntiles) {
    int rc;
    const int64_t nn = n < 1 ? 1 : n;
    if ((rc = grow(v->rec, v->cap_rec, nn))) return rc;
    if ((rc = grow(v->exact, v->cap_ex, nn))) return rc;
    if ((rc = grow(v->acc, v->cap_acc, nn))) return rc;
    if ((rc = grow(v->rect, v->cap_rect, nn))) return rc;
    if ((rc = grow(v->z64, v->cap_z, nn))) return rc;
    if ((rc = grow(v->flags, v->cap_flags, nn))) return rc;
    for (int b = 0; b < 2; ++b) {
        if ((rc = grow(v->keys[b], v->cap_keys[b], nn))) return rc;
        if ((rc = grow(v->vals[b], v->cap_vals[b], nn))) return rc;
    }
    if ((rc = grow(v->tcount, v->cap_tc, (nn + kProjThreads - 1) / kProjThreads))) return rc;
    if ((rc = grow(v->grad2d, v->cap_grad, nn * 16, /*zero=*/true))) return rc;
    if ((rc = grow(v->aux, v->cap_aux, npx))) return rc;
    if ((rc = grow(v->amb, v->cap_amb, npx))) return rc;
    if (v->pcap == 0) v->pcap = 4 * nn < 65536 ? 65536 : 4 * nn;  // first guess; regrown on overflow
    for (int b = 0; b < 2; ++b) {
        if ((rc = grow(v->pkeys[b], v->cap_pk[b], v->pcap))) return rc;
        if ((rc = grow(v->pvals[b], v->cap_pv[b], v->pcap))) return rc;
    }
    if ((rc = grow(v->bstream, v->cap_bs, 16 * v->pcap))) return rc;
    if ((rc = grow(v->bcount, v->cap_bc, 16 * (int64_t)ntiles))) return rc;
    return layout_sync(v, nn, v->pcap, ntiles);
}

// The loss of a fused forward + backward (s2d_forward_backward)
struct FusedLoss {
    const s2d_loss *loss;
    float *grads;
    double *loss_accum;
    cudaEvent_t wait;
};

int view_forward(s2d_view *v, cudaStream_t s, const float *params, int64_t n, const double pose[8],
                 const s2d_camera *cam, const s2d_raster_config *cfg, const s2d_image *out,
                 float *max_all, float *max_marked, const uint8_t *mask, const FusedLoss *fl = nullptr) {
    int rc = validate_camera(cam);
    if (rc) return rc;
    if (!cfg) return fail(S2D_ERR_INVALID, "raster config is NULL");
    if (cfg->splat_mode != S2D_SPLAT_AFFINE && cfg->splat_mode != S2D_SPLAT_RAY)
        return fail(S2D_ERR_INVALID, "unknown splat_mode");
    if (!pose) return fail(S2D_ERR_INVALID, "pose is NULL");
    if (n < 0 || n >= (int64_t)1 << 30) return fail(S2D_ERR_INVALID, "surfel count out of range");
    if (n > 0 && !params) return fail(S2D_ERR_INVALID, "params is NULL");
    if (!(pose[0] > 0) || !std::isfinite(pose[0])) return fail(S2D_ERR_INVALID, "pose scale must be positive");
    if (!out) return fail(S2D_ERR_INVALID, "image is NULL");
    const int64_t npx = (int64_t)cam->width * cam->height;
    ViewParams P;
    make_view_params(pose, *cam, *cfg, n, P);
    if (v->shard > 0 && v->shard < n) P.shard = v->shard;
    const int ntiles = P.ntx * P.nty;
    if ((rc = ensure_capacity(v, n, npx, ntiles))) return rc;
    v->has_fwd = false;
    S2D_CUDA(cudaMemsetAsync(v->sync, 0, v->sr.bytes, s));
    s2d_view::TimedCall tc{};
    tc.kind = fl ? 2 : 0;
    auto mark = [&]() {
        if (v->timing && tc.n < 6) {
            tc.e[tc.n] = v->take_event();
            cudaEventRecord(tc.e[tc.n++], s);
        }
    };
    mark();
    SyncRegion &sr = v->sr;
    // the depth sort and the pair emission run over the drawn surfels: on-screen with a
    // non-empty integer bbox (an empty bbox touches no pixel, _raster_kernels.py:32-34)
    int *d_v = sr.n_drawn;
    if (n > 0) {
        ProjectArgs pa;
        pa.P = P;
        pa.params = params;
        pa.rec = v->rec;
        pa.exact = v->exact;
        pa.acc = v->acc;
        pa.rect = v->rect;
        pa.z64 = v->z64;
        pa.flags = v->flags;
        pa.stats = sr.stats;
        pa.key_range = sr.key_range;
        // k_project leaves each tile's drawn pairs in its own segment of keys[1] / vals[1];
        // k_compact_hist concatenates them in index order into keys[0] / vals[0]
        pa.keys = v->keys[1];
        pa.vals = v->vals[1];
        pa.tcount = v->tcount;
        pa.ccount = sr.ccount;
        launch_project(pa, s);
        mark();
        // depth order: the drawn surfels' keys rebased to 24 bits, 3 stable 8-bit passes, then
        // k_tie_fix orders equal keys by (z64, index)
        launch_compact_hist(v->keys[1], v->vals[1], v->tcount, sr.ccount, n, sr.key_range, v->keys[0], v->vals[0],
                            sr.depth_hist, sr.n_drawn, s);
        const int64_t sort_tiles = (n + kSortTile - 1) / kSortTile + 1;
        int cur = 0;
        for (int p = 0; p < 3; ++p) {
            launch_onesweep(v->keys[cur], v->vals[cur], v->keys[cur ^ 1], v->vals[cur ^ 1], d_v, (int)n,
                            kRadixBits * p, sr.depth_hist + p * kRadix,
                            sr.depth_status + (size_t)p * sort_tiles * kRadix, sr.tickets + 1 + p, s);
            cur ^= 1;
        }
        // (the other ping-pong buffers are free now: the long-run list and the merge scratch)
        launch_tie_fix(v->keys[cur], v->vals[cur], v->z64, d_v, (int)n, sr.tie_ctl, v->vals[cur ^ 1],
                       v->keys[cur ^ 1], s);
        v->order_buf = cur;
        mark();
        // tile binning: pairs emitted in depth order, then stable sort by tile id
        const int tbits = bits_for(ntiles);
        const int ppass = passes_for_bits(tbits);
        EmitArgs ea;
        ea.order = v->vals[cur];
        ea.rect = v->rect;
        ea.d_v = d_v;
        ea.cap_v = (int)n;
        ea.ntx = P.ntx;
        ea.pair_passes = ppass;
        ea.pkeys = v->pkeys[0];
        ea.pvals = v->pvals[0];
        ea.pcap = (uint32_t)v->pcap;
        ea.stats = sr.stats;
        ea.status = sr.emit_status;
        ea.ticket = sr.tickets + 5;
        ea.pair_hist = sr.pair_hist;
        launch_scan_emit(ea, s);
        const int64_t psort_tiles = (v->pcap + kSortTile - 1) / kSortTile + 1;
        int pc = 0;
        for (int p = 0; p < ppass; ++p) {
            launch_onesweep(v->pkeys[pc], v->pvals[pc], v->pkeys[pc ^ 1], v->pvals[pc ^ 1],
                            &sr.stats->pairs_stored, (int)v->pcap, kRadixBits * p, sr.pair_hist + p * kRadix,
                            sr.pair_status + (size_t)p * psort_tiles * kRadix, sr.tickets + 6 + p, s);
            pc ^= 1;
        }
        v->pair_buf = pc;
        launch_tile_ranges(v->pkeys[pc], &sr.stats->pairs, (uint32_t)v->pcap, sr.ranges, s);
        S2D_CHECK_LAUNCH();
    } else {
        mark();
        mark();
    }
    mark();
    RasterArgs ra;
    memset(&ra, 0, sizeof(ra));
    ra.P = P;
    ra.params = params;
    ra.ranges = sr.ranges;
    ra.pair_ids = v->pvals[v->pair_buf];
    ra.pair_keys = v->pkeys[v->pair_buf];
    ra.bstream = v->bstream;
    ra.bcount = v->bcount;
    ra.rec = v->rec;
    ra.exact = v->exact;
    ra.acc = v->acc;
    ra.rect = v->rect;
    ra.aux = v->aux;
    ra.color = out->color;
    ra.depth = out->depth;
    ra.accum = out->accumulation;
    ra.normal = out->normal;
    ra.max_w = out->max_w;
    ra.arg_w = out->arg_w;
    ra.max_all = max_all;
    ra.max_marked = max_marked;
    ra.mask = mask;
    ra.stats = sr.stats;
    ra.amb_count = sr.amb_count;
    ra.amb_list = v->amb;
    if (fl) {
        ra.loss_kind = fl->loss->kind;
        ra.depth_mask = fl->loss->depth_mask;
        ra.w_rgb = fl->loss->w_rgb;
        ra.w_depth = fl->loss->w_depth;
        ra.target_rgb = fl->loss->target_rgb;
        ra.target_depth = fl->loss->target_depth;
        ra.grad2d = v->grad2d;
        ra.loss_accum = fl->loss_accum;
        if (fl->wait) S2D_CUDA(cudaStreamWaitEvent(s, fl->wait, 0));
        launch_raster_fused(ra, s);
        S2D_CHECK_LAUNCH();
        mark();
        if (n > 0) {
            ProjectBwdArgs pb;
            pb.P = P;
            pb.params = params;
            pb.flags = v->flags;
            pb.rect = v->rect;
            pb.grad2d = v->grad2d;
            pb.g2_stride = g2_stride(P.mode == S2D_SPLAT_RAY, false);  // k_raster_fused: no external seeds
            pb.grads = fl->grads;
            launch_project_backward(pb, s);
            S2D_CHECK_LAUNCH();
        }
        mark();
    } else {
        launch_raster_forward(ra, s);
        S2D_CHECK_LAUNCH();
        mark();
    }
    if (v->timing) v->timed.push_back(tc);
    v->P = P;
    v->n = n;
    v->has_fwd = fl == nullptr;
    v->last_stream = s;
    return S2D_OK;
}

}  // namespace

extern "C" {

const char *s2d_last_error(void) { return g_err.c_str(); }

int32_t s2d_version(void) { return 200; }

int s2d_ctx_create(int32_t device, s2d_ctx **out) {
    if (!out) return fail(S2D_ERR_INVALID, "out is NULL");
    int ndev = 0;
    S2D_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(S2D_ERR_INVALID, "no such CUDA device");
    S2D_CUDA(cudaSetDevice(device));
    s2d_ctx *c = new s2d_ctx;
    c->device = device;
    *out = c;
    return S2D_OK;
}

int s2d_ctx_destroy(s2d_ctx *ctx) {
    delete ctx;
    return S2D_OK;
}

int s2d_view_create(s2d_ctx *ctx, s2d_view **out) {
    if (!ctx || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    s2d_view *v = new s2d_view;
    v->ctx = ctx;
    *out = v;
    return S2D_OK;
}

int s2d_view_destroy(s2d_view *v) {
    if (!v) return S2D_OK;
    void *ptrs[] = {v->rec, v->exact, v->acc, v->rect, v->z64, v->flags, v->keys[0], v->keys[1], v->vals[0], v->vals[1],
                    v->pkeys[0], v->pkeys[1], v->pvals[0], v->pvals[1], v->bstream, v->bcount, v->grad2d, v->aux, v->amb, v->tcount, v->sync,
                    v->h_params_dev, v->h_img_dev};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (v->h_pin) cudaFreeHost(v->h_pin);
    for (auto &tc : v->timed)
        for (int k = 0; k < tc.n; ++k) cudaEventDestroy(tc.e[k]);
    for (cudaEvent_t e : v->free_events) cudaEventDestroy(e);
    delete v;
    return S2D_OK;
}

int s2d_view_stats_device(s2d_view *v, s2d_view_stats **out) {
    if (!v || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    if (!v->sync) return fail(S2D_ERR_STATE, "view has no forward yet");
    *out = v->sr.stats;
    return S2D_OK;
}

int s2d_view_stats_host(s2d_view *v, s2d_view_stats *out) {
    if (!v || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    if (!v->sync) {
        memset(out, 0, sizeof(*out));
        return S2D_OK;
    }
    S2D_CUDA(cudaStreamSynchronize(v->last_stream));
    S2D_CUDA(cudaMemcpy(out, v->sr.stats, sizeof(*out), cudaMemcpyDeviceToHost));
    return S2D_OK;
}

int s2d_view_stats_accumulate(s2d_view *v, void *stream, s2d_view_stats *acc_device) {
    if (!v || !acc_device) return fail(S2D_ERR_INVALID, "NULL argument");
    if (!v->sync) return fail(S2D_ERR_STATE, "view has no forward yet");
    count_launch();
    k_stats_accumulate<<<1, 1, 0, (cudaStream_t)stream>>>(v->sr.stats, acc_device);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_view_reserve_pairs(s2d_view *v, int64_t pairs) {
    if (!v) return fail(S2D_ERR_INVALID, "NULL view");
    if (pairs > ((int64_t)1 << 30)) return fail(S2D_ERR_INVALID, "pair capacity too large");
    v->pcap = pairs < 1024 ? 1024 : pairs;
    return S2D_OK;
}

int s2d_view_set_layout(s2d_view *v, int64_t shard_surfels) {
    if (!v) return fail(S2D_ERR_INVALID, "NULL view");
    if (shard_surfels < 0 || shard_surfels >= ((int64_t)1 << 30)) return fail(S2D_ERR_INVALID, "bad shard size");
    v->shard = shard_surfels;
    return S2D_OK;
}

int64_t s2d_launch_count(void) { return s2d::g_launches.load(); }

int s2d_view_set_timing(s2d_view *v, int32_t enable) {
    if (!v) return fail(S2D_ERR_INVALID, "NULL view");
    v->timing = enable != 0;
    return S2D_OK;
}

int s2d_view_timing(s2d_view *v, double out[8], int32_t reset) {
    if (!v || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    for (auto &tc : v->timed) {
        if (tc.n < 2) continue;
        S2D_CUDA(cudaEventSynchronize(tc.e[tc.n - 1]));
        for (int k = 0; k + 1 < tc.n; ++k) {
            float ms = 0.f;
            S2D_CUDA(cudaEventElapsedTime(&ms, tc.e[k], tc.e[k + 1]));
            // fused: project, sort, binning, raster (fused, as phase 3), projection backward
            const int phase = tc.kind == 0 ? k : tc.kind == 1 ? 4 + k : (k < 4 ? k : 5);
            if (phase < 6) v->phase_ms[phase] += ms;
        }
        if (tc.kind != 1) v->n_fwd_timed++;
        if (tc.kind != 0) v->n_bwd_timed++;
        for (int k = 0; k < tc.n; ++k) v->free_events.push_back(tc.e[k]);
    }
    v->timed.clear();
    for (int k = 0; k < 6; ++k) out[k] = v->phase_ms[k];
    out[6] = (double)v->n_fwd_timed;
    out[7] = (double)v->n_bwd_timed;
    if (reset) {
        for (int k = 0; k < 6; ++k) v->phase_ms[k] = 0;
        v->n_fwd_timed = v->n_bwd_timed = 0;
    }
    return S2D_OK;
}

int s2d_pose_inverse(const double pose_c2w[8], double out[8]) {
    if (!pose_c2w || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    h_pk_inverse(pose_c2w, out);
    return S2D_OK;
}

int s2d_forward(s2d_view *v, void *stream, const float *params, int64_t n, const double pose_c2w[8],
                const s2d_camera *cam, const s2d_raster_config *cfg, const s2d_image *out,
                float *max_all, float *max_marked, const uint8_t *mask) {
    if (!v) return fail(S2D_ERR_INVALID, "NULL view");
    return view_forward(v, (cudaStream_t)stream, params, n, pose_c2w, cam, cfg, out, max_all, max_marked,
                        mask);
}

int s2d_backward(s2d_view *v, void *stream, const float *params, int64_t n, const s2d_image *image,
                 const s2d_loss *loss, float *grads, double *loss_accum) {
    if (!v || !image || !loss) return fail(S2D_ERR_INVALID, "NULL argument");
    if (!v->has_fwd) return fail(S2D_ERR_STATE, "backward without a forward on this view");
    if (n != v->n) return fail(S2D_ERR_STATE, "surfel count differs from the forward");
    if (n > 0 && !grads) return fail(S2D_ERR_INVALID, "grads is NULL");
    if (loss->kind != S2D_LOSS_EXTERNAL) {
        if (!loss->target_rgb || !loss->target_depth)
            return fail(S2D_ERR_INVALID, "loss targets are NULL");
        if (!image->color || !image->depth || !image->accumulation)
            return fail(S2D_ERR_INVALID, "loss needs the forward color/depth/accumulation");
        if (loss->kind != S2D_LOSS_MSE && loss->kind != S2D_LOSS_L1)
            return fail(S2D_ERR_INVALID, "unknown loss kind");
    }
    cudaStream_t s = (cudaStream_t)stream;
    s2d_view::TimedCall tc{};
    tc.kind = 1;
    auto mark = [&]() {
        if (v->timing && tc.n < 6) {
            tc.e[tc.n] = v->take_event();
            cudaEventRecord(tc.e[tc.n++], s);
        }
    };
    mark();
    RasterArgs ra;
    memset(&ra, 0, sizeof(ra));
    ra.P = v->P;
    ra.params = params;
    ra.ranges = v->sr.ranges;
    ra.pair_ids = v->pvals[v->pair_buf];
    ra.pair_keys = v->pkeys[v->pair_buf];
    ra.bstream = v->bstream;
    ra.bcount = v->bcount;
    ra.rec = v->rec;
    ra.exact = v->exact;
    ra.acc = v->acc;
    ra.rect = v->rect;
    ra.aux = v->aux;
    ra.color = image->color;
    ra.depth = image->depth;
    ra.accum = image->accumulation;
    ra.normal = image->normal;
    ra.stats = v->sr.stats;
    ra.loss_kind = loss->kind;
    ra.depth_mask = loss->depth_mask;
    ra.w_rgb = loss->w_rgb;
    ra.w_depth = loss->w_depth;
    ra.target_rgb = loss->target_rgb;
    ra.target_depth = loss->target_depth;
    ra.d_color = loss->d_color;
    ra.d_depth = loss->d_depth;
    ra.d_normal = loss->d_normal;
    ra.d_accum = loss->d_accumulation;
    ra.grad2d = v->grad2d;
    ra.loss_accum = loss_accum;
    ra.amb_count = v->sr.amb_count;
    ra.amb_list = v->amb;
    // a loss over the depth mask: re-decide the float32-ambiguous mask pixels in float64 first
    const bool uses_mask = (loss->kind == S2D_LOSS_MSE && loss->w_depth != 0.0) ||
                           (loss->kind == S2D_LOSS_L1 && loss->depth_mask);
    if (uses_mask && n > 0) launch_mask_fixup(ra, s);
    launch_raster_backward(ra, s);
    mark();
    if (n > 0) {
        ProjectBwdArgs pb;
        pb.P = v->P;
        pb.params = params;
        pb.flags = v->flags;
        pb.rect = v->rect;
        pb.grad2d = v->grad2d;
        // the row width launch_raster_backward's kernel wrote (k_raster_bwd<kExt, kRay>)
        const bool ext = loss->kind == S2D_LOSS_EXTERNAL && (loss->d_normal != nullptr || loss->d_accumulation != nullptr);
        pb.g2_stride = g2_stride(v->P.mode == S2D_SPLAT_RAY, ext);
        pb.grads = grads;
        launch_project_backward(pb, s);
    }
    S2D_CHECK_LAUNCH();
    mark();
    if (v->timing) v->timed.push_back(tc);
    v->last_stream = s;
    return S2D_OK;
}

int s2d_forward_backward(s2d_view *v, void *stream, const float *params, int64_t n, const double pose_c2w[8],
                         const s2d_camera *cam, const s2d_raster_config *cfg, const s2d_image *out,
                         const s2d_loss *loss, float *grads, double *loss_accum, void *wait_event) {
    if (!v || !loss) return fail(S2D_ERR_INVALID, "NULL argument");
    if (n > 0 && !grads) return fail(S2D_ERR_INVALID, "grads is NULL");
    const bool fusable = (loss->kind == S2D_LOSS_L1 && !loss->depth_mask) ||
                         (loss->kind == S2D_LOSS_MSE && loss->w_depth == 0.0);
    cudaStream_t s = (cudaStream_t)stream;
    if (!fusable) {
        // the seeds need the whole image's depth-mask count first: two kernels
        int rc = view_forward(v, s, params, n, pose_c2w, cam, cfg, out, nullptr, nullptr, nullptr);
        if (rc) return rc;
        if (wait_event) S2D_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)wait_event, 0));
        return s2d_backward(v, stream, params, n, out, loss, grads, loss_accum);
    }
    if (!loss->target_rgb || !loss->target_depth) return fail(S2D_ERR_INVALID, "loss targets are NULL");
    s2d_image none;
    memset(&none, 0, sizeof(none));
    const FusedLoss fl{loss, grads, loss_accum, (cudaEvent_t)wait_event};
    return view_forward(v, s, params, n, pose_c2w, cam, cfg, out ? out : &none, nullptr, nullptr, nullptr, &fl);
}

int s2d_adam_step(void *stream, float *params, const float *grads, float *m1, float *m2, int64_t n,
                  int64_t step, const s2d_adam_config *cfg, const uint8_t *mask) {
    return s2d_adam_step_gated(stream, params, grads, m1, m2, n, step, cfg, mask, nullptr);
}

int s2d_adam_step_gated(void *stream, float *params, const float *grads, float *m1, float *m2, int64_t n,
                        int64_t step, const s2d_adam_config *cfg, const uint8_t *mask, const int32_t *skip) {
    if (!cfg) return fail(S2D_ERR_INVALID, "adam config is NULL");
    if (step < 1) return fail(S2D_ERR_INVALID, "adam step is 1-based");
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (n == 0) return S2D_OK;
    if (!params || !grads || !m1 || !m2) return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_adam(params, grads, m1, m2, n, step, *cfg, mask, skip, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_refine_gd(void *stream, float *params, const float *params0, const float *grads, int64_t n, double step,
                  const uint8_t *mask) {
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (!(step >= 0.0) || !std::isfinite(step)) return fail(S2D_ERR_INVALID, "step must be finite and >= 0");
    if (n == 0) return S2D_OK;
    if (!params || !params0 || !grads) return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_refine_gd(params + 9 * n, params0 + 9 * n, grads + 9 * n, n, step, mask, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_refine_gnorm(void *stream, const float *grads, int64_t n, const uint8_t *mask, float *out) {
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (!out) return fail(S2D_ERR_INVALID, "NULL buffer");
    S2D_CUDA(cudaMemsetAsync(out, 0, sizeof(float), (cudaStream_t)stream));
    if (n == 0) return S2D_OK;
    if (!grads) return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_refine_gnorm(grads + 9 * n, n, mask, out, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_view_inspect(s2d_view *v, s2d_view_debug *out) {
    if (!v || !out) return fail(S2D_ERR_INVALID, "NULL argument");
    if (!v->has_fwd) return fail(S2D_ERR_STATE, "no forward on this view");
    out->order = v->vals[v->order_buf];
    S2D_CUDA(cudaMemcpy(&out->drawn, v->sr.n_drawn, sizeof(int), cudaMemcpyDeviceToHost));
    out->pair_tiles = v->pkeys[v->pair_buf];
    out->pair_ids = v->pvals[v->pair_buf];
    out->ranges = reinterpret_cast<int32_t *>(v->sr.ranges);
    out->bbox = reinterpret_cast<int16_t *>(v->rect);
    out->z = v->z64;
    out->flags = v->flags;
    out->records = reinterpret_cast<float *>(v->rec);
    out->pixel_state = reinterpret_cast<int32_t *>(v->aux);
    out->ntiles = v->P.ntx * v->P.nty;
    out->tiles_x = v->P.ntx;
    out->pair_capacity = v->pcap;
    out->stream_lengths = v->bcount;
    out->streams = reinterpret_cast<const uint32_t *>(v->bstream);
    return S2D_OK;
}

int s2d_render_host(s2d_view *v, void *stream, const double *means, const double *quats, const double *scales,
                    const double *opacities, const double *colors, int64_t n, const double pose_c2w[8],
                    const s2d_camera *cam, const s2d_raster_config *cfg, double *color, double *depth,
                    double *accumulation, double *normal, int32_t *degenerate_skipped) {
    if (!v) return fail(S2D_ERR_INVALID, "NULL view");
    int rc = validate_camera(cam);
    if (rc) return rc;
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (n > 0 && !(means && quats && scales && opacities && colors))
        return fail(S2D_ERR_INVALID, "NULL surfel array");
    const int64_t npx = (int64_t)cam->width * cam->height;
    const int64_t np = 13 * (n < 1 ? 1 : n);
    // one grow-only pinned staging buffer per view: the float32 packed block, then the images
    const size_t need = (size_t)(np + 8 * npx) * sizeof(float);
    if (v->cap_pin < need) {
        if (v->h_pin) cudaFreeHost(v->h_pin);
        v->h_pin = nullptr;
        v->cap_pin = 0;
        S2D_CUDA(cudaMallocHost(&v->h_pin, need));
        v->cap_pin = need;
    }
    float *hp = v->h_pin;
    for (int64_t i = 0; i < 3 * n; ++i) hp[i] = (float)means[i];
    for (int64_t i = 0; i < 4 * n; ++i) hp[3 * n + i] = (float)quats[i];
    for (int64_t i = 0; i < 2 * n; ++i) hp[7 * n + i] = (float)scales[i];
    for (int64_t i = 0; i < n; ++i) hp[9 * n + i] = (float)opacities[i];
    for (int64_t i = 0; i < 3 * n; ++i) hp[10 * n + i] = (float)colors[i];
    float *himg = hp + np;
    if ((rc = grow(v->h_params_dev, v->cap_hp, np))) return rc;
    if ((rc = grow(v->h_img_dev, v->cap_himg, 8 * npx))) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    S2D_CUDA(cudaMemcpyAsync(v->h_params_dev, hp, (size_t)np * sizeof(float), cudaMemcpyHostToDevice, s));
    s2d_image img;
    memset(&img, 0, sizeof(img));
    img.color = v->h_img_dev;
    img.depth = v->h_img_dev + 3 * npx;
    img.accumulation = v->h_img_dev + 4 * npx;
    img.normal = v->h_img_dev + 5 * npx;
    for (int attempt = 0;; ++attempt) {
        if ((rc = view_forward(v, s, v->h_params_dev, n, pose_c2w, cam, cfg, &img, nullptr, nullptr, nullptr)))
            return rc;
        s2d_view_stats st;
        S2D_CUDA(cudaMemcpyAsync(&st, v->sr.stats, sizeof(st), cudaMemcpyDeviceToHost, s));
        S2D_CUDA(cudaStreamSynchronize(s));
        if (!st.overflow) {
            if (degenerate_skipped) *degenerate_skipped = st.degenerate;
            break;
        }
        if (attempt == 3) return fail(S2D_ERR_STATE, "pair capacity could not be sized");
        v->pcap = (int64_t)st.pairs + st.pairs / 4 + 1024;
    }
    S2D_CUDA(cudaMemcpyAsync(himg, v->h_img_dev, (size_t)8 * npx * sizeof(float), cudaMemcpyDeviceToHost, s));
    S2D_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < 3 * npx; ++i) {
        if (color) color[i] = himg[i];
        if (normal) normal[i] = himg[5 * npx + i];
    }
    for (int64_t i = 0; i < npx; ++i) {
        if (depth) depth[i] = himg[3 * npx + i];
        if (accumulation) accumulation[i] = himg[4 * npx + i];
    }
    return S2D_OK;
}

int s2d_transform_surfels(void *stream, const double pose[8], const float *params_in, int64_t n,
                          float *params_out) {
    if (!pose) return fail(S2D_ERR_INVALID, "pose is NULL");
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (!(pose[0] > 0) || !std::isfinite(pose[0])) return fail(S2D_ERR_INVALID, "pose scale must be positive");
    if (n == 0) return S2D_OK;
    if (!params_in || !params_out) return fail(S2D_ERR_INVALID, "NULL buffer");
    if (params_in == params_out) return fail(S2D_ERR_INVALID, "params_in and params_out must not alias");
    launch_transform(params_in, params_out, n, pose, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_fuse_gate(void *stream, const float *accumulation, const s2d_camera *cam, const float *params, int64_t n,
                  double accum_threshold, uint8_t *keep) {
    int rc = validate_camera(cam);
    if (rc) return rc;
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (!(accum_threshold > 0.0 && accum_threshold < 1.0))
        return fail(S2D_ERR_INVALID, "accum_threshold must be in (0, 1)");  // FusionConfig (mapper.py:57-58)
    if (n == 0) return S2D_OK;
    if (!accumulation || !params || !keep) return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_fuse_gate(accumulation, *cam, params, n, accum_threshold, keep, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_prune_mark(void *stream, const float *color, const float *depth, const float *accumulation,
                   const float *observed_rgb, const float *observed_depth, int64_t npx, double rgb_error,
                   double depth_error_frac, uint8_t *marked) {
    if (npx < 0) return fail(S2D_ERR_INVALID, "negative pixel count");
    if (!(rgb_error > 0.0) || !(depth_error_frac > 0.0))
        return fail(S2D_ERR_INVALID, "prune thresholds must be positive");  // FusionConfig (mapper.py:59-61)
    if (npx == 0) return S2D_OK;
    if (!color || !depth || !accumulation || !observed_rgb || !observed_depth || !marked)
        return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_prune_mark(color, depth, accumulation, observed_rgb, observed_depth, npx, rgb_error, depth_error_frac,
                      marked, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

int s2d_prune_keep(void *stream, const float *max_marked, int64_t n, double contribution_floor, uint8_t *keep) {
    if (n < 0) return fail(S2D_ERR_INVALID, "negative n");
    if (!(contribution_floor > 0.0)) return fail(S2D_ERR_INVALID, "prune thresholds must be positive");
    if (n == 0) return S2D_OK;
    if (!max_marked || !keep) return fail(S2D_ERR_INVALID, "NULL buffer");
    launch_prune_keep(max_marked, n, contribution_floor, keep, (cudaStream_t)stream);
    S2D_CHECK_LAUNCH();
    return S2D_OK;
}

}  // extern "C"
