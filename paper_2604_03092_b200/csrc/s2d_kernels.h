// s2d_kernels.h — host-callable launchers for the device kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/surfel2d.h"
#include "s2d_device.cuh"

namespace s2d {

extern std::atomic<int64_t> g_launches;
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

constexpr int kSortThreads = 256;
#ifndef S2D_SORT_ITEMS
#define S2D_SORT_ITEMS 16
#endif
constexpr int kSortItems = S2D_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;  // keys per onesweep CTA
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
#ifndef S2D_PROJ_THREADS
#define S2D_PROJ_THREADS 128
#endif
constexpr int kProjThreads = S2D_PROJ_THREADS;  // surfels per projection CTA (one per thread)
constexpr int kCompactTiles = 32;                // projection tiles per k_compact_hist CTA
#ifndef S2D_EMIT_ITEMS
#define S2D_EMIT_ITEMS 4
#endif
constexpr int kEmitItems = S2D_EMIT_ITEMS;
constexpr int kEmitTile = 256 * kEmitItems;
#ifndef S2D_EMIT_STAGE
#define S2D_EMIT_STAGE 4096
#endif
constexpr int kEmitStage = S2D_EMIT_STAGE;  // pairs a scan/emit CTA stages in shared memory (8 B each)

// Zeroed-per-view scratch ("sync region"): look-back status words, tickets,
// radix histograms, tile ranges, stats.  One memset per view.
struct SyncRegion {
    s2d_view_stats *stats;     // device stats (first, 32 B)
    int *tickets;              // [16]
    int *n_drawn;              // on-screen surfels with a non-empty integer bbox (the sorted set)
    uint32_t *key_range;       // [2]: ~min, max depth key
    uint32_t *depth_hist;      // [3 * kRadix]
    uint32_t *depth_status;    // [3][ceil(n / kSortTile) * kRadix]
    uint32_t *emit_status;     // [ceil(n / kEmitTile)]
    uint32_t *pair_hist;       // [2 * kRadix]
    uint32_t *pair_status;     // [2][ceil(pcap / kSortTile) * kRadix]
    int *amb_count;            // pixels listed for k_mask_fixup
    uint32_t *ccount;          // [ceil(n / kProjThreads / kCompactTiles)] drawn surfels per chunk
    uint32_t *tie_ctl;         // [3]: long-run count, inversion-in-a-long-run flag, CTA ticket (k_tie_fix)
    int2 *ranges;              // [ntiles]
    size_t bytes;
};

struct ProjectArgs {
    ViewParams P;
    const float *params;
    SplatRecord *rec;
    ExactRec *exact;
    AccurateRec *acc;
    short4 *rect;
    double *z64;
    uint8_t *flags;
    uint32_t *keys;       // [n]: tile t's drawn (key, index) pairs at [t kProjThreads, + tcount[t])
    uint32_t *vals;
    uint32_t *tcount;     // [ceil(n / kProjThreads)] drawn surfels per projection tile
    uint32_t *ccount;     // [ceil(n / kProjThreads / kCompactTiles)] drawn per chunk (sync region, zeroed)
    s2d_view_stats *stats;
    uint32_t *key_range;  // [~min, max] of on-screen depth keys (sync region, zeroed)
};
void launch_project(const ProjectArgs &a, cudaStream_t s);

// order-preserving concatenation of k_project's per-tile pairs, key rebase, digit histograms
void launch_compact_hist(const uint32_t *skeys, const uint32_t *svals, const uint32_t *tcount,
                         const uint32_t *ccount, int64_t n, const uint32_t *key_range, uint32_t *keys,
                         uint32_t *vals, uint32_t *hist, int *n_drawn, cudaStream_t s);
// one stable 8-bit LSD pass over the *d_n entries (cap: capacity the grid is sized for)
void launch_onesweep(const uint32_t *kin, const uint32_t *vin, uint32_t *kout, uint32_t *vout,
                     const int *d_n, int cap, int shift, const uint32_t *hist_pass,
                     uint32_t *status, int *ticket, cudaStream_t s);
// ctl: 3 zeroed words; list: >= cap / 64 + 1 words; scratch: cap words (may not alias keys / vals)
void launch_tie_fix(const uint32_t *keys, uint32_t *vals, const double *z64, const int *d_n, int cap,
                    uint32_t *ctl, uint32_t *list, uint32_t *scratch, cudaStream_t s);

struct EmitArgs {
    const uint32_t *order;
    const short4 *rect;
    const int *d_v;
    int cap_v;
    int ntx;
    int pair_passes;
    uint32_t *pkeys;
    uint32_t *pvals;
    uint32_t pcap;
    s2d_view_stats *stats;
    uint32_t *status;
    int *ticket;
    uint32_t *pair_hist;
};
void launch_scan_emit(const EmitArgs &a, cudaStream_t s);
void launch_tile_ranges(const uint32_t *pkeys, const int *d_p, uint32_t pcap, int2 *ranges,
                        cudaStream_t s);

struct RasterArgs {
    ViewParams P;
    const float *params;
    const int2 *ranges;
    const uint32_t *pair_ids;
    uint32_t *pair_keys;  // tile | bbox warp-block mask << 16
    // Forward -> backward work lists: warp w of tile t appends, in list order, one (surfel id,
    // lane mask of the block's pixels that blended it, lane mask of those whose weight was
    // clamped, 0) entry per pair its pixels blended, at
    // bstream[16 ranges[t].x + (2 w + h) (ranges[t].y - ranges[t].x) ...]: the stream of column
    // half h of warp w's block; bcount[16 t + 2 w + h] = its entries.
    uint4 *bstream;
    int *bcount;
    const SplatRecord *rec;
    const ExactRec *exact;
    const AccurateRec *acc;
    const short4 *rect;
    int2 *aux;  // per pixel (last list position, float bits of T before it)
    // forward outputs (forward writes, backward reads)
    float *color, *depth, *accum, *normal, *max_w;
    int32_t *arg_w;
    float *max_all, *max_marked;
    const uint8_t *mask;
    s2d_view_stats *stats;
    // backward
    int loss_kind, depth_mask;
    double w_rgb, w_depth;
    const float *target_rgb, *target_depth;
    const float *d_color, *d_depth, *d_normal, *d_accum;
    float *grad2d;  // [n][16] per-view 2D gradients, rows of g2_stride(ray, ext) floats (raster.cu)
    double *loss_accum;
    // pixels whose float32 depth-mask decision is within the error band (k_mask_fixup)
    int *amb_count;  // sync region (zeroed per view)
    int *amb_list;   // [H*W]
};
void launch_raster_forward(const RasterArgs &a, cudaStream_t s);
void launch_raster_backward(const RasterArgs &a, cudaStream_t s);
// forward + loss seeds + backward traversal in one kernel (colour/depth losses without the
// whole-image depth mask); needs a.target_rgb / a.target_depth / a.grad2d
void launch_raster_fused(const RasterArgs &a, cudaStream_t s);
// float64 re-decision of the ambiguous depth-mask pixels (before a masked loss's backward)
void launch_mask_fixup(const RasterArgs &a, cudaStream_t s);

struct ProjectBwdArgs {
    ViewParams P;
    const float *params;
    const uint8_t *flags;
    const short4 *rect;  // per-surfel bbox (ray mode: reference corner of the 2D gradients)
    float *grad2d;
    float *grads;
    int g2_stride;  // floats per surfel in grad2d, as the raster backward wrote them (g2_stride())
};
// Floats per surfel of the 2D-gradient rows: the affine mode's 10 values (+ 3 normal values
// with external normal / accumulation seeds, 13 in ray mode, 16 with both) in rows of 12 or 16.
constexpr int g2_stride(bool ray, bool ext) { return (ray || ext) ? 16 : 12; }
void launch_project_backward(const ProjectBwdArgs &a, cudaStream_t s);

// skip (device, nullable): the step is a no-op when *skip != 0 (a view of it overflowed)
void launch_adam(float *params, const float *grads, float *m1, float *m2, int64_t n, int64_t step,
                 const s2d_adam_config &cfg, const uint8_t *mask, const int32_t *skip, cudaStream_t s);

// mapper.refine's backtracking GD step and gradient norm on the opacity + colour block (optim.cu)
void launch_refine_gd(float *x, const float *x0, const float *g, int64_t n, double step, const uint8_t *mask,
                      cudaStream_t s);
void launch_refine_gnorm(const float *g, int64_t n, const uint8_t *mask, float *out, cudaStream_t s);

// map maintenance (map.cu)
void launch_transform(const float *in, float *out, int64_t n, const double pose[8], cudaStream_t s);
void launch_fuse_gate(const float *acc, const s2d_camera &cam, const float *params, int64_t n, double thr,
                      uint8_t *keep, cudaStream_t s);
void launch_prune_mark(const float *color, const float *depth, const float *acc, const float *orgb,
                       const float *odep, int64_t npx, double rgb_err, double depth_frac, uint8_t *marked,
                       cudaStream_t s);
void launch_prune_keep(const float *max_marked, int64_t n, double floor_, uint8_t *keep, cudaStream_t s);

// number of 8-bit digit passes needed for keys < 2^bits
inline int passes_for_bits(int bits) { return bits <= 0 ? 1 : (bits + kRadixBits - 1) / kRadixBits; }

}  // namespace s2d
