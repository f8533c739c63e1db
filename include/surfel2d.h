/*
 * surfel2d.h — C ABI of the B200 2D-Gaussian-surfel render/refine path.
 *
 * Drop-in boundary.  The reference's operator layer is the
 * numba module ``surfelslam._raster_kernels`` imported as ``_k`` by
 * ``surfelslam.rasterizer`` (rasterizer.py:15), driven by ``_render_state``
 * (rasterizer.py:301-331).  Each entry point below names the reference
 * interface it replaces.  Plain C types only: device pointers, sizes, a
 * cudaStream_t passed as void*.  No torch types.
 *
 * Conventions
 *  - Surfel parameters live in ONE packed float32 device block of 13*n floats,
 *    laid out [means 3n | quats 4n (wxyz) | scales 2n | opacities n | colors 3n]
 *    (the reference's SurfelArrays fields, rasterizer.py:71-82, in float32).
 *  - Poses are camera->world packed Sim(3) [s, tx, ty, tz, qw, qx, qy, qz]
 *    (geometry.py:8-11); the library inverts them in float64 exactly like
 *    pk_inverse (geometry.py:188-195).
 *  - Images are row-major (H, W[, 3]) float32; pixel (row y, col x) samples the
 *    image plane at (x, y) (rasterizer.py:27).
 *  - Every call is stream-ordered and asynchronous unless it says otherwise.
 *  - Return value: S2D_OK or an error code; s2d_last_error() gives a
 *    thread-local message.  Degenerate surfels are counted, not errors
 *    (rasterizer.py:244).
 */
#ifndef SURFEL2D_H_
#define SURFEL2D_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2D_OK 0
#define S2D_ERR_INVALID 1 /* bad argument (reference raises ValueError) */
#define S2D_ERR_CUDA 2    /* CUDA runtime error */
#define S2D_ERR_OOM 3     /* device allocation failed */
#define S2D_ERR_STATE 4   /* backward without a matching forward */

#define S2D_LOSS_MSE 0      /* reference render_loss (rasterizer.py:346-357) */
#define S2D_LOSS_L1 1       /* L1 RGB + w_depth * L1 depth (BASELINE configs 2,4,5) */
#define S2D_LOSS_EXTERNAL 2 /* caller supplies dL/d(color, depth, normal, accumulation) */

/* CameraIntrinsics (rasterizer.py:25-46) */
typedef struct s2d_camera {
    double fx, fy, cx, cy;
    int32_t width, height;
} s2d_camera;

/* RasterConfig (rasterizer.py:150-171) */
typedef struct s2d_raster_config {
    double weight_clamp;              /* 0.999 */
    double termination_transmittance; /* 1e-4 */
    double footprint_sigma;           /* 3.0 -> Mahalanobis cut sigma^2 */
    double near_plane;                /* 1e-3 */
    double max_condition;             /* 1e8 */
    double max_view_angle_deg;        /* 80 */
    double center_margin_frac;        /* 0.5 */
    int32_t splat_mode;               /* S2D_SPLAT_AFFINE (the reference) or S2D_SPLAT_RAY */
    int32_t reserved;
} s2d_raster_config;

/* Splat footprint models.  AFFINE is the reference's: the tangent-plane covariance pushed
 * through the projection Jacobian (rasterizer.py:212-225), evaluated as |M^-1 d|^2 with
 * M = J Bc; every parity claim is about this mode.  RAY intersects each pixel's ray with
 * the surfel plane exactly (the 2D-Gaussian-splatting homography: (u, v, 1/z) ~
 * (K [t_u t_v p])^-1 (x, y, 1)), blends the intersection depth, and has no reference
 * counterpart. */
#define S2D_SPLAT_AFFINE 0
#define S2D_SPLAT_RAY 1

/* RenderBuffers (rasterizer.py:174-179) + the new normal channel; NULL = not wanted */
typedef struct s2d_image {
    float *color;        /* (H,W,3) */
    float *depth;        /* (H,W) un-normalised expected depth */
    float *accumulation; /* (H,W) 1 - transmittance */
    float *normal;       /* (H,W,3) alpha-blended camera-frame normal (N1) */
    float *max_w;        /* (H,W) render_with_argmax max weight (rasterizer.py:340-343) */
    int32_t *arg_w;      /* (H,W) input index of max-weight surfel, -1 if none */
} s2d_image;

/* Per-view counters, readable after the stream is synchronised. */
typedef struct s2d_view_stats {
    int32_t visible;     /* V: on-screen surfels (rasterizer.py:318) */
    int32_t pairs;       /* P: (16x16 tile, surfel) pairs */
    int32_t degenerate;  /* RenderBuffers.degenerate_skipped */
    int32_t n_mask;      /* pixels with accumulation > 0.5 */
    int32_t overflow;    /* pair capacity exceeded (view must be re-run; handled internally) */
    int32_t guard_hits;  /* float64 re-checks taken at the 3-sigma cut / weight clamp */
    int32_t pairs_stored; /* min(pairs, capacity) (internal) */
    int32_t blended;     /* E: (pair, 8x4 pixel block) entries with >= 1 blended pixel (backward work) */
} s2d_view_stats;

/* Introspection of the last forward of a view (device pointers; parity tests). */
typedef struct s2d_view_debug {
    const uint32_t *order;      /* (drawn,) input indices in depth order (rasterizer.py:318-320) of the
                                   on-screen surfels whose integer bbox is non-empty */
    const uint32_t *pair_tiles; /* (P,) tile id (low 16 bits; bits 16-23: warp-block cull mask), sorted */
    const uint32_t *pair_ids;   /* (P,) surfel index of each pair: per-tile lists in depth order */
    const int32_t *ranges;      /* (ntiles, 2) [start, end) into the pair arrays */
    const int16_t *bbox;        /* (n, 4) x0, x1, y0, y1 (valid where flags & 4) */
    const double *z;            /* (n,) float64 camera depth (valid where flags & 4) */
    const uint8_t *flags;       /* (n,) bit0 in_front, bit1 valid, bit2 on_screen, bit3 drawn (non-empty bbox) */
    const float *records;       /* (n, 16) splat records */
    const int32_t *pixel_state; /* (H*W, 2) number of blended pairs, float bits of the final T */
    int32_t ntiles, tiles_x;
    int64_t pair_capacity;
    int32_t drawn; /* length of `order` (copied to the host by s2d_view_inspect; synchronous) */
    int32_t reserved;
    const int32_t *stream_lengths; /* (ntiles, 8, 2) blend-stream entries per (tile, 8x4 warp block,
                                      column half): the backward's work list lengths */
    const uint32_t *streams;       /* blend streams, 4 words per entry (surfel, blend lane mask, clamp
                                      lane mask, flags); half h of block w of tile t starts at entry
                                      16 ranges[t].start + (2 w + h) (ranges[t].end - ranges[t].start) */
} s2d_view_debug;

/* Loss definition for the backward pass (seeds fused into the backward kernel) */
typedef struct s2d_loss {
    int32_t kind;          /* S2D_LOSS_* */
    int32_t depth_mask;    /* 1: depth term only over accumulation > 0.5 (reference) */
    double w_rgb;          /* LossWeights.mse for MSE; RGB weight for L1 */
    double w_depth;        /* LossWeights.depth */
    const float *target_rgb;   /* (H,W,3) device */
    const float *target_depth; /* (H,W) device */
    /* S2D_LOSS_EXTERNAL: per-pixel upstream gradients (device, any may be NULL) */
    const float *d_color, *d_depth, *d_normal, *d_accumulation;
} s2d_loss;

typedef struct s2d_adam_config {
    double lr_means, lr_rest; /* 1e-3 / 5e-3 (BASELINE config 4) */
    double beta1, beta2, eps; /* 0.9, 0.999, 1e-8 (torch.optim.Adam) */
    double scale_min;         /* post-step clamp of tangent scales */
} s2d_adam_config;

typedef struct s2d_ctx s2d_ctx;   /* per-device context (module handles) */
typedef struct s2d_view s2d_view; /* per-view workspace + forward state */

/* thread-local message of the last failing call */
const char *s2d_last_error(void);
int32_t s2d_version(void); /* 200: s2d_render_host takes a stream */

int s2d_ctx_create(int32_t device, s2d_ctx **out);
int s2d_ctx_destroy(s2d_ctx *ctx);

/* A view owns its workspace arena (grow-only; no per-call cudaMalloc once sized). */
int s2d_view_create(s2d_ctx *ctx, s2d_view **out);
int s2d_view_destroy(s2d_view *view);
/* device pointer of the view's s2d_view_stats (valid until destroy) */
int s2d_view_stats_device(s2d_view *view, s2d_view_stats **out);
/* host copy of the stats; synchronises the view's last stream */
int s2d_view_stats_host(s2d_view *view, s2d_view_stats *out);

/* acc_device (device s2d_view_stats) <- combine with this view's stats, stream-ordered:
 * visible/pairs/pairs_stored = max, degenerate/n_mask/guard_hits = sum, overflow = or.
 * Lets a multi-view step check capacity once per iteration instead of per view. */
int s2d_view_stats_accumulate(s2d_view *view, void *stream, s2d_view_stats *acc_device);
/* set the (tile, surfel) pair capacity used by the next forward (>= 1024); after
 * stats.overflow the caller re-runs the view with a larger capacity */
int s2d_view_reserve_pairs(s2d_view *view, int64_t pairs);
/* Layout of the packed parameter and gradient blocks the view's s2d_forward / s2d_backward read
 * and write: W = ceil(n / c) shards of c = shard_surfels surfels, shard s holding surfels
 * [s c, (s + 1) c) as [means 3c | quats 4c | scales 2c | opacities c | colors 3c] (13 W c floats).
 * 0 or c >= n is the plain layout of the header comment.  With the optimizer sharded over W
 * ranks (c = ceil(n / W)) each rank's slice is contiguous: one reduce-scatter of the gradient
 * block and one in-place all-gather of the parameters (replaces the sum at mapper.py:300-307). */
int s2d_view_set_layout(s2d_view *view, int64_t shard_surfels);
int s2d_view_inspect(s2d_view *view, s2d_view_debug *out);

/* Number of kernels this library has launched in this process (all devices). */
int64_t s2d_launch_count(void);

/* Phase timing: when enabled, s2d_forward/s2d_backward record CUDA events between
 * their kernels on the launching stream; s2d_view_timing synchronises and returns
 * the accumulated milliseconds per phase since the last reset:
 *  [0] project  [1] depth sort (hist, 4 passes, tie fix)  [2] scan+emit, tile sort, ranges
 *  [3] raster forward  [4] raster backward  [5] projection backward
 * and the number of timed forwards in out[6], backwards in out[7]. */
int s2d_view_set_timing(s2d_view *view, int32_t enable);
int s2d_view_timing(s2d_view *view, double out[8], int32_t reset);

/* float64 pose inverse exactly as pk_inverse (geometry.py:188-195); out[8] */
int s2d_pose_inverse(const double pose_c2w[8], double out[8]);

/*
 * Forward render of n surfels (packed float32 params, device) from one view.
 * Replaces _render_state + _k.blend_forward (rasterizer.py:301-331,
 * _raster_kernels.py:22-55): projection, depth order, tile binning, blend.
 * Keeps the sorted tile lists and per-pixel state in `view` for s2d_backward.
 * Optional per_surfel_max (max_all, max_marked; (n,) float, device, zeroed by
 * the caller) + pixel mask (H,W) uint8 replace _k.max_blend_weights
 * (_raster_kernels.py:116-147) when non-NULL.
 */
int s2d_forward(s2d_view *view, void *stream, const float *params, int64_t n,
                const double pose_c2w[8], const s2d_camera *cam, const s2d_raster_config *cfg,
                const s2d_image *out, float *max_all, float *max_marked, const uint8_t *mask);

/*
 * Backward of the last s2d_forward of `view`: loss seeds, reverse-order blend
 * backward, projection backward.  Replaces rasterizer.grad_color_opacity
 * (rasterizer.py:360-399, _k.blend_gradients _raster_kernels.py:58-113) and
 * adds the geometry gradients.  ACCUMULATES (+=, atomically) into grads
 * (packed 13*n float32, device), so summing views needs no extra pass
 * (mapper.py:300-307) and views in flight on several streams, each with its
 * own s2d_view, may share one gradient block.
 * loss_accum (device double, nullable) receives += the view's loss value.
 * `image` must be the forward's outputs (color/depth/accumulation/normal as
 * the loss needs them).
 */
int s2d_backward(s2d_view *view, void *stream, const float *params, int64_t n,
                 const s2d_image *image, const s2d_loss *loss, float *grads, double *loss_accum);

/*
 * s2d_forward + s2d_backward in one call for the losses that need no whole-image
 * reduction before their seeds: L1 without the depth mask, and MSE with w_depth = 0
 * (rasterizer.py:360-380).  The compositing and the reverse traversal run in one kernel, each
 * warp back-propagating its pixel block right after rendering it (no image round trip).
 * `out` (nullable) receives color / depth / accumulation where those fields are non-NULL
 * (normal / max_w / arg_w are not rendered on this path); `wait_event`
 * (cudaEvent_t, nullable) is waited for before the loss targets are read, e.g. their
 * upload.  Any other loss falls back to s2d_forward + s2d_backward with `out`, which must
 * then be complete.  ACCUMULATES into grads like s2d_backward.  The view's forward state is
 * consumed: run s2d_forward again before an s2d_backward.  On the one-kernel path the view's
 * stats.n_mask is the float32 count of accumulation > 0.5 (no loss on that path reads it; the
 * depth-mask losses re-decide it in float64, as s2d_backward does).
 */
int s2d_forward_backward(s2d_view *view, void *stream, const float *params, int64_t n,
                         const double pose_c2w[8], const s2d_camera *cam, const s2d_raster_config *cfg,
                         const s2d_image *out, const s2d_loss *loss, float *grads, double *loss_accum,
                         void *wait_event);

/*
 * Fused Adam step + post-step projection on the packed parameter block
 * (replaces the GD update of mapper.py:330-335; D5): m1, m2 are packed 13*n
 * moments.  step is 1-based.  mask (n uint8, nullable) restricts the update
 * to targeted surfels (mapper.py:286,324-325).
 */
int s2d_adam_step(void *stream, float *params, const float *grads, float *m1, float *m2, int64_t n,
                  int64_t step, const s2d_adam_config *cfg, const uint8_t *mask);
/* The same step, skipped on the device when *skip != 0 (device int32, nullable; e.g. the
 * overflow word of an s2d_view_stats accumulated over the iteration's views): a refine
 * iteration can be queued without a host round trip and re-run if a view overflowed. */
int s2d_adam_step_gated(void *stream, float *params, const float *grads, float *m1, float *m2, int64_t n,
                        int64_t step, const s2d_adam_config *cfg, const uint8_t *mask, const int32_t *skip);

/*
 * mapper.refine's backtracking trial (mapper.py:319-335) on the packed block's opacity +
 * colour part (the contiguous floats [9n, 13n)): params = clip(params0 - step * grads, 0, 1),
 * grads taken as 0 outside `mask` (n uint8, nullable; mapper.py:320-321).  Every surfel is
 * clipped, like the reference's np.clip over the whole arrays.  Stream-ordered.
 */
int s2d_refine_gd(void *stream, float *params, const float *params0, const float *grads, int64_t n, double step,
                  const uint8_t *mask);
/* *out (device float) <- max |grads| over the masked surfels' opacity + colour gradients, the
 * L-inf norm of mapper.py:322.  Stream-ordered. */
int s2d_refine_gnorm(void *stream, const float *grads, int64_t n, const uint8_t *mask, float *out);

/*
 * Host-buffer entry point for non-Python callers: float64 numpy-layout
 * SurfelArrays fields in, float64 RenderBuffers out (what rasterizer.render
 * returns, rasterizer.py:334-337; replaces _render_state + _k.blend_forward,
 * rasterizer.py:301-331), host<->device copies inside through a pinned staging
 * buffer the view keeps (grow-only).  Runs on `stream` (NULL: the legacy default
 * stream) and returns after synchronising it.  Output pointers may be NULL.
 */
int s2d_render_host(s2d_view *view, void *stream, const double *means, const double *quats,
                    const double *scales, const double *opacities, const double *colors, int64_t n,
                    const double pose_c2w[8], const s2d_camera *cam, const s2d_raster_config *cfg,
                    double *color, double *depth, double *accumulation, double *normal,
                    int32_t *degenerate_skipped);

/* ---- map maintenance around the render path ---- */

/*
 * transform_surfels (mapper.py:184-197): params_out = Sim(3) `pose` applied to the packed
 * block params_in (n surfels, device; may not alias): means by pk_act (geometry.py:198-199),
 * rotations left-composed and canonicalised (geometry.py:39-50, 71-84), scales times the
 * pose scale, opacity/colour copied.  float64 arithmetic in the reference's order, rounded
 * to float32 once.
 */
int s2d_transform_surfels(void *stream, const double pose[8], const float *params_in, int64_t n,
                          float *params_out);

/*
 * fuse's accumulation gate (mapper.py:212-224): keep[i] = 1 when candidate i (camera-frame
 * packed block, device) falls outside the image or its own pixel round(f x / z + c) of the
 * map's rendered accumulation (H, W) is below accum_threshold.
 */
int s2d_fuse_gate(void *stream, const float *accumulation, const s2d_camera *cam, const float *params,
                  int64_t n, double accum_threshold, uint8_t *keep);

/*
 * prune's error mask (mapper.py:246-253) over npx pixels: marked = accumulation > 0.5 and
 * (max_c |color - observed_rgb| > rgb_error or (observed_depth > 0 and
 * |depth / max(accumulation, 1e-12) - observed_depth| > depth_error_frac * observed_depth)).
 */
int s2d_prune_mark(void *stream, const float *color, const float *depth, const float *accumulation,
                   const float *observed_rgb, const float *observed_depth, int64_t npx, double rgb_error,
                   double depth_error_frac, uint8_t *marked);

/* prune's victim test (mapper.py:255-256): keep[i] = !(max_marked[i] > contribution_floor). */
int s2d_prune_keep(void *stream, const float *max_marked, int64_t n, double contribution_floor,
                   uint8_t *keep);

#ifdef __cplusplus
}
#endif
#endif /* SURFEL2D_H_ */
