/*
 * rcgs.h -- C ABI of the B200 (sm_100a) ReCoGS recolor hot path.
 *
 * The reference (`splattint`, /root/reference/pkg/src/splattint) is a pure
 * Python package with no native seam: its "plugin interface" is the set of
 * module-level functions re-exported by splattint/__init__.py:4-99 and bound
 * by name in the callers (optimize.py:23-28, recolor.py:16-18,
 * session.py:19-48).  Each entry point below is the native half of one of those
 * functions; the Python package `paper_2511_18441_b200` binds them with ctypes
 * and keeps the reference's names, argument meaning and
 * error behaviour.
 *
 * Conventions
 *  - Plain C types only: raw device pointers ("d_" prefix), host pointers
 *    ("h_" prefix), sizes, and a cudaStream_t passed as void*.
 *  - Every call returns an int status (RCGS_OK on success) and never throws;
 *    rcgs_last_error() gives the message of the last failure on this thread.
 *    RCGS_EINVAL maps to splattint.errors.ValidationError (errors.py:16-17),
 *    RCGS_ECUDA to SplattintError (errors.py:4-5).
 *  - Caller-owned: SH coefficients, Adam moments, images, masks, gradients.
 *    Library-owned: opaque scene and per-view handles (stream-ordered device
 *    allocations), released with the matching *_destroy call.
 *  - Images are HWC float32 (H, W, 3) unless stated; SH is (N, 16, 3) float32.
 */
#ifndef RCGS_H
#define RCGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCGS_OK 0
#define RCGS_EINVAL 1      /* precondition violated (ValidationError)            */
#define RCGS_ECUDA 2       /* CUDA runtime failure (SplattintError)              */
#define RCGS_ENOMEM 3      /* device allocation failed (SplattintError)          */

#define RCGS_VERSION 1

typedef struct rcgs_scene rcgs_scene; /* device geometry: fp64 positions, cov3d, opacity */
typedef struct rcgs_view rcgs_view;   /* one camera's preprocessed + binned gaussians     */

/* Pinhole camera + world->camera pose (scene.py:34-75). */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R[9]; /* row-major rotation, x_cam = R x_world + t */
    double t[3];
} rcgs_camera;

/* RasterizerConfig (render.py:54-66). */
typedef struct {
    double near_clip, alpha_clamp, alpha_skip, transmittance_floor;
    double covariance_dilation, footprint_sigmas;
} rcgs_raster_config;

/* OptimizerConfig (optimize.py:33-41), minus the loss weight. */
typedef struct {
    double lr_dc, lr_rest, beta1, beta2, eps;
} rcgs_adam_config;

typedef struct {
    int64_t n_gaussians;  /* N                                               */
    int64_t n_kept;       /* K: survivors of near clip + 3-sigma cull         */
    int64_t n_pairs;      /* (gaussian, tile) pairs after binning              */
    int32_t tiles_x, tiles_y, tile_size;
    int32_t sort_bits;    /* depth-key bits actually radix-sorted              */
} rcgs_view_info;

int rcgs_version(void);
/* Checked builds (-DRCGS_CHECKED): number of device bound-check failures since
 * the last reset; RCGS_EINVAL in release builds. */
int rcgs_debug_violations(uint64_t* h_count, int reset);
/* Checked builds: run one device check that fails when fail != 0 (self-test). */
int rcgs_debug_selftest(int fail);
const char* rcgs_last_error(void);
/* Pre-grow the device's stream-ordered memory pool (used for the per-view and
 * temporary buffers) to `bytes`, so steady-state steps never map new memory. */
int rcgs_pool_reserve(int64_t bytes, void* stream);

/* ---- scene (replaces the geometry half of splattint.Scene, scene.py:126-186) -------- */
/* Copies fp64 positions (N,3), opacities (N,) and derives the view-independent 3D
 * covariance R S S^T R^T (render.py:95-100) from unit quaternions (N,4) and scales
 * (N,3).  All inputs are device pointers; the handle owns its copies. */
int rcgs_scene_create(const double* d_positions, const double* d_rotations,
                      const double* d_scales, const double* d_opacities, int64_t n,
                      int sh_degree, void* stream, rcgs_scene** out);
int rcgs_scene_destroy(rcgs_scene* scene, void* stream);

/* ---- per-view preprocess + tile binning (render.py:172-229 _project_scene) ---------- */
/* K1 fp64 projection + 3-sigma cull, stable depth radix sort of the kept gaussians
 * (bit-exact render.py:216 order), opacity-aware tile footprints, (tile|depth) pair
 * sort and tile ranges.  Synchronises `stream` twice (kept count, pair count). */
int rcgs_view_create(const rcgs_scene* scene, const rcgs_camera* cam,
                     const rcgs_raster_config* cfg, void* stream, rcgs_view** out);
int rcgs_view_info_get(const rcgs_view* view, rcgs_view_info* out);
int rcgs_view_destroy(rcgs_view* view, void* stream);
/* Kept gaussians front to back: scene index (K,) int64 and view-space z (K,) fp64. */
int rcgs_view_kept(const rcgs_view* view, int64_t* d_index, double* d_depth, void* stream);
/* Tile bins: [start, end) into the pair list per 16x16 tile, row-major (tiles_y,
 * tiles_x, 2) uint32 (the reference's per-tile index lists, render.py binning). */
int rcgs_view_ranges(const rcgs_view* view, uint32_t* d_ranges, void* stream);
/* The binned pair list (n_pairs,) uint32: scene indices, sorted by (tile, depth
 * rank); tile t's list is d_pair_g[ranges[t].start, ranges[t].end) -- the
 * reference's global depth order (render.py:216) restricted to the gaussians
 * whose opacity-aware footprint touches the tile (render.py:263-272). */
int rcgs_view_pairs(const rcgs_view* view, uint32_t* d_pair_g, void* stream);
/* Per kept gaussian in depth order, the fp64 operands of every exact decision
 * (K,6): mean2d x, y, conic a, b, c and opacity (render.py:181-223), bit-identical
 * to the reference's numpy values. */
int rcgs_view_exact(const rcgs_view* view, double* d_out, void* stream);

/* SH basis (K,16) fp64 along each kept gaussian's view direction and the channel
 * activation flags (K,3) uint8 from the last rcgs_view_color (ForwardCapture.basis /
 * .active, render.py:88-89).  Either output may be NULL. */
int rcgs_view_basis(const rcgs_view* view, double* d_basis, uint8_t* d_active, void* stream);

/* SH colour of the kept gaussians (render.py:209-214) from SH (N,16,3) fp32;
 * must be called before render/backward whenever SH changed. */
int rcgs_view_color(rcgs_view* view, const float* d_sh, void* stream);

/* ---- rasteriser (render.py:263-334) -------------------------------------------------- */
/* layout 0 = HWC (H,W,3), 1 = CHW (3,H,W); d_t_final (H,W) may be NULL. */
int rcgs_render(const rcgs_view* view, const float* h_background3, int layout,
                float* d_image, float* d_t_final, void* stream);
/* rcgs_render that also keeps the view's composite weights w = alpha * T (they
 * depend on geometry and camera only): rcgs_backward then streams them instead
 * of re-traversing the tile lists, and later renders of the view are an SpMV.
 * Results are bit-identical to the traversal paths.  Reserves up to
 * 8 * pairs * 132 bytes (~2.8 GB at 1080p / 1M gaussians), freed with the view. */
/* Viewer frame (session.py:381-405 render_rgba, protocol.py:29-38 image_to_rgba)
 * in one pass: the view composited with a zero background, where d_overlay (H,W)
 * uint8 != 0 blended (1 - strength) * img + strength * highlight in fp64, then
 * rint(clip(x, 0, 1) * 255) into d_rgba (H,W,4) uint8 with alpha 255 --
 * bit-identical to image_to_rgba(overlay(render)) on the host.  d_overlay may be
 * NULL (no selection). */
int rcgs_render_rgba(const rcgs_view* view, const uint8_t* d_overlay, const double* h_highlight3,
                     double strength, uint8_t* d_rgba, void* stream);
int rcgs_render_train(rcgs_view* view, const float* h_bg3, int layout, float* d_image, float* d_t_final,
                      void* stream);
/* Keep the composite weights recorded by rcgs_render_train resident with the
 * view (a compact copy, ~130 B per record; ~314 MB at 1080p / 1M gaussians)
 * instead of in the shared per-step arena: every later render / backward of the
 * view streams them (views reused across steps, e.g. a refit over a fixed set of
 * training cameras).  Synchronises `stream` once (record count). */
int rcgs_view_keep_records(rcgs_view* view, void* stream);

/* depth_from_gaussians (render.py:373-398): (H,W) fp64, +inf where T never drops
 * below tau at a composited gaussian.  d_cross (H,W) int32 = kept rank or -1, may be NULL. */
int rcgs_depth(const rcgs_view* view, double tau, double* d_depth, int32_t* d_cross,
               void* stream);

/* render_forward contribution lists (render.py:337-370).  Call with d_* = NULL to
 * get the count in *h_count, then again with buffers of that size.  Order:
 * pixel-major, then front to back (identical to the reference's np.nonzero). */
int rcgs_capture(const rcgs_view* view, int64_t* h_count, int64_t* d_pixel, int64_t* d_kept,
                 double* d_weight, void* stream);

/* Instrumentation: while d_counters30 != NULL every raster launch of the process
 * accumulates, at row `mode` (0 render, 1 depth, 2 backward, 3 mask hits, 4/5
 * capture), {evaluated pixel-entry pairs, composited pairs, warp blocks processed,
 * warp blocks skipped, warp-level entry iterations} into the (6, 5) uint64 array;
 * pass NULL to switch off.  Feeds the benchmark's compute roofline (one atomic
 * per warp block, <1% overhead).  The recording forward also fills [25] / [26] with
 * static list statistics: entries passing each 8x4 block's cull, and entries
 * passing each 8x8 region's cull (planning data for a two-pixels-per-lane raster). */
int rcgs_raster_counters(uint64_t* d_counters30);

/* Diagnostics: while d_trace != NULL every raster launch with at most max_items
 * work items (8x4 pixel blocks) overwrites, per item, 8 uint32 {start ns, end ns
 * (globaltimer low word), SM id, warp entry iterations, evaluated pixel-entry
 * pairs, fp64 gate-band alpha evaluations, exact transmittance re-walks, tile};
 * the load-balance probe (tools/raster_trace.py) reads it. */
int rcgs_raster_trace(uint32_t* d_trace, int64_t max_items);

/* Measured FP32 FFMA throughput of this device in FLOP/s (2 per FFMA): the
 * denominator of the rasteriser's compute roofline. */
int rcgs_fp32_peak(int32_t iters, double* h_flops, void* stream);

/* ---- loss + image gradient (losses.py:68-134), fp64 arithmetic ---------------------- */
/* d_loss3 (device, fp64) receives {l1, ssim, total}.  d_grad (H,W,3) fp32 gets
 * d total / d image, exactly zero when image == target (losses.py:127-130).
 * lam == 0 skips SSIM (images may then be smaller than 11 px). */
int rcgs_loss_grad(const float* d_image, const float* d_target, int32_t height, int32_t width,
                   double lam, double* d_loss3, float* d_grad, void* stream);

/* Float64 images and gradient (the host-facing losses API: bit-faithful sign and
 * array_equal semantics on float64 inputs). */
int rcgs_loss_grad_f64(const double* d_image, const double* d_target, int32_t height,
                       int32_t width, double lam, double* d_loss3, double* d_grad, void* stream);

/* ---- SH backward (backward.py:22-40) ------------------------------------------------ */
/* Per-gaussian channel sums acc[i,ch] = active[i,ch] * sum_p g[p,ch] * w_ip over the
 * view's composited contributions, written densely as d_acc (N,3) fp32 (zero for
 * culled gaussians).  Deterministic (no float atomics).  If d_nonfinite != NULL it
 * is OR-ed with 1 when any sum is non-finite. */
int rcgs_backward(const rcgs_view* view, const float* d_grad_image, float* d_acc,
                  int32_t* d_nonfinite, void* stream);

/* Expand a view's acc into the dense (N,16,3) gradient basis_k(dir_i) * acc[i,ch]. */
int rcgs_sh_grad(const rcgs_scene* scene, const float* d_acc, const double* h_center3,
                 float* d_grad, void* stream);

/* ---- Adam (optimize.py:59-83) -------------------------------------------------------- */
/* Fused gradient expansion + Adam over all N x 48 coefficients.  The gradient is
 * (1/G) sum_v basis(dir_{v,i}) (x) acc_v[i] for G views (G == 1 is the reference
 * iteration); d_accs points to G device pointers (host array).  If *d_reject != 0 the
 * update is skipped (non-finite gradient, optimize.py:72-74); otherwise the device
 * step counter *d_step is advanced.  With d_reject_record non-null the flag is
 * consumed for a pipelined caller: 1.0 / 0.0 (rejected or not) is written there
 * and *d_reject is reset to 0 for the next step, on the device. */
int rcgs_adam_fused(const rcgs_scene* scene, float* d_sh, float* d_m, float* d_v,
                    const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                    const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                    double* d_reject_record, void* stream);
/* rcgs_adam_fused + the colour pass of `next_view` (the view the next optimizer
 * step renders, render.py:209-214) evaluated from the updated SH tiles while they
 * are in shared memory: saves the colour kernel's full SH read.  Equivalent to
 * rcgs_adam_fused followed by rcgs_view_color(next_view, d_sh) (bit-identical),
 * including on a rejected step (SH unchanged, view still coloured). */
int rcgs_adam_fused_next(const rcgs_scene* scene, float* d_sh, float* d_m, float* d_v,
                         const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                         const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                         double* d_reject_record, rcgs_view* next_view, void* stream);
/* Snapshot publication (optimize.py:221-238): when the step commits with a step
 * count that is a multiple of `every`, the updated SH tiles are also written to
 * d_snapshot (bulk stores from the same shared-memory tiles, no extra read) and
 * the step count to *d_snapshot_step -- in stream order, exactly the
 * post-step-k scene the reference publishes, with no host round trip. */
typedef struct {
    float* d_snapshot;          /* (N,16,3) fp32 published copy                  */
    int64_t* d_snapshot_step;   /* step count of the published copy (may be NULL) */
    int64_t every;              /* snapshot_every (> 0)                           */
} rcgs_adam_publish;
/* rcgs_adam_fused / rcgs_adam_fused_next (next_view may be NULL) with optional
 * snapshot publication (publish may be NULL) and optional exact tile skipping:
 * d_tile_state (ceil(N/64) uint32, caller-owned, zero-initialised together with
 * m = v = 0; set to all-ones whenever m/v/SH are written from outside) marks the
 * 64-gaussian tiles whose Adam state may be nonzero.  A tile whose state is 0
 * and whose acc is 0 in every view is left untouched -- bit-identical to the
 * dense update, which maps (theta, 0, 0, g = 0) to itself.  NULL = dense. */
int rcgs_adam_fused_ex(const rcgs_scene* scene, float* d_sh, float* d_m, float* d_v,
                       const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                       const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                       double* d_reject_record, rcgs_view* next_view, const rcgs_adam_publish* publish,
                       uint32_t* d_tile_state, void* stream);
/* Dense Adam on an explicit gradient (N,16,3) (adam_step API). */
int rcgs_adam_dense(float* d_params, float* d_m, float* d_v, const float* d_grads, int64_t n,
                    const rcgs_adam_config* cfg, const int32_t* d_reject, int64_t* d_step,
                    void* stream);
/* OR 1 into *d_flag if any of d_x[0..count) is non-finite. */
int rcgs_nonfinite_check(const float* d_x, int64_t count, int32_t* d_flag, void* stream);

/* ---- stereo depth (stereo.py:61-219) ------------------------------------------------------ */
/* match_disparity (stereo.py:142-161): ZNCC block matching of two (H,W,channels)
 * float32/float64 (elem_bytes 4/8, both alike) images (gray = channel mean) with parabolic sub-pixel refinement and
 * the left-right check; transpose != 0 matches along the image columns (the
 * vertical pair, stereo.py:207-209).  Writes the (H,W) float64 disparity, -1 where
 * invalid; bit-identical to the reference for the same images (the box means
 * restate scipy.ndimage.uniform_filter's running sums).  variance_floor_sq is the
 * host's variance_floor ** 2.  Asynchronous on `stream` (workspace from the pool). */
int rcgs_stereo_match(const void* d_left, const void* d_right, int32_t height, int32_t width,
                      int32_t channels_left, int32_t channels_right, int32_t elem_bytes, int32_t transpose, int32_t max_disparity, int32_t window_radius,
                      double variance_floor, double variance_floor_sq, double lr_tolerance, double* d_disparity,
                      void* stream);
/* Diagnostics: count operands t where the matcher's fused division by the window
 * size differs from IEEE t / size (n pseudo-random t over 64 binades); must be 0. */
int rcgs_stereo_div_check(int32_t size, int64_t n, uint64_t seed, int64_t* h_mismatches, void* stream);
/* disparity_to_depth + aggregate_hv (+ estimate_depth's backfill when d_fallback is
 * non-null) over n pixels (stereo.py:164-219): fx_baseline = fx * baseline. */
int rcgs_stereo_depth(const double* d_disp_h, const double* d_disp_v, int64_t n, double fx_baseline,
                      double fy_baseline, double min_disparity, const double* d_fallback, double* d_depth,
                      void* stream);

/* ---- scene checkpoints (scene_io.py:108-153) --------------------------------------------- */
/* Decode n raw float32 PLY vertex rows of row_floats floats (property positions
 * in h_offsets59: x y z, rot_0..3, f_dc_0..2, f_rest_0..44, opacity, scale_0..2)
 * into fp64 positions (N,3), normalised fp64 rotations (N,4) and fp32 SH
 * (N,16,3) (channel-major f_rest transposed), values identical to the reference
 * loader; h_first_bad7 receives the first vertex with a non-finite position /
 * opacity / scale / rotation / f_dc / f_rest and the first zero-norm quaternion
 * (-1 if none).  Synchronises `stream`. */
int rcgs_ply_decode(const float* d_rows, int64_t n, int32_t row_floats, const int32_t* h_offsets59,
                    double* d_pos, double* d_rot, float* d_sh, int64_t* h_first_bad7, void* stream);
/* Write the 48 SH columns of n checkpoint rows (same offsets as rcgs_ply_decode) from
 * the device SH (scene_io.py:156-166): float32(d_base + (d_new - d_old)) in fp64 when
 * d_base (N,16,3 fp64) is given -- the published snapshot's value, optimize.py:226-238 --
 * else d_new.  The other columns of d_rows are left as they are.  Asynchronous. */
int rcgs_ply_encode_sh(const double* d_base, const float* d_old, const float* d_new, int64_t n,
                       int32_t row_floats, const int32_t* h_offsets59, float* d_rows, void* stream);

/* ---- select-from-mask outlier statistics (selection.py:155-181) ---------------------- */
/* knn_mean_distances: per point of the (m,3) fp64 cloud, the mean distance to its
 * k nearest neighbours (self excluded), bit-identical to scipy cKDTree.query(k+1)
 * + numpy mean (unfused squared distances, correctly rounded sqrt, numpy's
 * pairwise summation); exact uniform-grid search.  1 <= k <= 32, m > k.
 * Synchronises `stream` twice (bounding box, cell-size sample). */
int rcgs_knn_mean_distances(const double* d_points, int64_t m, int32_t k, double* d_means, void* stream);

/* ---- selection pass (selection.py:184-235, recolor.py:30-81) ------------------------- */
/* Stamp quad x quad squares of the visible cloud points into d_mask (H,W) uint8
 * (caller zero-fills); visibility z <= depth * (1 + tol), fp64, bit-exact. */
int rcgs_project_cloud(const double* d_points, int64_t m, const rcgs_camera* cam,
                       const double* d_depth, int32_t quad, double tol, uint8_t* d_mask,
                       void* stream);
/* out = mask ? clip(image * tint, 0, 1) : image, for npix HWC pixels. */
int rcgs_apply_recolor(const float* d_image, const uint8_t* d_mask, int64_t npix,
                       const float* h_tint3, float* d_out, void* stream);
/* fp64 variant for host-facing datasets (bit-exact recolor.py:30-39). */
int rcgs_apply_recolor_f64(const double* d_image, const uint8_t* d_mask, int64_t npix,
                           const double* h_tint3, double* d_out, void* stream);
/* Per-gaussian mask statistics of one view, accumulated into the outputs:
 * d_hits[i] += #{masked pixels p with w_ip > 0}; d_wsum[i] += round(2^32 * sum w_ip)
 * (integer, so order-independent and exact across views and ranks). */
int rcgs_mask_hits(const rcgs_view* view, const uint8_t* d_mask, int32_t* d_hits,
                   uint64_t* d_wsum, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RCGS_H */
