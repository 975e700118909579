/*
 * gsx.h -- C ABI of the B200-native RayGaussX render path (libgsx.so).
 *
 * The reference (`gsray`, pure Python) has no FFI; its drop-in boundary is the
 * Python API re-exported by /root/reference/pkg/src/gsray/__init__.py:6-52.
 * Each entry point below replaces one reference function (cited), and the
 * Python host package `paper_2509_07782_b200` binds them with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every device buffer (inputs, outputs and
 *    the opaque arenas / workspaces) is allocated and owned by the caller; the
 *    library keeps no global mutable state and never allocates device memory.
 *    Size queries (`*_bytes`) come first.
 *  - All calls are stream-ordered on `stream` (a cudaStream_t; 0 = legacy
 *    default stream) and reentrant.  Host structs passed by pointer are read
 *    at call time.
 *  - Errors are integer status codes, never exceptions across the ABI.  The
 *    Python side maps them to the reference exception types
 *    (errors.py:4-41).  Data-dependent errors (validation, overflow) are
 *    reported through a caller-provided device status word that the host
 *    reads after the stream synchronizes.
 *  - Record layout (scene_io.py:26-44): 87 float32 per primitive,
 *      mean[0:3] quat(w,x,y,z)[3:7] scales[7:10] sigma~[10] sh 9x3 [11:38]
 *      sg_axis 7x3 [38:59] sg_sharp 7 [59:66] sg_amp 7x3 [66:87].
 *    Gradients use the same layout and storage order.
 */
#ifndef GSX_H
#define GSX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSX_FLOATS_PER_RECORD 87
#define GSX_ABI_VERSION 3

typedef enum {
  GSX_OK = 0,
  GSX_ERR_EMPTY = 1,      /* EmptyScene (errors.py:13-14, scene.py:31-32) */
  GSX_ERR_VALIDATION = 2, /* ValidationError(record) (errors.py:34-41, scene.py:37-41) */
  GSX_ERR_OVERFLOW = 3,   /* BufferOverflow(count, capacity) (errors.py:17-23) */
  GSX_ERR_ARG = 4,        /* ValueError: bad argument / config (renderer.py:41-49) */
  GSX_ERR_CUDA = 5,       /* CUDA launch / runtime failure */
  GSX_ERR_STACK = 6       /* traversal stack exhausted (tree deeper than supported) */
} gsx_status;

/* RenderConfig, field for field (renderer.py:27-39). */
typedef struct {
  double dt;
  int64_t n_s;
  double t_eps;
  int64_t mode; /* 0 = "uniform", 1 = "adaptive" */
  double beta;
  double dt_min;
  double dt_max;
  int64_t ess;
  int64_t tile_size;       /* accepted; pixels are tile-size invariant (renderer.py:399-401) */
  double background[3];
  int64_t buffer_capacity; /* accepted; overflow splitting is bitwise neutral (renderer.py:361-371) */
  /* extension (no RenderConfig counterpart): warp traversal of camera
     renders, 0 = by focal length (packet cone for focal >= 1024 px), 1 =
     packet cone, 2 = per-lane packet.  Pixels do not depend on it. */
  int64_t traversal;
  /* extension: per-sample sums of the screened camera forward (with a
     workspace), 0 = shared memory (16 warps / SM, no spills), 1 = registers
     (32 warps / SM).  Pixels do not depend on it; which is faster depends on
     the device's memory latency (renderer.autotune picks per workload). */
  int64_t sums;
  /* extension: pass 2 of gsx_render_backward_logged, 0 = by the log's mean
     lanes per entry, 1 = compacted (lane, primitive) pairs, 2 = all lanes per
     entry.  Gradients agree to fp32 summation order. */
  int64_t pass2;
} gsx_render_cfg;

/* Camera (renderer.py:109-145): camera-to-world rotation R (row-major, from the
   normalized scalar-first quaternion), centre, focal length in pixels. */
typedef struct {
  double R[9];
  double center[3];
  double focal;
  int64_t width;
  int64_t height;
  double t_near;
  double t_far;
} gsx_camera;

/* RenderStats counters (renderer.py:69-78 order) + two algorithmic-work
   counters for the roofline: pairs = sum over composited
   segments of (#samples x #AABB candidates), i.e. the reference's density
   evaluations; composited = samples with sigma > 0. */
typedef struct {
  uint64_t rays, samples, segments, segments_skipped, closest_hit_calls, node_visits,
      aabb_hits, ellipsoid_hits, pairs, composited;
} gsx_stats;

/* FP32 issue-rate calibration: a dependent-FFMA loop over the whole device.
   Writes sink (one float per thread, grid*block) and returns flops through
   *flops.  Used by bench.py to measure the FP32 roofline denominator. */
int gsx_calibrate_fp32(int64_t iters, float* sink, double* flops, void* stream);
/* SFU issue-rate calibration: 8 independent MUFU.EX2 chains per thread over
   the whole device; *ops = exponentials executed.  The SFU roofline
   denominator of bench.py. */
int gsx_calibrate_sfu(int64_t iters, float* sink, double* ops, void* stream);

/* Device status word written by kernels: {status, record/count, capacity, pad}. */
typedef struct {
  int64_t code;
  int64_t index;
  int64_t count;
  int64_t capacity;
} gsx_dev_status;

const char* gsx_status_string(int status);
int gsx_abi_version(void);
/* CUDA error string of the last failing call on this thread ("" if none). */
const char* gsx_last_cuda_error(void);

/* ---- scene arena ------------------------------------------------------------
 * Replaces Scene._rebuild (scene.py:48-69) + GaussianShape/AppearanceCoeffs
 * ingestion (geometry.py:77-87, appearance.py:62-76).  The arena holds, for N
 * primitives in storage order: fp64 AABBs + fp64 iso_inv (parity queries),
 * fp32 render SoA (mean/sigma, iso_inv rows, log2-scaled k), fp32 outward-rounded
 * AABBs and the 76-float appearance block, plus the fp64 scene bounds.       */
size_t gsx_scene_arena_bytes(int64_t n);

/* params: [n,87] f32 device.  Validates every record (sigma~ > sigma_eps,
 * nonzero quaternion / SG axes, sharpness >= 0) into *dev_status, computes the
 * derived arrays and the fp64 scene bounds (bounds are also copied to
 * host_bounds[6] = lo xyz, hi xyz after a stream synchronize when non-NULL). */
int gsx_prepare(const float* params, int64_t n, double sigma_eps, void* arena,
                gsx_dev_status* dev_status, double* host_bounds, void* stream);

/* Copy derived per-primitive arrays out (testing / host mirrors).
 * which: 0 aabb_lo f64[n,3], 1 aabb_hi f64[n,3], 2 iso_inv f64[n,9],
 *        3 log_ratio f64[n], 4 bounds f64[6]. */
int gsx_scene_get(const void* arena, int64_t n, int which, void* out_device, void* stream);

/* ---- Morton reorder (spatial.py:81-92, scene.py:97-105) ------------------ */
/* codes[i] = morton_encode(quantize_points(means[i], lo, hi)), fp64 exact. */
int gsx_morton_codes(const double* means, int64_t n, const double* lo3, const double* hi3,
                     uint64_t* codes, void* stream);
/* Same, reading means straight from the [n,87] f32 records. */
int gsx_morton_codes_records(const float* params, int64_t n, const double* lo3,
                             const double* hi3, uint64_t* codes, void* stream);
/* morton_encode of integer coordinates (spatial.py:48-64); out of range -> dev_status ARG. */
int gsx_morton_encode(const int64_t* q, int64_t n, uint64_t* codes, gsx_dev_status* dev_status,
                      void* stream);
int gsx_morton_decode(const uint64_t* codes, int64_t n, int64_t* q, void* stream);

/* Stable LSD radix sort of 64-bit keys (np.argsort(kind="stable"), spatial.py:92).
 * perm_out[p] = original index stored at p; keys_out sorted. */
size_t gsx_sort_workspace_bytes(int64_t n);
int gsx_sort_codes(const uint64_t* keys_in, int64_t n, uint64_t* keys_out, int64_t* perm_out,
                   void* workspace, void* stream);

/* apply_permutation (scene.py:74-80): out[p,:] = params[perm[p],:];
 * uids_out[p] = uids_in[perm[p]] (either uid pointer may be NULL). */
int gsx_permute(const float* params, const int64_t* uids_in, const int64_t* perm, int64_t n,
                float* params_out, int64_t* uids_out, void* stream);

/* ---- LBVH (replaces Bvh spatial.py:126-211) ------------------------------
 * Karras LBVH over the primitives sorted by Morton code: sorted_codes[k] is
 * the code of primitive perm[k] (perm NULL = identity, i.e. storage already
 * in Morton order after reorder_by_morton), with a bottom-up refit of fp32
 * outward-rounded boxes.  Child boxes live in the parent node (64 B per
 * internal node); leaves reference storage indices. */
size_t gsx_bvh_arena_bytes(int64_t n);
size_t gsx_bvh_workspace_bytes(int64_t n);
int gsx_bvh_build(const void* scene_arena, const uint64_t* sorted_codes, const int64_t* perm,
                  int64_t n, void* bvh_arena, void* workspace, void* stream);
/* export for tests: node child boxes f32 [n-1, 2, 2, 3], children i32 [n-1, 2]
 * (>= 0 internal node, < 0 leaf ~prim), parent i32 [2n-1]. */
/* Rebuild the 4-wide nodes of bvh_arena from its binary nodes (for a binary
 * tree written by another builder: root = node 0, children in .w, leaves
 * ~index); workspace as for gsx_bvh_build. */
int gsx_bvh_collapse(void* bvh_arena, int64_t n, void* workspace, void* stream);
int gsx_bvh_export(const void* bvh_arena, int64_t n, float* boxes, int32_t* children,
                   int32_t* parents, void* stream);

/* ---- parity queries (fp64 exact) ------------------------------------------
 * queries: [m,8] f64 (o xyz, d xyz, t0, t1) device.
 * collect: Bvh.segment_overlaps (spatial.py:215-247) -- the exact candidate
 * SET (ascending storage index) of every primitive whose AABB slab interval
 * overlaps [t0,t1]; counts[m] always written, idx[m,capacity] filled up to
 * capacity, overflowing queries flagged in *dev_status (first one).
 * closest: closest_hit (spatial.py:309-354); t_out[m] (NaN = None). */
int gsx_collect_segments(const void* scene_arena, const void* bvh_arena, int64_t n,
                         const double* queries, int64_t m, int64_t capacity, int64_t* counts,
                         int64_t* idx, gsx_dev_status* dev_status, void* stream);
int gsx_closest_hit(const void* scene_arena, const void* bvh_arena, int64_t n,
                    const double* queries, int64_t m, double* t_out, void* stream);

/* ---- forward render (render_image renderer.py:396-437 / march_ray :263-285)
 * Camera variant: renders the 16x16 tiles at tile-sequence positions
 * tile_begin + k*tile_stride (k = 0,1,...) of the image (multi-GPU: rank r of
 * G uses tile_begin=r, tile_stride=G).  The sequence is row-major for
 * tile_stride 1 and visits the tile rows centre-out for tile_stride > 1
 * (gsx_tile_at in csrc/gsx_common.cuh); every rank set is a partition.  rgb [H,W,3] f32, depth [H,W] f32 (sum_j w_j t_j),
 * trans [H,W] f32 (exp(-optical depth)); pixels outside the tile set are not
 * written.  stats (device gsx_stats) may be NULL.
 * Rays variant: rays [m,8] f64 (o, d, t_near, t_far); clip != 0 applies
 * clip_ray_to_scene (renderer.py:160-175) first; outputs rgb [m,3], depth [m],
 * trans [m].
 * ws (nullable, ws_bytes >= gsx_render_workspace_bytes(n)) is a caller-owned
 * per-call workspace: with it the camera forward first computes every
 * primitive's image-space silhouette for this camera and screens the warp
 * candidate lists with it (pixels unchanged, fewer per-lane setups).  Two
 * concurrent renders need two workspaces.
 * dev_status (nullable): GSX_ERR_STACK if a traversal stack overflowed (the
 * frame is then incomplete). */
size_t gsx_render_workspace_bytes(int64_t n);
/* Row-major tile id at tile-sequence position s of a camera launch with
 * tile_stride `stride` over a tiles_x x tiles_y grid of 16x16 tiles (the
 * order gsx_render_forward / _logged / backward use; -1 if out of range).
 * Host-only: hosts that shard or gather frames query it instead of copying
 * the order. */
int64_t gsx_tile_id(int64_t s, int64_t tiles_x, int64_t tiles_y, int64_t stride);
int gsx_render_forward(const void* scene_arena, const void* bvh_arena, int64_t n,
                       const gsx_camera* cam, const gsx_render_cfg* cfg, int64_t tile_begin,
                       int64_t tile_stride, float* rgb, float* depth, float* trans,
                       gsx_stats* stats, void* ws, int64_t ws_bytes, gsx_dev_status* dev_status,
                       void* stream);
int gsx_render_rays(const void* scene_arena, const void* bvh_arena, int64_t n,
                    const double* rays, int64_t m, int clip, const gsx_render_cfg* cfg,
                    float* rgb, float* depth, float* trans, gsx_stats* stats,
                    gsx_dev_status* dev_status, void* stream);

/* ---- dense oracles (renderer.py:440-493, appearance.py:107-134), float64 ----
 * gsx_reference_rays: reference_integrate per ray (clip = 0: the ray's own
 * [t_near, t_far]) or reference_render's clip_ray_to_scene + integrate per
 * pixel ray (clip = 1; a miss gives the background): midpoint quadrature at
 * fine_dt against every primitive -- no BVH, no skipping, no termination --
 * composited as renderer.py:472-480.  rays [m,8] f64 (o, d, t_near, t_far),
 * background[3], rgb [m,3] f64.  params = the [N,87] f32 records the arena
 * was prepared from.
 * gsx_eval_fields: mixture density sigma [m] and density-weighted radiance
 * color [m,3] (f64) at points [m,3] for directions dirs [m,3], over every
 * primitive or the storage indices active [n_active] (an out-of-range index:
 * GSX_ERR_ARG in dev_status).  Zero density gives black. */
int gsx_reference_rays(const void* scene_arena, const float* params, int64_t n,
                       const double* rays, int64_t m, int clip, double fine_dt,
                       const double* background, double* rgb, void* stream);
int gsx_eval_fields(const void* scene_arena, const float* params, int64_t n,
                    const double* points, const double* dirs, int64_t m,
                    const int64_t* active, int64_t n_active, double* sigma, double* color,
                    gsx_dev_status* dev_status, void* stream);

/* Per-ray RenderStats: per_ray [m,10] u64 = (ray?, samples, segments,
 * segments_skipped, closest_hit_calls, node_visits, aabb_hits, ellipsoid_hits,
 * pairs, composited) of each ray (bench.false_positive_fraction
 * bench.py:181-198 needs them per ray); outputs as gsx_render_rays. */
int gsx_render_rays_stats(const void* scene_arena, const void* bvh_arena, int64_t n,
                          const double* rays, int64_t m, int clip, const gsx_render_cfg* cfg,
                          float* rgb, float* depth, float* trans, uint64_t* per_ray,
                          gsx_dev_status* dev_status, void* stream);

/* ---- backward (no reference counterpart: SURVEY.md Appendix C) -------------
 * Replays the forward march of the same tiles, and accumulates (atomically,
 * with warp-shuffle pre-reduction) dL/dparams into grad [n,87] f32 in record
 * layout / storage order.  rgb/depth/trans are the forward outputs;
 * dL_drgb [H,W,3], dL_ddepth [H,W], dL_dtrans [H,W] (either of the last two
 * may be NULL = zero). */
int gsx_render_backward(const void* scene_arena, const void* bvh_arena, const float* params,
                        int64_t n, const gsx_camera* cam, const gsx_render_cfg* cfg,
                        int64_t tile_begin, int64_t tile_stride, const float* rgb,
                        const float* depth, const float* trans, const float* dL_drgb,
                        const float* dL_ddepth, const float* dL_dtrans, float* grad,
                        gsx_dev_status* dev_status, void* stream);

/* ---- march log (training; no reference counterpart) --------------------------
 * A training forward can record, per warp, the candidate lists (with the mask
 * of lanes that used each entry) and per-sample sums it computes into a
 * device arena (`log`, log_bytes); the logged backward then skips the replay
 * traversal and density pass, and picks its pass-2 strategy (all lanes per
 * entry, or compacted (lane, primitive) pairs) on the device from the log's
 * lanes-per-entry statistics.  Warps whose records do
 * not fit are flagged and replayed by gsx_render_backward's kernel inside
 * gsx_render_backward_logged, so any capacity >= gsx_march_log_min_bytes is
 * correct; gsx_march_log_usage (synchronizes `stream`) reports the bytes the
 * last forward needed and whether it overflowed.  The backward must use the
 * same camera, cfg, tiles and scene as the logged forward.  ws / ws_bytes:
 * as gsx_render_forward (nullable; with it the logged forward is the
 * silhouette-screened kernel too). */
int64_t gsx_march_log_min_bytes(const gsx_camera* cam, int64_t tile_begin, int64_t tile_stride);
int gsx_render_forward_logged(const void* scene_arena, const void* bvh_arena, int64_t n,
                              const gsx_camera* cam, const gsx_render_cfg* cfg,
                              int64_t tile_begin, int64_t tile_stride, float* rgb, float* depth,
                              float* trans, void* log, int64_t log_bytes, void* ws,
                              int64_t ws_bytes, gsx_dev_status* dev_status, void* stream);
int gsx_render_backward_logged(const void* scene_arena, const void* bvh_arena,
                               const float* params, int64_t n, const gsx_camera* cam,
                               const gsx_render_cfg* cfg, int64_t tile_begin, int64_t tile_stride,
                               const float* rgb, const float* depth, const float* trans,
                               const float* dL_drgb, const float* dL_ddepth,
                               const float* dL_dtrans, const void* log, float* grad,
                               gsx_dev_status* dev_status, void* stream);
int gsx_march_log_usage(const void* log, int64_t* used_bytes, int* overflow, void* stream);

/* ---- training-step kernels ---------------------------------------------------
 * Image loss (densify.py:139-153 image_loss, :99-132 _ssim): [h,w,c] float32
 * images, L = (1-mix) L1 + mix (1-SSIM)/2 with scipy gaussian_filter(sigma 1.5,
 * truncate 3.5, mode 'reflect') statistics and a 5-px crop; h, w >= 11.
 * dL_drendered (may be NULL) receives dL/d rendered; host_out (may be NULL,
 * synchronizes the stream) receives {L, L1, SSIM}. */
size_t gsx_image_loss_workspace_bytes(int64_t h, int64_t w, int64_t c);
int gsx_image_loss(const float* rendered, const float* target, int64_t h, int64_t w, int64_t c,
                   double mix, float* dL_drendered, double* host_out, void* workspace,
                   void* stream);
/* Isotropic loss (geometry.py:215-233): *loss_dev (device double) receives
 * sum_i max(r_max,i - r0, 0) (divide by n for L_s); grad (may be NULL)
 * accumulates lambda_s dL_s/ds into the scale slots [7:10] of [n,87]. */
int gsx_iso_loss(const float* params, int64_t n, double r0, double lambda_s, float* grad,
                 double* loss_dev, void* stream);
/* Fused Adam over [n,87] records; lr87 = per-record-slot learning rates, lo87 =
 * per-slot lower bounds projected after the update (device, 87 floats each). */
int gsx_adam_step(float* params, const float* grad, float* m, float* v, int64_t n,
                  const float* lr87, const float* lo87, double beta1, double beta2, double eps,
                  int64_t step, void* stream);

/* ---- densification statistics (densify.py:49-83, observe_scene :190-204) ----
 * Observe one camera from the analytic gradient grad [n,87] (after the
 * multi-GPU all-reduce): for each observed primitive i (indices[0..m) or all
 * n when indices is NULL) sum_raw[i] += |dL/dmu_i|, sum_weighted[i] +=
 * alpha_i |dL/dmu_i| with alpha_i = |mu_i - center| / focal, counts[i] += 1
 * (float64 / int64 device arrays, GradAccumulator.observe semantics;
 * center is a host double[3]).  criteria: crit_* [n] u8 = counts >= 1 and
 * mean > tau (criterion_old: raw, criterion_new: weighted; either may be
 * NULL). */
int gsx_densify_observe(const float* grad, const float* params, int64_t n, const int64_t* indices,
                        int64_t m, const double* center, double focal, double* sum_raw,
                        double* sum_weighted, int64_t* counts, void* stream);
/* neighbor_density (densify.py:86-97): counts[i] = number of OTHER means
 * within the closed ball |mu_j - mu_i| <= radius (fp64 distances of the f32
 * means, exact BVH pruning), int64 [n] device. */
int gsx_neighbor_density(const void* scene_arena, const void* bvh_arena, int64_t n, double radius,
                         int64_t* counts, gsx_dev_status* dev_status, void* stream);
int gsx_densify_criteria(const double* sum_raw, const double* sum_weighted, const int64_t* counts,
                         int64_t n, double tau, uint8_t* crit_old, uint8_t* crit_new,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSX_H */
