/*
 * rgbid_b200.h — C-ABI of the B200-native RGBiD-SLAM front-end hot path.
 *
 * This is the drop-in boundary for the reference's front-end entry points
 * (namespace rgbid, /root/reference/proj/include/rgbid/{alignment,warping,fusion,camera}.hpp).  The reference
 * has no FFI of its own: its "plugin surface" is plain C++ free functions.  The
 * C++ drop-in (paper_1807_08271_b200/dropin/) implements
 * those functions with their exact signatures on top of this header, so a
 * maintainer replaces src/{alignment,warping,fusion}.cpp (and the hot part of
 * src/camera.cpp) by the drop-in sources and links librgbid_b200.so.
 *
 * Conventions (all entry points):
 *  - images are row-major fp64, width*height elements, NaN/inf = hole
 *    (reference inc/image.hpp:11-47);
 *  - poses are rgbid_pose {R row-major 3x3, t}, X_A = R X_B + t
 *    (reference inc/geometry.hpp:20-39);
 *  - host pointers unless a name says _dev; no exceptions cross the boundary:
 *    every function returns an rgbid_status;
 *  - one rgbid_ctx per host thread (it owns one CUDA stream + workspaces);
 *    calls on a ctx are synchronous unless named _async.
 *  - the library never falls back to the CPU: without a usable sm_100 device
 *    rgbid_ctx_create returns RGBID_E_CUDA.
 */
#ifndef RGBID_B200_H
#define RGBID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGBID_MAX_LEVELS 8

typedef enum {
  RGBID_OK = 0,
  RGBID_E_DEGENERATE = 1, /* DegenerateAlignmentError (inc/alignment.hpp:82-86); spectrum filled */
  RGBID_E_CUDA = 2,       /* CUDA error / no device */
  RGBID_E_ARG = 3,        /* invalid argument (std::invalid_argument in the reference) */
  RGBID_E_OOM = 4         /* device allocation failed */
} rgbid_status;

/* reference Intrinsics (inc/camera.hpp:16-41); k (distortion) is carried but the
 * hot path, like the reference, never applies it. */
typedef struct {
  double fx, fy, cx, cy;
  double k[5];
  int width, height;
} rgbid_intrinsics;

/* reference Pose (inc/geometry.hpp:22-39): R row-major, X_A = R X_B + t */
typedef struct {
  double R[9];
  double t[3];
} rgbid_pose;

/* reference AlignmentConfig (inc/alignment.hpp:88-96).  iterations[level] for
 * level < n_iterations, else 5 (src/alignment.cpp:373-374). */
typedef struct {
  int levels;
  int n_iterations;
  int iterations[RGBID_MAX_LEVELS];
  double convergence_eps;
  double lambda_n_min;
  double bilateral_sigma_space;
  double bilateral_sigma_intensity;
  double bilateral_sigma_depth;
} rgbid_align_config;

/* reference TDistParams (inc/alignment.hpp:28-33) */
typedef struct {
  double mu, sigma, nu;
} rgbid_tdist;

/* reference LevelLog (inc/alignment.hpp:66-70) */
typedef struct {
  int level, iterations;
  double final_cost;
} rgbid_level_log;

/* reference AlignmentResult (inc/alignment.hpp:72-80) + error payload */
typedef struct {
  rgbid_pose T_AB;
  double cov[36]; /* row-major 6x6, (translation, rotation) */
  int converged;
  int cov_degenerate;
  int n_levels;
  rgbid_level_log level_log[RGBID_MAX_LEVELS]; /* coarse to fine, like the reference */
  rgbid_tdist tdist_intensity;
  rgbid_tdist tdist_depth;
  double spectrum[6]; /* DegenerateAlignmentError::spectrum when status == RGBID_E_DEGENERATE */
  int status;         /* rgbid_status of this alignment (batched calls) */
  int total_iterations;
} rgbid_align_result;

/* One IRLS iteration, for step-level parity checks (restates the locals of
 * src/alignment.cpp:377-401; build_system is file-static in the reference). */
typedef struct {
  int level, iter;
  long long n_jets, n_depth;
  rgbid_tdist tI, tW; /* after build_system: tI.nu = max(nu_I, nu_W) */
  double H[36];       /* row-major; GPU fills upper triangle and mirrors it */
  double b[6];
  double cost;
  double xi[6];
  rgbid_pose T_after;
} rgbid_iter_trace;

/* reference DepthIntrinsics (inc/camera.hpp:45-51) */
typedef struct {
  double beta0, beta1;
  double q0[9], q1[9];
  double p0[2];
} rgbid_depth_intrinsics;

typedef struct rgbid_ctx rgbid_ctx;
typedef struct rgbid_frame rgbid_frame; /* device-resident (I, W) pair + cached pyramid */

/* ---- context ---------------------------------------------------------- */
const char* rgbid_version(void);
const char* rgbid_status_string(int status);
int rgbid_ctx_create(int device, rgbid_ctx** out);
int rgbid_ctx_destroy(rgbid_ctx* ctx);
/* last CUDA error text for this ctx (empty when none) */
const char* rgbid_ctx_last_error(rgbid_ctx* ctx);
/* count of this library's kernel launches on ctx since creation */
long long rgbid_ctx_kernel_launches(rgbid_ctx* ctx);
/* waits for all of ctx's streams; completes pending async batch chunks */
int rgbid_ctx_synchronize(rgbid_ctx* ctx);
/* stream used by ctx (cudaStream_t, as void*) */
void* rgbid_ctx_stream(rgbid_ctx* ctx);
/* Per-kernel CUDA-event timing of every library launch (graphs are bypassed
 * while enabled).  kernel_stats writes {"name": [launches, total_ms], ...} JSON
 * and returns the buffer size needed. */
int rgbid_ctx_set_profiling(rgbid_ctx* ctx, int enable);
int rgbid_ctx_reset_stats(rgbid_ctx* ctx);
int rgbid_ctx_kernel_stats(rgbid_ctx* ctx, char* buf, int cap);
/* bytes this ctx copied host->device / device->host since the last reset */
int rgbid_ctx_transfer_bytes(rgbid_ctx* ctx, long long* h2d, long long* d2h);

/* ---- device frames ------------------------------------------------------ */
/* FrameData (inc/alignment.hpp:14-18) uploaded once; I may be NULL (depth only). */
int rgbid_frame_create(rgbid_ctx* ctx, int width, int height, rgbid_frame** out);
int rgbid_frame_upload(rgbid_ctx* ctx, rgbid_frame* f, const double* I, const double* W);
int rgbid_frame_download(rgbid_ctx* ctx, const rgbid_frame* f, double* I, double* W);
/* Frame ingest from the sensor wire format — load_frame's decode (src/dataset.cpp:97-116):
 * bgr (w*h*3 u8, may be NULL) -> gray (0.299R + 0.587G + 0.114B)/255; depth (w*h u16)
 * -> scale/raw with raw 0 -> hole, scale = depth_scale / depth_factor (5000 for TUM).
 * Uploads 5 B/px instead of 16 B/px of fp64 maps. */
int rgbid_frame_decode(rgbid_ctx* ctx, rgbid_frame* f, const uint8_t* bgr, const uint16_t* depth,
                       double scale);
/* device pointers of the frame's level-0 maps (for zero-copy producers) */
int rgbid_frame_device_ptrs(rgbid_frame* f, double** I_dev, double** W_dev);
int rgbid_frame_destroy(rgbid_ctx* ctx, rgbid_frame* f);
/* mark the cached pyramid stale (the producer wrote new maps in place) */
int rgbid_frame_invalidate(rgbid_frame* f);

/* ---- hot-path entry points (reference signatures noted) ---------------- */

/* Pyramid build_pyramid(const FrameData&, const Intrinsics&, int)  — src/alignment.cpp:9-30.
 * out_I/out_W: `levels` host buffers of (w>>l)x(h>>l) (level 0 copied); K_out: levels entries. */
int rgbid_build_pyramid(rgbid_ctx* ctx, const double* I, const double* W, int width, int height,
                        const rgbid_intrinsics* K, int levels, double** out_I, double** out_W,
                        rgbid_intrinsics* K_out);

/* WarpedFrame inverse_geometric_warp(I_B, W_B, W_A, T_AB, K) — src/warping.cpp:76-114.
 * I_B/W_B are width_b x height_b; W_A and all outputs are width x height. */
int rgbid_inverse_geometric_warp(rgbid_ctx* ctx, const double* I_B, const double* W_B,
                                 int width_b, int height_b, const double* W_A, int width,
                                 int height, const rgbid_pose* T_AB, const rgbid_intrinsics* K,
                                 double* out_I, double* out_W, double* out_map_x,
                                 double* out_map_y);

/* AlignmentResult align(a, b, K, init, config) — src/alignment.cpp:367-409. */
int rgbid_align(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                const rgbid_intrinsics* K, const rgbid_pose* init, const rgbid_align_config* cfg,
                rgbid_align_result* result);
/* Same, host buffers in (uploads inside the call). */
int rgbid_align_host(rgbid_ctx* ctx, const double* I_A, const double* W_A, const double* I_B,
                     const double* W_B, int width, int height, const rgbid_intrinsics* K,
                     const rgbid_pose* init, const rgbid_align_config* cfg,
                     rgbid_align_result* result);
/* Step-level trace of the last rgbid_align/rgbid_align_batch item 0 on ctx
 * (max_entries records; returns the count in *n). */
int rgbid_last_align_trace(rgbid_ctx* ctx, rgbid_iter_trace* out, int max_entries, int* n);

/* Batched independent alignments (config 5): pairs[i] = (a[i], b[i]).  All frames
 * the same size.  inits may be NULL (identity).  results[i].status per pair; the
 * call returns RGBID_OK unless an argument/CUDA error occurred. */
int rgbid_align_batch(rgbid_ctx* ctx, int n, const rgbid_frame* const* a,
                      const rgbid_frame* const* b, const rgbid_intrinsics* K,
                      const rgbid_pose* inits, const rgbid_align_config* cfg,
                      rgbid_align_result* results);
/* How rgbid_align_batch splits n pairs: *n_chunks chunks of <= *chunk slots
 * (1024 cap, RGBID_BATCH_SLOTS overrides), executed as co-scheduled chunk pairs
 * on the ctx's two lanes; a batch of >= 64 pairs is always split in two so the
 * lanes overlap.  Host-only (no device needed). */
int rgbid_batch_plan(int n, int* chunk, int* n_chunks);
/* Batched alignments from HOST buffers (end-to-end path): pair i reads
 * I_A[i], W_A[i], I_B[i], W_B[i] (each width*height doubles, pinned memory
 * recommended).  Uploads are pipelined with compute in chunks of `chunk` pairs. */
int rgbid_align_batch_host(rgbid_ctx* ctx, int n, const double* const* I_A,
                           const double* const* W_A, const double* const* I_B,
                           const double* const* W_B, int width, int height,
                           const rgbid_intrinsics* K, const rgbid_pose* inits,
                           const rgbid_align_config* cfg, int chunk,
                           rgbid_align_result* results);
/* Streaming form of rgbid_align_batch_host: returns once every chunk is enqueued;
 * the last chunks (one per stream) may still be running, and their entries of
 * `results` (and the host buffers they read) must stay valid until the next
 * rgbid_align_batch_host_async / rgbid_align_batch_host call on ctx RETURNS (it
 * completes every chunk of the previous call before returning), or until
 * rgbid_align_batch_host_wait / rgbid_ctx_synchronize / any synchronous align
 * call on ctx.  Consecutive calls overlap one batch's first uploads with the
 * previous batch's last chunks. */
int rgbid_align_batch_host_async(rgbid_ctx* ctx, int n, const double* const* I_A,
                                 const double* const* W_A, const double* const* I_B,
                                 const double* const* W_B, int width, int height,
                                 const rgbid_intrinsics* K, const rgbid_pose* inits,
                                 const rgbid_align_config* cfg, int chunk,
                                 rgbid_align_result* results);
/* Completes every chunk a previous async call left in flight (results written). */
int rgbid_align_batch_host_wait(rgbid_ctx* ctx);

/* Mat6 filtered_hessian_covariance(a, b, K, T_AB, config, &degenerate) — src/alignment.cpp:411-436 */
int rgbid_filtered_hessian_covariance(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                                      const rgbid_intrinsics* K, const rgbid_pose* T_AB,
                                      const rgbid_align_config* cfg, double* cov36,
                                      int* degenerate);
/* Image<double> bilateral_filter(img, sigma_space, sigma_range) — src/alignment.cpp:252-277 */
int rgbid_bilateral_filter(rgbid_ctx* ctx, const double* img, int width, int height,
                           double sigma_space, double sigma_range, double* out);

/* void integrate_frame(Keyframe*, frame, T_kf_frame, K, sigma_w) — src/fusion.cpp:68-95.
 * Keyframe maps (kf_W, kf_C) are updated in place (host buffers); kf_I untouched,
 * exactly as the reference. */
int rgbid_integrate_frame(rgbid_ctx* ctx, double* kf_W, double* kf_C, const double* frame_I,
                          const double* frame_W, int width, int height,
                          const rgbid_pose* T_kf_frame, const rgbid_intrinsics* K,
                          double sigma_w);
/* k sequential integrate_frame calls fused into one kernel (bit-identical to k
 * calls: per-pixel state depends only on the same pixel).  Device-resident
 * keyframe (kf frame's W + C map) and frames. */
int rgbid_integrate_frames(rgbid_ctx* ctx, rgbid_frame* kf, double* kf_C_dev, int k,
                           const rgbid_frame* const* frames, const rgbid_pose* T_kf_frames,
                           const rgbid_intrinsics* K, double sigma_w);

/* CovisibilityResult covisibility_ratio(a, b, T_BA, K, sigma_w) — src/fusion.cpp:26-66.
 * counts[4] = {valid_ab, visible_ab, valid_ba, visible_ba} (optional). */
int rgbid_covisibility_ratio(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                             const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                             double* ratio, int* empty_frame, long long* counts);

/* InverseDepthMap correct_inverse_depth(W_m, dintr, intr, spatial) — src/camera.cpp:62-81 */
int rgbid_correct_inverse_depth(rgbid_ctx* ctx, const double* W_m, int width, int height,
                                const rgbid_depth_intrinsics* d, const rgbid_intrinsics* K,
                                int spatial, double* out);
/* InverseDepthMap forward_register(W_A, T_BA, K_A, K_B) — src/warping.cpp:20-74.
 * out is K_B->width x K_B->height. */
int rgbid_forward_register(rgbid_ctx* ctx, const double* W_A, int width, int height,
                           const rgbid_pose* T_BA, const rgbid_intrinsics* K_A,
                           const rgbid_intrinsics* K_B, double* out);

/* ---- distorted sensors (config 4 with k != 0) ---------------------------- */
/* Image<double> inverse_warp(src, f_w, w, h) (src/warping.cpp:8-18) with the
 * rectification map f_w(p) = project(K, ((x - cx) / fx, (y - cy) / fy, 1)) =
 * K distort(K^-1 p) (src/camera.cpp:11-22,41-45), applied to both maps
 * of a device frame (dst != src, both K->width x K->height). */
int rgbid_rectify_frame(rgbid_ctx* ctx, const rgbid_frame* src, const rgbid_intrinsics* K,
                        rgbid_frame* dst);
/* The same for one host image. */
int rgbid_rectify(rgbid_ctx* ctx, const double* src, int width, int height,
                  const rgbid_intrinsics* K, double* out);
/* std::optional<Vec2> undistort(K, m_d) (src/camera.cpp:24-39) for n normalized points
 * m_d[2i], m_d[2i+1]; ok[i] = 0 where the reference returns std::nullopt. */
int rgbid_undistort_points(rgbid_ctx* ctx, const double* m_d, long long n,
                           const rgbid_intrinsics* K, double* m_u, unsigned char* ok);

/* ---- front-end odometry driver (config 3) -------------------------------- */
/* Restates Pipeline::process_frame / track / fuse_and_maybe_switch
 * (src/pipeline.cpp:120-247) without the back-end; frames, reference and
 * keyframe state resident in HBM. */
typedef struct {
  rgbid_align_config align;       /* PipelineConfig::alignment */
  double keyframe_covisibility;   /* 0.7 (inc/pipeline.hpp:80) */
  double reference_covisibility;  /* 0.9 (inc/pipeline.hpp:81) */
  int buffer_capacity;            /* 30 (inc/pipeline.hpp:84) */
} rgbid_frontend_config;

/* FrameEstimate (inc/pipeline.hpp:25-31) */
typedef struct {
  double timestamp;
  rgbid_pose T_W_k;
  double cov[36]; /* step covariance, left-referenced in the previous frame */
  int lost;
  int keyframe_id; /* >= 0 when this frame started a keyframe */
} rgbid_frame_estimate;

typedef struct rgbid_frontend rgbid_frontend;
int rgbid_frontend_default_config(rgbid_frontend_config* cfg);
int rgbid_frontend_create(rgbid_ctx* ctx, const rgbid_intrinsics* K,
                          const rgbid_frontend_config* cfg, rgbid_frontend** out);
int rgbid_frontend_destroy(rgbid_frontend* fe);
/* Pipeline::process_frame(frame, timestamp); *est = the frame's estimate */
int rgbid_frontend_process(rgbid_frontend* fe, const double* I, const double* W, double timestamp,
                           rgbid_frame_estimate* est);
/* flush: absorb the open keyframe's buffered frames (Pipeline::finish front half) */
int rgbid_frontend_finish(rgbid_frontend* fe);
int rgbid_frontend_trajectory(rgbid_frontend* fe, rgbid_frame_estimate* out, int max, int* n);
int rgbid_frontend_keyframes(rgbid_frontend* fe, int* frame_index, int max, int* n);
int rgbid_frontend_current_keyframe(rgbid_frontend* fe, double* W, double* C, rgbid_pose* T_W_kf,
                                    int* id);

/* device helpers */
int rgbid_frame_copy(rgbid_ctx* ctx, rgbid_frame* dst, const rgbid_frame* src);
int rgbid_fill(rgbid_ctx* ctx, double* dev, long long n, double value);

/* ---- remaining drop-in entry points (not on the align hot path) --------- */
/* inverse_warp's sampling (src/warping.cpp:8-18): out(i) = bilinear(src, map_x(i), map_y(i))
 * for a coordinate map the caller evaluated from its f_w. */
int rgbid_remap_bilinear(rgbid_ctx* ctx, const double* src, int width, int height,
                         const double* map_x, const double* map_y, int out_width, int out_height,
                         double* out);
/* std::vector<PixelJet> residuals_and_jacobians(a, warped_b, K, lambda_n_min) —
 * src/alignment.cpp:195-250.  jets: records {x, y, r_I, r_W, J_I[6], J_W[6], lambda_n}
 * in row-major order; returns the jet count (negative rgbid_status on error). */
long long rgbid_residuals_and_jacobians(rgbid_ctx* ctx, const double* I_A, const double* W_A,
                                        const double* I_Bw, const double* W_Bw, int width,
                                        int height, const rgbid_intrinsics* K,
                                        double lambda_n_min, double* jets,
                                        unsigned char* has_depth, long long cap);
/* TDistParams estimate_location_scale(residuals, nu) — src/alignment.cpp:61-101 */
int rgbid_estimate_location_scale(rgbid_ctx* ctx, const double* r, long long n, double nu,
                                  rgbid_tdist* out);
/* double estimate_nu(residuals, mu, sigma) — src/alignment.cpp:109-127 */
int rgbid_estimate_nu(rgbid_ctx* ctx, const double* r, long long n, double mu, double sigma,
                      double* nu);

/* ---- self tests ---------------------------------------------------------- */
/* Bitwise check of the warp's reciprocal-based correctly-rounded division
 * against IEEE division on n random operand pairs; *mismatches must be 0. */
int rgbid_selftest_division(rgbid_ctx* ctx, unsigned long long n, unsigned long long seed,
                            unsigned long long* mismatches);

/* measured FP64 FMA throughput of this device (TFLOP/s, FMA = 2 flops): the
 * roofline denominator of the FP64-issue-bound Student-t kernel */
int rgbid_measure_fp64_peak(rgbid_ctx* ctx, double* tflops);

/* ---- loop-closure dense refinement ------------------- */
/* reference LoopConstraint (include/rgbid/loop.hpp:19-26) */
typedef struct {
  int i, j;          /* keyframe ids (i = query, j = match) */
  rgbid_pose T_ij;   /* pose of j in i's frame */
  double info[36];   /* row-major 6x6, symmetrised cov^-1 */
  int inliers;
  double hull_fraction;
  double score;
} rgbid_loop_constraint;

/* std::optional<LoopConstraint> make_loop_constraint(kf_i, kf_j, T_init, K, geom, config,
 * align_config) — src/loop.cpp:174-203, the back-end's second caller of align.  The
 * place-recognition inputs (geom.inliers, geom.hull_fraction) pass through.  A
 * degenerate alignment or a refined covisibility below min_covisibility (0.3 by default,
 * include/rgbid/loop.hpp:46) gives *accepted = 0 (std::nullopt) and RGBID_OK.  Runs on
 * ctx's stream: a second context on another host thread refines loops concurrently
 * with the front-end. */
int rgbid_make_loop_constraint(rgbid_ctx* ctx, const rgbid_frame* kf_i, const rgbid_frame* kf_j,
                               int id_i, int id_j, const rgbid_intrinsics* K,
                               const rgbid_pose* T_init, const rgbid_align_config* cfg,
                               double min_covisibility, int inliers, double hull_fraction,
                               rgbid_loop_constraint* out, int* accepted);

/* ---- normals and map export --------------------------- */
/* NormalMap normal_map(W, K) — src/segmentation.cpp:10-57.  Host buffers, w x h each;
 * holes propagate (NaN), degenerate pixels get -e_z. */
int rgbid_normal_map(rgbid_ctx* ctx, const double* W, int width, int height,
                     const rgbid_intrinsics* K, double* nx, double* ny, double* nz);

/* PointCloud export_map(keyframes, K, voxel) — src/pipeline.cpp:463-527.
 * Keyframe k: intensity I[k], inverse depth W[k] (host, width x height), pose T_W_kf[k].
 * points: capacity x 3 doubles (x, y, z), colors: capacity x 3 bytes (r, g, b).
 * *n = points in the cloud; if it exceeds capacity nothing is written and
 * RGBID_E_ARG is returned (n_kf * width * height always suffices). */
int rgbid_export_map(rgbid_ctx* ctx, int n_kf, const double* const* I, const double* const* W,
                     int width, int height, const rgbid_pose* T_W_kf, const rgbid_intrinsics* K,
                     double voxel, double* points, unsigned char* colors, long long capacity,
                     long long* n);

/* ---- synthetic inputs (restates /root/reference/proj/tests/synthetic.hpp) ---- */
/* render_plane(K, T_WC, n, d) with plane_texture evaluated at tex_scale * (X, Y) */
int rgbid_synth_render_plane(const rgbid_intrinsics* K, const rgbid_pose* T_WC, const double n[3],
                             double d, double tex_scale, double* I, double* W);
/* random_pose(std::mt19937(seed) advanced by `skip` poses, t_scale, angle_scale) */
int rgbid_synth_random_pose(uint32_t seed, int skip, double t_scale, double angle_scale,
                            rgbid_pose* out);
/* I += N(0, sigma_i), W += N(0, sigma_w) on valid pixels, std::mt19937(seed) */
int rgbid_synth_add_noise(double* I, double* W, int width, int height, uint32_t seed,
                          double sigma_i, double sigma_w);
/* Device-side generation of batch pair i (bench): renders A and B of
 * pair (seed_base + i) directly into frames a and b. variant 0 = clean,
 * 1 = noisy + 20% near occluder (counter-based Gaussian noise), 2 = variant 1 +
 * 5% W / 2% I seeded holes and a width/32-pixel W border band.
 * The hole pattern is integer-hashed: identical to rgbid_synth_pair_host's. */
int rgbid_synth_pair_device(rgbid_ctx* ctx, rgbid_frame* a, rgbid_frame* b,
                            const rgbid_intrinsics* K, uint32_t pair_seed, int variant,
                            rgbid_pose* T_AB_truth);
/* The same pair on the host (host libm: equal to the device rendering up to the
 * last bits of sin/cos/log): the reference arm's inputs, generated without the GPU. */
int rgbid_synth_pair_host(const rgbid_intrinsics* K, uint32_t pair_seed, int variant, double* I_A,
                          double* W_A, double* I_B, double* W_B, rgbid_pose* T_AB_truth);

#ifdef __cplusplus
}
#endif

#endif /* RGBID_B200_H */
