/*
 * planestereo_c.h — C ABI of the B200-native planestereo hot path.
 *
 * This is the drop-in boundary.  The reference (`/root/reference/proj`, a C++20
 * static library) has no FFI; its public interface is the C++ header API in
 * namespace `planestereo`.  Each entry point below replaces one reference
 * function (cited file:line, relative to the reference's `proj/`), and the C++
 * headers under `include/planestereo/` re-create that header API on top of
 * this ABI, so a user of the reference recompiles against
 * them unchanged.
 *
 * Conventions
 *   - plain pointers and sizes; no torch or C++ types cross this boundary;
 *   - all image-shaped buffers are row-major, stride = width, P = width*height;
 *   - the caller owns every host buffer; a ps_ctx owns device memory, streams
 *     and pinned staging and must not be used by two threads at once;
 *   - every function returns a ps_status; on failure ps_last_error() holds
 *     the message (the C++ layer rethrows the matching planestereo:: error,
 *     include/planestereo/error.hpp).
 */
#ifndef PLANESTEREO_C_H
#define PLANESTEREO_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field-for-field mirror of planestereo::PipelineConfig
 * (proj/include/planestereo/config.hpp:8-34); 44-byte POD. */
typedef struct ps_config {
    int iterations;           /* config.hpp:10  default 1   */
    int max_disparity;        /* config.hpp:12  default 128 */
    float cost_low;           /* config.hpp:14  default 0.25f */
    float cost_high;          /* config.hpp:16  default 0.5f  */
    int gradient_threshold;   /* config.hpp:18  default 20  */
    int occupancy_cell_size;  /* config.hpp:20  default 32  */
    int corner_threshold;     /* config.hpp:22  default 20  */
    int per_bin_cap;          /* config.hpp:24  default 5   */
    float sparse_accept_cost; /* config.hpp:26  default 0.25f */
    float uniqueness_ratio;   /* config.hpp:28  default 0.9f  */
    int threads;              /* config.hpp:30  default 1 (host threads; GPU ignores) */
} ps_config;

/* Mirror of planestereo::IterationStats (proj/include/planestereo/pipeline.hpp:50-58). */
typedef struct ps_iter_stats {
    int iteration;
    int support_count;
    int triangle_count;
    int occupancy_cell_size;
    double mean_cost;
    int valid_count;
    double millis;
} ps_iter_stats;

/* 1:1 with the exception classes of proj/include/planestereo/error.hpp:9-72. */
typedef enum ps_status {
    PS_OK = 0,
    PS_ERROR = 1,                   /* planestereo::Error (generic)        error.hpp:9  */
    PS_INVALID_CONFIG = 2,          /* InvalidConfig                       error.hpp:14 */
    PS_DIMENSION_TOO_SMALL = 3,     /* DimensionTooSmall                   error.hpp:19 */
    PS_DIMENSION_MISMATCH = 4,      /* DimensionMismatch                   error.hpp:24 */
    PS_FEWER_THAN_THREE_POINTS = 5, /* FewerThanThreePoints                error.hpp:29 */
    PS_DEGENERATE_TRIANGLE = 6,     /* DegenerateTriangle                  error.hpp:34 */
    PS_SEEDING_FAILED = 7,          /* SeedingFailed                       error.hpp:39 */
    PS_CUDA_ERROR = 8,              /* device failure (no reference analogue) */
    PS_NO_DEVICE = 9,               /* no sm_100 device / extension not usable */
    PS_CAPACITY = 10,               /* caller buffer too small (count written) */
    PS_NEGATIVE_DISPARITY = 11,     /* NegativeDisparity                   error.hpp:54 */
    PS_EMPTY_CLOUD = 12,            /* EmptyCloud                          error.hpp:59 */
    PS_NO_OVERLAP = 13,             /* NoOverlap                           error.hpp:64 */
    PS_INVALID_PLANE = 14           /* InvalidPlane                        error.hpp:69 */
} ps_status;

/* Run flags. */
#define PS_RUN_UNCHECKED_CELL 0x1u /* skip only the power-of-two cell rule of
                                      PipelineConfig::validate (proj/src/config.cpp:27-30);
                                      needed by BASELINE grids 10 and 6 */

typedef struct ps_ctx ps_ctx;

/* Called after every iteration of ps_run with host copies of the running
 * state (mirror of planestereo::IterationObserver, pipeline.hpp:98-99). */
typedef void (*ps_observer_fn)(int iteration, const float* final_disparity,
                               const uint8_t* final_valid, const float* final_cost,
                               int width, int height, void* user);

/* ---------------------------------------------------------------- context */
const char* ps_version(void);
ps_status ps_ctx_create(int device, ps_ctx** out);
void ps_ctx_destroy(ps_ctx* ctx);
/* Message of the last failure on this thread (ctx may be NULL). */
const char* ps_last_error(const ps_ctx* ctx);
void ps_config_default(ps_config* cfg);
/* PipelineConfig::validate (proj/src/config.cpp:17-49); flags as in ps_run. */
ps_status ps_config_validate(const ps_config* cfg, unsigned flags);

/* --------------------------------------------------------------- pipeline */
/* planestereo::run (proj/src/pipeline.cpp:131-203) for one rectified pair.
 * Outputs are caller-allocated P-sized arrays (any may be NULL);
 * trace has cfg->iterations entries (may be NULL). */
ps_status ps_run(ps_ctx* ctx, const uint8_t* left, const uint8_t* right, int width, int height,
                 const ps_config* cfg, unsigned flags, float* disparity, uint8_t* disparity_valid,
                 float* cost, float* dense, uint8_t* dense_valid, ps_iter_stats* trace,
                 ps_observer_fn observer, void* user);

/* Batched run over n_frames independent pairs (frames stacked, stride P).
 * Per-frame status goes to frame_status[n_frames] (PS_SEEDING_FAILED for a
 * frame whose seeding failed; its outputs are left untouched).  Outputs are
 * strided by P per frame, trace by cfg->iterations per frame; any may be NULL.
 * Returns the first non-OK frame status, or a context-level error. */
ps_status ps_run_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                       int width, int height, const ps_config* cfg, unsigned flags,
                       float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                       uint8_t* dense_valid, ps_iter_stats* trace, int* frame_status);

/* The same batch sharded over n_ctx contexts — one per GPU of the box
 * — from one process: an even split into contiguous blocks
 * (sizes differ by at most one frame), each block run by ps_run_batch on its
 * context from its own host thread.  Frames never interact, so no collective
 * is involved.  Same arguments and per-frame outputs as ps_run_batch;
 * returns the first context-level error (in context order), else the first
 * non-OK frame status.  The contexts must be distinct. */
ps_status ps_run_batch_multi(ps_ctx* const* ctxs, int n_ctx, int n_frames, const uint8_t* left,
                             const uint8_t* right, int width, int height, const ps_config* cfg,
                             unsigned flags, float* disparity, uint8_t* disparity_valid,
                             float* cost, float* dense, uint8_t* dense_valid,
                             ps_iter_stats* trace, int* frame_status);

/* Device-resident variant used to time the pipeline with inputs already in
 * HBM: ps_upload_batch copies the pairs into ctx-owned device memory,
 * ps_run_resident runs the pipeline on them (no host copies of images or
 * outputs; only the host Delaunay exchange), ps_download_batch copies the
 * outputs of the last resident run back. */
ps_status ps_upload_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                          int width, int height);
ps_status ps_run_resident(ps_ctx* ctx, const ps_config* cfg, unsigned flags);
ps_status ps_download_batch(ps_ctx* ctx, float* disparity, uint8_t* disparity_valid,
                            float* cost, float* dense, uint8_t* dense_valid,
                            ps_iter_stats* trace, int* frame_status);

/* Support list of one frame of the last run (the list used by the last
 * iteration; trace[i].support_count gives each iteration's prefix length). */
ps_status ps_get_supports(ps_ctx* ctx, int frame, int* u, int* v, double* d, int capacity,
                          int* count);

/* ------------------------------------------------------- kernel telemetry */
typedef struct ps_kernel_stat {
    char name[32];
    int launches;
    double total_ms;         /* CUDA-event time summed over launches */
    double algorithmic_bytes;/* SURVEY 8(d) bytes summed over launches */
} ps_kernel_stat;
/* Enables per-launch CUDA-event timing of the engine kernels (on the stream
 * each kernel is launched on). */
ps_status ps_set_profiling(ps_ctx* ctx, int enabled);
/* At most `groups` frame groups (CUDA streams) in flight; default 8.  With 1
 * the device stages run back to back, so kernel times are isolated. */
ps_status ps_set_max_groups(ps_ctx* ctx, int groups);
/* Host worker threads of the context's Delaunay pool (affinity CPUs / local
 * ranks, or PS_HOST_THREADS). */
ps_status ps_get_host_threads(ps_ctx* ctx, int* threads);
ps_status ps_reset_kernel_stats(ps_ctx* ctx);
ps_status ps_get_kernel_stats(ps_ctx* ctx, ps_kernel_stat* out, int capacity, int* count);
/* Kernel launches issued by this context since creation. */
long long ps_launch_count(const ps_ctx* ctx);
/* The context's CUDA stream (a cudaStream_t), so callers can bracket a
 * pipeline run with their own CUDA events on the stream it runs on. */
void* ps_ctx_stream(const ps_ctx* ctx);

/* ------------------------------------------------------------ stage API */
/* gradientMask (proj/src/image.cpp:43-60): member[P] in {0,1}; count = M. */
ps_status ps_gradient_mask(ps_ctx* ctx, const uint8_t* image, int width, int height,
                           int threshold, uint8_t* member, int* count);
/* censusTransform (proj/src/census.cpp:10-41). */
ps_status ps_census(ps_ctx* ctx, const uint8_t* image, int width, int height, uint32_t* out);
/* detectCandidates (proj/src/sparse.cpp:84-146); at most 120*per_bin_cap results. */
ps_status ps_detect_candidates(ps_ctx* ctx, const uint8_t* image, int width, int height,
                               const ps_config* cfg, int* u, int* v, float* score,
                               int capacity, int* count);
/* matchEpipolar over census fields (proj/src/sparse.cpp:148-195). */
ps_status ps_match_epipolar(ps_ctx* ctx, const uint32_t* census_left,
                            const uint32_t* census_right, int width, int height,
                            const int* cand_u, const int* cand_v, int n_candidates,
                            const ps_config* cfg, int* u, int* v, double* d, int capacity,
                            int* count);
/* delaunayTriangulate (proj/src/delaunay.cpp:288-325): positively oriented
 * index triples into the input list, in the reference's own order and
 * rotation; tris has room for 3*capacity ints.  Host code (exact integer
 * predicates). */
ps_status ps_delaunay(const int* u, const int* v, int n, int* tris, int capacity, int* n_tris);
/* Same triangle set, in radial-sweep order (the engine's fast path; triangle
 * order and rotation are not part of the Delaunay contract). */
ps_status ps_delaunay_fast(const int* u, const int* v, int n, int* tris, int capacity,
                           int* n_tris);
/* DisparityMesh ctor (proj/src/mesh.cpp:44-123): per-triangle planes (a,b,c)
 * and the P-sized triangle lookup (-1 outside). */
ps_status ps_mesh_build(ps_ctx* ctx, const int* u, const int* v, const double* d, int n_points,
                        const int* tris, int n_tris, int width, int height, double* planes,
                        int32_t* lookup);
/* interpolate (proj/src/mesh.cpp:149-182): mask==NULL evaluates every pixel. */
ps_status ps_interpolate(ps_ctx* ctx, const int32_t* lookup, const double* planes, int n_tris,
                         int width, int height, const uint8_t* mask, float max_disparity,
                         float* value, uint8_t* valid);
/* costEvaluation (proj/src/pipeline.cpp:33-54). */
ps_status ps_cost_evaluation(ps_ctx* ctx, const uint32_t* census_left,
                             const uint32_t* census_right, int width, int height,
                             const float* interp, const uint8_t* interp_valid,
                             const uint8_t* mask, float* cost);

/* One occupancy cell (mirror of planestereo::OccupancyCell, pipeline.hpp:17-23). */
typedef struct ps_cell {
    int u;
    int v;
    float disparity;
    float cost;
    int occupied;
} ps_cell;
/* disparityRefinement (proj/src/pipeline.cpp:56-86): folds costs into the
 * running state (in/out) and fills the two grids, each
 * ceil(W/cell) x ceil(H/cell) cells, row-major. */
ps_status ps_refinement(ps_ctx* ctx, const float* interp, const uint8_t* interp_valid,
                        const float* cost, float* final_disparity, uint8_t* final_valid,
                        float* final_cost, const uint8_t* mask, int width, int height,
                        int cell_size, const ps_config* cfg, ps_cell* confident,
                        ps_cell* invalid);
/* supportResampling (proj/src/pipeline.cpp:88-129). */
ps_status ps_support_resampling(ps_ctx* ctx, const ps_cell* confident, const ps_cell* invalid,
                                int cell_size, const int* sup_u, const int* sup_v,
                                const double* sup_d, int n_supports,
                                const uint32_t* census_left, const uint32_t* census_right,
                                int width, int height, const ps_config* cfg, int* u, int* v,
                                double* d, int capacity, int* count);

/* wtaOracle (proj/include/planestereo/synth.hpp:52-56, proj/src/synth.cpp:171-198):
 * per mask pixel the cost-minimal integer disparity in
 * [0, min(max_disparity, u - 2)] (max_disparity inclusive), ties toward the
 * smaller d; off-mask pixels get cost 1.0 and no disparity.  The census of
 * both views is computed on the device. */
ps_status ps_wta_oracle(ps_ctx* ctx, const uint8_t* left, const uint8_t* right, int width,
                        int height, const uint8_t* mask, int max_disparity, float* disparity,
                        uint8_t* disparity_valid, float* cost);
/* The same over n_frames pairs stacked frame after frame, with each frame's
 * mask = gradientMask(left, gradient_threshold): the dense WTA baseline of a
 * batch (outputs n_frames * width * height each). */
ps_status ps_wta_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                       int width, int height, int gradient_threshold, int max_disparity,
                       float* disparity, uint8_t* disparity_valid, float* cost);

/* ------------------------------------------------------ output encoders */
/* Rasters of the reference's io module (proj/src/io.cpp), computed on the
 * device; the file containers (PNG/PFM/PLY headers) are the caller's.
 *   KITTI 16-bit, writeKittiPng :349-368 — 2 bytes per pixel, row-major, the
 *     PNG row bytes: big-endian raw = clamp(lround(d*256), 1, 65535), 0 =
 *     invalid; PS_NEGATIVE_DISPARITY (message names the first one) if a valid
 *     disparity is negative.
 *   PFM, writePfm :311-329 — binary32 per pixel, rows bottom-up, invalid -1.0.
 *   point cloud, exportPointCloud :395-454 — the vertex list: xyz (3 floats)
 *     and intensity of each valid pixel with d >= min_disparity, row-major;
 *     PS_EMPTY_CLOUD when there is none, PS_INVALID_CONFIG for a bad calib.
 * The batch forms encode n_frames maps stacked frame after frame. */
typedef struct ps_calib { /* CameraCalib, proj/include/planestereo/io.hpp:17-24 */
    double focal;    /* pixels, > 0 */
    double baseline; /* meters, > 0 */
    double cx;
    double cy;
} ps_calib;
ps_status ps_encode_kitti16(ps_ctx* ctx, const float* disparity, const uint8_t* valid, int width,
                            int height, int n_frames, uint8_t* out);
ps_status ps_encode_pfm(ps_ctx* ctx, const float* disparity, const uint8_t* valid, int width,
                        int height, int n_frames, float* out);
ps_status ps_point_cloud(ps_ctx* ctx, const float* disparity, const uint8_t* valid,
                         const uint8_t* image, int width, int height, const ps_calib* calib,
                         double min_disparity, float* xyz, uint8_t* intensity, int capacity,
                         int* count);
/* The same over the last run's results in device memory (no map D2H):
 * which = PS_MAP_DISPARITY (the final disparity) or PS_MAP_DENSE (the dense
 * interpolation); a frame whose seeding failed encodes as all-invalid.  The
 * point cloud uses that frame's left image. */
#define PS_MAP_DISPARITY 0
#define PS_MAP_DENSE 1
ps_status ps_download_kitti16(ps_ctx* ctx, int which, uint8_t* out);
ps_status ps_download_pfm(ps_ctx* ctx, int which, float* out);
ps_status ps_download_point_cloud(ps_ctx* ctx, int frame, int which, const ps_calib* calib,
                                  double min_disparity, float* xyz, uint8_t* intensity,
                                  int capacity, int* count);

/* ------------------------------------------------------------ evaluation */
/* accuracy (proj/include/planestereo/eval.hpp:15-29, proj/src/eval.cpp:19-70)
 * of n_frames predictions against ground truth, on the device: per frame,
 * over the pixels valid in both maps (and inside mask, when not NULL),
 * evaluated[f], mean_abs_error[f] (the reference's row-major binary64 sum /
 * evaluated) and fractions[f * n_thresholds + k] = #{err < thresholds[k]} /
 * evaluated; n_thresholds <= 16.  PS_NO_OVERLAP (NoOverlap) if a frame has no
 * jointly valid pixel — the other frames are still filled. */
ps_status ps_accuracy(ps_ctx* ctx, int n_frames, const float* prediction,
                      const uint8_t* prediction_valid, const float* ground_truth,
                      const uint8_t* ground_truth_valid, const uint8_t* mask, int width,
                      int height, const double* thresholds, int n_thresholds, double* fractions,
                      long long* evaluated, double* mean_abs_error);
/* The same for the last run's results in device memory (which = PS_MAP_*),
 * ground truth given on the host for every frame of the batch; use_mask != 0
 * restricts to the run's gradient mask (accuracy(prediction, gt, mask, ...)). */
ps_status ps_download_accuracy(ps_ctx* ctx, int which, const float* ground_truth,
                               const uint8_t* ground_truth_valid, int use_mask,
                               const double* thresholds, int n_thresholds, double* fractions,
                               long long* evaluated, double* mean_abs_error);

/* ------------------------------------------------- synthetic stereo pairs */
/* Seeded BASELINE-style generator; bench/test fixture, not on
 * the hot path.  gt may be NULL. */
typedef struct ps_synth_params {
    int width;
    int height;
    int n_planes;       /* random planar patches */
    int max_disparity;  /* disparities lie in [0, max_disparity-1] */
    int ground;         /* 1: bottom ground region with disparity rising with v */
    float noise_sigma;  /* Gaussian noise added to the right view */
    uint32_t seed;
} ps_synth_params;
ps_status ps_synth_pair(const ps_synth_params* params, uint8_t* left, uint8_t* right, float* gt);
/* n_frames pairs with seeds params->seed + i, generated on `threads` host threads. */
ps_status ps_synth_batch(const ps_synth_params* params, int n_frames, int threads, uint8_t* left,
                         uint8_t* right);

/* The same generator on the device (bit-identical bytes, up to a 1-ulp
 * difference of the device log/cos in the Gaussian noise, which in practice
 * never changes a rounded byte): n_frames pairs with seeds params->seed + i,
 * returned in host buffers (gt may be NULL). */
ps_status ps_synth_batch_gpu(ps_ctx* ctx, const ps_synth_params* params, int n_frames,
                             uint8_t* left, uint8_t* right, float* gt);
/* ... or generated straight into the context's batch input buffers (as if
 * ps_upload_batch had uploaded them): feeds ps_run_resident with no host
 * generation and no host->device copy. */
ps_status ps_synth_resident(ps_ctx* ctx, const ps_synth_params* params, int n_frames);

/* renderScene (proj/include/planestereo/synth.hpp:13-50, proj/src/synth.cpp:
 * 46-169) on the device: band-limited noise textures from mt19937(seed) and
 * mt19937(seed+1), the left one forward-mapped into the right by the
 * piecewise-planar ground truth (nearest wins; losers occluded, sources
 * leaving the image invalid).  Regions must partition the image (PS_ERROR
 * otherwise, with the reference's messages); a plane outside
 * [0, max_disparity) inside its region is PS_INVALID_PLANE. */
typedef struct ps_scene_region { /* SceneRegion: [u0,u1) x [v0,v1), d = a*u + b*v + c */
    int u0;
    int v0;
    int u1;
    int v1;
    double a;
    double b;
    double c;
} ps_scene_region;
ps_status ps_render_scene(ps_ctx* ctx, int width, int height, float max_disparity, uint32_t seed,
                          const ps_scene_region* regions, int n_regions, uint8_t* left,
                          uint8_t* right, float* ground_truth, uint8_t* ground_truth_valid,
                          uint8_t* occluded);

#ifdef __cplusplus
}
#endif

#endif /* PLANESTEREO_C_H */
