/*
 * ps_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithm for the planestereo hot
 * path (/root/reference/proj, cited file:line relative to proj/).  It is the
 * parity checker for the CUDA product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product library never links or calls it.
 *
 * Pinned against the reference itself: oracle/Makefile also compiles the
 * reference sources into oracle/_ref/libps_ref.so (same entry points with an
 * `ref_` prefix, see ref_shim.cpp) and tests/test_oracle.py diffs the two on
 * seeded inputs and on the committed golden fixtures in tests/golden/.
 */
#ifndef PS_ORACLE_H
#define PS_ORACLE_H

#include <stdint.h>

#include "planestereo_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* gradientMask, proj/src/image.cpp:43-60. Returns M. */
int orc_gradient_mask(const uint8_t* img, int w, int h, int threshold, uint8_t* member);
/* censusTransform, proj/src/census.cpp:10-41. */
void orc_census(const uint8_t* img, int w, int h, uint32_t* out);
/* detectCandidates, proj/src/sparse.cpp:84-146. Returns count (<= cap). */
int orc_detect_candidates(const uint8_t* img, int w, int h, const ps_config* cfg, int* u, int* v,
                          float* score, int cap);
/* matchEpipolar (census overload), proj/src/sparse.cpp:148-195. Returns count. */
int orc_match_epipolar(const uint32_t* cl, const uint32_t* cr, int w, int h, const int* cu,
                       const int* cv, int n, const ps_config* cfg, int* su, int* sv, double* sd);
/* orient2d / inCircleSign, proj/src/delaunay.cpp:11-41. */
long long orc_orient2d(int au, int av, int bu, int bv, int cu, int cv);
int orc_incircle_sign(int au, int av, int bu, int bv, int cu, int cv, int du, int dv);
/* delaunayTriangulate, proj/src/delaunay.cpp:288-325.  tris needs room for
 * 3*(2n) ints.  Returns the triangle count, -1 on coordinate overflow. */
int orc_delaunay(const int* u, const int* v, int n, int* tris);
/* fitPlane, proj/src/mesh.cpp:12-26.  Returns 0, or -1 if degenerate. */
int orc_fit_plane(int u1, int v1, double d1, int u2, int v2, double d2, int u3, int v3, double d3,
                  double* abc);
/* DisparityMesh ctor + rasterize, proj/src/mesh.cpp:44-123. Returns 0 / -1. */
int orc_mesh_build(const int* u, const int* v, const double* d, const int* tris, int nt, int w,
                   int h, double* planes, int32_t* lookup);
/* interpolate, proj/src/mesh.cpp:149-182 (mask NULL = full image). */
void orc_interpolate(const int32_t* lookup, const double* planes, int w, int h,
                     const uint8_t* mask, float max_disparity, float* value, uint8_t* valid);
/* costEvaluation, proj/src/pipeline.cpp:33-54. */
/* wtaOracle, proj/src/synth.cpp:171-198: per mask pixel the first cost-minimal
 * d in [0, min(nd, u - 2)]; cost 1.0 and invalid elsewhere. */
void orc_wta(const uint8_t* left, const uint8_t* right, int w, int h, const uint8_t* mask, int nd,
             float* disparity, uint8_t* valid, float* cost);
/* Output encoders of proj/src/io.cpp (rasters only; the containers are text).
 * writeKittiPng :349-368 -> 2 bytes/pixel big-endian, returns the index of
 * the first negative valid disparity (row-major) or -1. */
long long orc_encode_kitti16(const float* d, const uint8_t* valid, int w, int h, uint8_t* out);
/* writePfm :311-329 -> rows bottom-up, invalid -1.0 */
void orc_encode_pfm(const float* d, const uint8_t* valid, int w, int h, float* out);
/* exportPointCloud :395-454 -> vertex count (xyz, intensity), -1 for a bad
 * calibration (InvalidConfig); count 0 is the caller's EmptyCloud. */
int orc_point_cloud(const float* d, const uint8_t* valid, const uint8_t* image, int w, int h,
                    const ps_calib* calib, double min_disparity, float* xyz, uint8_t* intensity);
/* accuracy, proj/src/eval.cpp:19-59 (mask may be NULL): PS_NO_OVERLAP when
 * no pixel is jointly valid. */
int orc_accuracy(const float* pred, const uint8_t* pred_valid, const float* gt,
                 const uint8_t* gt_valid, const uint8_t* mask, int w, int h,
                 const double* thresholds, int n_thr, double* fractions, long long* evaluated,
                 double* mean_abs_error);
void orc_cost_evaluation(const uint32_t* cl, const uint32_t* cr, int w, int h, const float* value,
                         const uint8_t* valid, const uint8_t* mask, float* cost);
/* disparityRefinement, proj/src/pipeline.cpp:56-86. */
void orc_refinement(const float* value, const uint8_t* valid, const float* cost, float* fd,
                    uint8_t* fv, float* fc, const uint8_t* mask, int w, int h, int cell,
                    const ps_config* cfg, ps_cell* confident, ps_cell* invalid);
/* supportResampling, proj/src/pipeline.cpp:88-129. Returns the new count. */
int orc_support_resampling(const ps_cell* confident, const ps_cell* invalid, int cell,
                           const int* su, const int* sv, const double* sd, int n,
                           const uint32_t* cl, const uint32_t* cr, int w, int h,
                           const ps_config* cfg, int* ou, int* ov, double* od, int cap);
/* Staged run(): proj/src/pipeline.cpp:131-203 with validate() optional
 * (validate=0 skips it entirely, as SURVEY App. B's staged driver does).
 * Returns a ps_status.  sup_* receive the last iteration's support list. */
int orc_run(const uint8_t* left, const uint8_t* right, int w, int h, const ps_config* cfg,
            int validate, float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
            uint8_t* dense_valid, ps_iter_stats* trace, int* sup_u, int* sup_v, double* sup_d,
            int sup_cap, int* sup_count);
/* n frames (stride w*h) on `threads` host threads, one frame per thread at a
 * time; outputs as orc_run (any may be NULL).  Used for the CPU baseline. */
int orc_run_batch(int n, const uint8_t* left, const uint8_t* right, int w, int h,
                  const ps_config* cfg, int threads, float* disparity, uint8_t* disparity_valid,
                  float* cost, float* dense, uint8_t* dense_valid, int* status);

#ifdef __cplusplus
}
#endif

#endif
