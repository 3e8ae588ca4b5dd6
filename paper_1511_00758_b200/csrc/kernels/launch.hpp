// launch.hpp — host-side launchers of the sm_100a kernels (one per kernel
// family).  Every launcher enqueues on `st` and returns the number of kernel
// launches it issued, so the engine can report its own launch count.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "planestereo_c.h"
#include "star_layout.hpp"

namespace ps {

// K1 — gradient mask + census(L) + census(R), fused over 128x8 tiles
// (proj/src/image.cpp:43-60, proj/src/census.cpp:10-41).  Any of mask / cl /
// cr / right may be null to skip that output.  `code` (optional) receives the
// initial per-pixel C_f state of the refinement: code_high on mask pixels
// (C_f = costHigh, pipeline.cpp:146), kCodeOff elsewhere.
int launch_frontend(const uint8_t* left, const uint8_t* right, FrameGeom g, int frames,
                    int grad_threshold, uint8_t* mask, uint32_t* cl, uint32_t* cr,
                    int* mask_count, cudaStream_t st, uint8_t* code = nullptr,
                    int code_high = 0);

// K2 — segment-test corners, 12x10 binning, per-bin top-`cap` and the
// global (score desc, v, u) sort (proj/src/sparse.cpp:84-146).
// Writes cand_u/v/score[f*cand_stride + i] and cand_count[f].
// `scratch` must hold frames*120*max_bin_pixels keys when cap > 8 (else unused).
int launch_candidates(const uint8_t* left, FrameGeom g, int frames, int corner_threshold,
                      int cap, unsigned long long* bin_keys, int* bin_count,
                      unsigned long long* scratch, long long scratch_stride, int* cand_u,
                      int* cand_v, float* cand_score, int* cand_count, int cand_stride,
                      cudaStream_t st);
long long candidate_scratch_stride(FrameGeom g);

// K3 — epipolar census matching, warp per candidate (proj/src/sparse.cpp:44-80,148-195).
int launch_match(const uint32_t* cl, const uint32_t* cr, FrameGeom g, int frames, int max_disp,
                 const CostTables& tab, const int* cand_u, const int* cand_v,
                 const int* cand_count, int cand_stride, int max_candidates, uint8_t* ok,
                 int* disp, int* costk, cudaStream_t st);

// Support list compaction of match results (seed path): supports of frame f
// are written at su/sv/sd[f*scap + base[f] + k] in candidate order; taken
// bits set; out_count[f] = base[f] + accepted (base may be null = 0).
int launch_emit_matches(const int* cand_u, const int* cand_v, const int* cand_count,
                        int cand_stride, int max_candidates, const uint8_t* ok, const int* disp,
                        FrameGeom g, int frames, uint32_t* taken, int* su, int* sv, double* sd,
                        int scap, const int* base, const int* base2, int* out_count,
                        int* chunk_buf, cudaStream_t st);

// K5+K6 — per-triangle plane fit (binary64, source order, no FMA;
// proj/src/mesh.cpp:12-26) and exact top-left rasterisation into the
// triangle lookup (mesh.cpp:58-107), with hull-vertex pinning (mesh.cpp:109-122)
// given as host-computed pin bits (3 per triangle, pins.cpp; may be null).
// Triangles are flat over frames: frame f owns [tri_off[f], tri_off[f+1]).
// The lookup must be preset to -1.
int launch_mesh(const int* tris, const int* tri_off, int frames, long long total_tris,
                const int* su, const int* sv, const double* sd, int scap, FrameGeom g,
                const uint8_t* pin_bits, double* planes, int32_t* lookup, int* err_flag,
                cudaStream_t st);
// Pipeline variant: rasterises the interpolated disparity itself
// (interpolate(), mesh.cpp:149-182) instead of the triangle id: dit[px] =
// binary32 plane value when 0 <= d < max_disp, NaN for invalid or outside the
// hull.  dit must be preset to NaN (memset 0xff).  tri_pitch > 0: frame f's
// triangles (and pin bytes) sit at f * tri_pitch in the arrays (one pitched
// copy per frame group) instead of flat at tri_off[f].
int launch_mesh_disparity(const int* tris, const int* tri_off, int frames, long long total_tris,
                          const int* su, const int* sv, const double* sd, int scap, FrameGeom g,
                          const uint8_t* pin_bits, float max_disp, float* dit, int* err_flag,
                          cudaStream_t st, long long tri_pitch = 0);

// K7 (+K9 when last) — fused interpolate / costEvaluation / disparityRefinement
// with per-cell packed-key atomicMin grids and the trace reduction
// (mesh.cpp:149-182, pipeline.cpp:33-86,183-191).
struct RefineArgs {
    FrameGeom g;
    int frames;
    const uint8_t* mask;
    const float* dit;  // interpolated disparity, NaN = invalid (launch_mesh_disparity)
    const uint32_t* cl;
    const uint32_t* cr;
    float max_disp;
    int cell;
    int cols;
    int cells_per_frame;  // cells of this iteration
    int cell_stride;      // per-frame stride of the grid arrays (>= cells_per_frame)
    uint8_t* code;  // C_f per pixel as a byte code (CostTables), updated in place
    float* Df;
    uint8_t* Dv;    // LAST only: D_f validity (code < code_high)
    float* Cf;      // LAST only: C_f as binary32
    unsigned long long* Cg;
    unsigned long long* Cb;
    unsigned long long* trace_sum;  // [frames] for this iteration (stride trace_stride)
    unsigned* trace_valid;
    int trace_stride;
    float* dense;       // LAST only
    uint8_t* dense_valid;
};
int launch_refine(const RefineArgs& a, const CostTables& tab, bool last, cudaStream_t st);

// K8 — resampling: confident cells (row-major) appended as supports,
// occupied invalid cells compacted into the re-match list
// (proj/src/pipeline.cpp:88-129).  S_old[f] is the current support count.
int launch_resample_confident(const unsigned long long* Cg, int cells_per_frame, int cell_stride,
                              FrameGeom g, int frames, const float* dit, uint32_t* taken, int* su,
                              int* sv, double* sd, int scap, const int* S_old, int* conf_count,
                              int* chunk_buf, cudaStream_t st);
int launch_resample_invalid(const unsigned long long* Cb, int cells_per_frame, int cell_stride,
                            FrameGeom g, int frames, int* rem_u, int* rem_v, int rem_stride,
                            int* rem_count, int* chunk_buf, cudaStream_t st);
// S[f] = S[f] + a[f] + b[f]
int launch_add_counts(int* S, const int* a, const int* b, int frames, cudaStream_t st);

// K4 on the device (star.cu, star_dt.cuh): per-frame exact Delaunay of the
// support lists of a frame group.  Arrays are frame-strided: supports and
// per-support scratch by scap, cells by gw*gh (+1 for cell_start), triangles
// and pin bytes by pitch, flags by flag_ints.  Flags per frame: [0] fail
// (the host replays the reference sweep for that frame), [1] rotation
// suspects (4 ints each at kStarSuspectBase: triangle, v0, v1, v2), [2] ints
// used and [3] count of the ambiguous hull vertices at kStarFanBase (vertex,
// n, then n counter-clockwise triangles of 3 vertex ids), [4] collinear set,
// [5] points deferred from pass 1 (k_star) to pass 2 (k_star_far).
struct StarArgs {
    const int* su;
    const int* sv;
    const double* sd;
    int scap;
    const int* S;  // device support counts
    int frames;
    int W, H;
    float max_disp;
    int gs, gw, gh;  // grid cell size and dimensions (cells of gs x gs pixels)
    int* cell_cnt;
    int* cell_start;
    int* cell_items;
    int* cell_xy;  // per cell_items position: (v << 16) | u of that point, -1 for a duplicate
    uint8_t* dup;
    int* pin_tri;  // per support: sorted vertex set of its pinned triangle or -1
    int* tris;
    long long pitch;  // triangle capacity per frame
    uint8_t* pins;
    int* tri_count;
    int* flags;
    int flag_ints, max_suspect, fan_base;  // star_flag_layout(scap)
    unsigned long long* col_key;  // per frame 2 * W: column extremes as (v, index) keys
    int* col_idx;                 // per frame 2 * W: their point indices (-1: empty column)
    int* hull;                    // per frame 2 * scap: hull successor / predecessor per point
    int* hull_tmp;                // per frame 8 * (2 * W + 2 * H + 8) ints: monotone-chain stacks
    int* hard;                    // per frame scap: points pass 1 deferred to pass 2 (count in flags[5])
    int phase2;                   // k_star's own radius-4 phase (1), else such points go to pass 2
    int hull_late;                // k_star's hull vertices in phase 2 (1) or where pass 1 finds them (0)
    int near;                     // k_star's radius-2 steps scan the point's near set first (1) or the box rows (0)
    int* ring;                    // per support kRingInts ints: its pass-1 star (count, then the (b, c)
                                  // of each triangle (p, b, c)); count -1: none; nullptr: not kept
};
// grid + stars + triangle list + hull pins; then the rotation check; then
// (after the host fixes: {frame, 0, tri, v0, v1, v2} rotation or {frame, 1,
// vertex, s0, s1, s2} pin) the pin bits.
int launch_star_mesh(const StarArgs& a, int max_points, cudaStream_t st);
int launch_star_check(const StarArgs& a, long long max_tris, cudaStream_t st);
int launch_star_finish(const StarArgs& a, const int* fixes, int n_fix, long long max_tris,
                       cudaStream_t st);

// Packs supports [S_prev[f], S_now[f]) of every frame into out (u,v pairs)
// and out_d (disparities) at off[f].
int launch_pack_new_supports(const int* su, const int* sv, const double* sd, int scap,
                             const int* S_prev, const int* S_now, const int* off, int frames,
                             int max_new, int2* out, double* out_d, cudaStream_t st);

// Stage-API helpers (single frame, host-visible semantics).
int launch_interpolate(const int32_t* lookup, const double* planes, FrameGeom g,
                       const uint8_t* mask, float max_disp, float* value, uint8_t* valid,
                       cudaStream_t st);
int launch_cost_eval(const uint32_t* cl, const uint32_t* cr, FrameGeom g, const float* value,
                     const uint8_t* valid, const uint8_t* mask, const CostTables& tab, float* cost,
                     cudaStream_t st);

}  // namespace ps

namespace ps {
int launch_fill_f32(float* p, long long n, float x, cudaStream_t st);

// Layout of ps_cell / planestereo::OccupancyCell marshalling (pipeline.hpp:17-23).
struct StageCell {
    int u;
    int v;
    float disparity;
    float cost;
    int occupied;
};
// disparityRefinement over user maps (stage.cu): final state in place, both
// grids (ceil(W/cell) x ceil(H/cell) cells) written to out_conf / out_inv.
int launch_stage_refine(FrameGeom g, const float* interp, const uint8_t* interp_valid,
                        const float* cost, const uint8_t* mask, float* fd, uint8_t* fv, float* fc,
                        int cell, float cost_low, float cost_high, unsigned long long* kg,
                        unsigned long long* kb, StageCell* out_conf, StageCell* out_inv,
                        cudaStream_t st);
// wtaOracle (proj/src/synth.cpp:171-198) over census fields of `frames`
// frames (wta.cu): disparity / validity / cost per pixel, cost 1.0 off-mask.
int launch_wta(const uint32_t* cl, const uint32_t* cr, const uint8_t* mask, FrameGeom g, int frames,
               int max_disparity, const CostTables& tab, float* disparity, uint8_t* valid,
               float* cost, cudaStream_t st);

// Output encoders (codecs.cu): KITTI 16-bit raster (big-endian words, 0 =
// invalid; neg_first <- smallest index of a negative valid disparity), PFM
// raster (bottom-up, -1 = invalid), and the ordered point-cloud vertex list.
// frame_ok[f] == 0 marks a frame with no result (all invalid); may be null.
int launch_kitti16(const float* d, const uint8_t* valid, const int* frame_ok, long long P, int frames,
                   uint16_t* out, unsigned long long* neg_first, cudaStream_t st);
int launch_pfm(const float* d, const uint8_t* valid, const int* frame_ok, int W, int H, int frames,
               float* out, cudaStream_t st);
int launch_point_cloud(const float* d, const uint8_t* valid, const uint8_t* image, int W, int H,
                       double focal, double baseline, double cx, double cy, double min_d,
                       float* xyz, uint8_t* intensity, int capacity, int* chunk_buf, int* count,
                       cudaStream_t st);

// accuracy (proj/src/eval.cpp:19-70) over `frames` maps (accuracy.cu):
// counts[f] = {evaluated, hits[0..n_thr)} (n_thr <= 16), err_sum[f] = the
// row-major sequential binary64 error sum.  mask may be null.
int launch_accuracy(const float* pred, const uint8_t* pred_valid, const float* gt,
                    const uint8_t* gt_valid, const uint8_t* mask, long long P, int frames,
                    const double* thresholds, int n_thr, unsigned long long* counts,
                    double* err_sum, cudaStream_t st);

// On-device scene generation (synth.cpp in kernels/): mt19937 output streams
// (one CTA per seed), the BASELINE generator of host/synth.cpp (same bytes),
// and the reference's renderScene (proj/src/synth.cpp:46-169).
struct SceneRegionDev {  // SceneRegion, proj/include/planestereo/synth.hpp:13-20
    int u0, v0, u1, v1;
    double a, b, c;
};
int launch_mt_streams(const uint32_t* seeds, int streams, long long n, long long stride,
                      uint32_t* out, cudaStream_t st);
long long baseline_stream_draws(int w, int h, int n_planes);
int launch_synth_baseline(const ps_synth_params& p, int frames, const uint32_t* stream,
                          long long stride, float* disp, unsigned long long* keys, uint8_t* left,
                          uint8_t* right, long long img_stride, cudaStream_t st);
int launch_render_scene(int w, int h, float max_disp, const SceneRegionDev* regions,
                        int n_regions, const uint32_t* stream_left, const uint32_t* stream_right,
                        int* tmp_a, int* tmp_b, int* minmax, unsigned long long* keys,
                        unsigned long long* bad, uint8_t* left, uint8_t* right, float* gt,
                        uint8_t* gt_valid, uint8_t* occluded, cudaStream_t st);

}  // namespace ps
