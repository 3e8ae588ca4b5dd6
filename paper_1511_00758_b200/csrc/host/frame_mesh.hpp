// frame_mesh.hpp — one frame's mesh for one iteration, as the reference
// builds it (planestereo::triangulate + DisparityMesh, proj/src/mesh.cpp:44-147),
// without replaying the reference's lexicographic sweep when it can be avoided.
//
// What the raster consumes from the reference's mesh is (1) the triangle SET,
// (2) each triangle's plane, fitted in the vertex rotation the sweep stored
// (mesh.cpp:12-26 sums three products in source order), and (3) for each
// hull vertex pixel the tie rule leaves uncovered, the FIRST incident
// triangle in the sweep's output order (mesh.cpp:109-122).
//
//  (1) comes from IncDT: the previous iteration's triangulation plus this
//      iteration's new supports (incdt.hpp).
//  (2) matters only when the three rotations round differently; integer
//      disparities (seeds, re-matched supports) are exact, so only triangles
//      with a fractional vertex are fitted three ways, and the rare ones
//      that differ get the sweep's rotation from SweepOrder.
//  (3) matters only when the incident planes give different binary32 D_it
//      bits at the vertex (a d = 0 hull vertex: ±1e-17); then SweepOrder
//      orders the incident triangles as the sweep's slots.
// Any inconsistency falls back to the exact replay (delaunay_lex).
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "../kernels/star_layout.hpp"
#include "delaunay.hpp"
#include "incdt.hpp"
#include "sweep_order.hpp"

namespace ps {

struct MeshStats {
    long long frames = 0;      // frame-iterations meshed
    long long fallbacks = 0;   // of which replayed with delaunay_lex
    long long first_iter = 0;  //   of which first-iteration meshes (by design, not a fallback)
    long long fb_device = 0;   //   because the device mesh flagged the frame (star overflow, capacity)
    long long fb_why[5] = {0, 0, 0, 0, 0};  // device causes: fan, search, degree, suspects, capacity
    long long fb_queries = 0;  //   because the order-query budget ran out
    long long fb_resolve = 0;  //   because SweepOrder could not certify a window
    double replay_ms = 0;      // time in delaunay_lex replays
    long long ambiguous = 0;   // hull-vertex pins resolved through SweepOrder
    long long rotations = 0;   // triangles whose rotation SweepOrder decided
    long long rot_checked = 0; // triangles fitted three ways
    double dt_ms = 0, check_ms = 0, order_ms = 0;
    double rot_ms = 0, pin_ms = 0, init_ms = 0;  // of order_ms: rotations, pins, SweepOrder::init
};

struct FrameMesh {
    IncDT dt;
    std::vector<int> u, v;   // the frame's support list so far
    std::vector<double> d;
    bool lex_only = false;   // PS_DELAUNAY=lex: always replay
    // scratch
    std::vector<int> ranks, rank_of, px, py, inc, q, stored;
    std::vector<uint64_t> birth;
    std::vector<uint8_t> rot_bad;
    SweepOrder so;
    void reset() {
        dt.reset();
        u.clear();
        v.clear();
        d.clear();
    }
};

// Meshes the frame's current support list (fm.u/v/d): writes up to `cap`
// triangles (3 support indices each, in the rotation the raster must fit) to
// `tris` and one pin byte per triangle (bit k: corner k is an uncovered
// vertex pixel pinned to this triangle).  Returns the triangle count, 0 for
// a degenerate set, -1 coordinate overflow, -2 internal error, -3 capacity.
int mesh_iteration(FrameMesh& fm, int width, int height, float max_disparity, int* tris, int cap,
                   uint8_t* pins, DelaunayWorkspace& ws, MeshStats& st);

// Host side of the device mesh (kernels/star.cu): the frame's flag record
// (layout.ints ints: rotation suspects and ambiguous hull vertices, see
// launch.hpp) is resolved into fixes appended to `fixes` as
// {frame, 0, triangle, v0, v1, v2} (the sweep's stored rotation) and
// {frame, 1, vertex, s0, s1, s2} (the pinned triangle's sorted vertex set).
// Returns false when the frame should be replayed instead (query budget or
// an inconsistency).
// par (optional) runs fn(i, scratch) for i in [0, n) on any threads, each
// concurrent call with its own scratch; budget_scale multiplies the order-
// query budget (queries that run in parallel cost less latency than the
// serial replay they avoid).
using ParallelQueries = std::function<void(int, const std::function<void(int, SweepOrder::Scratch&)>&)>;
bool resolve_device_flags(FrameMesh& fm, const int* flags, const StarFlagLayout& layout, int frame, int width, int height,
                          float max_disparity, std::vector<int>& fixes, DelaunayWorkspace& ws,
                          MeshStats& st, const ParallelQueries* par = nullptr, int budget_scale = 1);

// The exact replay (delaunay_lex + the sweep's pins) into caller buffers.
int replay_mesh(FrameMesh& fm, int width, int height, int* tris, int cap, uint8_t* pins,
                DelaunayWorkspace& ws, MeshStats& st);

}  // namespace ps
