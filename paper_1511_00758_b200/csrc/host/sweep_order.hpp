// sweep_order.hpp — the reference sweep's slot order and vertex rotation of
// individual triangles, without replaying the sweep.
//
// planestereo::delaunayTriangulate (proj/src/delaunay.cpp:50-325) inserts the
// points in lexicographic order; every insertion appends one triangle slot per
// strictly visible hull edge (:196-208) and rewrites existing slots in place by
// Lawson flips (:221-274).  The output is the slot array, so a triangle's
// position in the list (which decides hull-vertex pins, mesh.cpp:109-122) and
// its stored vertex rotation (which can decide fitPlane's rounding,
// mesh.cpp:12-26) are history, not geometry.  Three facts make that history
// local:
//
//  1. The triangles a point p destroys are its strict-in-circle cavity in
//     DT(Q<p), the Delaunay triangulation of the points before p, and that
//     cavity is a tree hanging off the fan, so the flip ORDER does not matter.
//  2. A flip (a,b,p)+(b,a,d) -> (a,d,p)+(d,b,p) keeps, in each slot, the
//     origin of the half-edge opposite p at its position: a fan slot of p keeps
//     the hull vertex x_{j+1}; a destroyed slot keeps the apex d it was entered
//     at, one position further on.  So a final triangle (t, p, o) (p its
//     lexicographic maximum, o the vertex after p counter-clockwise) sits in
//     the fan slot j of p when o = x_{j+1} on p's visible hull chain, and
//     otherwise in the slot of sigma, the triangle of DT(Q<p) at o that
//     contains the direction o -> p, with o moved one position forward.
//  3. DT(Q<p) near o is the Delaunay triangulation of the prefix points in a
//     window around o, certified by checking that no prefix point outside the
//     window lies in sigma's closed circumdisk (the triangulation is the
//     unique one of the lex-max perturbed in-circle test, delaunay.cpp).
//
// query() follows that chain back to a fan slot, then unwinds the rotations.
// The slot index order is the order of (birth point rank, fan position).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "delaunay.hpp"

namespace ps {

class SweepOrder {
public:
    // Mutable state of one query (window points, replay slots and history):
    // queries on the same SweepOrder may run concurrently, one Scratch each.
    struct Scratch;

    // px/py: the lexicographically sorted, deduplicated points (ranks 0..m-1).
    void init(const int* px, const int* py, int m);
    // Triangle with ranks (a, b, c), counter-clockwise (orient > 0), of the
    // final triangulation.  On success: birth = (rank << 32) | fan position of
    // the slot the sweep leaves it in (ordered like the slot indices), and
    // stored[0..2] = its ranks in the sweep's stored rotation.  Returns false
    // if the chain could not be followed (the caller then replays the sweep).
    bool query(int a, int b, int c, uint64_t& birth, int stored[3]) { return query(a, b, c, birth, stored, own()); }
    bool query(int a, int b, int c, uint64_t& birth, int stored[3], Scratch& S) const;
    bool query_steps(int a, int b, int c, uint64_t& birth, int stored[3], Scratch& S, int max_steps,
                     bool& more) const;

    // The same for a group of final triangles (ranks, counter-clockwise, 3 per
    // triangle) by replaying the sweep on the points of a window around them
    // and following each triangle's slot history there, every history entry
    // certified against the full prefix (no prefix point outside the window
    // in its closed circumdisk) and every fan birth checked against the full
    // hull; the window doubles until all certify.  Returns false only when
    // even the whole set fails (an inconsistency: the caller replays).
    bool resolve(const int* tris, int count, uint64_t* birth, int* stored) {
        return resolve(tris, count, birth, stored, own());
    }
    bool resolve(const int* tris, int count, uint64_t* birth, int* stored, Scratch& S) const;

    // the scratch of the single-threaded entry points (and their statistics)
    Scratch& scratch() { return own(); }
    const Scratch& stats() { return own(); }

private:
    long long orient(int a, int b, int c) const {
        return ((long long)x_[b] - x_[a]) * ((long long)y_[c] - y_[a]) -
               ((long long)y_[b] - y_[a]) * ((long long)x_[c] - x_[a]);
    }
    int incircle(int a, int b, int c, int d) const;  // exact sign
    int hull_prev(int o, int p) const;                     // CCW predecessor of o on hull(Q<p), -1 if none
    int fan_index(int o, int p) const;                     // j with o = x_{j+1} on p's visible chain, else -1
    bool window_triangle(int o, int p, int out[3], Scratch& S) const;  // sigma (ranks, CCW)
    // true if no point of rank < p outside the box [u0,u1]x[v0,v1] lies in the
    // closed circumdisk of the CCW triangle (a, b, c); grows the box to cover
    // the offenders otherwise
    bool disk_clear(int a, int b, int c, int p, int& u0, int& u1, int& v0, int& v1, int grow) const;
    bool replay(int u0, int u1, int v0, int v1, int last, Scratch& S) const;  // ranks <= last only
    bool resolve_windows(const int* tris, int count, uint64_t* birth, int* stored, Scratch& S) const;  // lex sweep of the window's points, with slot history

    const int* x_ = nullptr;
    const int* y_ = nullptr;
    int m_ = 0;
    int apex_ = -1;   // first point off the leading collinear run (delaunay.cpp:67-79)
    bool side_pos_ = true;
    int minx_ = 0, maxx_ = 0, miny_ = 0, maxy_ = 0;
    bool wide_ = false;
    // Andrew's monotone chains over the lexicographic order, collinear points
    // kept: below pointers are set at push time, so the chain at time p is the
    // list reachable from p - 1; pop time = rank whose processing removed it.
    std::vector<int> belowL_, popL_, belowU_, popU_;
    // bucket grid of ranks (increasing within a bucket)
    int bs_ = 16, bw_ = 0, bh_ = 0;
    std::vector<int> bstart_, bitems_;
    std::vector<int> stk_, bcell_, bfill_;  // init scratch
    Scratch& own();
    std::unique_ptr<Scratch> own_;
};

struct SweepOrder::Scratch {
    std::vector<int> wu_, wv_, wrank_, wtris_;  // window points
    // replay state (window ranks; slot = 4 * index, half-edge = 4 * slot + k)
    struct Slot {
        int v[3];
        int n[3];
        int birth;  // window index of the inserting point (apex for the leading fan)
        int fan;    // fan position within the window's visible chain
        int hist;   // latest history entry, -1 if never eaten
        int eaten;  // window index of the last point that ate it
        int x0;     // a fan slot's first hull vertex x_j at birth (window index)
    };
    struct Hist {
        int time;   // window index of the eating point
        int v[3];   // contents just before it was eaten
        int prev;
    };
    std::vector<Slot> rs_;
    std::vector<Hist> rh_;
    std::vector<int> rrank_, rhn_, rhp_, rhe_, rstack_;
    int rapex_ = -1;
    DelaunayWorkspace ws_;
    long long window_points = 0, replay_points = 0;  // statistics
    int windows = 0, replays = 0;
    long long fast_calls = 0, fast_hits = 0;  // resolve() calls, triangles answered without a window
};

}  // namespace ps
