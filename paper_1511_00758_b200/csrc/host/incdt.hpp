// incdt.hpp — incremental exact Delaunay triangulation of a growing support
// list, one per frame, kept across the iterations of a run.
//
// planestereo::run re-triangulates the whole support list every iteration
// (proj/src/pipeline.cpp:161 -> delaunayTriangulate, delaunay.cpp:288-325),
// and the list only grows: iteration i+1's supports are iteration i's plus
// the resampled ones (pipeline.cpp:88-129).  The triangle SET is the unique
// Delaunay triangulation under the lexicographic-maximum perturbation of the
// in-circle test (delaunay.cpp here), which does not depend
// on the insertion order, so each iteration only inserts its new supports
// into the previous triangulation: point location by a visibility walk from
// the last insertion (new supports arrive in row-major cell order), a 1->3,
// 2->4 or hull fan split, then Lawson flips with the perturbed predicate.
// Coincident points keep the first occurrence (delaunay.cpp:303-311).
#pragma once

#include <cstdint>
#include <vector>

namespace ps {

class IncDT {
public:
    // Forget everything (a new frame / run).
    void reset();
    // Append the points idx0..n-1 of (u, v) (indices into the frame's support
    // list; the arrays hold every support so far) to the triangulation.
    // Returns false on a coordinate >= 2^20 (the reference's bound) or an
    // internal inconsistency.
    bool extend(const int* u, const int* v, int n);

    int triangles() const { return int(T_.size()); }
    // triangle t: vertices (counter-clockwise) and twin half-edges; half-edge
    // e = 4t + k runs from vertex k to vertex k+1 (mod 3), -1 = hull
    int vert(int t, int k) const { return T_[t].v[k]; }
    int twin(int e) const { return T_[e >> 2].n[e & 3]; }
    int hull_start() const { return hull0_; }      // a hull vertex, -1 if < 1 triangle
    int hull_next(int v) const { return hnext_[v]; }
    int hull_edge(int v) const { return hedge_[v]; }  // half-edge v -> hull_next(v)
    bool degenerate() const { return T_.empty(); }  // fewer than 3 non-collinear points

    long long flips = 0, tests = 0, walk_steps = 0, stale = 0;  // statistics

private:
    struct alignas(32) Tri {
        int v[3];
        int n[3];
        int pad[2];
    };
    struct Pt {
        int x, y;
    };
    int& V(int e) { return T_[e >> 2].v[e & 3]; }
    int& N(int e) { return T_[e >> 2].n[e & 3]; }
    long long orient(int a, int b, int c) const {
        const Pt A = P_[a], B = P_[b], C = P_[c];
        return ((long long)B.x - A.x) * ((long long)C.y - A.y) - ((long long)B.y - A.y) * ((long long)C.x - A.x);
    }
    bool inside(int a, int b, int c, int d);  // perturbed strict in-circle
    int add(int a, int b, int c, int na, int nb, int nc);
    void link(int e, int f) {
        N(e) = f;
        if (f >= 0) N(f) = e;
    }
    void legalize();
    bool insert(int p);
    bool start(int n);  // first non-degenerate triangle from the pending points

    std::vector<Pt> P_;  // points seen so far (indices < nv_)
    int nv_ = 0;
    bool wide_ = false;
    std::vector<Tri> T_;
    std::vector<int> hnext_, hprev_, hedge_;
    std::vector<int> stack_;
    std::vector<int> pending_;  // points waiting for a non-degenerate start
    // walk starts: a triangle holding each vertex when it was inserted (may go
    // stale; checked before use) and the last vertex inserted per 8x8 bucket
    std::vector<int> vtri_, bucket_;
    int bx0_ = 0, by0_ = 0, bw_ = 0, bh_ = 0;
    int last_ = 0;  // triangle to start walks from otherwise
    int lastp_ = -1;  // the last point inserted
    int hull0_ = -1;
};

}  // namespace ps
