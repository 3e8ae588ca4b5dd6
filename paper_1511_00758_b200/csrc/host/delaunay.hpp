// delaunay.hpp — exact Delaunay triangulation of integer pixel coordinates.
//
// Replaces planestereo::delaunayTriangulate (proj/src/delaunay.cpp:288-325).
// Contract: the output TRIANGLE SET equals the reference's;
// triangle order and per-triangle rotation are not contractual.  The set is
// the unique Delaunay subdivision with every cocircular cell triangulated so
// that each interior diagonal avoids the lexicographically largest vertex of
// its quad — what a lexicographic insertion with strict in-circle flips
// produces, because the newly inserted point is always the lexicographic
// maximum of every quad it tests.
#pragma once

#include <cstdint>
#include <vector>

namespace ps {

// One triangle slot of the lexicographic sweep (delaunay_lex.cpp).
struct alignas(32) LexTri {
    int v[3];
    int n[3];
    int pad[2];
};

struct DelaunayWorkspace {
    std::vector<uint64_t> key, key_tmp;
    std::vector<int> ord, ord_tmp;
    std::vector<int> kept;
    std::vector<int> px, py;
    std::vector<int> tv, tn;  // triangle vertices / neighbour half-edges (radial sweep)
    std::vector<LexTri> lex;  // triangle slots (lexicographic sweep)
    std::vector<int> hnext, hprev, hedge;
    std::vector<int> stack;
    std::vector<uint8_t> covered;  // mesh_pins scratch
    std::vector<float> first;
};

// Lexicographic (u, v) order with coincident points removed, first
// occurrence kept (delaunay.cpp:296-311): ws.kept[0..m) = original indices.
void lex_order(const int* u, const int* v, int n, DelaunayWorkspace& ws, int& minx, int& miny,
               int& m, int& spanx, int& spany);

// Returns the number of triangles (index triples into the input written to
// `tris`, 3 ints each, positively oriented: orient2d > 0), 0 for fewer than
// three distinct points or a collinear set, -1 if a coordinate has
// |c| >= 2^20 (the reference's exactness bound, delaunay.cpp:289-294).
int delaunay(const int* u, const int* v, int n, std::vector<int>& tris, DelaunayWorkspace& ws);

// Same set, in the reference's own triangle order and rotation (lexicographic
// sweep, delaunay_lex.cpp): ~4x more in-circle tests than the radial sweep,
// but cache-friendly, so only ~15% slower; the engine uses it because the
// order decides hull-vertex pins and the rotation decides fitPlane rounding.
int delaunay_lex(const int* u, const int* v, int n, std::vector<int>& tris, DelaunayWorkspace& ws);
// The same into a caller buffer of capacity triangles (3 ints each); -3 when
// the triangulation has more.
int delaunay_lex(const int* u, const int* v, int n, int* tris, int capacity, DelaunayWorkspace& ws);

// Hull-vertex pinning (mesh.cpp:109-122) for this triangle list: pin_bits[t]
// bit k set when corner k of triangle t is an uncovered vertex pixel whose
// first incident triangle is t (pins.cpp).
// The same pin bits for the triangulation delaunay_lex() just left in `ws`
// (its triangle list, ntri triangles), visiting only hull vertices.
void lex_hull_pins(const DelaunayWorkspace& ws, int ntri, int width, int height,
                   std::vector<uint8_t>& pin_bits);
void lex_hull_pins(const DelaunayWorkspace& ws, int ntri, int width, int height, uint8_t* pin_bits);

void mesh_pins(const int* u, const int* v, int n, const int* tris, int nt, int width, int height,
               std::vector<uint8_t>& state, std::vector<uint8_t>& pin_bits);

}  // namespace ps
