// pins.cpp — hull-vertex pinning decided on the host, from the exact tie rule.
//
// The reference pins every vertex pixel left uncovered by the top-left tie
// rule to its FIRST incident triangle (proj/src/mesh.cpp:109-122).  A vertex
// pixel lies on two edges of each incident triangle (edge value 0) and
// strictly inside the third, so it is covered by that triangle iff both
// incident edges accept ties (mesh.cpp:80); only hull vertices can end up
// uncovered.  mesh_pins() marks, per triangle, the corners that pin (3 bits),
// which the raster kernel stores directly.
//
// It also answers whether the triangle ORDER matters for this mesh: if all
// incident triangles of every uncovered vertex evaluate to the same binary32
// disparity there, any order reproduces the reference; if two differ
// (typically d = 0 with plane values of +-1e-17, which decides 0 <= d < ND),
// the frame must use the reference's own order (delaunay_lex).  Arithmetic is
// the reference's: fitPlane in binary64 in source order without FMA
// (mesh.cpp:12-26; this file is compiled with -ffp-contract=off), plane
// evaluation ((a*u)+(b*v))+c then a binary32 rounding (mesh.hpp:19, mesh.cpp:158).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "delaunay.hpp"

namespace ps {

namespace {

bool tie_accept(int xi, int yi, int xj, int yj) {
    // edge i->j accepts pixels on it (mesh.cpp:80)
    return (yj < yi) || (yj == yi && xj > xi);
}

float plane_at_vertex(const int* u, const int* v, const double* d, const int* t, int k) {
    const long long u1 = u[t[0]], u2 = u[t[1]], u3 = u[t[2]];
    const long long w1 = v[t[0]], w2 = v[t[1]], w3 = v[t[2]];
    const long long det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    if (det == 0) return 0.0f;
    const double d1 = d[t[0]], d2 = d[t[1]], d3 = d[t[2]];
    const double dA = d1 * double(w2 - w3) + d2 * double(w3 - w1) + d3 * double(w1 - w2);
    const double dB = double(u1) * (d2 - d3) + double(u2) * (d3 - d1) + double(u3) * (d1 - d2);
    const double dC = d1 * double(u2 * w3 - u3 * w2) - d2 * double(u1 * w3 - u3 * w1) +
                      d3 * double(u1 * w2 - u2 * w1);
    const double a = dA / double(det), b = dB / double(det), c = dC / double(det);
    const double s = a * double(u[t[k]]) + b * double(v[t[k]]);
    return float(s + c);
}

}  // namespace

// fitPlane (mesh.cpp:12-26) sums three exact products in source order; the
// sums, and with them the plane, depend on the vertex rotation only if one of
// them rounds.  Supports carry float-representable disparities, so every
// term is a multiple of 2^E (E = lowest mantissa bit over the non-zero d's);
// if every sum's magnitude bound stays below 2^(E+52), all of fitPlane's
// additions are exact and every rotation yields bit-identical planes.  Fails
// only for meshes mixing tiny (~1e-15, d = 0 plane noise) and large
// disparities in one triangle; those frames take the reference's own order
// and rotation (delaunay_lex).
bool planes_rotation_exact(const int* u, const int* v, const double* d, const int* tris, int nt) {
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        int emin = 1 << 20;
        double dmax = 0.0;
        for (int k = 0; k < 3; ++k) {
            const double x = d[tr[k]];
            if (x == 0.0) continue;
            const float fx = float(x);
            emin = std::min(emin, std::ilogb(fx) - 23);
            dmax = std::max(dmax, std::fabs(x));
        }
        if (dmax == 0.0) continue;
        double umax = 0.0, wmax = 0.0;
        for (int k = 0; k < 3; ++k) {
            umax = std::max(umax, std::fabs(double(u[tr[k]])));
            wmax = std::max(wmax, std::fabs(double(v[tr[k]])));
        }
        // |detA| <= 3*dmax*2*wmax, |detB| <= 3*umax*2*dmax, |detC| <= 3*dmax*2*umax*wmax
        const double bound = 6.0 * dmax * std::max(std::max(umax, wmax), umax * wmax) + 6.0 * dmax;
        if (bound >= std::ldexp(1.0, emin + 52)) return false;
    }
    return true;
}

bool mesh_pins(const int* u, const int* v, const double* d, int n, const int* tris, int nt,
               int width, int height, float max_disp, bool check_order,
               std::vector<uint8_t>& state, std::vector<float>& first,
               std::vector<uint8_t>& pin_bits) {
    // state: 0 = not (yet) seen uncovered, 1 = covered, 2 = uncovered and pinned
    state.assign(n, 0);
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        for (int k = 0; k < 3; ++k) {
            const int p = tr[k], q = tr[(k + 1) % 3], r = tr[(k + 2) % 3];
            if (tie_accept(u[r], v[r], u[p], v[p]) && tie_accept(u[p], v[p], u[q], v[q]))
                state[p] = 1;
        }
    }
    pin_bits.assign(nt, 0);
    if (check_order) first.assign(n, 0.0f);
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        for (int k = 0; k < 3; ++k) {
            const int p = tr[k];
            if (state[p] == 1) continue;
            if (u[p] < 0 || u[p] >= width || v[p] < 0 || v[p] >= height) continue;
            if (state[p] == 0) {
                state[p] = 2;
                pin_bits[t] |= uint8_t(1u << k);  // first incident triangle
                if (check_order) first[p] = plane_at_vertex(u, v, d, tr, k);
            } else if (check_order) {
                // Only the validity decision can propagate (sentinel vs census
                // cost -> C_f, grids, supports): two valid values differ by a
                // rounding of the exact vertex disparity (~1e-17 at d = 0) and
                // give the same lround column and cost; that residue stays in
                // D_f / dense, inside the 1e-3 px tolerance.
                const float val = plane_at_vertex(u, v, d, tr, k);
                const bool a = val >= 0.0f && val < max_disp;
                const bool b = first[p] >= 0.0f && first[p] < max_disp;
                if (a != b) return true;
            }
        }
    }
    return false;
}

}  // namespace ps
