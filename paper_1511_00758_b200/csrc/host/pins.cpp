// pins.cpp — hull-vertex pinning decided on the host, from the exact tie rule.
//
// The reference pins every vertex pixel left uncovered by the top-left tie
// rule to its FIRST incident triangle (proj/src/mesh.cpp:109-122).  A vertex
// pixel lies on two edges of each incident triangle (edge value 0) and
// strictly inside the third, so it is covered by that triangle iff both
// incident edges accept ties (mesh.cpp:80); only hull vertices can end up
// uncovered.  mesh_pins() marks, per triangle, the corners that pin (3 bits),
// which the raster kernel stores directly (no atomics, no extra pass).
//
// "First" is in the triangle order of the list; the engine triangulates with
// delaunay_lex(), whose order and vertex rotation are the reference's, so the
// pinned triangle — and with it the sign of a plane value of +-1e-17 at a
// d = 0 hull vertex, which decides its validity — is the reference's.
#include <vector>

#include "delaunay.hpp"

namespace ps {

namespace {

bool tie_accept(int xi, int yi, int xj, int yj) {
    // edge i->j accepts pixels on it (mesh.cpp:80)
    return (yj < yi) || (yj == yi && xj > xi);
}

}  // namespace

void mesh_pins(const int* u, const int* v, int n, const int* tris, int nt, int width, int height,
               std::vector<uint8_t>& state, std::vector<uint8_t>& pin_bits) {
    // state: 0 = uncovered and not yet pinned, 1 = covered, 2 = pinned
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
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        for (int k = 0; k < 3; ++k) {
            const int p = tr[k];
            if (state[p] != 0) continue;
            if (u[p] < 0 || u[p] >= width || v[p] < 0 || v[p] >= height) continue;
            state[p] = 2;
            pin_bits[t] |= uint8_t(1u << k);  // first incident triangle
        }
    }
}

}  // namespace ps
