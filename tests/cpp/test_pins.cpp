// test_pins.cpp — lex_hull_pins() (hull-vertex walk over the sweep's final
// half-edges) against mesh_pins() (all triangles, pins.cpp) on random and
// lattice point sets (lattices give cocircular cells).  Host code only; run by
// tests/test_delaunay.py.
#include "delaunay.hpp"
#include <cstdio>
#include <random>
#include <vector>
#include <chrono>
int main() {
    std::mt19937 rng(1);
    long long bad = 0, sets = 0, pinned = 0;
    double t_mesh = 0, t_lex = 0;
    for (int it = 0; it < 3000; ++it) {
        const int W = 20 + rng() % 200, H = 20 + rng() % 150;
        const int n = 3 + rng() % (it < 2000 ? 60 : 3000);
        const int step = 1 + rng() % 4;
        std::vector<int> u(n), v(n);
        for (int i = 0; i < n; ++i) {
            if (it % 3 == 0) { u[i] = (rng() % (W / step)) * step; v[i] = (rng() % (H / step)) * step; }
            else { u[i] = rng() % W; v[i] = rng() % H; }
        }
        ps::DelaunayWorkspace ws; std::vector<int> tris; std::vector<uint8_t> st, p1, p2;
        const int nt = ps::delaunay_lex(u.data(), v.data(), n, tris, ws);
        if (nt <= 0) continue;
        auto a = std::chrono::steady_clock::now();
        ps::mesh_pins(u.data(), v.data(), n, tris.data(), nt, W, H, st, p1);
        auto b = std::chrono::steady_clock::now();
        ps::lex_hull_pins(ws, nt, W, H, p2);
        auto c = std::chrono::steady_clock::now();
        t_mesh += std::chrono::duration<double, std::milli>(b - a).count();
        t_lex += std::chrono::duration<double, std::milli>(c - b).count();
        ++sets;
        for (int t = 0; t < nt; ++t) pinned += p1[t] != 0;
        if (p1 != p2) { ++bad; if (bad < 5) printf("mismatch set %d n=%d nt=%d\n", it, n, nt); }
    }
    printf("sets %lld mismatches %lld pinned-tris %lld  mesh_pins %.2f ms  lex_hull_pins %.2f ms\n", sets, bad, pinned, t_mesh, t_lex);
    return bad != 0;
}
