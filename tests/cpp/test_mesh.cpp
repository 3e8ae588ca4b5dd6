// test_mesh.cpp — host mesh builder (frame_mesh.cpp) against the exact
// reference-order sweep (delaunay_lex, itself checked array-for-array against
// the compiled reference in tests/test_delaunay.py).
//
//   test_mesh [--synthetic N] synthetic sets (N, default 1500) (lattices, random, fractional and
//                             tiny disparities, d = 0 hull vertices), grown in
//                             several batches like the pipeline's support list
//   test_mesh FILE.sup ...    support lists dumped from pipeline runs
//                             (tests/test_mesh.py writes them with the oracle)
//
// Checks, per set and batch:
//  * SweepOrder::resolve on the triangles around sampled vertices gives the
//    sweep's slot order and stored rotation;
//  * mesh_iteration's triangles are the same set, each plane (fitPlane's three
//    numerators) has the same bits as in the sweep's rotation or, where the
//    rotations round differently, gives the same binary32 D_it at every pixel
//    the triangle covers, and every uncovered hull-vertex pixel gets the same
//    D_it bits as the sweep's pin.
// Prints "ok <sets> <checks>" and exits 0, or prints the first failures.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <vector>

#include "delaunay.hpp"
#include "frame_mesh.hpp"
#include "sweep_order.hpp"

using namespace ps;

namespace {

int failures = 0;
long long checks = 0, sets = 0;

struct Plane {
    double A, B, C;
    long long det;
};

Plane fitp(const std::vector<int>& u, const std::vector<int>& v, const std::vector<double>& d, int i,
           int j, int k) {
    const long long u1 = u[i], u2 = u[j], u3 = u[k], w1 = v[i], w2 = v[j], w3 = v[k];
    const double d1 = d[i], d2 = d[j], d3 = d[k];
    Plane p;
    p.det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    p.A = d1 * double(w2 - w3) + d2 * double(w3 - w1) + d3 * double(w1 - w2);
    p.B = double(u1) * (d2 - d3) + double(u2) * (d3 - d1) + double(u3) * (d1 - d2);
    p.C = d1 * double(u2 * w3 - u3 * w2) - d2 * double(u1 * w3 - u3 * w1) + d3 * double(u1 * w2 - u2 * w1);
    return p;
}

uint32_t dit(const Plane& p, int u, int v, float nd) {
    const double a = p.A / double(p.det), b = p.B / double(p.det), c = p.C / double(p.det);
    const float x = float((a * u + b * v) + c);
    if (!(x >= 0.0f && x < nd)) return 0x7fc00000u;
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    return bits;
}

long long floor_div(long long a, long long b) {
    long long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

// D_it bits of plane pa vs pb at every pixel the triangle covers under the
// top-left rule (mesh.cpp:58-104) and at its vertex pixels
bool same_dit(const std::vector<int>& u, const std::vector<int>& v, const int* t, const Plane& pa,
              const Plane& pb, int W, int H, float nd) {
    const int x[3] = {u[t[0]], u[t[1]], u[t[2]]}, y[3] = {v[t[0]], v[t[1]], v[t[2]]};
    for (int q = 0; q < 3; ++q)
        if (dit(pa, x[q], y[q], nd) != dit(pb, x[q], y[q], nd)) return false;
    for (int vv = std::max(0, std::min({y[0], y[1], y[2]})); vv <= std::min(H - 1, std::max({y[0], y[1], y[2]})); ++vv) {
        long long lo = 0, hi = W - 1;
        bool empty = false;
        for (int a = 0; a < 3 && !empty; ++a) {
            const int b = (a + 1) % 3;
            const long long A = y[a] - y[b];
            const long long bias = ((y[b] < y[a]) || (y[b] == y[a] && x[b] > x[a])) ? 0 : 1;
            const long long K = (long long)(x[b] - x[a]) * (vv - y[a]) + (long long)(y[b] - y[a]) * x[a];
            if (A > 0) lo = std::max(lo, -floor_div(K - bias, A));
            else if (A < 0) hi = std::min(hi, floor_div(K - bias, -A));
            else if (K < bias) empty = true;
        }
        for (long long uu = lo; !empty && uu <= hi; ++uu)
            if (dit(pa, int(uu), vv, nd) != dit(pb, int(uu), vv, nd)) return false;
    }
    return true;
}

std::array<int, 3> key(const int* t) {
    std::array<int, 3> k = {t[0], t[1], t[2]};
    std::sort(k.begin(), k.end());
    return k;
}

void fail(const char* tag, const char* what) {
    if (++failures <= 10) std::printf("FAIL %s: %s\n", tag, what);
}

// mesh_iteration vs delaunay_lex + lex_hull_pins on one support list
void compare_mesh(FrameMesh& fm, int W, int H, float nd, const char* tag) {
    const int n = int(fm.u.size());
    const int cap = 2 * n + 8;
    std::vector<int> ta(3 * size_t(cap)), tb(3 * size_t(cap));
    std::vector<uint8_t> pa(cap), pb(cap);
    DelaunayWorkspace wa, wb;
    MeshStats st;
    const int na = mesh_iteration(fm, W, H, nd, ta.data(), cap, pa.data(), wa, st);
    if (std::getenv("TEST_MESH_VERBOSE"))
        std::printf("  stats: rot_checked %lld rotations %lld ambiguous %lld fallbacks %lld order %.1f ms replays %d pts %lld windows %d\n",
                    st.rot_checked, st.rotations, st.ambiguous, st.fallbacks, st.order_ms, fm.so.stats().replays, fm.so.stats().replay_points, fm.so.stats().windows);
    const int nb = delaunay_lex(fm.u.data(), fm.v.data(), n, tb.data(), cap, wb);
    if (nb > 0) lex_hull_pins(wb, nb, W, H, pb.data());
    ++sets;
    if (na != nb) return fail(tag, "triangle count");
    std::map<std::array<int, 3>, int> where;
    for (int t = 0; t < nb; ++t) where[key(&tb[3 * t])] = t;
    std::map<int, uint32_t> pin_a, pin_b;  // vertex -> pinned D_it bits
    for (int t = 0; t < na; ++t) {
        auto it = where.find(key(&ta[3 * t]));
        ++checks;
        if (it == where.end()) return fail(tag, "triangle set");
        const int s = it->second;
        const Plane pa_ = fitp(fm.u, fm.v, fm.d, ta[3 * t], ta[3 * t + 1], ta[3 * t + 2]);
        const Plane pb_ = fitp(fm.u, fm.v, fm.d, tb[3 * s], tb[3 * s + 1], tb[3 * s + 2]);
        if ((std::memcmp(&pa_.A, &pb_.A, 8) || std::memcmp(&pa_.B, &pb_.B, 8) || std::memcmp(&pa_.C, &pb_.C, 8)) &&
            !same_dit(fm.u, fm.v, &ta[3 * t], pa_, pb_, W, H, nd))
            return fail(tag, "D_it of a rotation-dependent plane");
        for (int k = 0; k < 3; ++k) {
            if (pa[t] >> k & 1) pin_a[ta[3 * t + k]] = dit(pa_, fm.u[ta[3 * t + k]], fm.v[ta[3 * t + k]], nd);
            if (pb[s] >> k & 1) pin_b[tb[3 * s + k]] = dit(pb_, fm.u[tb[3 * s + k]], fm.v[tb[3 * s + k]], nd);
        }
    }
    ++checks;
    if (pin_a != pin_b) return fail(tag, "pinned hull-vertex D_it");
}

// SweepOrder::resolve on the triangles around sampled vertices vs the sweep
void compare_order(const std::vector<int>& u, const std::vector<int>& v, int stride, const char* tag) {
    const int n = int(u.size());
    DelaunayWorkspace ws;
    std::vector<int> tb;
    const int nt = delaunay_lex(u.data(), v.data(), n, tb, ws);
    if (nt <= 0) return;
    int minx, miny, m, sx, sy;
    DelaunayWorkspace wo;
    lex_order(u.data(), v.data(), n, wo, minx, miny, m, sx, sy);
    std::vector<int> rank_of(n, -1), px(m), py(m);
    for (int r = 0; r < m; ++r) {
        rank_of[wo.kept[r]] = r;
        px[r] = u[wo.kept[r]];
        py[r] = v[wo.kept[r]];
    }
    SweepOrder so;
    so.init(px.data(), py.data(), m);
    std::vector<std::vector<int>> inc(n);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) inc[tb[3 * t + k]].push_back(t);
    ++sets;
    for (int x = 0; x < n; x += stride) {
        if (inc[x].empty()) continue;
        std::vector<int> q, s(3 * inc[x].size());
        std::vector<uint64_t> b(inc[x].size());
        for (int t : inc[x]) {
            // present each triangle starting at its smallest rank (not the sweep's rotation)
            int r[3] = {rank_of[tb[3 * t]], rank_of[tb[3 * t + 1]], rank_of[tb[3 * t + 2]]};
            int k = 0;
            if (r[1] < r[k]) k = 1;
            if (r[2] < r[k]) k = 2;
            for (int j = 0; j < 3; ++j) q.push_back(r[(k + j) % 3]);
        }
        if (!so.resolve(q.data(), int(inc[x].size()), b.data(), s.data())) return fail(tag, "resolve failed");
        for (size_t i = 0; i < inc[x].size(); ++i) {
            const int t = inc[x][i];
            ++checks;
            for (int k = 0; k < 3; ++k)
                if (wo.kept[s[3 * i + k]] != tb[3 * t + k]) return fail(tag, "stored rotation");
            for (size_t j = 0; j < inc[x].size(); ++j)
                if ((inc[x][j] < t) != (b[j] < b[i])) return fail(tag, "slot order");
        }
    }
}

float pick_d(std::mt19937& rng, float nd, int tiny_odds) {
    if (rng() % tiny_odds == 0) return float(std::ldexp(double(rng() % 1000 + 1), -60));  // tiny (rotation)
    switch (rng() % 8) {
    case 0: return 0.0f;                                   // d = 0 supports (pins)
    case 1: return float(rng() % 3);
    case 2: return float(std::ldexp(double(rng() % 7 + 1), -2));
    case 3: case 4: return float(rng() % int(nd));
    default: return float((rng() % 100000) / 100000.0 * nd);
    }
}

void synthetic(int count) {
    std::mt19937 rng(20261020);
    for (int it = 0; it < count; ++it) {
        const int W = 24 + rng() % 80, H = 16 + rng() % 60;
        const float nd = float(4 + rng() % 60);
        const int step = 1 + rng() % 4;
        // tiny disparities (rotation-dependent planes) are rare in real meshes;
        // a few sets have many, which exercises the replay fallback
        const int tiny_odds = it % 10 == 0 ? 8 : 400;
        FrameMesh fm;
        fm.reset();
        std::vector<int> cuts;
        // three batches: coarse lattice, finer lattice, random fill
        for (int b = 0; b < 3; ++b) {
            const int s = b == 0 ? 3 * step : b == 1 ? step + 1 : 1;
            for (int y = 2; y < H - 2; y += s)
                for (int x = 2; x < W - 2; x += s)
                    if (rng() % 3 != 0) {
                        fm.u.push_back(x + (b == 2 ? int(rng() % 2) : 0));
                        fm.v.push_back(y);
                        fm.d.push_back(double(pick_d(rng, nd, tiny_odds)));
                    }
            if (rng() % 4 == 0 && !fm.u.empty()) {  // a duplicate coordinate
                const int k = rng() % fm.u.size();
                fm.u.push_back(fm.u[k]);
                fm.v.push_back(fm.v[k]);
                fm.d.push_back(double(pick_d(rng, nd, tiny_odds)));
            }
            if (fm.u.size() < 3) continue;
            char tag[64];
            std::snprintf(tag, sizeof tag, "synthetic %d batch %d", it, b);
            if (std::getenv("TEST_MESH_VERBOSE")) { std::printf("%s n=%zu\n", tag, fm.u.size()); std::fflush(stdout); }
            compare_mesh(fm, W, H, nd, tag);
            if (std::getenv("TEST_MESH_VERBOSE")) { std::printf("  mesh done\n"); std::fflush(stdout); }
            if (b == 2 && it % 5 == 0) compare_order(fm.u, fm.v, std::max<int>(1, int(fm.u.size()) / 200), tag);
        }
    }
}

void from_file(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(path, "cannot open");
    int hdr[5];
    bool ok = std::fread(hdr, 4, 5, f) == 5;
    const int W = hdr[0], H = hdr[1], ND = hdr[2], its = hdr[3], n = hdr[4];
    std::vector<int> cnt(its), u(n), v(n);
    std::vector<double> d(n);
    ok = ok && std::fread(cnt.data(), 4, its, f) == size_t(its) && std::fread(u.data(), 4, n, f) == size_t(n) &&
         std::fread(v.data(), 4, n, f) == size_t(n) && std::fread(d.data(), 8, n, f) == size_t(n);
    std::fclose(f);
    if (!ok) return fail(path, "short file");
    FrameMesh fm;
    fm.reset();
    for (int i = 0; i < its; ++i) {
        fm.u.assign(u.begin(), u.begin() + cnt[i]);
        fm.v.assign(v.begin(), v.begin() + cnt[i]);
        fm.d.assign(d.begin(), d.begin() + cnt[i]);
        char tag[256];
        std::snprintf(tag, sizeof tag, "%s iteration %d", path, i + 1);
        compare_mesh(fm, W, H, float(ND), tag);
    }
    std::vector<int> uu(u.begin(), u.begin() + cnt[its - 1]), vv(v.begin(), v.begin() + cnt[its - 1]);
    compare_order(uu, vv, std::max(1, int(uu.size()) / 300), path);
}

}  // namespace

int main(int argc, char** argv) {
    // test_mesh [--synthetic N] [FILE.sup ...]
    int a = 1;
    if (argc == 1) synthetic(1500);
    if (argc > 2 && std::strcmp(argv[1], "--synthetic") == 0) {
        synthetic(std::atoi(argv[2]));
        a = 3;
    }
    for (; a < argc; ++a) from_file(argv[a]);
    if (failures) {
        std::printf("%d failures (%lld sets, %lld checks)\n", failures, sets, checks);
        return 1;
    }
    std::printf("ok %lld %lld\n", sets, checks);
    return 0;
}
