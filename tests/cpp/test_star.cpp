// test_star.cpp — the device Delaunay (kernels/star_dt.cuh, per-point stars)
// run on the CPU, against the reference-order sweep's triangle set
// (delaunay_lex, array-for-array equal to the compiled reference).
//
//   test_star [--no-local | --tiled] [--synthetic N] [FILE.sup ...]
// Prints "ok <sets> <triangles>" and exits 0, or the first failures.
static long long g_near_steps = 0, g_near_miss = 0, g_near_none = 0;
#define PS_NEAR_STATS(miss) (++g_near_steps, g_near_miss += (miss))
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_1511_00758_b200/csrc/kernels/star_dt.cuh"
#include "delaunay.hpp"

using namespace ps;

namespace {

int failures = 0;
int radius = 2;  // gather radius of the local pass (--no-local: every search on the grid)
bool tiled = false;  // --tiled: the device's tiled pass 1
long long sets = 0, tris_checked = 0;

void fail(const char* tag, const char* what) {
    if (++failures <= 10) std::printf("FAIL %s: %s\n", tag, what);
}

std::vector<std::array<int, 3>> star_triangles(const std::vector<int>& u, const std::vector<int>& v,
                                               bool& ok) {
    const int n = int(u.size());
    ok = true;
    std::vector<std::array<int, 3>> out;
    if (n < 3) return out;
    int minx = u[0], maxx = u[0], miny = v[0], maxy = v[0];
    for (int i = 1; i < n; ++i) {
        minx = std::min(minx, u[i]);
        maxx = std::max(maxx, u[i]);
        miny = std::min(miny, v[i]);
        maxy = std::max(maxy, v[i]);
    }
    const double area = double(maxx - minx + 1) * double(maxy - miny + 1);
    int gs = std::max(1, int(std::lround(std::sqrt(2.0 * area / n))));
    const int gw = (maxx - minx) / gs + 1, gh = (maxy - miny) / gs + 1;
    std::vector<int> start(size_t(gw) * gh + 1, 0), items(n);
    for (int i = 0; i < n; ++i) ++start[size_t((v[i] - miny) / gs) * gw + (u[i] - minx) / gs + 1];
    for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int i = 0; i < n; ++i) items[fill[size_t((v[i] - miny) / gs) * gw + (u[i] - minx) / gs]++] = i;
    std::vector<uint8_t> dup(n, 0);
    for (int c = 0; c + 1 < int(start.size()); ++c)
        for (int a = start[c]; a < start[c + 1]; ++a)
            for (int b = start[c]; b < a; ++b) {
                const int i = items[a], j = items[b];
                if (u[i] == u[j] && v[i] == v[j]) dup[std::max(i, j)] = 1;
            }
    // column extremes: smallest / largest v, smallest index on ties (never a dup)
    std::vector<int> lo(maxx - minx + 1, -1), hi(maxx - minx + 1, -1);
    for (int i = 0; i < n; ++i) {
        int& l = lo[u[i] - minx];
        if (l < 0 || v[i] < v[l] || (v[i] == v[l] && i < l)) l = i;
        int& h = hi[u[i] - minx];
        if (h < 0 || v[i] > v[h] || (v[i] == v[h] && i < h)) h = i;
    }
    std::vector<int> hn(n, -1), hp(n, -1), c1(n + 2 * (maxx - minx + 1) + 8), c2(c1.size());
    star::Grid g{u.data(), v.data(), dup.data(), start.data(), items.data(), n, minx, miny, maxx, maxy,
                 gs, gw, gh, lo.data(), hi.data(), hn.data(), hp.data(), 0, 1.0 / gs};
    g.flat = star::build_hull(g, c1.data(), c2.data(), hn.data(), hp.data());
    star::Local L;
    int lidx[star::kLocalMax], ldxy[star::kLocalMax];
    L.idx = lidx;
    L.dxy = ldxy;
    if (tiled) {
        // the device's pass 1 (star.cu k_star): tiles of cells with a halo in
        // "shared memory", radius 2 then 4, the grid search for the rest
        const int tw = (gw + star::kTileCells - 1) / star::kTileCells, th = (gh + star::kTileCells - 1) / star::kTileCells;
        constexpr int RC = star::kTileRegion * star::kTileRegion;
        std::vector<int> rs(RC + 1), rxy, rid;
        for (int ty = 0; ty < th; ++ty)
            for (int tx = 0; tx < tw; ++tx) {
                const int cx0 = tx * star::kTileCells - star::kTileHalo, cy0 = ty * star::kTileCells - star::kTileHalo;
                rxy.clear();
                rid.clear();
                for (int c = 0; c < RC; ++c) {
                    rs[c] = int(rxy.size());
                    const int gx = cx0 + c % star::kTileRegion, gy = cy0 + c / star::kTileRegion;
                    if (gx < 0 || gy < 0 || gx >= gw || gy >= gh) continue;
                    for (int k = start[size_t(gy) * gw + gx]; k < start[size_t(gy) * gw + gx + 1]; ++k) {
                        const int s = items[k];
                        if (dup[s]) continue;
                        rxy.push_back(((v[s] - (miny + cy0 * gs)) << 16) | (u[s] - (minx + cx0 * gs)));
                        rid.push_back(s);
                    }
                }
                rs[RC] = int(rxy.size());
                const star::Tile T{rs.data(), rxy.data(), rid.data(), cx0, cy0};
                for (int ry = star::kTileHalo; ry < star::kTileHalo + star::kTileCells; ++ry)
                    for (int rx = star::kTileHalo; rx < star::kTileHalo + star::kTileCells; ++rx) {
                        const int c = ry * star::kTileRegion + rx;
                        for (int i = rs[c]; i < rs[c + 1]; ++i) {
                            const int p = rid[i];
                            const star::TilePoint P{p, cx0 + rx, cy0 + ry, rxy[i] & 0xffff, rxy[i] >> 16, u[p], v[p], hp[p], hn[p]};
                            int tb[2 * 16];
                            bool closed;
                            int nl[star::kNearCap];
                            star::Near N{nl, 1, -1, 0};
                            if (!star::near_build(g, T, P, N)) {
                                N.n = -1;
                                ++g_near_none;
                            }
                            int k = star::tile_walk_near(g, T, P, N, closed, tb, 16);
                            if (k == -4) k = star::tile_walk(g, T, P, 4, closed, tb, 16);
                            if (k >= 0) {
                                for (int j = 0; j < k; ++j)
                                    if (p < tb[2 * j] && p < tb[2 * j + 1]) out.push_back({p, tb[2 * j], tb[2 * j + 1]});
                                continue;
                            }
                            star::Local none;
                            none.complete = false;
                            k = star::walk_star(g, none, p, closed, [&](int a, int b, int c2) {
                                if (a < b && a < c2) out.push_back({a, b, c2});
                            });
                            if (k == -2) {
                                ok = false;
                                return out;
                            }
                        }
                    }
            }
        return out;
    }
    for (int p = 0; p < n; ++p) {
        bool closed;
        star::gather(g, p, radius, L);
        if (radius < 0) L.complete = false;
        const int k = star::walk_star(g, L, p, closed, [&](int a, int b, int c) {
            if (a < b && a < c) out.push_back({a, b, c});
        });
        if (k == -2) {
            ok = false;
            return out;
        }
    }
    return out;
}

void compare(const std::vector<int>& u, const std::vector<int>& v, const char* tag) {
    ++sets;
    bool ok;
    auto got = star_triangles(u, v, ok);
    if (!ok) return fail(tag, "star search failed");
    DelaunayWorkspace ws;
    std::vector<int> tb;
    const int nt = delaunay_lex(u.data(), v.data(), int(u.size()), tb, ws);
    std::vector<std::array<int, 3>> want;
    for (int t = 0; t < std::max(nt, 0); ++t) {
        std::array<int, 3> k = {tb[3 * t], tb[3 * t + 1], tb[3 * t + 2]};
        // the star emits (min, next ccw, next): rotate to the smallest index first
        int m = 0;
        if (k[1] < k[m]) m = 1;
        if (k[2] < k[m]) m = 2;
        want.push_back({k[m], k[(m + 1) % 3], k[(m + 2) % 3]});
    }
    std::sort(got.begin(), got.end());
    std::sort(want.begin(), want.end());
    tris_checked += long(want.size());
    if (got != want) {
        char msg[128];
        std::snprintf(msg, sizeof msg, "triangle set differs (%zu vs %zu)", got.size(), want.size());
        fail(tag, msg);
    }
}

void synthetic(int count) {
    std::mt19937 rng(7);
    for (int it = 0; it < count; ++it) {
        std::vector<int> u, v;
        if (it % 3 != 2) {  // lattices (cocircular cells), jittered or not, with holes
            const int L = 3 + rng() % 14, step = 1 + rng() % 4;
            const double keep = 0.3 + 0.7 * (rng() % 1000) / 1000.0;
            const bool jit = rng() % 3 == 0;
            for (int i = 0; i < L; ++i)
                for (int j = 0; j < L; ++j)
                    if ((rng() % 1000) / 1000.0 < keep) {
                        u.push_back(i * step + (jit ? int(rng() % 2) : 0));
                        v.push_back(j * step + (jit ? int(rng() % 2) : 0));
                    }
        } else {  // random points in a small square (collinear and cocircular subsets)
            const int n = 3 + rng() % 300, R = 3 + rng() % 40;
            for (int i = 0; i < n; ++i) {
                u.push_back(rng() % R);
                v.push_back(rng() % R);
            }
        }
        std::vector<int> idx(u.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = int(i);
        std::shuffle(idx.begin(), idx.end(), rng);
        std::vector<int> uu, vv;
        for (int i : idx) {
            uu.push_back(u[i]);
            vv.push_back(v[i]);
        }
        char tag[64];
        std::snprintf(tag, sizeof tag, "synthetic %d", it);
        compare(uu, vv, tag);
    }
}

void from_file(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(path, "cannot open");
    int hdr[5];
    bool ok = std::fread(hdr, 4, 5, f) == 5;
    const int its = hdr[3], n = hdr[4];
    std::vector<int> cnt(its), u(n), v(n);
    ok = ok && std::fread(cnt.data(), 4, its, f) == size_t(its) && std::fread(u.data(), 4, n, f) == size_t(n) &&
         std::fread(v.data(), 4, n, f) == size_t(n);
    std::fclose(f);
    if (!ok) return fail(path, "short file");
    for (int i = 0; i < its; ++i) {
        char tag[256];
        std::snprintf(tag, sizeof tag, "%s iteration %d", path, i + 1);
        compare(std::vector<int>(u.begin(), u.begin() + cnt[i]), std::vector<int>(v.begin(), v.begin() + cnt[i]), tag);
    }
}

}  // namespace

int main(int argc, char** argv) {
    int a = 1;
    if (argc > 1 && (std::strcmp(argv[1], "--no-local") == 0 || std::strcmp(argv[1], "--tiled") == 0)) {
        if (argv[1][2] == 'n') radius = -1;
        else tiled = true;
        ++argv;
        --argc;
    }
    if (argc == 1) synthetic(3000);
    if (argc > 2 && std::strcmp(argv[1], "--synthetic") == 0) {
        synthetic(std::atoi(argv[2]));
        a = 3;
    }
    for (; a < argc; ++a) from_file(argv[a]);
    if (failures) {
        std::printf("%d failures (%lld sets)\n", failures, sets);
        return 1;
    }
    if (g_near_steps)
        std::printf("near set: %lld steps, %lld not certified, %lld points without one\n", g_near_steps, g_near_miss,
                    g_near_none);
    std::printf("ok %lld %lld\n", sets, tris_checked);
    return 0;
}
