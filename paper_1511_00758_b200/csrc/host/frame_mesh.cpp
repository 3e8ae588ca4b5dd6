// frame_mesh.cpp — see frame_mesh.hpp.
#include "frame_mesh.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace ps {

namespace {

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// IncDT half-edges: e = 4t + k
inline int nxt(int e) { return (e & 3) == 2 ? e - 2 : e + 1; }
inline int prv(int e) { return (e & 3) == 0 ? e + 2 : e - 1; }

// fitPlane (proj/src/mesh.cpp:12-26), numerators in source order; this file is
// built with -ffp-contract=off, so every step rounds like the reference's.
struct Fit {
    double A, B, C;
    long long det;
};

inline Fit fit(const FrameMesh& fm, int i, int j, int k) {
    const long long u1 = fm.u[i], u2 = fm.u[j], u3 = fm.u[k];
    const long long w1 = fm.v[i], w2 = fm.v[j], w3 = fm.v[k];
    const double d1 = fm.d[i], d2 = fm.d[j], d3 = fm.d[k];
    Fit f;
    f.det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    f.A = d1 * double(w2 - w3) + d2 * double(w3 - w1) + d3 * double(w1 - w2);
    f.B = double(u1) * (d2 - d3) + double(u2) * (d3 - d1) + double(u3) * (d1 - d2);
    f.C = d1 * double(u2 * w3 - u3 * w2) - d2 * double(u1 * w3 - u3 * w1) +
          d3 * double(u1 * w2 - u2 * w1);
    return f;
}

inline bool same_bits(const Fit& a, const Fit& b) {
    return std::memcmp(&a.A, &b.A, 8) == 0 && std::memcmp(&a.B, &b.B, 8) == 0 &&
           std::memcmp(&a.C, &b.C, 8) == 0;
}

// D_it at (u, v) as the raster stores it: binary32 bits, or NaN when invalid
// (mesh.cpp:149-164: d = float(a*u + b*v + c), valid iff 0 <= d < ND).
inline uint32_t dit_bits(const Fit& f, int u, int v, float nd) {
    const double a = f.A / double(f.det), b = f.B / double(f.det), c = f.C / double(f.det);
    const double s = (a * double(u) + b * double(v)) + c;
    const float d = float(s);
    if (!(d >= 0.0f && d < nd)) return 0x7fc00000u;
    uint32_t bits;
    std::memcpy(&bits, &d, 4);
    return bits;
}

// Order-query budget per frame-iteration.  Each query replays windows of
// the sweep; past the budget the whole replay is cheaper.  Measured (one
// host core): VGA ~20 k supports, query ~0.05 ms vs replay 3-8 ms; 1080p
// 465 k, 45 ms vs 1.4 s; 4K 5.8 M, ~170 ms vs ~30 s: the ratio grows slowly
// with the point count.  PS_MAX_QUERIES overrides it (probing).
int max_queries(int n) {
    static const int env = [] {
        const char* e = std::getenv("PS_MAX_QUERIES");
        return e ? std::atoi(e) : -1;
    }();
    if (env >= 0) return env;
    return 32 + n / 32768;
}

long long floor_div(long long a, long long b) {  // mesh.cpp:30-36
    long long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

// Whether the three rotations of a triangle whose fitted planes differ in
// their binary64 bits still give the same binary32 D_it at every pixel the
// triangle covers (the top-left rule of mesh.cpp:58-104) and at its vertex
// pixels (pins): then the rotation the sweep stored cannot show in any output.
bool rotations_equivalent(const FrameMesh& fm, int i, int j, int k, const Fit f[3], int width,
                          int height, float nd) {
    const int x[3] = {fm.u[i], fm.u[j], fm.u[k]}, y[3] = {fm.v[i], fm.v[j], fm.v[k]};
    auto same_at = [&](int u, int v) {
        const uint32_t b0 = dit_bits(f[0], u, v, nd);
        return dit_bits(f[1], u, v, nd) == b0 && dit_bits(f[2], u, v, nd) == b0;
    };
    for (int q = 0; q < 3; ++q)
        if (x[q] >= 0 && x[q] < width && y[q] >= 0 && y[q] < height && !same_at(x[q], y[q])) return false;
    long long A[3], bias[3];
    for (int a = 0; a < 3; ++a) {
        const int b = (a + 1) % 3;
        A[a] = y[a] - y[b];
        bias[a] = ((y[b] < y[a]) || (y[b] == y[a] && x[b] > x[a])) ? 0 : 1;
    }
    const int vmin = std::max(0, std::min({y[0], y[1], y[2]}));
    const int vmax = std::min(height - 1, std::max({y[0], y[1], y[2]}));
    for (int v = vmin; v <= vmax; ++v) {
        long long lo = 0, hi = width - 1;
        bool empty = false;
        for (int a = 0; a < 3 && !empty; ++a) {
            const int b = (a + 1) % 3;
            const long long K = (long long)(x[b] - x[a]) * (v - y[a]) + (long long)(y[b] - y[a]) * x[a];
            if (A[a] > 0) lo = std::max(lo, -floor_div(K - bias[a], A[a]));
            else if (A[a] < 0) hi = std::min(hi, floor_div(K - bias[a], -A[a]));
            else if (K < bias[a]) empty = true;
        }
        if (empty) continue;
        for (long long u = lo; u <= hi; ++u)
            if (!same_at(int(u), v)) return false;
    }
    return true;
}

inline bool integral(double x) { return x == std::floor(x) && std::fabs(x) < 1e9; }

inline bool tie_accept(int xi, int yi, int xj, int yj) {
    return (yj < yi) || (yj == yi && xj > xi);  // mesh.cpp:80
}

int replay(FrameMesh& fm, int width, int height, int* tris, int cap, uint8_t* pins,
           DelaunayWorkspace& ws, MeshStats& st) {
    ++st.fallbacks;
    const double t0 = now_ms();
    const int n = int(fm.u.size());
    const int t = delaunay_lex(fm.u.data(), fm.v.data(), n, tris, cap, ws);
    if (t > 0) lex_hull_pins(ws, t, width, height, pins);
    st.replay_ms += now_ms() - t0;
    return t;
}

}  // namespace

int replay_mesh(FrameMesh& fm, int width, int height, int* tris, int cap, uint8_t* pins,
                DelaunayWorkspace& ws, MeshStats& st) {
    return replay(fm, width, height, tris, cap, pins, ws, st);
}

bool resolve_device_flags(FrameMesh& fm, const int* flags, const StarFlagLayout& layout, int frame, int width, int height,
                          float max_disparity, std::vector<int>& fixes, DelaunayWorkspace& ws,
                          MeshStats& st, const ParallelQueries* par, int budget_scale) {
    ++st.frames;
    const int n = int(fm.u.size());
    const int budget = max_queries(n) * std::max(1, budget_scale);
    const int n_sus = flags[1];
    const int n_amb = flags[3];
    const int* sus = flags + kStarSuspectBase;
    const int* fan = flags + layout.fan_base;
    bool have_order = false;
    auto build_order = [&] {
        if (have_order) return;
        const double ti = now_ms();
        int minx, miny, m, spanx, spany;
        lex_order(fm.u.data(), fm.v.data(), n, ws, minx, miny, m, spanx, spany);
        fm.ranks.assign(ws.kept.begin(), ws.kept.begin() + m);
        fm.rank_of.assign(n, -1);
        fm.px.resize(m);
        fm.py.resize(m);
        for (int r = 0; r < m; ++r) {
            fm.rank_of[fm.ranks[r]] = r;
            fm.px[r] = fm.u[fm.ranks[r]];
            fm.py[r] = fm.v[fm.ranks[r]];
        }
        fm.so.init(fm.px.data(), fm.py.data(), m);
        have_order = true;
        st.init_ms += now_ms() - ti;
    };
    auto sorted3 = [](int a, int b, int c) {
        if (a > b) std::swap(a, b);
        if (b > c) std::swap(b, c);
        if (a > b) std::swap(a, b);
        return std::array<int, 3>{a, b, c};
    };
    int queries = 0;
    // (2) rotation suspects: does any covered pixel see the difference?  The
    // suspects that need the sweep's rotation are collected first, their
    // order queries run (possibly on several host threads: each query is
    // independent given the frame's SweepOrder), then the fixes are written
    // in suspect order, so the result does not depend on the schedule.
    std::vector<std::pair<std::array<int, 3>, std::array<int, 3>>> rotated;  // vertex set -> stored order
    std::vector<std::array<int, 4>> need;  // (triangle, i, j, k)
    for (int q = 0; q < n_sus; ++q) {
        const int t = sus[4 * q], i = sus[4 * q + 1], j = sus[4 * q + 2], k = sus[4 * q + 3];
        if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n) return false;
        ++st.rot_checked;
        const Fit f3[3] = {fit(fm, i, j, k), fit(fm, j, k, i), fit(fm, k, i, j)};
        if (rotations_equivalent(fm, i, j, k, f3, width, height, max_disparity)) continue;
        need.push_back({t, i, j, k});
    }
    queries = int(need.size());
    if (queries > budget) {
        ++st.fb_queries;
        return false;
    }
    if (!need.empty()) {
        const double to = now_ms();
        build_order();
        std::vector<std::array<int, 3>> s3(need.size());
        std::vector<uint8_t> okq(need.size(), 0);
        auto one = [&](int q, SweepOrder::Scratch& S) {
            int r3[3] = {fm.rank_of[need[q][1]], fm.rank_of[need[q][2]], fm.rank_of[need[q][3]]};
            uint64_t b;
            okq[q] = fm.so.resolve(r3, 1, &b, s3[q].data(), S) ? 1 : 0;
        };
        if (par && need.size() > 1) {
            (*par)(int(need.size()), one);
        } else {
            for (int q = 0; q < int(need.size()); ++q) one(q, fm.so.scratch());
        }
        st.order_ms += now_ms() - to;
        st.rot_ms += now_ms() - to;
        for (size_t q = 0; q < need.size(); ++q) {
            if (!okq[q]) {
                ++st.fb_resolve;
                return false;
            }
            const int v0 = fm.ranks[s3[q][0]], v1 = fm.ranks[s3[q][1]], v2 = fm.ranks[s3[q][2]];
            fixes.insert(fixes.end(), {frame, 0, need[q][0], v0, v1, v2});
            rotated.push_back({sorted3(need[q][1], need[q][2], need[q][3]), {v0, v1, v2}});
            ++st.rotations;
        }
    }
    // (3) ambiguous hull vertices: the incident triangle the sweep stored first
    for (int a = 0, at = 0; a < n_amb; ++a) {
        const int h = fan[at], cnt = fan[at + 1];
        const int* tr = fan + at + 2;
        at += 2 + 3 * cnt;
        if (h < 0 || h >= n || cnt <= 0) return false;
        std::vector<std::array<int, 3>> inc(cnt);
        uint32_t first = 0;
        bool agree = true;
        for (int i = 0; i < cnt; ++i) {
            int x = tr[3 * i], y = tr[3 * i + 1], z = tr[3 * i + 2];
            // stored rotation: the host's fix, else the device's (smallest first)
            std::array<int, 3> key = sorted3(x, y, z), order;
            bool found = false;
            for (const auto& rr : rotated)
                if (rr.first == key) {
                    order = rr.second;
                    found = true;
                }
            if (!found) {
                while (!(x < y && x < z)) {
                    const int tmp = x;
                    x = y;
                    y = z;
                    z = tmp;
                }
                order = {x, y, z};
            }
            inc[i] = order;
            const uint32_t bits = dit_bits(fit(fm, order[0], order[1], order[2]), fm.u[h], fm.v[h], max_disparity);
            if (i == 0) first = bits;
            else if (bits != first) agree = false;
        }
        int pick = 0;
        if (!agree) {
            if (++queries > budget) {
                ++st.fb_queries;
                return false;
            }
            const double to = now_ms();
            build_order();
            std::vector<int> r3(3 * size_t(cnt)), s3(3 * size_t(cnt));
            fm.birth.resize(cnt);
            for (int i = 0; i < cnt; ++i) {
                // counter-clockwise as the device wrote it (the set is what matters)
                r3[3 * i] = fm.rank_of[tr[3 * i]];
                r3[3 * i + 1] = fm.rank_of[tr[3 * i + 1]];
                r3[3 * i + 2] = fm.rank_of[tr[3 * i + 2]];
            }
            const bool ok = fm.so.resolve(r3.data(), cnt, fm.birth.data(), s3.data());
            st.order_ms += now_ms() - to;
            st.pin_ms += now_ms() - to;
            if (!ok) {
                ++st.fb_resolve;
                return false;
            }
            for (int i = 1; i < cnt; ++i)
                if (fm.birth[i] < fm.birth[pick]) pick = i;
            ++st.ambiguous;
        }
        const auto s = sorted3(inc[pick][0], inc[pick][1], inc[pick][2]);
        fixes.insert(fixes.end(), {frame, 1, h, s[0], s[1], s[2]});
    }
    return true;
}

int mesh_iteration(FrameMesh& fm, int width, int height, float max_disparity, int* tris, int cap,
                   uint8_t* pins, DelaunayWorkspace& ws, MeshStats& st) {
    ++st.frames;
    const int n = int(fm.u.size());
    if (fm.lex_only) return replay(fm, width, height, tris, cap, pins, ws, st);
    double t0 = now_ms();
    if (!fm.dt.extend(fm.u.data(), fm.v.data(), n)) {
        for (int i = 0; i < n; ++i)
            if (std::abs(fm.u[i]) >= (1 << 20) || std::abs(fm.v[i]) >= (1 << 20)) return -1;
        fm.lex_only = true;  // internal inconsistency: exact replay from now on
        return replay(fm, width, height, tris, cap, pins, ws, st);
    }
    if (fm.dt.degenerate()) return 0;
    const int nt = fm.dt.triangles();
    if (nt > cap) return -3;
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = fm.dt.vert(t, k);
    double t1 = now_ms();
    st.dt_ms += t1 - t0;

    // (2) rotation: fractional-vertex triangles fitted three ways
    fm.q.clear();  // triangles whose rotation must come from the sweep
    for (int t = 0; t < nt; ++t) {
        const int i = tris[3 * t], j = tris[3 * t + 1], k = tris[3 * t + 2];
        if (integral(fm.d[i]) && integral(fm.d[j]) && integral(fm.d[k])) continue;
        ++st.rot_checked;
        const Fit f3[3] = {fit(fm, i, j, k), fit(fm, j, k, i), fit(fm, k, i, j)};
        if ((!same_bits(f3[0], f3[1]) || !same_bits(f3[0], f3[2])) &&
            !rotations_equivalent(fm, i, j, k, f3, width, height, max_disparity))
            fm.q.push_back(t);
    }

    bool have_order = false;
    auto build_order = [&]() -> bool {
        if (have_order) return true;
        int minx, miny, m, spanx, spany;
        lex_order(fm.u.data(), fm.v.data(), n, ws, minx, miny, m, spanx, spany);
        fm.ranks.assign(ws.kept.begin(), ws.kept.begin() + m);
        fm.rank_of.assign(n, -1);
        fm.px.resize(m);
        fm.py.resize(m);
        for (int r = 0; r < m; ++r) {
            fm.rank_of[fm.ranks[r]] = r;
            fm.px[r] = fm.u[fm.ranks[r]];
            fm.py[r] = fm.v[fm.ranks[r]];
        }
        fm.so.init(fm.px.data(), fm.py.data(), m);
        have_order = true;
        return true;
    };

    // Each order query replays a window of the sweep: past a handful the
    // whole replay is cheaper (real meshes need 0-2 per frame-iteration).
    if (int(fm.q.size()) > max_queries(n)) return replay(fm, width, height, tris, cap, pins, ws, st);
    int queries = int(fm.q.size());
    if (!fm.q.empty()) {
        const double to = now_ms();
        build_order();
        const std::vector<int> rot = fm.q;
        for (const int t : rot) {
            int r3[3] = {fm.rank_of[tris[3 * t]], fm.rank_of[tris[3 * t + 1]], fm.rank_of[tris[3 * t + 2]]};
            uint64_t b;
            int s3[3];
            if (!fm.so.resolve(r3, 1, &b, s3)) {
                st.order_ms += now_ms() - to;
                return replay(fm, width, height, tris, cap, pins, ws, st);
            }
            for (int k = 0; k < 3; ++k) tris[3 * t + k] = fm.ranks[s3[k]];
            ++st.rotations;
        }
        st.order_ms += now_ms() - to;
    }

    // (3) pins: walk the hull; an uncovered vertex pixel whose incident planes
    // disagree takes the incident triangle the sweep stored first
    std::memset(pins, 0, size_t(nt));
    auto tv = [&](int e) { return fm.dt.vert(e >> 2, e & 3); };
    const int h0 = fm.dt.hull_start();
    int guard = 0;
    for (int h = h0; h >= 0;) {
        if (++guard > n + 1) return replay(fm, width, height, tris, cap, pins, ws, st);
        bool covered = false;
        fm.inc.clear();
        for (int g = fm.dt.hull_edge(h); g >= 0;) {  // g: h -> q, triangle on its left
            const int q = tv(nxt(g)), r = tv(prv(g));
            if (tie_accept(fm.u[r], fm.v[r], fm.u[h], fm.v[h]) &&
                tie_accept(fm.u[h], fm.v[h], fm.u[q], fm.v[q])) {
                covered = true;
                break;
            }
            fm.inc.push_back(g >> 2);
            g = fm.dt.twin(prv(g));  // twin of r -> h: the next triangle around h
            if (int(fm.inc.size()) > nt) return replay(fm, width, height, tris, cap, pins, ws, st);
        }
        const int hu = fm.u[h], hv = fm.v[h];
        if (!covered && !fm.inc.empty() && hu >= 0 && hu < width && hv >= 0 && hv < height) {
            uint32_t first = 0;
            bool agree = true;
            for (size_t i = 0; i < fm.inc.size(); ++i) {
                const int t = fm.inc[i];
                const uint32_t bits = dit_bits(fit(fm, tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]), hu, hv, max_disparity);
                if (i == 0) first = bits;
                else if (bits != first) agree = false;
            }
            int pin_t = fm.inc[0];
            if (!agree && ++queries > max_queries(n)) return replay(fm, width, height, tris, cap, pins, ws, st);
            if (!agree) {
                const double to = now_ms();
                build_order();
                const int cnt = int(fm.inc.size());
                std::vector<int> r3(3 * size_t(cnt)), s3(3 * size_t(cnt));
                fm.birth.resize(cnt);
                for (int i = 0; i < cnt; ++i)
                    for (int k = 0; k < 3; ++k) r3[3 * i + k] = fm.rank_of[fm.dt.vert(fm.inc[i], k)];
                const bool ok = fm.so.resolve(r3.data(), cnt, fm.birth.data(), s3.data());
                st.order_ms += now_ms() - to;
                if (!ok) return replay(fm, width, height, tris, cap, pins, ws, st);
                int best = 0;
                for (int i = 1; i < cnt; ++i)
                    if (fm.birth[i] < fm.birth[best]) best = i;
                pin_t = fm.inc[best];
                ++st.ambiguous;
            }
            for (int k = 0; k < 3; ++k)
                if (tris[3 * pin_t + k] == h) pins[pin_t] |= uint8_t(1u << k);
        }
        h = fm.dt.hull_next(h);
        if (h == h0) break;
    }
    st.check_ms += now_ms() - t1;
    return nt;
}

}  // namespace ps
