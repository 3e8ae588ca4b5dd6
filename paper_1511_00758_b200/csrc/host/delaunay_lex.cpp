// delaunay_lex.cpp — lexicographic-sweep Delaunay in the reference's order.
//
// Same triangle SET as delaunay() (delaunay.cpp) but also the same triangle
// ORDER and vertex rotation as planestereo::delaunayTriangulate
// (proj/src/delaunay.cpp:288-325), because it performs the same sequence of
// textbook operations: points inserted in (u, v) order, each new point fanned
// to its strictly visible hull chain from the first to the last edge, Lawson
// flips of the edges opposite the new point in LIFO order with a strict
// in-circle test, and a flipped pair (a,b,c)+(b,a,d) rewritten in place as
// (a,d,c)+(d,b,c).  Checked array-for-array against the compiled reference
// (tests/test_delaunay.py).
//
// The order matters downstream in two places: an uncovered hull vertex pixel
// takes its FIRST incident triangle (mesh.cpp:109-122), and fitPlane's binary64
// rounding depends on the vertex rotation (the plane offset is anchored at the
// first vertex).  The engine therefore always triangulates with this sweep;
// it is also the order of the public ps_delaunay().
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "delaunay.hpp"

namespace ps {

namespace {

// Half-edge e = 4 * slot + k (k = 0..2): one 32-byte record per triangle slot
// holds its vertices and neighbour half-edges (one cache line per flip side).
inline int lnext(int e) { return (e & 3) == 2 ? e - 2 : e + 1; }

struct LexSweep {
    const int* x;
    const int* y;
    LexTri* T;
    int* hnext;
    int* hprev;
    int* hedge;
    std::vector<int>* stack;
    int ntri = 0;
    bool wide = false;

    int& V(int e) const { return T[e >> 2].v[e & 3]; }
    int& N(int e) const { return T[e >> 2].n[e & 3]; }

    long long orient(int a, int b, int c) const {
        const long long abx = (long long)x[b] - x[a], aby = (long long)y[b] - y[a];
        const long long acx = (long long)x[c] - x[a], acy = (long long)y[c] - y[a];
        return abx * acy - aby * acx;
    }

    bool inside(int a, int b, int c, int d) const {
        const long long adx = (long long)x[a] - x[d], ady = (long long)y[a] - y[d];
        const long long bdx = (long long)x[b] - x[d], bdy = (long long)y[b] - y[d];
        const long long cdx = (long long)x[c] - x[d], cdy = (long long)y[c] - y[d];
        const long long aq = adx * adx + ady * ady;
        const long long bq = bdx * bdx + bdy * bdy;
        const long long cq = cdx * cdx + cdy * cdy;
        if (!wide) {
            return adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                       aq * (bdx * cdy - cdx * bdy) > 0;
        }
        using W = __int128;
        return W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                   W(aq) * (W(bdx) * cdy - W(cdx) * bdy) > 0;
    }

    int add(int a, int b, int c, int na, int nb, int nc) {
        const int e = 4 * ntri;
        LexTri& r = T[ntri++];
        r.v[0] = a;
        r.v[1] = b;
        r.v[2] = c;
        r.n[0] = na;
        r.n[1] = nb;
        r.n[2] = nc;
        if (na >= 0) N(na) = e;
        if (nb >= 0) N(nb) = e + 1;
        if (nc >= 0) N(nc) = e + 2;
        return e;
    }

    void hull(int a, int b) {
        hnext[a] = b;
        hprev[b] = a;
    }

    void legalize() {
        while (!stack->empty()) {
            const int e = stack->back();
            stack->pop_back();
            const int f = N(e);
            if (f < 0) continue;
            const int e1 = lnext(e), e2 = lnext(e1);
            const int f1 = lnext(f), f2 = lnext(f1);
            const int a = V(e), b = V(e1), c = V(e2), d = V(f2);
            if (!inside(a, b, c, d)) continue;  // strict: cocircular never flips
            const int ne1 = N(e1), nf1 = N(f1), nf2 = N(f2);
            V(e1) = d;
            V(f) = d;
            V(f1) = b;
            V(f2) = c;
            N(e) = nf1;
            if (nf1 >= 0) N(nf1) = e; else hedge[a] = e;
            N(e1) = f2;
            N(f2) = e1;
            N(f) = nf2;
            if (nf2 >= 0) N(nf2) = f; else hedge[d] = f;
            N(f1) = ne1;
            if (ne1 >= 0) N(ne1) = f1; else hedge[b] = f1;
            // edges incident to the new point (f1, e2) are locally Delaunay
            // and never flip; only the two opposite edges are re-examined
            stack->push_back(e);
            stack->push_back(f);
        }
    }

    bool visible(int a, int p) const { return orient(a, hnext[a], p) < 0; }

    bool insert(int p) {
        const int q = p - 1;  // lexicographic max so far: on the hull
        int a, b;
        if (visible(q, p)) {
            a = q;
            b = hnext[q];
        } else if (visible(hprev[q], p)) {
            a = hprev[q];
            b = q;
        } else {
            return false;
        }
        while (hnext[b] != a && visible(b, p)) b = hnext[b];
        while (hprev[a] != b && visible(hprev[a], p)) a = hprev[a];
        int prevE1 = -1, firstE0 = -1;
        for (int xv = a; xv != b;) {
            const int xn = hnext[xv];
            const int e = add(xv, p, xn, prevE1, -1, hedge[xv]);
            if (firstE0 < 0) firstE0 = e;
            prevE1 = e + 1;
            stack->push_back(e + 2);
            xv = xn;
        }
        hull(a, p);
        hull(p, b);
        hedge[a] = firstE0;
        hedge[p] = prevE1;
        legalize();
        return true;
    }
};

}  // namespace

void lex_order(const int* u, const int* v, int n, DelaunayWorkspace& ws, int& minx, int& miny,
               int& m, int& spanx, int& spany);

namespace {
int lex_sweep(const int* u, const int* v, int n, DelaunayWorkspace& ws);
}  // namespace

int delaunay_lex(const int* u, const int* v, int n, std::vector<int>& tris,
                 DelaunayWorkspace& ws) {
    tris.clear();
    const int nt = lex_sweep(u, v, n, ws);
    if (nt <= 0) return nt;
    tris.resize(3 * std::size_t(nt));
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = ws.kept[ws.lex[t].v[k]];
    return nt;
}

int delaunay_lex(const int* u, const int* v, int n, int* tris, int capacity,
                 DelaunayWorkspace& ws) {
    const int nt = lex_sweep(u, v, n, ws);
    if (nt <= 0) return nt;
    if (nt > capacity) return -3;
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = ws.kept[ws.lex[t].v[k]];
    return nt;
}

namespace {
// The sweep itself: triangles left in ws.lex[0..ntri), vertex ids into ws.kept.
int lex_sweep(const int* u, const int* v, int n, DelaunayWorkspace& ws) {
    constexpr int kLimit = 1 << 20;
    for (int i = 0; i < n; ++i)
        if (std::abs(u[i]) >= kLimit || std::abs(v[i]) >= kLimit) return -1;
    if (n < 3) return 0;
    int minx, miny, m, spanx, spany;
    lex_order(u, v, n, ws, minx, miny, m, spanx, spany);  // sorted + deduplicated in ws.kept
    if (m < 3) return 0;
    ws.px.resize(m);
    ws.py.resize(m);
    for (int i = 0; i < m; ++i) {
        ws.px[i] = u[ws.kept[i]];
        ws.py[i] = v[ws.kept[i]];
    }
    ws.lex.resize(2 * std::size_t(m));  // T <= 2m - 5
    ws.hnext.assign(m, -1);
    ws.hprev.assign(m, -1);
    ws.hedge.assign(m, -1);
    ws.stack.clear();
    LexSweep s{ws.px.data(), ws.py.data(), ws.lex.data(), ws.hnext.data(),
               ws.hprev.data(), ws.hedge.data(), &ws.stack};
    s.wide = spanx >= (1 << 14) || spany >= (1 << 14);

    int k = 2;
    while (k < m && s.orient(0, 1, k) == 0) ++k;
    if (k == m) return 0;
    const int apex = k;
    if (s.orient(0, 1, apex) > 0) {
        int prevE1 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = s.add(j, j + 1, apex, -1, -1, prevE1);
            if (j == 0) s.hedge[apex] = e + 2;
            s.hedge[j] = e;
            prevE1 = e + 1;
        }
        s.hedge[k - 1] = prevE1;
        for (int j = 0; j + 1 < k; ++j) s.hull(j, j + 1);
        s.hull(k - 1, apex);
        s.hull(apex, 0);
    } else {
        int prevE2 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = s.add(j + 1, j, apex, -1, prevE2, -1);
            if (j == 0) s.hedge[0] = e + 1;
            s.hedge[j + 1] = e;
            prevE2 = e + 2;
        }
        s.hedge[apex] = prevE2;
        for (int j = 0; j + 1 < k; ++j) s.hull(j + 1, j);
        s.hull(0, apex);
        s.hull(apex, k - 1);
    }
    for (int p = apex + 1; p < m; ++p)
        if (!s.insert(p)) return -2;
    return s.ntri;
}
}  // namespace

namespace {

bool tie_accept(int xi, int yi, int xj, int yj) {
    // edge i->j accepts pixels on it (mesh.cpp:80)
    return (yj < yi) || (yj == yi && xj > xi);
}

}  // namespace

// mesh_pins() for the triangulation delaunay_lex() just left in `ws`, from
// its final half-edge state: only hull vertices can be uncovered by the tie
// rule (an interior vertex pixel belongs to exactly one of the triangles
// around it), so only their incident triangles are visited — a walk around
// each hull vertex from its hull half-edge — instead of all T triangles.
void lex_hull_pins(const DelaunayWorkspace& ws, int ntri, int width, int height,
                   std::vector<uint8_t>& pin_bits) {
    pin_bits.assign(std::max(ntri, 0), 0);
    if (ntri > 0) lex_hull_pins(ws, ntri, width, height, pin_bits.data());
}

void lex_hull_pins(const DelaunayWorkspace& ws, int ntri, int width, int height, uint8_t* pin_bits) {
    if (ntri <= 0) return;
    std::memset(pin_bits, 0, std::size_t(ntri));
    const LexTri* T = ws.lex.data();
    auto V = [&](int e) { return T[e >> 2].v[e & 3]; };
    auto N = [&](int e) { return T[e >> 2].n[e & 3]; };
    const int* x = ws.px.data();
    const int* y = ws.py.data();
    int h = 0;  // the lexicographic minimum is a hull vertex
    do {
        bool covered = false;
        int first = -1, corner = 0;
        for (int g = ws.hedge[h];;) {  // g: half-edge h -> q, its triangle on the left
            const int gin = lnext(lnext(g));  // r -> h
            const int q = V(lnext(g)), r = V(gin);
            if (tie_accept(x[r], y[r], x[h], y[h]) && tie_accept(x[h], y[h], x[q], y[q])) {
                covered = true;
                break;
            }
            if (first < 0 || (g >> 2) < first) {
                first = g >> 2;
                corner = g & 3;
            }
            const int tw = N(gin);
            if (tw < 0) break;  // r -> h is the incoming hull edge
            g = tw;
        }
        if (!covered && first >= 0 && x[h] >= 0 && x[h] < width && y[h] >= 0 && y[h] < height)
            pin_bits[first] |= uint8_t(1u << corner);
        h = ws.hnext[h];
    } while (h != 0);
}

}  // namespace ps
