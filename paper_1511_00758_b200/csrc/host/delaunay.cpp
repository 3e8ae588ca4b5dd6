// delaunay.cpp — exact lexicographic-sweep Delaunay for pixel coordinates.
//
// Same output set as planestereo::delaunayTriangulate
// (proj/src/delaunay.cpp:288-325; see delaunay.hpp for the contract), built
// for the per-frame, per-iteration host step of the B200 engine:
//   * LSD radix sort of 43-bit (u,v) keys (stable, so equal coordinates keep
//     input order and the first occurrence wins, as in delaunay.cpp:303-311);
//   * points arrive in lexicographic order, so each new point is outside the
//     current hull and the previous point is a hull vertex with an incident
//     visible edge: the visible chain is found by walking both ways from it,
//     O(#visible edges) per insertion (no full hull scan);
//   * Lawson flips only of edges opposite the new point, with a strict exact
//     in-circle test: the new point is the lexicographic maximum of every
//     quad it tests, which is exactly the cocircular tie rule of the
//     reference's output;
//   * exact predicates: int64 everywhere when the bounding box spans < 2^14
//     px (in-circle magnitude < 2^60), __int128 otherwise.
#include "delaunay.hpp"

#include <cstdlib>

namespace ps {

namespace {

inline int nxt(int e) { return (e % 3 == 2) ? e - 2 : e + 1; }
inline int prv(int e) { return (e % 3 == 0) ? e + 2 : e - 1; }

struct Sweep {
    const int* x;
    const int* y;
    int* tv;
    int* tn;
    int* hnext;
    int* hprev;
    int* hedge;
    std::vector<int>* stack;
    int ntri = 0;
    bool wide = false;

    long long orient(int a, int b, int c) const {
        const long long abx = (long long)x[b] - x[a], aby = (long long)y[b] - y[a];
        const long long acx = (long long)x[c] - x[a], acy = (long long)y[c] - y[a];
        return abx * acy - aby * acx;
    }

    // > 0 iff d lies strictly inside the circumcircle of CCW (a,b,c).
    bool inside(int a, int b, int c, int d) const {
        const long long adx = (long long)x[a] - x[d], ady = (long long)y[a] - y[d];
        const long long bdx = (long long)x[b] - x[d], bdy = (long long)y[b] - y[d];
        const long long cdx = (long long)x[c] - x[d], cdy = (long long)y[c] - y[d];
        const long long aq = adx * adx + ady * ady;
        const long long bq = bdx * bdx + bdy * bdy;
        const long long cq = cdx * cdx + cdy * cdy;
        if (!wide) {
            const long long det = adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                                  aq * (bdx * cdy - cdx * bdy);
            return det > 0;
        }
        using W = __int128;
        const W det = W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                      W(aq) * (W(bdx) * cdy - W(cdx) * bdy);
        return det > 0;
    }

    int add(int a, int b, int c, int na, int nb, int nc) {
        const int e = 3 * ntri++;
        tv[e] = a;
        tv[e + 1] = b;
        tv[e + 2] = c;
        tn[e] = na;
        tn[e + 1] = nb;
        tn[e + 2] = nc;
        if (na >= 0) tn[na] = e;
        if (nb >= 0) tn[nb] = e + 1;
        if (nc >= 0) tn[nc] = e + 2;
        return e;
    }

    void hull(int a, int b) {
        hnext[a] = b;
        hprev[b] = a;
    }

    // Edge e has the new point as its opposite apex (tv[prv(e)]).
    void legalize() {
        while (!stack->empty()) {
            const int e = stack->back();
            stack->pop_back();
            const int f = tn[e];
            if (f < 0) continue;
            const int e1 = nxt(e), e2 = nxt(e1);
            const int f1 = nxt(f), f2 = nxt(f1);
            const int a = tv[e], b = tv[e1], c = tv[e2], d = tv[f2];
            if (!inside(a, b, c, d)) continue;
            const int ne1 = tn[e1], ne2 = tn[e2], nf1 = tn[f1], nf2 = tn[f2];
            // (a,b,c)+(b,a,d) -> (a,d,c)+(d,b,c); c is the new point.
            tv[e] = a;
            tv[e1] = d;
            tv[e2] = c;
            tv[f] = d;
            tv[f1] = b;
            tv[f2] = c;
            tn[e] = nf1;
            if (nf1 >= 0) tn[nf1] = e; else hedge[a] = e;
            tn[e1] = f2;
            tn[f2] = e1;
            tn[e2] = ne2;  // unchanged slot (c->a)
            tn[f] = nf2;
            if (nf2 >= 0) tn[nf2] = f; else hedge[d] = f;
            tn[f1] = ne1;
            if (ne1 >= 0) tn[ne1] = f1; else hedge[b] = f1;
            stack->push_back(e);
            stack->push_back(f);
        }
    }

    bool visible(int a, int p) const { return orient(a, hnext[a], p) < 0; }

    bool insert(int p) {
        const int q = p - 1;  // previous point: lexicographic max so far, on the hull
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

void radix_sort_keys(std::vector<uint64_t>& key, std::vector<int>& ord, std::vector<uint64_t>& kt,
                     std::vector<int>& ot, int n, int bits) {
    kt.resize(n);
    ot.resize(n);
    uint32_t count[1 << 16];
    for (int shift = 0; shift < bits; shift += 16) {
        std::fill(count, count + (1 << 16), 0u);
        for (int i = 0; i < n; ++i) ++count[(key[i] >> shift) & 0xffff];
        uint32_t sum = 0;
        for (int d = 0; d < (1 << 16); ++d) {
            const uint32_t c = count[d];
            count[d] = sum;
            sum += c;
        }
        for (int i = 0; i < n; ++i) {
            const uint32_t pos = count[(key[i] >> shift) & 0xffff]++;
            kt[pos] = key[i];
            ot[pos] = ord[i];
        }
        key.swap(kt);
        ord.swap(ot);
    }
}

}  // namespace

int delaunay(const int* u, const int* v, int n, std::vector<int>& tris, DelaunayWorkspace& ws) {
    tris.clear();
    constexpr int kLimit = 1 << 20;
    int minx = kLimit, maxx = -kLimit, miny = kLimit, maxy = -kLimit;
    for (int i = 0; i < n; ++i) {
        if (std::abs(u[i]) >= kLimit || std::abs(v[i]) >= kLimit) return -1;
        minx = u[i] < minx ? u[i] : minx;
        maxx = u[i] > maxx ? u[i] : maxx;
        miny = v[i] < miny ? v[i] : miny;
        maxy = v[i] > maxy ? v[i] : maxy;
    }
    if (n < 3) return 0;

    ws.key.resize(n);
    ws.ord.resize(n);
    for (int i = 0; i < n; ++i) {
        ws.key[i] = (uint64_t(uint32_t(u[i] - minx)) << 21) | uint64_t(uint32_t(v[i] - miny));
        ws.ord[i] = i;
    }
    int bits = 21;
    while ((1ll << (bits - 21)) <= (long long)(maxx - minx)) ++bits;
    radix_sort_keys(ws.key, ws.ord, ws.key_tmp, ws.ord_tmp, n, bits);

    ws.kept.resize(n);
    ws.px.resize(n);
    ws.py.resize(n);
    int m = 0;
    for (int i = 0; i < n; ++i) {
        if (m > 0 && ws.key[i] == ws.key[i - 1]) continue;  // coincident: first occurrence wins
        const int idx = ws.ord[i];
        ws.kept[m] = idx;
        ws.px[m] = u[idx];
        ws.py[m] = v[idx];
        ++m;
    }
    if (m < 3) return 0;

    ws.tv.resize(6 * std::size_t(m));
    ws.tn.resize(6 * std::size_t(m));
    ws.hnext.assign(m, -1);
    ws.hprev.assign(m, -1);
    ws.hedge.assign(m, -1);
    ws.stack.clear();
    Sweep s{ws.px.data(), ws.py.data(), ws.tv.data(), ws.tn.data(), ws.hnext.data(),
            ws.hprev.data(), ws.hedge.data(), &ws.stack};
    s.wide = (maxx - minx) >= (1 << 14) || (maxy - miny) >= (1 << 14);

    // Collinear prefix: points 0..k-1 on one line, point k off it.
    int k = 2;
    while (k < m && s.orient(0, 1, k) == 0) ++k;
    if (k == m) return 0;  // collinear set
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
    for (int p = apex + 1; p < m; ++p) {
        if (!s.insert(p)) return -2;  // cannot happen for lexicographic input
    }

    tris.resize(3 * std::size_t(s.ntri));
    for (int e = 0; e < 3 * s.ntri; ++e) tris[e] = ws.kept[ws.tv[e]];
    return s.ntri;
}

}  // namespace ps
