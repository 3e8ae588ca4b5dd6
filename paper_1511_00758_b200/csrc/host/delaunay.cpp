// delaunay.cpp — exact radial-sweep Delaunay for pixel coordinates.
//
// Same output set as planestereo::delaunayTriangulate
// (proj/src/delaunay.cpp:288-325; see delaunay.hpp for the contract), built
// for the per-frame, per-iteration host step of the B200 engine.
//
// Why not the reference's lexicographic sweep: inserting points in (u, v)
// order along grid-like support sets creates long slivers that are flipped
// again and again (measured: ~17 flips and ~36 in-circle tests per point on
// a VGA support set).  Here points are inserted in order of exact squared
// distance from an integer centre instead (a radial sweep): every new point
// is strictly outside the current hull (all earlier points lie in a closed
// disc it is on or outside of), a hull vertex near the right angle is found
// through an angular hash, and Lawson flips restore the Delaunay property
// (~1-3 flips per point).
//
// Because the insertion order is no longer lexicographic, cocircular ties are
// decided by an explicit symbolic perturbation instead of by the order: of
// the four points of a cocircular quad, the lexicographically largest is
// treated as lifted above the common circle.  That makes every cocircular
// diagonal avoid the lex-max vertex of its quad, which is exactly the rule
// the reference's output obeys, and the perturbed
// predicate defines a unique triangulation, so the result is independent of
// the insertion order.  Collinear hull points stay vertices (strict
// visibility), as in the reference.
//
// Predicates are exact: int64 when the bounding box spans < 2^14 px
// (in-circle magnitude < 2^60), __int128 otherwise.
#include "delaunay.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace ps {

namespace {

inline int nxt(int e) { return (e % 3 == 2) ? e - 2 : e + 1; }

struct Sweep {
    const int* x;
    const int* y;
    int* tv;
    int* tn;
    int* hnext;
    int* hprev;
    int* hedge;
    std::vector<int>* stack;
    std::vector<int>* hash;
    int cx = 0, cy = 0;
    int ntri = 0;
    bool wide = false;

    long long orient(int a, int b, int c) const {
        const long long abx = (long long)x[b] - x[a], aby = (long long)y[b] - y[a];
        const long long acx = (long long)x[c] - x[a], acy = (long long)y[c] - y[a];
        return abx * acy - aby * acx;
    }

    int incircle_sign(int a, int b, int c, int d) const {
        const long long adx = (long long)x[a] - x[d], ady = (long long)y[a] - y[d];
        const long long bdx = (long long)x[b] - x[d], bdy = (long long)y[b] - y[d];
        const long long cdx = (long long)x[c] - x[d], cdy = (long long)y[c] - y[d];
        const long long aq = adx * adx + ady * ady;
        const long long bq = bdx * bdx + bdy * bdy;
        const long long cq = cdx * cdx + cdy * cdy;
        if (!wide) {
            const long long det = adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                                  aq * (bdx * cdy - cdx * bdy);
            return (det > 0) - (det < 0);
        }
        using W = __int128;
        const W det = W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                      W(aq) * (W(bdx) * cdy - W(cdx) * bdy);
        return (det > 0) - (det < 0);
    }

    bool lex_less(int a, int b) const { return x[a] < x[b] || (x[a] == x[b] && y[a] < y[b]); }

    // d strictly inside the circumcircle of CCW (a,b,c), with cocircular ties
    // broken by lifting the lexicographically largest of the four points.
    bool inside(int a, int b, int c, int d) const {
        const int s = incircle_sign(a, b, c, d);
        if (s != 0) return s > 0;
        int m = a;
        if (lex_less(m, b)) m = b;
        if (lex_less(m, c)) m = c;
        if (lex_less(m, d)) m = d;
        if (m == d) return false;
        // the lifted vertex m pulls the plane through a,b,c up: d is inside iff
        // its barycentric coordinate for m is positive.
        if (m == a) return orient(b, c, d) > 0;
        if (m == b) return orient(c, a, d) > 0;
        return orient(a, b, d) > 0;
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

    int hash_key(int p) const {
        const double dx = double(x[p] - cx), dy = double(y[p] - cy);
        const double s = std::fabs(dx) + std::fabs(dy);
        double ang = 0.0;
        if (s > 0.0) {
            const double q = dx / s;
            ang = (dy > 0.0 ? 3.0 - q : 1.0 + q) * 0.25;  // pseudo-angle in [0, 1)
        }
        const int n = int(hash->size());
        int k = int(ang * n);
        return k >= n ? n - 1 : (k < 0 ? 0 : k);
    }

    // Edge e: a->b with apex c = the new point, twin f: b->a with apex d.
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
            // (a,b,c)+(b,a,d) -> (a,d,c)+(d,b,c)
            tv[e1] = d;
            tv[f] = d;
            tv[f1] = b;
            tv[f2] = c;
            tn[e] = nf1;
            if (nf1 >= 0) tn[nf1] = e; else hedge[a] = e;
            tn[e1] = f2;
            tn[f2] = e1;
            tn[e2] = ne2;
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
        // start from a hull vertex near p's angle (stale hash entries are skipped)
        const int n = int(hash->size());
        const int key = hash_key(p);
        int start = -1;
        for (int j = 0; j < n; ++j) {
            const int s = (*hash)[(key + j) % n];
            if (s >= 0 && hnext[s] >= 0) {
                start = s;
                break;
            }
        }
        if (start < 0) return false;
        start = hprev[start];
        int e = start;
        while (!visible(e, p)) {
            e = hnext[e];
            if (e == start) return false;  // p not strictly outside: cannot happen
        }
        int a = e, b = hnext[e];
        while (hnext[b] != a && visible(b, p)) b = hnext[b];
        while (hprev[a] != b && visible(hprev[a], p)) a = hprev[a];
        int prevE1 = -1, firstE0 = -1;
        for (int xv = a; xv != b;) {
            const int xn = hnext[xv];
            const int t = add(xv, p, xn, prevE1, -1, hedge[xv]);
            if (firstE0 < 0) firstE0 = t;
            prevE1 = t + 1;
            stack->push_back(t + 2);
            if (xv != a) hnext[xv] = hprev[xv] = -1;  // left the hull
            xv = xn;
        }
        hull(a, p);
        hull(p, b);
        hedge[a] = firstE0;
        hedge[p] = prevE1;
        (*hash)[hash_key(p)] = p;
        (*hash)[hash_key(a)] = a;
        legalize();
        return true;
    }
};

void radix_sort_keys(std::vector<uint64_t>& key, std::vector<int>& ord, std::vector<uint64_t>& kt,
                     std::vector<int>& ot, int n, int bits) {
    kt.resize(n);
    ot.resize(n);
    constexpr int kDigit = 11;
    constexpr int kBuckets = 1 << kDigit;
    uint32_t count[kBuckets];
    for (int shift = 0; shift < bits; shift += kDigit) {
        std::fill(count, count + kBuckets, 0u);
        for (int i = 0; i < n; ++i) ++count[(key[i] >> shift) & (kBuckets - 1)];
        uint32_t sum = 0;
        for (int d = 0; d < kBuckets; ++d) {
            const uint32_t c = count[d];
            count[d] = sum;
            sum += c;
        }
        for (int i = 0; i < n; ++i) {
            const uint32_t pos = count[(key[i] >> shift) & (kBuckets - 1)]++;
            kt[pos] = key[i];
            ot[pos] = ord[i];
        }
        key.swap(kt);
        ord.swap(ot);
    }
}

int bit_width(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

}  // namespace

// Lexicographic (u, v) order with coincident points removed, first occurrence
// kept (delaunay.cpp:296-311): ws.kept[0..m) = original indices.  Stable LSD
// radix sort on 43-bit keys, so equal coordinates keep input order.
void lex_order(const int* u, const int* v, int n, DelaunayWorkspace& ws, int& minx, int& miny,
               int& m, int& spanx, int& spany) {
    minx = u[0];
    miny = v[0];
    int maxx = u[0], maxy = v[0];
    for (int i = 1; i < n; ++i) {
        minx = std::min(minx, u[i]);
        maxx = std::max(maxx, u[i]);
        miny = std::min(miny, v[i]);
        maxy = std::max(maxy, v[i]);
    }
    spanx = maxx - minx;
    spany = maxy - miny;
    ws.key.resize(n);
    ws.ord.resize(n);
    for (int i = 0; i < n; ++i) {
        ws.key[i] = (uint64_t(uint32_t(u[i] - minx)) << 21) | uint64_t(uint32_t(v[i] - miny));
        ws.ord[i] = i;
    }
    radix_sort_keys(ws.key, ws.ord, ws.key_tmp, ws.ord_tmp, n, 21 + bit_width(uint64_t(spanx)));
    ws.kept.resize(n);
    m = 0;
    for (int i = 0; i < n; ++i) {
        if (m > 0 && ws.key[i] == ws.key[i - 1]) continue;
        ws.kept[m++] = ws.ord[i];
    }
}

int delaunay(const int* u, const int* v, int n, std::vector<int>& tris, DelaunayWorkspace& ws) {
    tris.clear();
    constexpr int kLimit = 1 << 20;
    for (int i = 0; i < n; ++i)
        if (std::abs(u[i]) >= kLimit || std::abs(v[i]) >= kLimit) return -1;
    if (n < 3) return 0;

    // 1. lexicographic order + dedup, first occurrence wins
    int minx, miny, m, spanx, spany;
    lex_order(u, v, n, ws, minx, miny, m, spanx, spany);
    if (m < 3) return 0;
    const int maxx = minx + spanx, maxy = miny + spany;

    // 2. radial order around an integer centre (stable: ties stay lexicographic)
    const int cx = minx + (maxx - minx) / 2, cy = miny + (maxy - miny) / 2;
    ws.key.resize(m);
    ws.ord.resize(m);
    uint64_t dmax = 0;
    for (int i = 0; i < m; ++i) {
        const long long dx = u[ws.kept[i]] - cx, dy = v[ws.kept[i]] - cy;
        ws.key[i] = uint64_t(dx * dx + dy * dy);
        dmax = std::max(dmax, ws.key[i]);
        ws.ord[i] = ws.kept[i];
    }
    radix_sort_keys(ws.key, ws.ord, ws.key_tmp, ws.ord_tmp, m, bit_width(dmax));
    ws.px.resize(m);
    ws.py.resize(m);
    for (int i = 0; i < m; ++i) {
        ws.px[i] = u[ws.ord[i]];
        ws.py[i] = v[ws.ord[i]];
    }

    ws.tv.resize(6 * std::size_t(m));
    ws.tn.resize(6 * std::size_t(m));
    ws.hnext.assign(m, -1);
    ws.hprev.assign(m, -1);
    ws.hedge.assign(m, -1);
    ws.stack.clear();
    int hs = int(std::ceil(std::sqrt(double(m))));
    std::vector<int>& hash = ws.kept;  // reuse storage: kept[] is no longer needed
    hash.assign(std::max(hs, 1), -1);
    Sweep s{ws.px.data(), ws.py.data(), ws.tv.data(), ws.tn.data(), ws.hnext.data(),
            ws.hprev.data(), ws.hedge.data(), &ws.stack, &hash};
    s.cx = cx;
    s.cy = cy;
    s.wide = (maxx - minx) >= (1 << 14) || (maxy - miny) >= (1 << 14);

    // 3. collinear prefix (in radial order) + first off-line point: a fan over
    //    the prefix sorted along its line (it is Delaunay as built).
    int k = 2;
    while (k < m && s.orient(0, 1, k) == 0) ++k;
    if (k == m) return 0;  // collinear set
    const int apex = k;
    std::vector<int> line(k);
    for (int i = 0; i < k; ++i) line[i] = i;
    std::sort(line.begin(), line.end(), [&](int a, int b) { return s.lex_less(a, b); });
    if (s.orient(line[0], line[1], apex) > 0) {
        int prevE1 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = s.add(line[j], line[j + 1], apex, -1, -1, prevE1);
            if (j == 0) s.hedge[apex] = e + 2;
            s.hedge[line[j]] = e;
            prevE1 = e + 1;
        }
        s.hedge[line[k - 1]] = prevE1;
        for (int j = 0; j + 1 < k; ++j) s.hull(line[j], line[j + 1]);
        s.hull(line[k - 1], apex);
        s.hull(apex, line[0]);
    } else {
        int prevE2 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = s.add(line[j + 1], line[j], apex, -1, prevE2, -1);
            if (j == 0) s.hedge[line[0]] = e + 1;
            s.hedge[line[j + 1]] = e;
            prevE2 = e + 2;
        }
        s.hedge[apex] = prevE2;
        for (int j = 0; j + 1 < k; ++j) s.hull(line[j + 1], line[j]);
        s.hull(line[0], apex);
        s.hull(apex, line[k - 1]);
    }
    for (int i = 0; i <= k; ++i) hash[s.hash_key(i)] = i;

    // 4. radial sweep
    for (int p = apex + 1; p < m; ++p) {
        if (!s.insert(p)) return -2;
    }

    tris.resize(3 * std::size_t(s.ntri));
    for (int e = 0; e < 3 * s.ntri; ++e) tris[e] = ws.ord[ws.tv[e]];
    return s.ntri;
}

}  // namespace ps
