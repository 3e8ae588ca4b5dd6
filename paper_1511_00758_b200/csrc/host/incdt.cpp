// incdt.cpp — see incdt.hpp.
//
// Half-edge e = 4t + k runs from V(e) to V(next(e)); triangles are 32-byte
// records (vertices + twins: one cache line per flip side), counter-clockwise
// (orient > 0); N(e) is the twin or -1 on the hull; a hull edge a -> b
// (interior on its left) is hedge[a], with hnext[a] = b.
#include "incdt.hpp"

#include <algorithm>
#include <cstdlib>

namespace ps {

namespace {
inline int nxt(int e) { return (e & 3) == 2 ? e - 2 : e + 1; }
inline int prv(int e) { return (e & 3) == 0 ? e + 2 : e - 1; }
}  // namespace

void IncDT::reset() {
    nv_ = 0;
    wide_ = false;
    P_.clear();
    T_.clear();
    hnext_.clear();
    hprev_.clear();
    hedge_.clear();
    stack_.clear();
    pending_.clear();
    vtri_.clear();
    bucket_.clear();
    bw_ = bh_ = 0;
    last_ = 0;
    lastp_ = -1;
    hull0_ = -1;
}

// delaunay.cpp's predicate: exact in-circle, cocircular ties broken by lifting
// the lexicographically largest of the four points.
bool IncDT::inside(int a, int b, int c, int d) {
    ++tests;
    const Pt A = P_[a], B = P_[b], Cc = P_[c], D = P_[d];
    const long long adx = (long long)A.x - D.x, ady = (long long)A.y - D.y;
    const long long bdx = (long long)B.x - D.x, bdy = (long long)B.y - D.y;
    const long long cdx = (long long)Cc.x - D.x, cdy = (long long)Cc.y - D.y;
    const long long aq = adx * adx + ady * ady;
    const long long bq = bdx * bdx + bdy * bdy;
    const long long cq = cdx * cdx + cdy * cdy;
    int s;
    if (!wide_) {
        const long long det = adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                              aq * (bdx * cdy - cdx * bdy);
        s = (det > 0) - (det < 0);
    } else {
        using W = __int128;
        const W det = W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                      W(aq) * (W(bdx) * cdy - W(cdx) * bdy);
        s = (det > 0) - (det < 0);
    }
    if (s != 0) return s > 0;
    auto lex_less = [&](int p, int q) {
        return P_[p].x < P_[q].x || (P_[p].x == P_[q].x && P_[p].y < P_[q].y);
    };
    int m = a;
    if (lex_less(m, b)) m = b;
    if (lex_less(m, c)) m = c;
    if (lex_less(m, d)) m = d;
    if (m == d) return false;
    if (m == a) return orient(b, c, d) > 0;
    if (m == b) return orient(c, a, d) > 0;
    return orient(a, b, d) > 0;
}

int IncDT::add(int a, int b, int c, int na, int nb, int nc) {
    const int e = 4 * int(T_.size());
    T_.push_back(Tri{{a, b, c}, {na, nb, nc}, {0, 0}});
    if (na >= 0) N(na) = e;
    if (nb >= 0) N(nb) = e + 1;
    if (nc >= 0) N(nc) = e + 2;
    return e;
}

// Lawson flips of the edges opposite the new point (LIFO), strict perturbed
// in-circle: (a,b,c)+(b,a,d) -> (a,d,c)+(d,b,c), as delaunay.cpp.
void IncDT::legalize() {
    while (!stack_.empty()) {
        const int e = stack_.back();
        stack_.pop_back();
        const int f = N(e);
        if (f < 0) continue;
        const int e1 = nxt(e), e2 = nxt(e1);
        const int f1 = nxt(f), f2 = nxt(f1);
        const int a = V(e), b = V(e1), c = V(e2), d = V(f2);
        if (!inside(a, b, c, d)) continue;
        ++flips;
        const int ne1 = N(e1), nf1 = N(f1), nf2 = N(f2);
        V(e1) = d;
        V(f) = d;
        V(f1) = b;
        V(f2) = c;
        link(e, nf1);
        if (nf1 < 0) hedge_[a] = e;
        link(e1, f2);
        link(f, nf2);
        if (nf2 < 0) hedge_[d] = f;
        link(f1, ne1);
        if (ne1 < 0) hedge_[b] = f1;
        stack_.push_back(e);
        stack_.push_back(f);
    }
}

bool IncDT::start(int) {
    // first point, first point elsewhere, first point off their line
    const int a = pending_[0];
    int b = -1, c = -1;
    for (int q : pending_) {
        if (b < 0) {
            if (P_[q].x != P_[a].x || P_[q].y != P_[a].y) b = q;
        } else if (orient(a, b, q) != 0) {
            c = q;
            break;
        }
    }
    if (c < 0) return true;  // still degenerate: keep waiting
    if (orient(a, b, c) < 0) std::swap(b, c);
    const int e = add(a, b, c, -1, -1, -1);
    hnext_[a] = b;
    hnext_[b] = c;
    hnext_[c] = a;
    hprev_[b] = a;
    hprev_[c] = b;
    hprev_[a] = c;
    hedge_[a] = e;
    hedge_[b] = e + 1;
    hedge_[c] = e + 2;
    hull0_ = a;
    last_ = 0;
    std::vector<int> rest;
    rest.swap(pending_);
    for (int q : rest)
        if (q != a && q != b && q != c && !insert(q)) return false;
    return true;
}

bool IncDT::insert(int p) {
    // visibility walk from the last triangle, or from one holding the last
    // vertex inserted in p's 8x8 bucket when p is not next to the last point
    int t = std::min(last_, triangles() - 1);
    int* bucket = nullptr;
    const Pt pp = P_[p];
    {
        const int bx = (pp.x - bx0_) >> 3, by = (pp.y - by0_) >> 3;
        if (bx >= 0 && bx < bw_ && by >= 0 && by < bh_) {
            bucket = &bucket_[size_t(by) * bw_ + bx];
            const int q = *bucket;
            const bool near_last =
                lastp_ >= 0 && std::abs(P_[lastp_].x - pp.x) + std::abs(P_[lastp_].y - pp.y) <= 6;
            if (q >= 0 && !near_last) {
                const int tq = vtri_[q];
                const Tri& T = T_[tq];
                if (T.v[0] == q || T.v[1] == q || T.v[2] == q) t = tq;
                else ++stale;
            }
        }
    }
    int out_edge = -1, on_edge = -1;
    for (int steps = 0;; ++steps) {
        if (steps > 4 * triangles() + 16) return false;
        ++walk_steps;
        const Tri& T = T_[t];
        const Pt A = P_[T.v[0]], B = P_[T.v[1]], Cc = P_[T.v[2]];
        const long long o0 = ((long long)B.x - A.x) * (pp.y - A.y) - ((long long)B.y - A.y) * (pp.x - A.x);
        const long long o1 = ((long long)Cc.x - B.x) * (pp.y - B.y) - ((long long)Cc.y - B.y) * (pp.x - B.x);
        const long long o2 = ((long long)A.x - Cc.x) * (pp.y - Cc.y) - ((long long)A.y - Cc.y) * (pp.x - Cc.x);
        const long long o[3] = {o0, o1, o2};
        // leave through the first separating edge, starting at a rotating index
        int neg = -1;
        for (int i = 0; i < 3 && neg < 0; ++i) {
            const int k = (steps + i) % 3;
            if (o[k] < 0) neg = k;
        }
        if (neg >= 0) {
            const int f = T.n[neg];
            if (f < 0) {
                out_edge = 4 * t + neg;
                break;
            }
            t = f >> 2;
            continue;
        }
        const int zeros = (o0 == 0) + (o1 == 0) + (o2 == 0);
        if (zeros >= 2) return true;  // coincides with a vertex: the first occurrence wins
        if (zeros == 1) on_edge = 4 * t + (o0 == 0 ? 0 : o1 == 0 ? 1 : 2);
        break;
    }

    if (out_edge >= 0) {  // outside the hull: fan to the strictly visible chain
        int a = V(out_edge), b = V(nxt(out_edge));
        auto visible = [&](int x) { return orient(x, hnext_[x], p) < 0; };
        while (hnext_[b] != a && visible(b)) b = hnext_[b];
        while (hprev_[a] != b && visible(hprev_[a])) a = hprev_[a];
        int prevE1 = -1, firstE0 = -1;
        for (int xv = a; xv != b;) {
            const int xn = hnext_[xv];
            const int e = add(xv, p, xn, prevE1, -1, hedge_[xv]);
            if (firstE0 < 0) firstE0 = e;
            prevE1 = e + 1;
            stack_.push_back(e + 2);
            if (xv != a) {
                hnext_[xv] = hprev_[xv] = hedge_[xv] = -1;  // left the hull
                if (hull0_ == xv) hull0_ = p;
            }
            xv = xn;
        }
        hnext_[a] = p;
        hprev_[p] = a;
        hnext_[p] = b;
        hprev_[b] = p;
        hedge_[a] = firstE0;
        hedge_[p] = prevE1;
        last_ = firstE0 >> 2;
    } else if (on_edge < 0) {  // strictly inside triangle t: 1 -> 3
        const int e0 = 4 * t;
        const int a = V(e0), b = V(e0 + 1), c = V(e0 + 2);
        const int nbc = N(e0 + 1), nca = N(e0 + 2);
        V(e0 + 2) = p;
        const int t1 = add(b, c, p, nbc, -1, -1);
        const int t2 = add(c, a, p, nca, -1, -1);
        link(e0 + 1, t1 + 2);
        link(t1 + 1, t2 + 2);
        link(t2 + 1, e0 + 2);
        if (nbc < 0) hedge_[b] = t1;
        if (nca < 0) hedge_[c] = t2;
        stack_.push_back(e0);
        stack_.push_back(t1);
        stack_.push_back(t2);
        last_ = t;
    } else {  // on the edge a -> b of t
        const int e = on_edge, tt = e >> 2;
        const int a = V(e), b = V(nxt(e)), c = V(prv(e));
        const int nbc = N(nxt(e)), nca = N(prv(e));
        const int f = N(e);
        const int e0 = 4 * tt;
        if (f < 0) {  // a hull edge: 1 -> 2, p joins the hull between a and b
            V(e0) = a;
            V(e0 + 1) = p;
            V(e0 + 2) = c;
            N(e0) = -1;
            link(e0 + 2, nca);
            const int t1 = add(p, b, c, -1, nbc, -1);
            link(e0 + 1, t1 + 2);
            if (nca < 0) hedge_[c] = e0 + 2;
            if (nbc < 0) hedge_[b] = t1 + 1;
            hnext_[a] = p;
            hprev_[p] = a;
            hnext_[p] = b;
            hprev_[b] = p;
            hedge_[a] = e0;
            hedge_[p] = t1;
            stack_.push_back(e0 + 2);
            stack_.push_back(t1 + 1);
        } else {  // 2 -> 4 with the twin triangle (b, a, d)
            const int s0 = 4 * (f >> 2);
            const int f1 = nxt(f), f2 = nxt(f1);
            const int d = V(f2);
            const int nad = N(f1), ndb = N(f2);
            V(e0) = a;
            V(e0 + 1) = p;
            V(e0 + 2) = c;
            V(s0) = b;
            V(s0 + 1) = p;
            V(s0 + 2) = d;
            N(e0) = N(e0 + 1) = N(s0) = N(s0 + 1) = -1;
            link(e0 + 2, nca);
            link(s0 + 2, ndb);
            const int t1 = add(p, b, c, -1, nbc, -1);
            const int t3 = add(p, a, d, -1, nad, -1);
            link(e0, t3);          // a->p | p->a
            link(e0 + 1, t1 + 2);  // p->c | c->p
            link(t1, s0);          // p->b | b->p
            link(s0 + 1, t3 + 2);  // p->d | d->p
            if (nca < 0) hedge_[c] = e0 + 2;
            if (nbc < 0) hedge_[b] = t1 + 1;
            if (ndb < 0) hedge_[d] = s0 + 2;
            if (nad < 0) hedge_[a] = t3 + 1;
            stack_.push_back(e0 + 2);
            stack_.push_back(t1 + 1);
            stack_.push_back(s0 + 2);
            stack_.push_back(t3 + 1);
        }
        last_ = tt;
    }
    legalize();
    vtri_[p] = last_;  // holds p: flips during its own insertion keep p in the slot
    lastp_ = p;
    if (bucket) *bucket = p;
    return true;
}

bool IncDT::extend(const int* u, const int* v, int n) {
    if (n <= nv_) return true;
    constexpr int kLimit = 1 << 20;
    for (int i = nv_; i < n; ++i)
        if (std::abs(u[i]) >= kLimit || std::abs(v[i]) >= kLimit) return false;
    P_.resize(n);
    for (int i = nv_; i < n; ++i) P_[i] = Pt{u[i], v[i]};
    int minx = P_[0].x, maxx = P_[0].x, miny = P_[0].y, maxy = P_[0].y;
    for (int i = 1; i < n; ++i) {
        minx = std::min(minx, P_[i].x);
        maxx = std::max(maxx, P_[i].x);
        miny = std::min(miny, P_[i].y);
        maxy = std::max(maxy, P_[i].y);
    }
    wide_ = (maxx - minx) >= (1 << 14) || (maxy - miny) >= (1 << 14);
    hnext_.resize(n, -1);
    hprev_.resize(n, -1);
    hedge_.resize(n, -1);
    vtri_.resize(n, 0);
    if (bw_ == 0 || minx < bx0_ || miny < by0_ || ((maxx - bx0_) >> 3) >= bw_ || ((maxy - by0_) >> 3) >= bh_) {
        // (re)size the hint buckets to the points' extent (the hints are only a start)
        bx0_ = minx;
        by0_ = miny;
        bw_ = ((maxx - minx) >> 3) + 1;
        bh_ = ((maxy - miny) >> 3) + 1;
        bucket_.assign(size_t(bw_) * bh_, -1);
    }
    T_.reserve(2 * size_t(n) + 8);
    for (int p = nv_; p < n; ++p) {
        if (T_.empty()) {
            pending_.push_back(p);
            if (pending_.size() >= 3 && !start(n)) return false;
            continue;
        }
        if (!insert(p)) return false;
    }
    nv_ = n;
    return true;
}

}  // namespace ps
