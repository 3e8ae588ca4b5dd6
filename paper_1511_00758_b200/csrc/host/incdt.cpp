// incdt.cpp — see incdt.hpp.
//
// Half-edge e = 3t + k runs from tv[e] to tv[next(e)]; triangles are
// counter-clockwise (orient > 0), tn[e] is the twin or -1 on the hull; a hull
// edge a -> b (interior on its left) is hedge[a], with hnext[a] = b.
#include "incdt.hpp"

#include <algorithm>
#include <cstdlib>

namespace ps {

namespace {
inline int nxt(int e) { return (e % 3 == 2) ? e - 2 : e + 1; }
inline int prv(int e) { return (e % 3 == 0) ? e + 2 : e - 1; }
}  // namespace

void IncDT::reset() {
    nv_ = 0;
    wide_ = false;
    tv_.clear();
    tn_.clear();
    hnext_.clear();
    hprev_.clear();
    hedge_.clear();
    stack_.clear();
    pending_.clear();
    vtri_.clear();
    bucket_.clear();
    bw_ = bh_ = 0;
    last_ = 0;
    hull0_ = -1;
}

// delaunay.cpp's predicate: exact in-circle, cocircular ties broken by lifting
// the lexicographically largest of the four points.
bool IncDT::inside(int a, int b, int c, int d) {
    ++tests;
    const long long adx = (long long)x_[a] - x_[d], ady = (long long)y_[a] - y_[d];
    const long long bdx = (long long)x_[b] - x_[d], bdy = (long long)y_[b] - y_[d];
    const long long cdx = (long long)x_[c] - x_[d], cdy = (long long)y_[c] - y_[d];
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
    auto lex_less = [&](int p, int q) { return x_[p] < x_[q] || (x_[p] == x_[q] && y_[p] < y_[q]); };
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
    const int e = int(tv_.size());
    tv_.push_back(a);
    tv_.push_back(b);
    tv_.push_back(c);
    tn_.push_back(na);
    tn_.push_back(nb);
    tn_.push_back(nc);
    if (na >= 0) tn_[na] = e;
    if (nb >= 0) tn_[nb] = e + 1;
    if (nc >= 0) tn_[nc] = e + 2;
    return e;
}

// Lawson flips of the edges opposite the new point (LIFO), strict perturbed
// in-circle: (a,b,c)+(b,a,d) -> (a,d,c)+(d,b,c), as delaunay.cpp.
void IncDT::legalize() {
    while (!stack_.empty()) {
        const int e = stack_.back();
        stack_.pop_back();
        const int f = tn_[e];
        if (f < 0) continue;
        const int e1 = nxt(e), e2 = nxt(e1);
        const int f1 = nxt(f), f2 = nxt(f1);
        const int a = tv_[e], b = tv_[e1], c = tv_[e2], d = tv_[f2];
        if (!inside(a, b, c, d)) continue;
        ++flips;
        const int ne1 = tn_[e1], nf1 = tn_[f1], nf2 = tn_[f2];
        tv_[e1] = d;
        tv_[f] = d;
        tv_[f1] = b;
        tv_[f2] = c;
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
            if (x_[q] != x_[a] || y_[q] != y_[a]) b = q;
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
    // visibility walk from a triangle of the last vertex inserted near p
    int t = std::min(last_, triangles() - 1);
    int* bucket = nullptr;
    {
        const int bx = (x_[p] - bx0_) >> 3, by = (y_[p] - by0_) >> 3;
        if (bx >= 0 && bx < bw_ && by >= 0 && by < bh_) {
            bucket = &bucket_[size_t(by) * bw_ + bx];
            const int q = *bucket;
            if (q >= 0) {
                const int tq = vtri_[q];
                if (tv_[3 * tq] == q || tv_[3 * tq + 1] == q || tv_[3 * tq + 2] == q) t = tq;
            }
        }
    }
    int out_edge = -1, on_edge = -1;
    for (int steps = 0;; ++steps) {
        if (steps > 4 * triangles() + 16) return false;
        ++walk_steps;
        const int e0 = 3 * t;
        long long o[3];
        int neg = -1, zeros = 0, zk = -1;
        for (int k = 0; k < 3; ++k) {
            o[k] = orient(tv_[e0 + k], tv_[e0 + (k + 1) % 3], p);
            if (o[k] == 0) {
                ++zeros;
                zk = k;
            }
        }
        // leave through the first separating edge, starting at a rotating index
        for (int i = 0; i < 3 && neg < 0; ++i) {
            const int k = (steps + i) % 3;
            if (o[k] < 0) neg = k;
        }
        if (neg >= 0) {
            const int f = tn_[e0 + neg];
            if (f < 0) {
                out_edge = e0 + neg;
                break;
            }
            t = f / 3;
            continue;
        }
        if (zeros >= 2) return true;  // coincides with a vertex: the first occurrence wins
        if (zeros == 1) on_edge = e0 + zk;
        break;
    }

    if (out_edge >= 0) {  // outside the hull: fan to the strictly visible chain
        int a = tv_[out_edge], b = tv_[nxt(out_edge)];
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
        last_ = firstE0 / 3;
    } else if (on_edge < 0) {  // strictly inside triangle t: 1 -> 3
        const int e0 = 3 * t;
        const int a = tv_[e0], b = tv_[e0 + 1], c = tv_[e0 + 2];
        const int nbc = tn_[e0 + 1], nca = tn_[e0 + 2];
        tv_[e0 + 2] = p;
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
        const int e = on_edge, tt = e / 3;
        const int a = tv_[e], b = tv_[nxt(e)], c = tv_[prv(e)];
        const int nbc = tn_[nxt(e)], nca = tn_[prv(e)];
        const int f = tn_[e];
        const int e0 = 3 * tt;
        if (f < 0) {  // a hull edge: 1 -> 2, p joins the hull between a and b
            tv_[e0] = a;
            tv_[e0 + 1] = p;
            tv_[e0 + 2] = c;
            tn_[e0] = -1;
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
            const int s0 = 3 * (f / 3);
            const int f1 = nxt(f), f2 = nxt(f1);
            const int d = tv_[f2];
            const int nad = tn_[f1], ndb = tn_[f2];
            tv_[e0] = a;
            tv_[e0 + 1] = p;
            tv_[e0 + 2] = c;
            tv_[s0] = b;
            tv_[s0 + 1] = p;
            tv_[s0 + 2] = d;
            tn_[e0] = tn_[e0 + 1] = tn_[s0] = tn_[s0 + 1] = -1;
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
    if (bucket) *bucket = p;
    return true;
}

bool IncDT::extend(const int* u, const int* v, int n) {
    x_ = u;
    y_ = v;
    if (n <= nv_) return true;
    constexpr int kLimit = 1 << 20;
    int minx = 0, maxx = 0, miny = 0, maxy = 0;
    for (int i = 0; i < n; ++i) {
        if (std::abs(u[i]) >= kLimit || std::abs(v[i]) >= kLimit) return false;
        if (i == 0 || u[i] < minx) minx = u[i];
        if (i == 0 || u[i] > maxx) maxx = u[i];
        if (i == 0 || v[i] < miny) miny = v[i];
        if (i == 0 || v[i] > maxy) maxy = v[i];
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
    tv_.reserve(6 * size_t(n));
    tn_.reserve(6 * size_t(n));
    for (int p = nv_; p < n; ++p) {
        if (tv_.empty()) {
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
