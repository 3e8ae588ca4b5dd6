// sweep_order.cpp — see sweep_order.hpp.
#include "sweep_order.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

namespace ps {

SweepOrder::Scratch& SweepOrder::own() {
    if (!own_) own_ = std::make_unique<Scratch>();
    return *own_;
}

void SweepOrder::init(const int* px, const int* py, int m) {
    x_ = px;
    y_ = py;
    m_ = m;
    apex_ = -1;
    if (m < 3) return;
    minx_ = maxx_ = px[0];
    miny_ = maxy_ = py[0];
    for (int i = 1; i < m; ++i) {
        minx_ = std::min(minx_, px[i]);
        maxx_ = std::max(maxx_, px[i]);
        miny_ = std::min(miny_, py[i]);
        maxy_ = std::max(maxy_, py[i]);
    }
    wide_ = (maxx_ - minx_) >= (1 << 14) || (maxy_ - miny_) >= (1 << 14);
    int k = 2;
    while (k < m && orient(0, 1, k) == 0) ++k;
    if (k == m) return;
    apex_ = k;
    side_pos_ = orient(0, 1, apex_) > 0;

    // Andrew's monotone chains (collinear points kept, as the sweep's strict
    // visibility keeps them on the hull): lower pops on a right turn, upper
    // on a left turn.
    // Both chains in one pass over the points (they are independent), raw
    // stacks; every entry of below*/pop* is written exactly once.
    belowL_.resize(m);
    belowU_.resize(m);
    popL_.resize(m);
    popU_.resize(m);
    stk_.resize(2 * size_t(m));
    int* sL = stk_.data();
    int* sU = sL + m;
    int nL = 0, nU = 0;
    const int* X = px;
    const int* Y = py;
    auto ori = [X, Y](int a, int b, int c) {
        return ((long long)X[b] - X[a]) * ((long long)Y[c] - Y[a]) - ((long long)Y[b] - Y[a]) * ((long long)X[c] - X[a]);
    };
    for (int r = 0; r < m; ++r) {
        popL_[r] = popU_[r] = INT_MAX;
        while (nL >= 2 && ori(sL[nL - 2], sL[nL - 1], r) < 0) popL_[sL[--nL]] = r;
        belowL_[r] = nL ? sL[nL - 1] : -1;
        sL[nL++] = r;
        while (nU >= 2 && ori(sU[nU - 2], sU[nU - 1], r) > 0) popU_[sU[--nU]] = r;
        belowU_[r] = nU ? sU[nU - 1] : -1;
        sU[nU++] = r;
    }

    // bucket grid: ranks are increasing within a bucket (filled in rank
    // order); power-of-two buckets, so the cell of a point is two shifts
    const int span = std::max(maxx_ - minx_, maxy_ - miny_) + 1;
    bs_ = 16;
    int sh = 4;
    while (bs_ < span / 512) {
        bs_ *= 2;
        ++sh;
    }
    bw_ = (maxx_ - minx_) / bs_ + 1;
    bh_ = (maxy_ - miny_) / bs_ + 1;
    bstart_.assign(size_t(bw_) * bh_ + 1, 0);
    bcell_.resize(m);
    for (int r = 0; r < m; ++r) {
        const int c = ((py[r] - miny_) >> sh) * bw_ + ((px[r] - minx_) >> sh);
        bcell_[r] = c;
        ++bstart_[size_t(c) + 1];
    }
    for (size_t i = 1; i < bstart_.size(); ++i) bstart_[i] += bstart_[i - 1];
    bitems_.resize(m);
    bfill_.assign(bstart_.begin(), bstart_.end() - 1);
    for (int r = 0; r < m; ++r) bitems_[bfill_[bcell_[r]]++] = r;
}

int SweepOrder::incircle(int a, int b, int c, int d) const {
    const long long adx = (long long)x_[a] - x_[d], ady = (long long)y_[a] - y_[d];
    const long long bdx = (long long)x_[b] - x_[d], bdy = (long long)y_[b] - y_[d];
    const long long cdx = (long long)x_[c] - x_[d], cdy = (long long)y_[c] - y_[d];
    const long long aq = adx * adx + ady * ady;
    const long long bq = bdx * bdx + bdy * bdy;
    const long long cq = cdx * cdx + cdy * cdy;
    if (!wide_) {
        const long long det = adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                              aq * (bdx * cdy - cdx * bdy);
        return (det > 0) - (det < 0);
    }
    using W = __int128;
    const W det = W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                  W(aq) * (W(bdx) * cdy - W(cdx) * bdy);
    return (det > 0) - (det < 0);
}

// Counter-clockwise predecessor of o on hull(Q<p): the lower chain runs left
// to right, the upper chain right to left, and they meet at rank 0 and p - 1.
int SweepOrder::hull_prev(int o, int p) const {
    if (o >= p) return -1;
    const bool onL = popL_[o] >= p, onU = popU_[o] >= p;
    if (onL && o != 0) return belowL_[o];
    if (!onU) return -1;
    // o on the upper chain (or o = 0): the element directly above it there
    for (int x = p - 1, steps = 0; x >= 0 && steps <= m_; x = belowU_[x], ++steps)
        if (belowU_[x] == o) return x;
    return -1;
}

int SweepOrder::fan_index(int o, int p) const {
    const int h = hull_prev(o, p);
    if (h < 0 || orient(h, o, p) >= 0) return -1;  // hull edge h->o not strictly visible
    int count = 0;
    for (int x = h; count <= m_; ++count) {
        const int hx = hull_prev(x, p);
        if (hx < 0 || orient(hx, x, p) >= 0) break;
        x = hx;
    }
    return count;
}

bool SweepOrder::disk_clear(int a, int b, int c, int p, int& u0, int& u1, int& v0, int& v1,
                            int grow) const {
    const double ax = x_[a], ay = y_[a];
    const double bxx = x_[b] - ax, byy = y_[b] - ay;
    const double cxx = x_[c] - ax, cyy = y_[c] - ay;
    const double D = 2.0 * (bxx * cyy - byy * cxx);
    const double bq = bxx * bxx + byy * byy, cq = cxx * cxx + cyy * cyy;
    const double ux = (cyy * bq - byy * cq) / D, uy = (bxx * cq - cxx * bq) / D;
    const double cx = ax + ux, cy = ay + uy;
    const double r = std::sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0;
    // fast path: the disk's bounding box (clipped to the prefix region) is inside the box
    const double right = double(x_[p]);
    if ((cx - r >= u0 || u0 <= minx_) && (cx + r <= u1 || u1 >= right) &&
        (cy - r >= v0 || v0 <= miny_) && (cy + r <= v1 || v1 >= maxy_))
        return true;
    bool clear = true;
    int nu0 = u0, nu1 = u1, nv0 = v0, nv1 = v1;
    const double ylo = std::max(double(miny_), cy - r), yhi = std::min(double(maxy_), cy + r);
    if (ylo > yhi) return true;
    const int rb0 = (int(std::floor(ylo)) - miny_) / bs_, rb1 = (int(std::floor(yhi)) - miny_) / bs_;
    for (int by = std::max(0, rb0); by <= std::min(bh_ - 1, rb1); ++by) {
        const double ry0 = miny_ + double(by) * bs_, ry1 = ry0 + bs_ - 1;
        double dy = 0.0;
        if (cy < ry0) dy = ry0 - cy;
        else if (cy > ry1) dy = cy - ry1;
        if (dy > r) continue;
        const double half = std::sqrt(std::max(0.0, r * r - dy * dy));
        const double xlo = std::max(double(minx_), cx - half);
        const double xhi = std::min(right, cx + half);
        if (xlo > xhi) continue;
        const int cb0 = std::max(0, (int(std::floor(xlo)) - minx_) / bs_);
        const int cb1 = std::min(bw_ - 1, (int(std::floor(xhi)) - minx_) / bs_);
        for (int bx = cb0; bx <= cb1; ++bx) {
            const int rx0 = minx_ + bx * bs_, rx1 = rx0 + bs_ - 1;
            if (rx0 >= u0 && rx1 <= u1 && int(ry0) >= v0 && int(ry1) <= v1) continue;
            const size_t bk = size_t(by) * bw_ + bx;
            for (int i = bstart_[bk]; i < bstart_[bk + 1]; ++i) {
                const int q = bitems_[i];
                if (q >= p) break;
                if (x_[q] >= u0 && x_[q] <= u1 && y_[q] >= v0 && y_[q] <= v1) continue;
                if (incircle(a, b, c, q) >= 0) {
                    clear = false;
                    nu0 = std::min(nu0, x_[q] - grow);
                    nu1 = std::max(nu1, x_[q] + grow);
                    nv0 = std::min(nv0, y_[q] - grow);
                    nv1 = std::max(nv1, y_[q] + grow);
                }
            }
        }
    }
    u0 = nu0;
    u1 = nu1;
    v0 = nv0;
    v1 = nv1;
    return clear;
}

bool SweepOrder::window_triangle(int o, int p, int out[3], Scratch& S) const {
    const int R0 = 2 * bs_;
    int u0 = std::min(x_[o], x_[p]) - R0, u1 = std::min(std::max(x_[o], x_[p]) + R0, x_[p]);
    int v0 = std::min(y_[o], y_[p]) - R0, v1 = std::max(y_[o], y_[p]) + R0;
    auto clamp_box = [&] {
        u0 = std::max(u0, minx_);
        v0 = std::max(v0, miny_);
        v1 = std::min(v1, maxy_);
        u1 = std::min(u1, x_[p]);
    };
    clamp_box();
    for (int attempt = 0; attempt < 24; ++attempt) {
        // prefix points (rank < p) in the box
        S.wu_.clear();
        S.wv_.clear();
        S.wrank_.clear();
        int io = -1;
        const int bx0 = (u0 - minx_) / bs_, bx1 = (u1 - minx_) / bs_;
        const int by0 = (v0 - miny_) / bs_, by1 = (v1 - miny_) / bs_;
        for (int by = by0; by <= by1; ++by)
            for (int bx = bx0; bx <= bx1; ++bx) {
                const size_t b = size_t(by) * bw_ + bx;
                for (int i = bstart_[b]; i < bstart_[b + 1]; ++i) {
                    const int r = bitems_[i];
                    if (r >= p) break;
                    if (x_[r] < u0 || x_[r] > u1 || y_[r] < v0 || y_[r] > v1) continue;
                    if (r == o) io = int(S.wrank_.size());
                    S.wu_.push_back(x_[r]);
                    S.wv_.push_back(y_[r]);
                    S.wrank_.push_back(r);
                }
            }
        ++S.windows;
        S.window_points += (long long)S.wrank_.size();
        int sigma[3] = {-1, -1, -1};
        const int nw = int(S.wrank_.size());
        if (io >= 0 && nw >= 3) {
            const int nt = delaunay(S.wu_.data(), S.wv_.data(), nw, S.wtris_, S.ws_);
            for (int t = 0; t < nt && sigma[0] < 0; ++t) {
                const int* tr = &S.wtris_[3 * size_t(t)];
                for (int k = 0; k < 3; ++k) {
                    if (tr[k] != io) continue;
                    const int a = S.wrank_[tr[(k + 1) % 3]], b = S.wrank_[tr[(k + 2) % 3]];
                    if (orient(o, a, p) > 0 && orient(o, p, b) > 0) {
                        sigma[0] = o;
                        sigma[1] = a;
                        sigma[2] = b;
                    }
                }
            }
        }
        if (sigma[0] < 0) {  // the window's hull cuts the direction off: grow
            const int g = R0 << (attempt + 1);
            u0 -= g;
            v0 -= g;
            v1 += g;
            u1 += g;
            clamp_box();
            if (u0 == minx_ && v0 == miny_ && v1 == maxy_ && u1 == x_[p] && attempt > 2 && nw >= 3 && io >= 0)
                return false;  // the whole prefix and still no triangle: inconsistent
            continue;
        }
        // certificate: no prefix point outside the box in sigma's closed disk
        const bool bad = !disk_clear(sigma[0], sigma[1], sigma[2], p, u0, u1, v0, v1, R0);
        if (!bad) {
            out[0] = sigma[0];
            out[1] = sigma[1];
            out[2] = sigma[2];
            return true;
        }
        clamp_box();
    }
    return false;
}

bool SweepOrder::query(int a, int b, int c, uint64_t& birth, int stored[3], Scratch& S) const {
    bool more = false;
    return query_steps(a, b, c, birth, stored, S, -1, more);
}

// query() following at most max_steps sigma steps (-1: no limit); `more` is
// set when the chain needs more (the result is then not written).
bool SweepOrder::query_steps(int a, int b, int c, uint64_t& birth, int stored[3], Scratch& S, int max_steps,
                             bool& more) const {
    more = false;
    if (apex_ < 0) return false;
    struct Step {
        int o, t, p;
    };
    std::vector<Step> chain;
    int T[3] = {a, b, c};
    int base[3];
    for (int guard = 0;; ++guard) {
        if (guard > m_) return false;
        int k = 0;
        if (T[1] > T[k]) k = 1;
        if (T[2] > T[k]) k = 2;
        const int p = T[k], o = T[(k + 1) % 3], t = T[(k + 2) % 3];
        if (p == apex_) {  // the leading fan (delaunay.cpp:123-164)
            const int j = std::min(t, o);
            if (std::max(t, o) != j + 1 || j + 1 >= apex_) return false;
            base[0] = side_pos_ ? j : j + 1;
            base[1] = side_pos_ ? j + 1 : j;
            base[2] = apex_;
            birth = (uint64_t(uint32_t(apex_)) << 32) | uint32_t(j);
            break;
        }
        const int j = fan_index(o, p);
        if (j >= 0) {  // fan slot j of p: stored (x_j .. t, p, x_{j+1} = o)
            base[0] = t;
            base[1] = p;
            base[2] = o;
            birth = (uint64_t(uint32_t(p)) << 32) | uint32_t(j);
            break;
        }
        if (max_steps >= 0 && int(chain.size()) >= max_steps) {
            more = true;
            return false;
        }
        int sigma[3];
        if (!window_triangle(o, p, sigma, S)) return false;
        chain.push_back({o, t, p});
        T[0] = sigma[0];
        T[1] = sigma[1];
        T[2] = sigma[2];
    }
    // unwind: the slot of sigma, with o one position forward, then t, p
    int cur[3] = {base[0], base[1], base[2]};
    for (size_t i = chain.size(); i-- > 0;) {
        const Step& s = chain[i];
        int k = -1;
        for (int q = 0; q < 3; ++q)
            if (cur[q] == s.o) k = q;
        if (k < 0) return false;
        int nx[3];
        nx[(k + 1) % 3] = s.o;
        nx[(k + 2) % 3] = s.t;
        nx[k] = s.p;
        cur[0] = nx[0];
        cur[1] = nx[1];
        cur[2] = nx[2];
    }
    stored[0] = cur[0];
    stored[1] = cur[1];
    stored[2] = cur[2];
    return true;
}

}  // namespace ps

namespace ps {

// The reference sweep (delaunay.cpp:50-284) over the window's points in rank
// order, recording for every slot the contents it had before each time it
// was eaten (a Lawson flip on the side not holding the new point).
bool SweepOrder::replay(int u0, int u1, int v0, int v1, int last, Scratch& S) const {
    S.rrank_.clear();
    const int bx0 = std::max(0, (u0 - minx_) / bs_), bx1 = std::min(bw_ - 1, (u1 - minx_) / bs_);
    const int by0 = std::max(0, (v0 - miny_) / bs_), by1 = std::min(bh_ - 1, (v1 - miny_) / bs_);
    for (int by = by0; by <= by1; ++by)
        for (int bx = bx0; bx <= bx1; ++bx) {
            const size_t b = size_t(by) * bw_ + bx;
            for (int i = bstart_[b]; i < bstart_[b + 1]; ++i) {
                const int r = bitems_[i];
                if (r > last) break;  // ranks increase within a bucket
                if (x_[r] >= u0 && x_[r] <= u1 && y_[r] >= v0 && y_[r] <= v1) S.rrank_.push_back(r);
            }
        }
    std::sort(S.rrank_.begin(), S.rrank_.end());
    const int n = int(S.rrank_.size());
    ++S.replays;
    S.replay_points += n;
    S.rs_.clear();
    S.rh_.clear();
    S.rapex_ = -1;
    if (n < 3) return false;
    const int* R = S.rrank_.data();
    auto ori = [&](int a, int b, int c) { return orient(R[a], R[b], R[c]); };
    int k = 2;
    while (k < n && ori(0, 1, k) == 0) ++k;
    if (k == n) return false;
    S.rapex_ = k;
    S.rhn_.assign(n, -1);
    S.rhp_.assign(n, -1);
    S.rhe_.assign(n, -1);
    S.rstack_.clear();
    S.rs_.reserve(2 * size_t(n));
    auto V = [&](int e) -> int& { return S.rs_[e >> 2].v[e & 3]; };
    auto N = [&](int e) -> int& { return S.rs_[e >> 2].n[e & 3]; };
    auto lnext = [](int e) { return (e & 3) == 2 ? e - 2 : e + 1; };
    auto add = [&](int a, int b, int c, int na, int nb, int nc, int birth, int fan) {
        const int e = 4 * int(S.rs_.size());
        S.rs_.push_back(Scratch::Slot{{a, b, c}, {na, nb, nc}, birth, fan, -1, -1, a});
        if (na >= 0) N(na) = e;
        if (nb >= 0) N(nb) = e + 1;
        if (nc >= 0) N(nc) = e + 2;
        return e;
    };
    auto hull = [&](int a, int b) {
        S.rhn_[a] = b;
        S.rhp_[b] = a;
    };
    const int apex = k;
    if (ori(0, 1, apex) > 0) {
        int prevE1 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = add(j, j + 1, apex, -1, -1, prevE1, apex, j);
            if (j == 0) S.rhe_[apex] = e + 2;
            S.rhe_[j] = e;
            prevE1 = e + 1;
        }
        S.rhe_[k - 1] = prevE1;
        for (int j = 0; j + 1 < k; ++j) hull(j, j + 1);
        hull(k - 1, apex);
        hull(apex, 0);
    } else {
        int prevE2 = -1;
        for (int j = 0; j + 1 < k; ++j) {
            const int e = add(j + 1, j, apex, -1, prevE2, -1, apex, j);
            if (j == 0) S.rhe_[0] = e + 1;
            S.rhe_[j + 1] = e;
            prevE2 = e + 2;
        }
        S.rhe_[apex] = prevE2;
        for (int j = 0; j + 1 < k; ++j) hull(j + 1, j);
        hull(0, apex);
        hull(apex, k - 1);
    }
    auto visible = [&](int a, int p) { return ori(a, S.rhn_[a], p) < 0; };
    for (int p = apex + 1; p < n; ++p) {
        const int q = p - 1;
        int a, b;
        if (visible(q, p)) {
            a = q;
            b = S.rhn_[q];
        } else if (visible(S.rhp_[q], p)) {
            a = S.rhp_[q];
            b = q;
        } else {
            return false;
        }
        while (S.rhn_[b] != a && visible(b, p)) b = S.rhn_[b];
        while (S.rhp_[a] != b && visible(S.rhp_[a], p)) a = S.rhp_[a];
        int prevE1 = -1, firstE0 = -1, j = 0;
        for (int xv = a; xv != b; ++j) {
            const int xn = S.rhn_[xv];
            const int e = add(xv, p, xn, prevE1, -1, S.rhe_[xv], p, j);
            if (firstE0 < 0) firstE0 = e;
            prevE1 = e + 1;
            S.rstack_.push_back(e + 2);
            xv = xn;
        }
        hull(a, p);
        hull(p, b);
        S.rhe_[a] = firstE0;
        S.rhe_[p] = prevE1;
        while (!S.rstack_.empty()) {
            const int e = S.rstack_.back();
            S.rstack_.pop_back();
            const int f = N(e);
            if (f < 0) continue;
            const int e1 = lnext(e), e2 = lnext(e1);
            const int f1 = lnext(f), f2 = lnext(f1);
            const int va = V(e), vb = V(e1), vc = V(e2), vd = V(f2);
            if (incircle(R[va], R[vb], R[vc], R[vd]) <= 0) continue;
            Scratch::Slot& F = S.rs_[f >> 2];
            if (F.eaten != p) {  // first time this insertion eats the slot
                S.rh_.push_back(Scratch::Hist{p, {F.v[0], F.v[1], F.v[2]}, F.hist});
                F.hist = int(S.rh_.size()) - 1;
                F.eaten = p;
            }
            const int ne1 = N(e1), nf1 = N(f1), nf2 = N(f2);
            V(e1) = vd;
            V(f) = vd;
            V(f1) = vb;
            V(f2) = vc;
            N(e) = nf1;
            if (nf1 >= 0) N(nf1) = e; else S.rhe_[va] = e;
            N(e1) = f2;
            N(f2) = e1;
            N(f) = nf2;
            if (nf2 >= 0) N(nf2) = f; else S.rhe_[vd] = f;
            N(f1) = ne1;
            if (ne1 >= 0) N(ne1) = f1; else S.rhe_[vb] = f1;
            S.rstack_.push_back(e);
            S.rstack_.push_back(f);
        }
    }
    return true;
}

bool SweepOrder::resolve(const int* tris, int count, uint64_t* birth, int* stored, Scratch& S) const {
    if (apex_ < 0) return false;
    if (count <= 0) return true;
    // Triangles left in a fan slot of their lexicographic maximum need no
    // window (query's first step, from the precomputed hull chains); only the
    // rest are resolved by window replays.
    std::vector<int> rest;
    for (int t = 0; t < count; ++t) {
        bool more = false;
        if (query_steps(tris[3 * t], tris[3 * t + 1], tris[3 * t + 2], birth[t], stored + 3 * t, S, 0, more))
            continue;
        if (!more) return false;
        rest.push_back(t);
    }
    ++S.fast_calls;
    S.fast_hits += count - int(rest.size());
    if (rest.empty()) return true;
    if (int(rest.size()) < count) {
        std::vector<int> sub(3 * rest.size()), ss(3 * rest.size());
        std::vector<uint64_t> sb(rest.size());
        for (size_t i = 0; i < rest.size(); ++i)
            for (int q = 0; q < 3; ++q) sub[3 * i + q] = tris[3 * rest[i] + q];
        if (!resolve_windows(sub.data(), int(rest.size()), sb.data(), ss.data(), S)) return false;
        for (size_t i = 0; i < rest.size(); ++i) {
            birth[rest[i]] = sb[i];
            for (int q = 0; q < 3; ++q) stored[3 * rest[i] + q] = ss[3 * i + q];
        }
        return true;
    }
    return resolve_windows(tris, count, birth, stored, S);
}

bool SweepOrder::resolve_windows(const int* tris, int count, uint64_t* birth, int* stored, Scratch& S) const {
    int bu0 = INT_MAX, bu1 = INT_MIN, bv0 = INT_MAX, bv1 = INT_MIN;
    // Only points up to the last vertex of the triangles matter: a final
    // triangle's slot is not touched after its last vertex is inserted, so
    // the window's sweep stops there (and its right edge is that column).
    int last = 0;
    for (int i = 0; i < 3 * count; ++i) last = std::max(last, tris[i]);
    const int xcap = x_[last];
    for (int i = 0; i < 3 * count; ++i) {
        bu0 = std::min(bu0, x_[tris[i]]);
        bu1 = std::max(bu1, x_[tris[i]]);
        bv0 = std::min(bv0, y_[tris[i]]);
        bv1 = std::max(bv1, y_[tris[i]]);
    }
    const double area = double(maxx_ - minx_ + 1) * double(maxy_ - miny_ + 1);
    int delta = std::max(8, int(2.0 * std::sqrt(area / m_)));
    std::vector<std::pair<uint64_t, int>> key;  // sorted vertex set -> slot
    int u0 = std::max(minx_, bu0 - delta), u1 = std::min(xcap, bu1 + delta);
    int v0, v1;
    // The sweep's slots are column-tall fans eaten point after point down the
    // column, so a window that cuts the columns is (nearly always) grown to
    // the full height anyway, one doubling per attempt (measured on BASELINE
    // config 2: 5-6 attempts, the last one full-height): start there.
    (void)bv0;
    (void)bv1;
    v0 = miny_;
    v1 = maxy_;
    for (int attempt = 0;; ++attempt) {
        // the window holds every point up to `last`: nothing to certify
        const bool whole = u0 <= minx_ && u1 >= xcap && v0 <= miny_ && v1 >= maxy_;
        // growth for the next attempt: towards the points that broke a
        // certificate, or uniformly when the window itself was too small
        int nu0 = u0, nu1 = u1, nv0 = v0, nv1 = v1;
        bool grow_all = false;
        bool gl = false, gr = false, gd = false, gu = false;  // directional growth requests
        const bool fallback = attempt >= 8;  // then finish chains in the full set instead
        const bool replayed = replay(u0, u1, v0, v1, last, S);
        bool ok = replayed;
        if (!replayed) grow_all = true;
        // the query triangles' slots: a linear scan for a few triangles, a
        // sorted key table for many
        const bool table = count > 8;
        if (replayed && table) {
            key.clear();
            for (size_t s = 0; s < S.rs_.size(); ++s) {
                int a = S.rrank_[S.rs_[s].v[0]], b = S.rrank_[S.rs_[s].v[1]], c = S.rrank_[S.rs_[s].v[2]];
                if (a > b) std::swap(a, b);
                if (b > c) std::swap(b, c);
                if (a > b) std::swap(a, b);
                key.push_back({(uint64_t(uint32_t(a)) << 42) ^ (uint64_t(uint32_t(b)) << 21) ^ uint64_t(uint32_t(c)), int(s)});
            }
            std::sort(key.begin(), key.end());
        }
        for (int t = 0; replayed && !grow_all && t < count; ++t) {
            int a = tris[3 * t], b = tris[3 * t + 1], c = tris[3 * t + 2];
            if (a > b) std::swap(a, b);
            if (b > c) std::swap(b, c);
            if (a > b) std::swap(a, b);
            int slot = -1;
            if (table) {
                const uint64_t kq = (uint64_t(uint32_t(a)) << 42) ^ (uint64_t(uint32_t(b)) << 21) ^ uint64_t(uint32_t(c));
                auto it = std::lower_bound(key.begin(), key.end(), std::make_pair(kq, -1));
                for (; it != key.end() && it->first == kq; ++it) {
                    const Scratch::Slot& SL = S.rs_[it->second];
                    int sa = S.rrank_[SL.v[0]], sb = S.rrank_[SL.v[1]], sc = S.rrank_[SL.v[2]];
                    if (sa > sb) std::swap(sa, sb);
                    if (sb > sc) std::swap(sb, sc);
                    if (sa > sb) std::swap(sa, sb);
                    if (sa == a && sb == b && sc == c) slot = it->second;
                }
            } else {
                // window indices of the three ranks (rrank_ is sorted)
                const auto wi = [&](int r) {
                    const auto it = std::lower_bound(S.rrank_.begin(), S.rrank_.end(), r);
                    return it != S.rrank_.end() && *it == r ? int(it - S.rrank_.begin()) : -1;
                };
                const int ia = wi(a), ib = wi(b), ic = wi(c);
                if (ia >= 0 && ib >= 0 && ic >= 0)
                    for (size_t q = 0; q < S.rs_.size() && slot < 0; ++q) {
                        const int* v = S.rs_[q].v;
                        const bool has_a = v[0] == ia || v[1] == ia || v[2] == ia;
                        const bool has_b = v[0] == ib || v[1] == ib || v[2] == ib;
                        const bool has_c = v[0] == ic || v[1] == ic || v[2] == ic;
                        if (has_a && has_b && has_c) slot = int(q);
                    }
            }
            if (slot < 0) {  // not a triangle of DT(window): the window is too small
                ok = false;
                grow_all = true;
                break;
            }
            const Scratch::Slot& SL = S.rs_[slot];
            // every eaten state must be a triangle of the full prefix DT
            int origin = SL.v[2];
            bool certified = true;
            for (int h = SL.hist; h >= 0; h = S.rh_[h].prev) {
                const Scratch::Hist& H = S.rh_[h];
                int cu0 = u0, cu1 = u1, cv0 = v0, cv1 = v1;
                if (!whole && !disk_clear(S.rrank_[H.v[0]], S.rrank_[H.v[1]], S.rrank_[H.v[2]], S.rrank_[H.time],
                                          cu0, cu1, cv0, cv1, 2 * bs_)) {
                    ok = certified = false;
                    nu0 = std::min(nu0, cu0);
                    nu1 = std::max(nu1, cu1);
                    nv0 = std::min(nv0, cv0);
                    nv1 = std::max(nv1, cv1);
                }
                origin = H.v[2];  // after the loop: the contents at the end of its birth
            }
            if (!certified) continue;  // collect every offender of this attempt
            const int pb = S.rrank_[SL.birth];
            // contents at the end of the birth insertion, in the window's rotation
            int b0[3] = {SL.v[0], SL.v[1], SL.v[2]};
            for (int h = SL.hist; h >= 0; h = S.rh_[h].prev)
                for (int q = 0; q < 3; ++q) b0[q] = S.rh_[h].v[q];
            uint64_t bkey;
            int shift = 0;  // window rotation -> the sweep's rotation
            const bool lead = SL.birth == S.rapex_;
            int jq = -1;
            if (whole) {
                jq = SL.fan;
            } else if (lead) {
                bool same = S.rapex_ == apex_ && pb == apex_;
                for (int i = 0; i <= S.rapex_ && same; ++i) same = S.rrank_[i] == i;
                if (same) jq = SL.fan;
            } else {
                jq = fan_index(S.rrank_[origin], pb);
                if (jq < 0 && !fallback) {
                    // the window's visible chain from pb (it faces right, toward the
                    // new point) is not the full prefix's: the window cut the
                    // columns at the sweep front, so grow it vertically
                    gd = gu = true;
                    ok = false;
                    continue;
                }
            }
            if (jq >= 0) {
                bkey = (uint64_t(uint32_t(pb)) << 32) | uint32_t(jq);
            } else {
                // born from a hull vertex of the window that is not one of the
                // full prefix's: follow the rest of the chain in the full set
                const int tb[3] = {S.rrank_[b0[0]], S.rrank_[b0[1]], S.rrank_[b0[2]]};
                int qs[3];
                if (!query(tb[0], tb[1], tb[2], bkey, qs, S)) return false;
                int pos = -1;
                for (int q = 0; q < 3; ++q)
                    if (qs[q] == tb[0]) pos = q;
                if (pos < 0) return false;
                shift = pos;  // qs[(i + shift) % 3] == tb[i]
            }
            int fin[3];
            for (int q = 0; q < 3; ++q) fin[(q + shift) % 3] = S.rrank_[SL.v[q]];
            birth[t] = bkey;
            stored[3 * t] = fin[0];
            stored[3 * t + 1] = fin[1];
            stored[3 * t + 2] = fin[2];
        }
        if (ok) return true;
        if (whole) return false;
        if (!grow_all && (gl || gr || gd || gu)) {
            const int gx = std::max(delta, (u1 - u0 + 1) / 2), gy = std::max(delta, (v1 - v0 + 1) / 2);
            if (gl) nu0 = std::min(nu0, u0 - gx);
            if (gr) nu1 = std::max(nu1, u1 + gx);
            if (gd) nv0 = std::min(nv0, v0 - gy);
            if (gu) nv1 = std::max(nv1, v1 + gy);
        }
        auto clamp_new = [&] {
            nu0 = std::max(minx_, nu0);
            nu1 = std::min(xcap, nu1);
            nv0 = std::max(miny_, nv0);
            nv1 = std::min(maxy_, nv1);
        };
        clamp_new();
        // uniform growth when asked, or when no directed growth could enlarge the window
        if (grow_all || (nu0 == u0 && nu1 == u1 && nv0 == v0 && nv1 == v1)) {
            delta *= 2;
            nu0 = std::min(nu0, u0 - delta);
            nu1 = std::max(nu1, u1 + delta);
            nv0 = std::min(nv0, v0 - delta);
            nv1 = std::max(nv1, v1 + delta);
            clamp_new();
        }
        u0 = nu0;
        u1 = nu1;
        v0 = nv0;
        v1 = nv1;
    }
}

}  // namespace ps
