// star_dt.cuh — K4 on the device: the exact Delaunay triangulation of a
// frame's support points as the union of per-point STARS, one thread per point.
//
// Replaces delaunayTriangulate's triangle set (proj/src/delaunay.cpp:288-325;
// SURVEY App. A.1): the unique Delaunay triangulation under the lexicographic-
// maximum perturbation of the in-circle test, which is what the reference's
// lexicographic sweep produces.  Because that triangulation is unique, each
// point can compute its own neighbours independently:
//   * the nearest other point q0 is a Delaunay neighbour (its closed diameter
//     disc holds no third point);
//   * given a Delaunay edge p -> q, the next neighbour counter-clockwise is the
//     point r left of p -> q whose circle through p, q, r is smallest in the
//     perturbed order (no other left point inside it) — a gift wrap;
//   * a uniform grid of the points bounds every search: first the points of
//     the cells around p (gathered once, coordinates relative to p); a
//     winner is final once every cell meeting its circumcircle has been
//     scanned (no point outside can beat it); no point lies left of p -> q
//     exactly when p -> q runs clockwise along the convex hull (build_hull).
// Hull vertices have a gap in their star; the wrap then also runs clockwise
// from q0.  Each triangle is emitted by its smallest vertex index.
//
// Predicates are exact in int64: coordinates are pixels, and a frame's span
// below 2^14 bounds the in-circle determinant by 2^60 (wider frames take the
// host path).  Written __host__ __device__ so the same code is unit-tested on
// the CPU against the sweep (tests/cpp/test_star.cpp).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define PS_HD __host__ __device__ __forceinline__
#else
#define PS_HD inline
#endif

namespace ps {
namespace star {

struct Grid {
    const int* u;           // support coordinates, list order
    const int* v;
    const uint8_t* dup;     // 1 = a coincident point with a smaller index exists (not a vertex)
    const int* cell_start;  // gw * gh + 1 prefix offsets
    const int* cell_items;  // point indices per cell, increasing
    int n;
    int minx, miny, maxx, maxy;  // bounding box of the points
    int gs;                      // cell size (pixels)
    int gw, gh;
    // per column x = minx + i (i < maxx - minx + 1): the points of smallest and
    // largest v (-1: none; the smallest index on ties, never a duplicate)
    const int* col_lo;
    const int* col_hi;
    // per point: its counter-clockwise successor / predecessor on the convex
    // hull boundary (collinear boundary points included, as the sweep keeps
    // them, delaunay.cpp:116-118), -1 off the hull (build_hull)
    const int* hnext;
    const int* hprev;
    int flat;    // every point on one line: no triangle at all
    double igs;  // 1 / gs
};

PS_HD long long orient(const Grid& g, int a, int b, int c) {
    return ((long long)g.u[b] - g.u[a]) * ((long long)g.v[c] - g.v[a]) -
           ((long long)g.v[b] - g.v[a]) * ((long long)g.u[c] - g.u[a]);
}

PS_HD bool lex_less(const Grid& g, int a, int b) {
    return g.u[a] < g.u[b] || (g.u[a] == g.u[b] && g.v[a] < g.v[b]);
}

// d strictly inside the circumcircle of CCW (a, b, c), cocircular ties broken
// by lifting the lexicographically largest of the four (delaunay.cpp, incdt.cpp).
PS_HD bool inside(const Grid& g, int a, int b, int c, int d) {
    const long long adx = (long long)g.u[a] - g.u[d], ady = (long long)g.v[a] - g.v[d];
    const long long bdx = (long long)g.u[b] - g.u[d], bdy = (long long)g.v[b] - g.v[d];
    const long long cdx = (long long)g.u[c] - g.u[d], cdy = (long long)g.v[c] - g.v[d];
    const long long aq = adx * adx + ady * ady;
    const long long bq = bdx * bdx + bdy * bdy;
    const long long cq = cdx * cdx + cdy * cdy;
    const long long det = adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) +
                          aq * (bdx * cdy - cdx * bdy);
    if (det != 0) return det > 0;
    int m = a;
    if (lex_less(g, m, b)) m = b;
    if (lex_less(g, m, c)) m = c;
    if (lex_less(g, m, d)) m = d;
    if (m == d) return false;
    if (m == a) return orient(g, b, c, d) > 0;
    if (m == b) return orient(g, c, a, d) > 0;
    return orient(g, a, b, d) > 0;
}

struct Box {
    int x0, y0, x1, y1;  // cell index range, inclusive
};

// (the cell searches are conservative by a pixel: a product by 1 / gs does)
PS_HD int cell_x(const Grid& g, double x) {
    int c = int(floor((x - g.minx) * g.igs));
    return c < 0 ? 0 : (c >= g.gw ? g.gw - 1 : c);
}
PS_HD int cell_y(const Grid& g, double y) {
    int c = int(floor((y - g.miny) * g.igs));
    return c < 0 ? 0 : (c >= g.gh ? g.gh - 1 : c);
}

PS_HD bool covers(const Box& outer, const Box& inner) {
    return outer.x0 <= inner.x0 && outer.y0 <= inner.y0 && outer.x1 >= inner.x1 && outer.y1 >= inner.y1;
}

PS_HD Box unite(const Box& a, const Box& b) {
    return Box{a.x0 < b.x0 ? a.x0 : b.x0, a.y0 < b.y0 ? a.y0 : b.y0, a.x1 > b.x1 ? a.x1 : b.x1,
               a.y1 > b.y1 ? a.y1 : b.y1};
}

// Scan the cells of `box` not in `done` (done may be empty: x0 > x1).
template <class F>
PS_HD void scan_new(const Grid& g, const Box& box, const Box& done, F&& f) {
    for (int cy = box.y0; cy <= box.y1; ++cy)
        for (int cx = box.x0; cx <= box.x1; ++cx) {
            if (done.x0 <= done.x1 && cx >= done.x0 && cx <= done.x1 && cy >= done.y0 && cy <= done.y1)
                continue;
            const int c = cy * g.gw + cx;
            for (int i = g.cell_start[c]; i < g.cell_start[c + 1]; ++i) f(g.cell_items[i]);
        }
}

// p -> q is a hull edge with the outside on `side` (left: side > 0): no
// point lies there.  Counter-clockwise the hull has its interior on the left.
PS_HD bool hull_edge(const Grid& g, int p, int q, int side) {
    return g.flat || (side > 0 ? g.hprev[p] == q : g.hnext[p] == q);
}

// The convex hull boundary of the frame's points, collinear points kept
// (Andrew's monotone chains over the lexicographic order, the order the
// reference's sweep inserts in).  Its points are the column extremes (a
// boundary point of a non-vertical hull edge has nothing below or above it
// in its column) and every point of the first and last columns; those are
// visited in (u, v) order through the grid (points of one cell sorted).
// lo/hi: scratch for the two chains (n + 2 * cols ints each is enough);
// hnext/hprev (n entries, preset to -1) receive the boundary cycle.  Returns
// 1 when all points lie on one line (no cycle is written), else 0.
PS_HD int build_hull(const Grid& g, int* lo, int* hi, int* hnext, int* hprev) {
    const int cols = g.maxx - g.minx + 1;
    // first and last occupied columns
    int c0 = -1, c1 = -1;
    for (int i = 0; i < cols; ++i)
        if (g.col_lo[i] >= 0) {
            if (c0 < 0) c0 = i;
            c1 = i;
        }
    if (c0 < 0) return 1;
    int nl = 0, nh = 0;
    auto push = [&](int s) {
        while (nl >= 2 && orient(g, lo[nl - 2], lo[nl - 1], s) < 0) --nl;
        lo[nl++] = s;
        while (nh >= 2 && orient(g, hi[nh - 2], hi[nh - 1], s) > 0) --nh;
        hi[nh++] = s;
    };
    auto whole_column = [&](int i) {  // every point of column minx + i, by v
        const int x = g.minx + i;
        const int cx = (x - g.minx) / g.gs;
        for (int cy = 0; cy < g.gh; ++cy) {
            const int c = cy * g.gw + cx;
            // the cell's points of this column in increasing v (distinct:
            // coincident points are duplicates), by repeated selection
            int last = -2147483647;
            for (;;) {
                int best = -1;
                for (int k = g.cell_start[c]; k < g.cell_start[c + 1]; ++k) {
                    const int s = g.cell_items[k];
                    if (g.u[s] != x || g.dup[s] || g.v[s] <= last) continue;
                    if (best < 0 || g.v[s] < g.v[best]) best = s;
                }
                if (best < 0) break;
                push(best);
                last = g.v[best];
            }
        }
    };
    whole_column(c0);
    for (int i = c0 + 1; i < c1; ++i) {
        const int a = g.col_lo[i], b = g.col_hi[i];
        if (a < 0) continue;
        push(a);
        if (b != a) push(b);
    }
    if (c1 != c0) whole_column(c1);
    if (nl < 2) return 1;
    // collinear set: the upper chain then holds the same line as the lower
    bool flat = true;
    for (int i = 1; i + 1 < nh && flat; ++i) flat = orient(g, hi[0], hi[nh - 1], hi[i]) == 0;
    for (int i = 1; i + 1 < nl && flat; ++i) flat = orient(g, lo[0], lo[nl - 1], lo[i]) == 0;
    if (flat) return 1;
    // counter-clockwise: the lower chain left to right, then the upper chain
    // right to left; they share their first and last points
    for (int i = 0; i + 1 < nl; ++i) {
        hnext[lo[i]] = lo[i + 1];
        hprev[lo[i + 1]] = lo[i];
    }
    for (int i = nh - 1; i > 0; --i) {
        hnext[hi[i]] = hi[i - 1];
        hprev[hi[i - 1]] = hi[i];
    }
    return 0;
}

// Circumcircle of the CCW triangle (a, b, c): centre and radius (with a
// margin, so a cell test never drops a point inside the exact circle).
struct Disc {
    double cx, cy, r;
};
PS_HD Disc disc_of(const Grid& g, int a, int b, int c) {
    const double ax = g.u[a], ay = g.v[a];
    const double bx = g.u[b] - ax, by = g.v[b] - ay, cx = g.u[c] - ax, cy = g.v[c] - ay;
    const double iD = 0.5 / (bx * cy - by * cx);
    const double bq = bx * bx + by * by, cq = cx * cx + cy * cy;
    const double ux = (cy * bq - by * cq) * iD, uy = (bx * cq - cx * bq) * iD;
    return Disc{ax + ux, ay + uy, sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0};
}
// Where a point beating the winner of a p -> q search can lie: inside the
// winner's circle and strictly on the search side of p -> q.  When the
// circle's centre is on the other side that part is the minor segment cut
// by the chord pq, which lies within its sagitta h of the chord (for the
// near-collinear triangles along the hull the circle is huge but h is
// tiny); else the circle's bounding box.  Pixel coordinates, a margin kept.
struct Region {
    double x0, y0, x1, y1;
};
PS_HD Region search_region(const Grid& g, int p, int q, int side, const Disc& d) {
    Region box{d.cx - d.r, d.cy - d.r, d.cx + d.r, d.cy + d.r};
    // the points' bounding box: where the circle pokes out of it, only the
    // part inside matters (the circle's extent across the box's bounds)
    if (box.x0 < g.minx) box.x0 = g.minx;
    if (box.x1 > g.maxx) box.x1 = g.maxx;
    if (box.y0 < g.miny) box.y0 = g.miny;
    if (box.y1 > g.maxy) box.y1 = g.maxy;
    {
        const double dx = d.cx < box.x0 ? box.x0 - d.cx : (d.cx > box.x1 ? d.cx - box.x1 : 0.0);
        const double dy = d.cy < box.y0 ? box.y0 - d.cy : (d.cy > box.y1 ? d.cy - box.y1 : 0.0);
        const double hy = sqrt(d.r * d.r > dx * dx ? d.r * d.r - dx * dx : 0.0) + 1.0;
        const double hx = sqrt(d.r * d.r > dy * dy ? d.r * d.r - dy * dy : 0.0) + 1.0;
        if (d.cy - hy > box.y0) box.y0 = d.cy - hy;
        if (d.cy + hy < box.y1) box.y1 = d.cy + hy;
        if (d.cx - hx > box.x0) box.x0 = d.cx - hx;
        if (d.cx + hx < box.x1) box.x1 = d.cx + hx;
    }
    const double pu = g.u[p], pv = g.v[p], qu = g.u[q], qv = g.v[q];
    const double ex = qu - pu, ey = qv - pv;
    const double cs = ex * (d.cy - pv) - ey * (d.cx - pu);  // > 0: centre left of p -> q
    if ((side > 0) == (cs > 0)) return box;
    const double r0 = (d.r - 1.0) / (1.0 + 1e-9);  // disc_of's radius without its margin
    const double a = 0.25 * (ex * ex + ey * ey);   // (half chord)^2
    const double h = a / (r0 + sqrt(r0 * r0 > a ? r0 * r0 - a : 0.0)) + 2.0;
    const double x0 = (pu < qu ? pu : qu) - h, x1 = (pu > qu ? pu : qu) + h;
    const double y0 = (pv < qv ? pv : qv) - h, y1 = (pv > qv ? pv : qv) + h;
    if (x0 > box.x0) box.x0 = x0;
    if (x1 < box.x1) box.x1 = x1;
    if (y0 > box.y0) box.y0 = y0;
    if (y1 < box.y1) box.y1 = y1;
    return box;
}
// squared distance from (x, y) to the pixel box of cell (cx, cy)
PS_HD double cell_dist2(const Grid& g, int cx, int cy, double x, double y) {
    const double x0 = g.minx + double(cx) * g.gs, x1 = x0 + g.gs - 1;
    const double y0 = g.miny + double(cy) * g.gs, y1 = y0 + g.gs - 1;
    const double dx = x < x0 ? x0 - x : (x > x1 ? x - x1 : 0.0);
    const double dy = y < y0 ? y0 - y : (y > y1 ? y - y1 : 0.0);
    return dx * dx + dy * dy;
}

// The cells of row cy from x0 to x1 (inclusive) except the column ranges
// [e0a, e0b] and [e1a, e1b] (empty when a > b), as runs of consecutive cells:
// a run's points are consecutive in cell_items, so `f(i0, i1)` receives
// item ranges — an empty stretch of a row costs one lookup, not one per cell.
template <class F>
PS_HD void row_runs(const Grid& g, int cy, int x0, int x1, int e0a, int e0b, int e1a, int e1b, F&& f) {
    if (e0a > e0b || (e1a <= e1b && e1a < e0a)) {
        const int ta = e0a, tb = e0b;
        e0a = e1a;
        e0b = e1b;
        e1a = ta;
        e1b = tb;
    }
    const int rb = cy * g.gw;
    int cur = x0;
    auto emit = [&](int a, int b) {
        const int i0 = g.cell_start[rb + a], i1 = g.cell_start[rb + b + 1];
        if (i0 < i1) f(i0, i1);
    };
    if (e0a <= e0b && e0b >= cur && e0a <= x1) {
        if (e0a > cur) emit(cur, e0a - 1);
        cur = e0b + 1 > cur ? e0b + 1 : cur;
    }
    if (e1a <= e1b && e1b >= cur && e1a <= x1 && cur <= x1) {
        if (e1a > cur) emit(cur, e1a - 1);
        cur = e1b + 1 > cur ? e1b + 1 : cur;
    }
    if (cur <= x1) emit(cur, x1);
}

// Clips the cell range [x0, x1] of the pixel-row band [ya, yb] to the cells
// that can hold a point strictly on the search side of p -> q (left for
// side > 0); false when none can.
PS_HD bool clip_side(const Grid& g, int p, int q, int side, double ya, double yb, int& x0, int& x1) {
    // side * (qx * (y - pv) - qy * (x - pu)) > 0, linear in x and y
    const double sg = side > 0 ? 1.0 : -1.0, pu = g.u[p], pv = g.v[p];
    const double qx = double(g.u[q]) - pu, qy = double(g.v[q]) - pv;
    const double ax = -sg * qy;
    const double b0 = sg * qx * (ya - pv) - ax * pu, b1 = sg * qx * (yb - pv) - ax * pu;
    const double bm = b0 > b1 ? b0 : b1;
    if (ax > 0) {
        const int c = cell_x(g, -bm / ax - 1.0);
        x0 = c > x0 ? c : x0;
    } else if (ax < 0) {
        const int c = cell_x(g, -bm / ax + 1.0);
        x1 = c < x1 ? c : x1;
    } else if (bm <= 0) {
        return false;
    }
    return x0 <= x1;
}

// The pencil of circles through p and q: relative to p, the circle through
// p, q and s has its centre at q / 2 + t(s) * perp(q), perp(q) = (-qy, qx),
// with t(s) = num(s) / (2 den(s)), num = |s|^2 - q.s, den = cross(q, s) (> 0
// left of p -> q).  A point s on the search side lies inside the circle of
// the current winner b exactly when t(s) < t(b) (left) or t(s) > t(b)
// (right); compared as num(s) * den(b) vs num(b) * den(s) — both dens share
// the side's sign — which is exact in int64 for offsets below 2^14.  Equal
// products: cocircular (the exact rule of inside() decides).
struct Pencil {
    long long num, den;
};
PS_HD Pencil pencil(long long qx, long long qy, long long sx, long long sy) {
    return Pencil{sx * (sx - qx) + sy * (sy - qy), qx * sy - qy * sx};
}
// +1: s beats b (strictly inside b's circle), -1: b stays, 0: cocircular
PS_HD int pencil_cmp(const Pencil& s, const Pencil& b, int side) {
    const long long l = s.num * b.den, r = b.num * s.den;
    if (l == r) return 0;
    return (side > 0 ? l < r : l > r) ? 1 : -1;
}

// Next star neighbour of p after q: counter-clockwise (side > 0: r left of
// p -> q, triangle (p, q, r)) or clockwise (side < 0: r right of p -> q,
// triangle (p, r, q)).  -1 if no point lies on that side (a hull edge), -2 if
// the search found nothing (an inconsistency).
// First the rings of cells around p and q (a far point from the column
// extremes if they hold none), then the cell rows outward from p's row, each read only over the chord of the
// current winner's circumcircle: a better point lies inside that circle on
// the same side of p -> q, and that part of the circle only shrinks as the
// winner improves (circles through p and q form a pencil), so a row skipped
// or cut with the circle of its time holds no later winner either.
PS_HD int next_neighbour(const Grid& g, int p, int q, int side) {
    if (hull_edge(g, p, q, side)) return -1;
    int r = -1;
    Disc d{0.0, 0.0, 0.0};
    const long long qx = (long long)g.u[q] - g.u[p], qy = (long long)g.v[q] - g.v[p];
    Pencil rb{0, 0};
    auto consider = [&](int s) {
        if (s == p || s == q || g.dup[s]) return;
        const Pencil ps = pencil(qx, qy, (long long)g.u[s] - g.u[p], (long long)g.v[s] - g.v[p]);
        if (side > 0 ? ps.den <= 0 : ps.den >= 0) return;
        if (r >= 0) {
            const int c = pencil_cmp(ps, rb, side);
            if (c < 0 || (c == 0 && !(side > 0 ? inside(g, p, q, r, s) : inside(g, p, r, q, s)))) return;
        }
        r = s;
        rb = ps;
        d = side > 0 ? disc_of(g, p, q, r) : disc_of(g, p, r, q);
    };
    // rings around p and around q until a candidate appears: the next
    // neighbour is next to p, or — in a long thin hull triangle — next to q
    const int pcx = cell_x(g, g.u[p]), pcy = cell_y(g, g.v[p]);
    const int qcx = cell_x(g, g.u[q]), qcy = cell_y(g, g.v[q]);
    const int maxr = g.gw > g.gh ? g.gw : g.gh;
    auto ring = [&](int ox, int oy, int k) {
        for (int cy = oy - k; cy <= oy + k; ++cy) {
            if (cy < 0 || cy >= g.gh) continue;
            const bool edge_row = cy == oy - k || cy == oy + k;
            for (int cx = ox - k; cx <= ox + k; cx += (edge_row || k == 0) ? 1 : 2 * k) {
                if (cx < 0 || cx >= g.gw) continue;
                const int c = cy * g.gw + cx;
                for (int i = g.cell_start[c]; i < g.cell_start[c + 1]; ++i) consider(g.cell_items[i]);
            }
        }
    };
    int k = 0;
    for (; k <= 2 && k <= maxr && r < 0; ++k) {
        ring(pcx, pcy, k);
        ring(qcx, qcy, k);
    }
    if (r < 0) {
        // nothing nearby: a far point on that side (a long thin triangle
        // along the hull); any one starts the circle search, and one exists
        // among the column extremes (they include every hull vertex)
        // (columns outward from p's: a near one keeps the first circle small)
        const int cols = g.maxx - g.minx + 1, c0 = g.u[p] - g.minx;
        for (int k2 = 0; r < 0 && (c0 - k2 >= 0 || c0 + k2 < cols); ++k2)
            for (int e = 0; e < 4 && r < 0; ++e) {
                const int i = e < 2 ? c0 - k2 : c0 + k2;
                if (i < 0 || i >= cols || (k2 == 0 && e >= 2)) continue;
                const int w = (e & 1) == 0 ? g.col_lo[i] : g.col_hi[i];
                if (w >= 0) consider(w);
            }
        if (r < 0) return -2;
    }
    const int done = k - 1;  // rings 0..done around both cells are read
    const int py = pcy;
    for (int t = 0;; ++t) {
        const Region reg = search_region(g, p, q, side, d);
        for (int sgn = 0; sgn < 2; ++sgn) {
            if (t == 0 && sgn == 1) continue;
            const int cy = sgn == 0 ? py + t : py - t;
            if (cy < 0 || cy >= g.gh) continue;
            const double ya = g.miny + double(cy) * g.gs, yb = ya + g.gs - 1;
            if (yb < reg.y0 || ya > reg.y1) continue;
            const double dy = d.cy < ya ? ya - d.cy : (d.cy > yb ? d.cy - yb : 0.0);
            if (dy > d.r) continue;
            const double half = sqrt(d.r * d.r - dy * dy);
            int x0 = cell_x(g, d.cx - half > reg.x0 ? d.cx - half : reg.x0);
            int x1 = cell_x(g, d.cx + half < reg.x1 ? d.cx + half : reg.x1);
            if (!clip_side(g, p, q, side, ya, yb, x0, x1)) continue;
            const bool rp = cy >= pcy - done && cy <= pcy + done, rq = cy >= qcy - done && cy <= qcy + done;
            row_runs(g, cy, x0, x1, rp ? pcx - done : 1, rp ? pcx + done : 0, rq ? qcx - done : 1,
                     rq ? qcx + done : 0, [&](int i0, int i1) {
                         for (int i = i0; i < i1; ++i) consider(g.cell_items[i]);
                     });
        }
        // stop once the next rows both ways lie outside the region (it only
        // shrinks as the winner improves: circles through p, q form a pencil)
        const Region now = search_region(g, p, q, side, d);
        const bool up = py - t <= 0 || g.miny + double(py - t) * g.gs - 1 < now.y0;
        const bool dn = py + t >= g.gh - 1 || g.miny + double(py + t + 1) * g.gs > now.y1;
        if (up && dn) break;
    }
    return r;
}

PS_HD int nearest(const Grid& g, int p) {
    const int px = cell_x(g, g.u[p]), py = cell_y(g, g.v[p]);
    int best = -1;
    long long bd = 0;
    const int maxr = (g.gw > g.gh ? g.gw : g.gh);
    for (int k = 0; k <= maxr; ++k) {
        // cells at Chebyshev ring k
        for (int cy = py - k; cy <= py + k; ++cy) {
            if (cy < 0 || cy >= g.gh) continue;
            const bool edge_row = cy == py - k || cy == py + k;
            for (int cx = px - k; cx <= px + k; cx += (edge_row || k == 0) ? 1 : 2 * k) {
                if (cx < 0 || cx >= g.gw) continue;
                const int c = cy * g.gw + cx;
                for (int i = g.cell_start[c]; i < g.cell_start[c + 1]; ++i) {
                    const int s = g.cell_items[i];
                    if (s == p || g.dup[s]) continue;
                    const long long dx = g.u[s] - g.u[p], dy = g.v[s] - g.v[p];
                    const long long d2 = dx * dx + dy * dy;
                    if (d2 == 0) continue;  // coincident (a dup of p or p of it)
                    if (best < 0 || d2 < bd || (d2 == bd && s < best)) {
                        best = s;
                        bd = d2;
                    }
                }
            }
        }
        // every point beyond ring k is at least k * gs away (in one axis)
        if (best >= 0 && (long long)k * g.gs * k * g.gs >= bd) break;
    }
    return best;
}

// ---- the fast path: the points of the cells around p gathered once, in
// coordinates relative to p; a search uses them alone when its answer is
// certified inside the gathered box (else it falls back to the grid search).
constexpr int kLocalMax = 64;

// Candidate storage is strided so the device can interleave a block's
// threads in shared memory (element i of thread t at [i * stride + t]).
struct Local {
    int n = 0;
    bool complete = true;  // every point of `box` was gathered
    Box box{1, 1, 0, 0};
    int* idx = nullptr;    // point index
    int* dxy = nullptr;    // (dy << 16) | (dx & 0xffff), relative to p
    int stride = 1;
    int cap = kLocalMax;   // capacity of idx / dxy
    PS_HD int id(int i) const { return idx[i * stride]; }
    PS_HD int dx(int i) const { return int(short(dxy[i * stride] & 0xffff)); }
    PS_HD int dy(int i) const { return dxy[i * stride] >> 16; }
};

PS_HD void gather(const Grid& g, int p, int radius, Local& L) {
    L.n = 0;
    if (g.maxx - g.minx >= 4096 || g.maxy - g.miny >= 4096 || radius * g.gs >= 16000) {
        L.complete = false;  // next_local's int32 bound / 16-bit offsets
        return;
    }
    const int px = cell_x(g, g.u[p]), py = cell_y(g, g.v[p]);
    L.box = Box{px - radius < 0 ? 0 : px - radius, py - radius < 0 ? 0 : py - radius,
                px + radius >= g.gw ? g.gw - 1 : px + radius, py + radius >= g.gh ? g.gh - 1 : py + radius};
    L.complete = true;
    for (int cy = L.box.y0; cy <= L.box.y1; ++cy)
        for (int cx = L.box.x0; cx <= L.box.x1; ++cx) {
            const int c = cy * g.gw + cx;
            for (int i = g.cell_start[c]; i < g.cell_start[c + 1]; ++i) {
                const int s = g.cell_items[i];
                if (s == p || g.dup[s]) continue;
                if (L.n == L.cap) {
                    L.complete = false;
                    return;
                }
                L.idx[L.n * L.stride] = s;
                L.dxy[L.n * L.stride] = ((g.v[s] - g.v[p]) << 16) | ((g.u[s] - g.u[p]) & 0xffff);
                ++L.n;
            }
        }
}

// The cells whose points could lie within the circle through p, q, r
// (relative coordinates; r, q counter-clockwise after p for side > 0).
PS_HD Box circle_box_rel(const Grid& g, int p, double qx, double qy, double rx, double ry) {
    const double iD = 0.5 / (qx * ry - qy * rx);
    const double qq = qx * qx + qy * qy, rr = rx * rx + ry * ry;
    const double ux = (ry * qq - qy * rr) * iD, uy = (qx * rr - rx * qq) * iD;
    const double rad = sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0;
    const double cx = g.u[p] + ux, cy = g.v[p] + uy;
    return Box{cell_x(g, cx - rad), cell_y(g, cy - rad), cell_x(g, cx + rad), cell_y(g, cy + rad)};
}

// Local next neighbour: -1 hull edge, -3 not certified (use the grid search).
PS_HD int next_local(const Grid& g, const Local& L, int p, int q, int side) {
    if (hull_edge(g, p, q, side)) return -1;
    if (!L.complete) return -3;
    // relative offsets below 2^12 (gather): every product below fits int32
    const int qx = g.u[q] - g.u[p], qy = g.v[q] - g.v[p];
    int bi = -1;
    int bnum = 0, bden = 0;
    for (int i = 0; i < L.n; ++i) {
        const int w = L.dxy[i * L.stride];
        const int sx = int(short(w & 0xffff)), sy = w >> 16;
        const int den = qx * sy - qy * sx;  // orient(p, q, s); q itself gives 0
        if (side > 0 ? den <= 0 : den >= 0) continue;
        const int num = sx * (sx - qx) + sy * (sy - qy);
        if (bi >= 0) {
            const long long l = (long long)num * bden, r = (long long)bnum * den;
            if (l == r) {  // cocircular: the exact perturbed rule
                const int s = L.id(i), b = L.id(bi);
                if (!(side > 0 ? inside(g, p, q, b, s) : inside(g, p, b, q, s))) continue;
            } else if (side > 0 ? l > r : l < r) {
                continue;
            }
        }
        bi = i;
        bnum = num;
        bden = den;
    }
    if (bi >= 0) {
        const double bx = L.dx(bi), by = L.dy(bi);
        const Box need = side > 0 ? circle_box_rel(g, p, double(qx), double(qy), bx, by)
                                  : circle_box_rel(g, p, bx, by, double(qx), double(qy));
        return covers(L.box, need) ? L.id(bi) : -3;
    }
    return -3;  // not a hull edge: the neighbour lies beyond the gathered cells
}

// Local nearest neighbour, certified when every point outside the gathered
// box is strictly farther; -3 otherwise.
PS_HD int nearest_local(const Grid& g, const Local& L, int p) {
    if (!L.complete) return -3;
    int best = -1;
    long long bd = 0;
    for (int i = 0; i < L.n; ++i) {
        const long long d2 = (long long)L.dx(i) * L.dx(i) + (long long)L.dy(i) * L.dy(i);
        if (d2 == 0) continue;
        const int s = L.id(i);
        if (best < 0 || d2 < bd || (d2 == bd && s < best)) {
            best = s;
            bd = d2;
        }
    }
    // distance from p to the outside of the box (sides on the grid edge have no outside)
    const long long px = g.u[p] - g.minx, py = g.v[p] - g.miny;  // grid-relative
    long long m = 1ll << 40;
    auto lower = [&](long long x) { m = x < m ? x : m; };
    if (L.box.x0 > 0) lower(px - (long long)L.box.x0 * g.gs + 1);
    if (L.box.y0 > 0) lower(py - (long long)L.box.y0 * g.gs + 1);
    if (L.box.x1 < g.gw - 1) lower((long long)(L.box.x1 + 1) * g.gs - px);
    if (L.box.y1 < g.gh - 1) lower((long long)(L.box.y1 + 1) * g.gs - py);
    if (best < 0) return m >= (1ll << 40) ? -1 : -3;
    return bd < m * m ? best : -3;
}

// inside() for a cocircular quadruple given by offsets from p: triangle
// (p, a, b) counter-clockwise, d the fourth point (all distinct); the same
// lifting of the lexicographically largest point.
PS_HD bool inside_tie_rel(int ax, int ay, int bx, int by, int dx, int dy) {
    // lexicographic maximum of p = (0, 0), a, b, d
    int mx = 0, my = 0, m = 0;
    auto take = [&](int x, int y, int k) {
        if (x > mx || (x == mx && y > my)) {
            mx = x;
            my = y;
            m = k;
        }
    };
    take(ax, ay, 1);
    take(bx, by, 2);
    take(dx, dy, 3);
    auto orient_rel = [](long long x0, long long y0, long long x1, long long y1, long long x2, long long y2) {
        return (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
    };
    if (m == 3) return false;
    if (m == 0) return orient_rel(ax, ay, bx, by, dx, dy) > 0;
    if (m == 1) return orient_rel(bx, by, 0, 0, dx, dy) > 0;
    return orient_rel(0, 0, ax, ay, dx, dy) > 0;
}

// ---- the tiled fast path (star.cu k_star): a block holds the points of a
// tile of cells plus a halo of kTileHalo cells in shared memory, compacted
// per cell (duplicates dropped) with coordinates relative to the region's
// pixel origin; a point's searches read the rows of its (2R+1)^2-cell box
// there as runs of consecutive entries.  Same certificates as Local.
constexpr int kTileCells = 8;  // tile width in cells
constexpr int kTileHalo = 4;   // halo (the largest search radius)
constexpr int kTileRegion = kTileCells + 2 * kTileHalo;

struct Tile {
    const int* start;  // kTileRegion^2 + 1 offsets into xy / id, region cells row-major
    const int* xy;     // (y << 16) | x relative to the region's pixel origin
    const int* id;     // point index
    int cx0, cy0;      // grid cell of region cell (0, 0) (may lie outside the grid)
};

// The point of p's walk state: its grid cell, region-relative pixel, absolute pixel.
struct TilePoint {
    int p, pcx, pcy, pxr, pyr, pu, pv;
    int hprev, hnext;  // hull neighbours (-1 off the hull)
};

// Rows of p's box of radius R (grid cells, clipped to the grid) in region
// coordinates: calls f(i0, i1) per row.
template <class F>
PS_HD void tile_box(const Grid& g, const Tile& T, const TilePoint& P, int R, Box& box, F&& f) {
    box = Box{P.pcx - R < 0 ? 0 : P.pcx - R, P.pcy - R < 0 ? 0 : P.pcy - R,
              P.pcx + R >= g.gw ? g.gw - 1 : P.pcx + R, P.pcy + R >= g.gh ? g.gh - 1 : P.pcy + R};
    const int x0 = box.x0 - T.cx0, x1 = box.x1 - T.cx0;
    for (int y = box.y0 - T.cy0; y <= box.y1 - T.cy0; ++y) {
        const int i0 = T.start[y * kTileRegion + x0], i1 = T.start[y * kTileRegion + x1 + 1];
        if (i0 < i1) f(i0, i1);
    }
}

// Nearest other point within the box, certified when every point outside
// is strictly farther; -1 no other point in the set, -3 not certified.
// (bx, by): its offset from p.
PS_HD int tile_nearest(const Grid& g, const Tile& T, const TilePoint& P, int R, int& bx, int& by) {
    int best = -1;
    int bd = 0;
    Box box;
    tile_box(g, T, P, R, box, [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            const int w = T.xy[i];
            const int sx = (w & 0xffff) - P.pxr, sy = (w >> 16) - P.pyr;
            const int d2 = sx * sx + sy * sy;
            if (d2 == 0) continue;  // p itself (duplicates are not in the region)
            if (best >= 0 && (d2 > bd || (d2 == bd && T.id[i] > best))) continue;
            best = T.id[i];
            bd = d2;
            bx = sx;
            by = sy;
        }
    });
    const long long px = P.pu - g.minx, py = P.pv - g.miny;
    long long m = 1ll << 40;
    auto lower = [&](long long x) { m = x < m ? x : m; };
    if (box.x0 > 0) lower(px - (long long)box.x0 * g.gs + 1);
    if (box.y0 > 0) lower(py - (long long)box.y0 * g.gs + 1);
    if (box.x1 < g.gw - 1) lower((long long)(box.x1 + 1) * g.gs - px);
    if (box.y1 < g.gh - 1) lower((long long)(box.y1 + 1) * g.gs - py);
    if (best < 0) return m >= (1ll << 40) ? -1 : -3;
    return (long long)bd < m * m ? best : -3;
}

// Next neighbour of p after q (offset (qx, qy)) within the box: -1 hull
// edge, -3 not certified; (bx, by): the winner's offset.
PS_HD int tile_next(const Grid& g, const Tile& T, const TilePoint& P, int R, int q, int qx, int qy, int side,
                    int& bx, int& by) {
    if (g.flat || (side > 0 ? P.hprev == q : P.hnext == q)) return -1;
    int bi = -1, bnum = 0, bden = 0;
    Box box;
    tile_box(g, T, P, R, box, [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            const int w = T.xy[i];
            const int sx = (w & 0xffff) - P.pxr, sy = (w >> 16) - P.pyr;
            const int den = qx * sy - qy * sx;  // orient(p, q, s); p and q give 0
            if (side > 0 ? den <= 0 : den >= 0) continue;
            const int num = sx * (sx - qx) + sy * (sy - qy);
            if (bi >= 0) {
                const long long l = (long long)num * bden, r = (long long)bnum * den;
                if (l == r) {  // cocircular
                    if (!(side > 0 ? inside_tie_rel(qx, qy, bx, by, sx, sy) : inside_tie_rel(bx, by, qx, qy, sx, sy)))
                        continue;
                } else if (side > 0 ? l > r : l < r) {
                    continue;
                }
            }
            bi = i;
            bnum = num;
            bden = den;
            bx = sx;
            by = sy;
        }
    });
    if (bi < 0) return -3;
    // the winner's circle must lie within the box
    const double qxd = qx, qyd = qy, rx = side > 0 ? bx : qx, ry = side > 0 ? by : qy;
    const double ax = side > 0 ? qxd : bx, ay = side > 0 ? qyd : by;
    const double iD = 0.5 / (ax * ry - ay * rx);
    const double aa = ax * ax + ay * ay, rr = rx * rx + ry * ry;
    const double ux = (ry * aa - ay * rr) * iD, uy = (ax * rr - rx * aa) * iD;
    const double rad = sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0;
    const double cx = P.pu + ux, cy = P.pv + uy;
    const Box need{cell_x(g, cx - rad), cell_y(g, cy - rad), cell_x(g, cx + rad), cell_y(g, cy + rad)};
    return covers(box, need) ? T.id[bi] : -3;
}

// p's star from the region with search radius R, into tb ((b, c) per
// triangle (p, b, c), counter-clockwise from the nearest neighbour, then
// clockwise for a hull vertex).  Returns the triangle count, -4 when a
// search is not certified within the box, -5 for more than `cap` triangles.
PS_HD int tile_walk(const Grid& g, const Tile& T, const TilePoint& P, int R, bool& closed, int* tb, int cap) {
    closed = false;
    int qx = 0, qy = 0;
    const int q0 = tile_nearest(g, T, P, R, qx, qy);
    if (q0 == -3) return -4;
    if (q0 < 0) return 0;
    const int q0x = qx, q0y = qy;
    int count = 0;
    for (int dir = 0; dir < 2; ++dir) {
        const int side = dir == 0 ? 1 : -1;
        int cur = q0, cx = q0x, cy = q0y;
        for (int guard = 0; guard <= g.n; ++guard) {
            int rx = 0, ry = 0;
            const int r = tile_next(g, T, P, R, cur, cx, cy, side, rx, ry);
            if (r == -3) return -4;
            if (r < 0) break;
            if (count == cap) return -5;
            tb[2 * count] = side > 0 ? cur : r;
            tb[2 * count + 1] = side > 0 ? r : cur;
            ++count;
            if (side > 0 && r == q0) {
                closed = true;
                return count;
            }
            cur = r;
            cx = rx;
            cy = ry;
        }
    }
    return count;
}

// ---- pass 1's common case: the near set.  The points of p's radius-2 box
// at squared distance below t2 <= (2 gs)^2 from p -- all of the set's points
// that close lie in that box -- are listed once per point (at most
// kNearCap, packed (x + 128) | (y + 128) << 8 | region index << 16, at
// list[j * stride]); each step then scans that short list instead of the box
// rows.  A winner over the list is the winner over the set when the circle
// through p, q and it has squared diameter below t2: a point beating it lies
// in (or on) that circle, so within the diameter of p, so in the list.  The
// certificate is exact integer arithmetic; a step it does not certify falls
// back to tile_next over the box.
constexpr int kNearCap = 32;

struct Near {
    int* list;
    int stride, n, t2;
};

// Builds p's near set: t2 the largest of 4, 3, 2, 1 gs^2 whose set fits
// kNearCap.  False (use the box) when none fits or the offsets would not
// pack (gs > 60).
PS_HD bool near_build(const Grid& g, const Tile& T, const TilePoint& P, Near& N) {
    if (g.gs > 60) return false;
    const int s2 = g.gs * g.gs;
    int c1 = 0, c2 = 0, c3 = 0, n = 0;
    Box box;
    tile_box(g, T, P, 2, box, [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            const int w = T.xy[i];
            const int sx = (w & 0xffff) - P.pxr, sy = (w >> 16) - P.pyr;
            const int d2 = sx * sx + sy * sy;
            if (d2 == 0 || d2 >= 4 * s2) continue;  // p itself (duplicates are not in the region)
            c1 += d2 < s2;
            c2 += d2 < 2 * s2;
            c3 += d2 < 3 * s2;
            if (n < kNearCap) N.list[n * N.stride] = (sx + 128) | ((sy + 128) << 8) | (i << 16);
            ++n;
        }
    });
    if (n <= kNearCap) {
        N.n = n;
        N.t2 = 4 * s2;
        return true;
    }
    const int t2 = c3 <= kNearCap ? 3 * s2 : c2 <= kNearCap ? 2 * s2 : c1 <= kNearCap ? s2 : 0;
    if (t2 == 0) return false;
    n = 0;
    tile_box(g, T, P, 2, box, [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i) {
            const int w = T.xy[i];
            const int sx = (w & 0xffff) - P.pxr, sy = (w >> 16) - P.pyr;
            const int d2 = sx * sx + sy * sy;
            if (d2 == 0 || d2 >= t2) continue;
            N.list[n * N.stride] = (sx + 128) | ((sy + 128) << 8) | (i << 16);
            ++n;
        }
    });
    N.n = n;
    N.t2 = t2;
    return true;
}

// Nearest other point from the near set, certified when closer than sqrt(t2).
PS_HD int near_nearest(const Tile& T, const Near& N, int& bx, int& by) {
    int best = -1, bd = 0;
    for (int j = 0; j < N.n; ++j) {
        const int w = N.list[j * N.stride];
        const int sx = (w & 0xff) - 128, sy = ((w >> 8) & 0xff) - 128;
        const int d2 = sx * sx + sy * sy;
        if (best >= 0 && d2 > bd) continue;
        const int id = T.id[w >> 16];
        if (best >= 0 && d2 == bd && id > best) continue;
        best = id;
        bd = d2;
        bx = sx;
        by = sy;
    }
    return best >= 0 && bd < N.t2 ? best : -3;
}

// tile_next over the near set: the winner's id, or -1 hull edge, -3 not
// certified (the caller then searches the box).
PS_HD int near_next(const Grid& g, const Tile& T, const TilePoint& P, const Near& N, int q, int qx, int qy, int side,
                    int& bx, int& by) {
    if (g.flat || (side > 0 ? P.hprev == q : P.hnext == q)) return -1;
    int bw = -1, bnum = 0, bden = 0;
    for (int j = 0; j < N.n; ++j) {
        const int w = N.list[j * N.stride];
        const int sx = (w & 0xff) - 128, sy = ((w >> 8) & 0xff) - 128;
        const int den = qx * sy - qy * sx;
        if (side > 0 ? den <= 0 : den >= 0) continue;
        const int num = sx * (sx - qx) + sy * (sy - qy);
        if (bw >= 0) {
            const long long l = (long long)num * bden, r = (long long)bnum * den;
            if (l == r) {
                if (!(side > 0 ? inside_tie_rel(qx, qy, bx, by, sx, sy) : inside_tie_rel(bx, by, qx, qy, sx, sy)))
                    continue;
            } else if (side > 0 ? l > r : l < r) {
                continue;
            }
        }
        bw = w;
        bnum = num;
        bden = den;
        bx = sx;
        by = sy;
    }
    if (bw < 0) return -3;
    // circle through p (the origin), a and b (counter-clockwise): centre
    // (nx, ny) / (2 cr), squared diameter (nx^2 + ny^2) / cr^2
    const long long ax = side > 0 ? qx : bx, ay = side > 0 ? qy : by;
    const long long cx = side > 0 ? bx : qx, cy = side > 0 ? by : qy;
    const long long aa = ax * ax + ay * ay, cc = cx * cx + cy * cy, cr = ax * cy - ay * cx;
    const long long nx = cy * aa - ay * cc, ny = ax * cc - cx * aa;
    return nx * nx + ny * ny < (long long)N.t2 * cr * cr ? T.id[bw >> 16] : -3;
}

// tile_walk at radius 2 through the near set (N.n < 0: no near set).
PS_HD int tile_walk_near(const Grid& g, const Tile& T, const TilePoint& P, const Near& N, bool& closed, int* tb,
                         int cap) {
    if (N.n < 0) return tile_walk(g, T, P, 2, closed, tb, cap);
    closed = false;
    int qx = 0, qy = 0;
    int q0 = near_nearest(T, N, qx, qy);
    if (q0 == -3) q0 = tile_nearest(g, T, P, 2, qx, qy);
    if (q0 == -3) return -4;
    if (q0 < 0) return 0;
    const int q0x = qx, q0y = qy;
    int count = 0;
    for (int dir = 0; dir < 2; ++dir) {
        const int side = dir == 0 ? 1 : -1;
        int cur = q0, cx = q0x, cy = q0y;
        for (int guard = 0; guard <= g.n; ++guard) {
            int rx = 0, ry = 0;
            int r = near_next(g, T, P, N, cur, cx, cy, side, rx, ry);
#ifdef PS_NEAR_STATS
            PS_NEAR_STATS(r == -3);
#endif
            if (r == -3) r = tile_next(g, T, P, 2, cur, cx, cy, side, rx, ry);
            if (r == -3) return -4;
            if (r < 0) break;
            if (count == cap) return -5;
            tb[2 * count] = side > 0 ? cur : r;
            tb[2 * count + 1] = side > 0 ? r : cur;
            ++count;
            if (side > 0 && r == q0) {
                closed = true;
                return count;
            }
            cur = r;
            cx = rx;
            cy = ry;
        }
    }
    return count;
}

// Walks the star of p and calls on_tri(a, b, c) for each incident triangle,
// counter-clockwise (a = p).  Returns the triangle count (0: p is not a
// vertex or the set is collinear around it), -2 if a search failed, or -4
// when more than `budget` steps needed the grid search (budget < 0: no
// limit; the device then hands p to a warp, star.cu).  `closed` tells
// whether the star is a full cycle; otherwise p is a hull vertex.
template <class F>
PS_HD int walk_star(const Grid& g, const Local& L, int p, bool& closed, F&& on_tri, int budget = -1) {
    closed = false;
    if (g.dup[p]) return 0;
    int q0 = nearest_local(g, L, p);
    if (q0 == -3) {
        if (budget == 0) return -4;
        if (budget > 0) --budget;
        q0 = nearest(g, p);
    }
    if (q0 < 0) return 0;
    bool over = false;
    auto step = [&](int q, int side) {
        const int r = next_local(g, L, p, q, side);
        if (r != -3) return r;
        if (budget == 0) {
            over = true;
            return -4;
        }
        if (budget > 0) --budget;
        return next_neighbour(g, p, q, side);
    };
    int count = 0;
    int cur = q0;
    for (int guard = 0; guard <= g.n; ++guard) {  // counter-clockwise from q0
        const int r = step(cur, +1);
        if (over) return -4;
        if (r == -2) return -2;
        if (r < 0) break;
        on_tri(p, cur, r);
        ++count;
        if (r == q0) {
            closed = true;
            return count;
        }
        cur = r;
    }
    cur = q0;
    for (int guard = 0; guard <= g.n; ++guard) {  // a hull vertex: clockwise from q0
        const int r = step(cur, -1);
        if (over) return -4;
        if (r == -2) return -2;
        if (r < 0) break;
        on_tri(p, r, cur);
        ++count;
        cur = r;
    }
    return count;
}

}  // namespace star
}  // namespace ps
