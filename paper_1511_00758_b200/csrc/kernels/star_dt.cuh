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
    int flat;  // every point on one line: no triangle at all
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

PS_HD int cell_x(const Grid& g, double x) {
    int c = int(floor((x - g.minx) / g.gs));
    return c < 0 ? 0 : (c >= g.gw ? g.gw - 1 : c);
}
PS_HD int cell_y(const Grid& g, double y) {
    int c = int(floor((y - g.miny) / g.gs));
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
    const double D = 2.0 * (bx * cy - by * cx);
    const double bq = bx * bx + by * by, cq = cx * cx + cy * cy;
    const double ux = (cy * bq - by * cq) / D, uy = (bx * cq - cx * bq) / D;
    return Disc{ax + ux, ay + uy, sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0};
}
// squared distance from (x, y) to the pixel box of cell (cx, cy)
PS_HD double cell_dist2(const Grid& g, int cx, int cy, double x, double y) {
    const double x0 = g.minx + double(cx) * g.gs, x1 = x0 + g.gs - 1;
    const double y0 = g.miny + double(cy) * g.gs, y1 = y0 + g.gs - 1;
    const double dx = x < x0 ? x0 - x : (x > x1 ? x - x1 : 0.0);
    const double dy = y < y0 ? y0 - y : (y > y1 ? y - y1 : 0.0);
    return dx * dx + dy * dy;
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
    auto consider = [&](int s) {
        if (s == p || s == q || g.dup[s]) return;
        const long long o = orient(g, p, q, s);
        if (side > 0 ? o <= 0 : o >= 0) return;
        if (r < 0 || (side > 0 ? inside(g, p, q, r, s) : inside(g, p, r, q, s))) {
            r = s;
            d = side > 0 ? disc_of(g, p, q, r) : disc_of(g, p, r, q);
        }
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
        const int cols = g.maxx - g.minx + 1;
        for (int i = 0; i < cols && r < 0; ++i)
            for (int e = 0; e < 2 && r < 0; ++e) {
                const int w = e == 0 ? g.col_lo[i] : g.col_hi[i];
                if (w >= 0) consider(w);
            }
        if (r < 0) return -2;
    }
    const int done = k - 1;  // rings 0..done around both cells are read
    auto read = [&](int cx, int cy) {
        return (cx >= pcx - done && cx <= pcx + done && cy >= pcy - done && cy <= pcy + done) ||
               (cx >= qcx - done && cx <= qcx + done && cy >= qcy - done && cy <= qcy + done);
    };
    const int py = pcy;
    for (int t = 0;; ++t) {
        bool any = false;
        for (int sgn = 0; sgn < 2; ++sgn) {
            if (t == 0 && sgn == 1) continue;
            const int cy = sgn == 0 ? py + t : py - t;
            if (cy < 0 || cy >= g.gh) continue;
            const double ya = g.miny + double(cy) * g.gs, yb = ya + g.gs - 1;
            const double dy = d.cy < ya ? ya - d.cy : (d.cy > yb ? d.cy - yb : 0.0);
            if (dy > d.r) continue;
            any = true;
            const double half = sqrt(d.r * d.r - dy * dy);
            const int x0 = cell_x(g, d.cx - half), x1 = cell_x(g, d.cx + half);
            for (int cx = x0; cx <= x1; ++cx) {
                if (read(cx, cy)) continue;
                const int c = cy * g.gw + cx;
                for (int i = g.cell_start[c]; i < g.cell_start[c + 1]; ++i) consider(g.cell_items[i]);
            }
        }
    // stop once both rows lie beyond the circle's vertical extent
        const double up = g.miny + double(py - t) * g.gs, dn = g.miny + double(py + t + 1) * g.gs - 1;
        if (!any && (py - t < 0 || up - 1 < d.cy - d.r) && (py + t >= g.gh || dn + 1 > d.cy + d.r)) break;
        if (py - t < 0 && py + t >= g.gh) break;
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
        L.complete = false;  // incircle_rel's exactness bound / 16-bit offsets
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

// s inside the circle through p (origin) and the counter-clockwise a, b:
// the lifted 3x3 determinant relative to p, exact in binary64 while the
// coordinates differ by < 2^12 (|det| < 2^52); 0 = cocircular -> exact rule.
PS_HD double incircle_rel(double ax, double ay, double bx, double by, double sx, double sy) {
    const double aq = ax * ax + ay * ay, bq = bx * bx + by * by, sq = sx * sx + sy * sy;
    return ax * (by * sq - sy * bq) - ay * (bx * sq - sx * bq) + aq * (bx * sy - sx * by);
}

// The cells whose points could lie within the circle through p, q, r
// (relative coordinates; r, q counter-clockwise after p for side > 0).
PS_HD Box circle_box_rel(const Grid& g, int p, double qx, double qy, double rx, double ry) {
    const double D = 2.0 * (qx * ry - qy * rx);
    const double qq = qx * qx + qy * qy, rr = rx * rx + ry * ry;
    const double ux = (ry * qq - qy * rr) / D, uy = (qx * rr - rx * qq) / D;
    const double rad = sqrt(ux * ux + uy * uy) * (1.0 + 1e-9) + 1.0;
    const double cx = g.u[p] + ux, cy = g.v[p] + uy;
    return Box{cell_x(g, cx - rad), cell_y(g, cy - rad), cell_x(g, cx + rad), cell_y(g, cy + rad)};
}

// Local next neighbour: -1 hull edge, -3 not certified (use the grid search).
PS_HD int next_local(const Grid& g, const Local& L, int p, int q, int side) {
    const long long qx = g.u[q] - g.u[p], qy = g.v[q] - g.v[p];
    int best = -1;
    if (hull_edge(g, p, q, side)) return -1;
    if (!L.complete) return -3;
    int bx = 0, by = 0;
    for (int i = 0; i < L.n; ++i) {
        const int s = L.id(i);
        if (s == q) continue;
        const int sx = L.dx(i), sy = L.dy(i);
        const long long o = qx * sy - qy * sx;  // orient(p, q, s)
        if (side > 0 ? o <= 0 : o >= 0) continue;
        if (best < 0) {
            best = s;
            bx = sx;
            by = sy;
            continue;
        }
        const double det = side > 0 ? incircle_rel(double(qx), double(qy), double(bx), double(by), double(sx), double(sy))
                                    : incircle_rel(double(bx), double(by), double(qx), double(qy), double(sx), double(sy));
        const bool in = det != 0.0 ? det < 0.0 : (side > 0 ? inside(g, p, q, best, s) : inside(g, p, best, q, s));
        if (in) {
            best = s;
            bx = sx;
            by = sy;
        }
    }
    if (best >= 0) {
        const Box need = side > 0 ? circle_box_rel(g, p, double(qx), double(qy), double(bx), double(by))
                                  : circle_box_rel(g, p, double(bx), double(by), double(qx), double(qy));
        return covers(L.box, need) ? best : -3;
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
