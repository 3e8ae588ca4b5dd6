/*
 * ps_oracle.c — TEST INFRASTRUCTURE ONLY (see ps_oracle.h).
 *
 * A plain-C restatement of the reference CPU path, one function per
 * reference function, each citing the reference file:line it restates
 * (paths relative to /root/reference/proj).  Compiled with
 * -O2 -ffp-contract=off and no -march so binary32/binary64 arithmetic is
 * evaluated exactly as the reference's default build evaluates it
 * (no FMA contraction in plane fitting/evaluation).
 */
#define _GNU_SOURCE
#include "ps_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define CENSUS_R 2   /* CensusField::kRadius, census.hpp:19 */
#define CENSUS_BITS 24
#define MASK_MARGIN 2 /* GradientMask::kMargin, image.hpp:50 */

static float census_cost(uint32_t a, uint32_t b) {
    /* census.hpp:45-47: float(popcount(a^b)) / 24.0f */
    return (float)__builtin_popcount(a ^ b) / (float)CENSUS_BITS;
}

/* ---------------------------------------------------------------- image.cpp:43-60 */
int orc_gradient_mask(const uint8_t* img, int w, int h, int threshold, uint8_t* member) {
    int count = 0;
    memset(member, 0, (size_t)w * h);
    for (int v = MASK_MARGIN; v < h - MASK_MARGIN; ++v) {
        const uint8_t* up = img + (size_t)(v - 1) * w;
        const uint8_t* mid = img + (size_t)v * w;
        const uint8_t* dn = img + (size_t)(v + 1) * w;
        for (int u = MASK_MARGIN; u < w - MASK_MARGIN; ++u) {
            int g = abs((int)mid[u + 1] - (int)mid[u - 1]) + abs((int)dn[u] - (int)up[u]);
            if (g >= threshold) {
                member[(size_t)v * w + u] = 1;
                ++count;
            }
        }
    }
    return count;
}

/* ---------------------------------------------------------------- census.cpp:10-41 */
void orc_census(const uint8_t* img, int w, int h, uint32_t* out) {
    memset(out, 0, sizeof(uint32_t) * (size_t)w * h);
    for (int v = CENSUS_R; v < h - CENSUS_R; ++v) {
        for (int u = CENSUS_R; u < w - CENSUS_R; ++u) {
            const uint8_t c = img[(size_t)v * w + u];
            uint32_t desc = 0;
            int bit = 0;
            for (int dv = -CENSUS_R; dv <= CENSUS_R; ++dv) {
                for (int du = -CENSUS_R; du <= CENSUS_R; ++du) {
                    if (dv == 0 && du == 0) continue;
                    desc |= (uint32_t)(img[(size_t)(v + dv) * w + (u + du)] < c) << bit;
                    ++bit;
                }
            }
            out[(size_t)v * w + u] = desc;
        }
    }
}

/* ---------------------------------------------------------------- sparse.cpp:12-146 */
/* Bresenham circle of radius 3, clockwise from 12 o'clock (sparse.cpp:12-15). */
static const int k_ring[16][2] = {{0, -3}, {1, -3}, {2, -2},  {3, -1},  {3, 0},  {3, 1},
                                  {2, 2},  {1, 3},  {0, 3},   {-1, 3},  {-2, 2}, {-3, 1},
                                  {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3}};

static int ring_has_arc(unsigned m16) {
    /* sparse.cpp:22-36: contiguous run >= 9 on the 16-ring */
    unsigned ring = m16 | (m16 << 16);
    int run = 0;
    for (int i = 0; i < 32; ++i) {
        if (ring & (1u << i)) {
            if (++run >= 9) return 1;
        } else {
            run = 0;
        }
    }
    return 0;
}

typedef struct {
    int u, v;
    float score;
    int bin;
} corner_t;

/* byScoreThenRowMajor, sparse.cpp:130-134 */
static int cmp_corner(const void* pa, const void* pb) {
    const corner_t* a = (const corner_t*)pa;
    const corner_t* b = (const corner_t*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    if (a->v != b->v) return a->v < b->v ? -1 : 1;
    if (a->u != b->u) return a->u < b->u ? -1 : 1;
    return 0;
}
static int cmp_corner_binned(const void* pa, const void* pb) {
    const corner_t* a = (const corner_t*)pa;
    const corner_t* b = (const corner_t*)pb;
    if (a->bin != b->bin) return a->bin < b->bin ? -1 : 1;
    return cmp_corner(pa, pb);
}

int orc_detect_candidates(const uint8_t* img, int w, int h, const ps_config* cfg, int* ou, int* ov,
                          float* oscore, int cap) {
    const int t = cfg->corner_threshold;
    size_t n = 0, capn = 1024;
    corner_t* all = (corner_t*)malloc(capn * sizeof(corner_t));
    for (int v = 3; v < h - 3; ++v) {
        for (int u = 3; u < w - 3; ++u) {
            const int c = img[(size_t)v * w + u];
            const int hi = c + t, lo = c - t;
            int nb = 0, nd = 0; /* compass pre-test, sparse.cpp:98-109 */
            for (int k = 0; k < 16; k += 4) {
                int p = img[(size_t)(v + k_ring[k][1]) * w + (u + k_ring[k][0])];
                nb += p > hi;
                nd += p < lo;
            }
            if (nb < 2 && nd < 2) continue;
            unsigned bright = 0, dark = 0;
            int score = 0;
            for (int k = 0; k < 16; ++k) {
                int p = img[(size_t)(v + k_ring[k][1]) * w + (u + k_ring[k][0])];
                bright |= (unsigned)(p > hi) << k;
                dark |= (unsigned)(p < lo) << k;
                int e = abs(p - c) - t;
                score += e > 0 ? e : 0;
            }
            if (!ring_has_arc(bright) && !ring_has_arc(dark)) continue;
            int bu = u * 12 / w; /* sparse.cpp:124-125 */
            if (bu > 11) bu = 11;
            int bv = v * 10 / h;
            if (bv > 9) bv = 9;
            if (n == capn) {
                capn *= 2;
                all = (corner_t*)realloc(all, capn * sizeof(corner_t));
            }
            all[n].u = u;
            all[n].v = v;
            all[n].score = (float)score;
            all[n].bin = bv * 12 + bu;
            ++n;
        }
    }
    /* per-bin sort + cap (sparse.cpp:137-143), then the global sort (:144) */
    qsort(all, n, sizeof(corner_t), cmp_corner_binned);
    size_t kept = 0;
    for (size_t i = 0; i < n;) {
        size_t j = i;
        while (j < n && all[j].bin == all[i].bin) ++j;
        size_t take = j - i;
        if ((long long)take > cfg->per_bin_cap) take = (size_t)cfg->per_bin_cap;
        for (size_t k = 0; k < take; ++k) all[kept++] = all[i + k];
        i = j;
    }
    qsort(all, kept, sizeof(corner_t), cmp_corner);
    int out = 0;
    for (size_t i = 0; i < kept && out < cap; ++i, ++out) {
        ou[out] = all[i].u;
        ov[out] = all[i].v;
        if (oscore) oscore[out] = all[i].score;
    }
    free(all);
    return out;
}

/* searchLeftToRight, sparse.cpp:44-64 */
static void search_l2r(const uint32_t* cl, const uint32_t* cr, int w, int u, int v, int dmax,
                       int* best_d, float* best_c, float* second_c) {
    const uint32_t ref = cl[(size_t)v * w + u];
    const uint32_t* row = cr + (size_t)v * w;
    int bd = -1;
    float bc = 2.0f, sc = 2.0f;
    for (int d = 0; d <= dmax; ++d) {
        float c = census_cost(ref, row[u - d]);
        if (c < bc) {
            bc = c;
            bd = d;
        }
    }
    for (int d = 0; d <= dmax; ++d) {
        if (abs(d - bd) <= 1) continue;
        float c = census_cost(ref, row[u - d]);
        if (c < sc) sc = c;
    }
    *best_d = bd;
    *best_c = bc;
    *second_c = sc;
}

/* searchRightToLeft, sparse.cpp:66-80 */
static int search_r2l(const uint32_t* cl, const uint32_t* cr, int w, int ur, int v, int dmax) {
    const uint32_t ref = cr[(size_t)v * w + ur];
    const uint32_t* row = cl + (size_t)v * w;
    int bd = 0;
    float bc = 2.0f;
    for (int d = 0; d <= dmax; ++d) {
        float c = census_cost(ref, row[ur + d]);
        if (c < bc) {
            bc = c;
            bd = d;
        }
    }
    return bd;
}

/* matchEpipolar, sparse.cpp:148-195 */
int orc_match_epipolar(const uint32_t* cl, const uint32_t* cr, int w, int h, const int* cu,
                       const int* cv, int n, const ps_config* cfg, int* su, int* sv, double* sd) {
    int* slot = (int*)malloc(sizeof(int) * (size_t)w * h); /* byPixel map */
    float* acc_cost = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (size_t i = 0; i < (size_t)w * h; ++i) slot[i] = -1;
    int count = 0;
    for (int i = 0; i < n; ++i) {
        const int u = cu[i], v = cv[i];
        if (!(u >= CENSUS_R && u < w - CENSUS_R && v >= CENSUS_R && v < h - CENSUS_R)) continue;
        int dmax = cfg->max_disparity - 1;
        if (u - CENSUS_R < dmax) dmax = u - CENSUS_R;
        if (dmax < 0) continue;
        int bd;
        float bc, sc;
        search_l2r(cl, cr, w, u, v, dmax, &bd, &bc, &sc);
        if (bd < 0 || bc > cfg->sparse_accept_cost) continue;
        if (sc <= 1.0f && bc > cfg->uniqueness_ratio * sc) continue;
        const int ur = u - bd;
        int back = cfg->max_disparity - 1;
        if (w - 1 - CENSUS_R - ur < back) back = w - 1 - CENSUS_R - ur;
        const int bk = search_r2l(cl, cr, w, ur, v, back);
        if (abs(ur + bk - u) > 1) continue;
        const size_t key = (size_t)v * w + u;
        if (slot[key] < 0) {
            slot[key] = count;
            su[count] = u;
            sv[count] = v;
            sd[count] = (double)bd;
            acc_cost[count] = bc;
            ++count;
        } else if (bc < acc_cost[slot[key]]) {
            sd[slot[key]] = (double)bd;
            acc_cost[slot[key]] = bc;
        }
    }
    free(slot);
    free(acc_cost);
    return count;
}

/* ---------------------------------------------------------------- delaunay.cpp */
/* orient2d, delaunay.cpp:11-17 */
long long orc_orient2d(int au, int av, int bu, int bv, int cu, int cv) {
    long long abx = (long long)bu - au, aby = (long long)bv - av;
    long long acx = (long long)cu - au, acy = (long long)cv - av;
    return abx * acy - aby * acx;
}

/* inCircleSign, delaunay.cpp:19-41 (exact, __int128) */
int orc_incircle_sign(int au, int av, int bu, int bv, int cu, int cv, int du, int dv) {
    long long adx = (long long)au - du, ady = (long long)av - dv;
    long long bdx = (long long)bu - du, bdy = (long long)bv - dv;
    long long cdx = (long long)cu - du, cdy = (long long)cv - dv;
    long long aq = adx * adx + ady * ady, bq = bdx * bdx + bdy * bdy, cq = cdx * cdx + cdy * cdy;
    __int128 det = (__int128)adx * ((__int128)bdy * cq - (__int128)cdy * bq) -
                   (__int128)ady * ((__int128)bdx * cq - (__int128)cdx * bq) +
                   (__int128)aq * ((__int128)bdx * cdy - (__int128)cdx * bdy);
    return det > 0 ? 1 : (det < 0 ? -1 : 0);
}

/* Lexicographic sweep with Lawson flips (delaunay.cpp:50-284), restated. */
typedef struct {
    int n;
    const int* pu;
    const int* pv;
    int* tri;   /* 3 vertex ids per triangle, half-edge e = 3t+i runs tri[e] -> tri[next(e)] */
    int* twin;  /* opposite half-edge or -1 */
    int ntri3;
    int* hnext; /* hull ring */
    int* hprev;
    int* hedge; /* half-edge of hull edge (v -> hnext[v]) */
    int* stack;
    int nstack, capstack;
    int last;
} sweep_t;

static int he_next(int e) { return e - e % 3 + (e + 1) % 3; }

static long long sw_orient(const sweep_t* s, int a, int b, int c) {
    return orc_orient2d(s->pu[a], s->pv[a], s->pu[b], s->pv[b], s->pu[c], s->pv[c]);
}

static void sw_push(sweep_t* s, int e) {
    if (s->nstack == s->capstack) {
        s->capstack = s->capstack ? 2 * s->capstack : 256;
        s->stack = (int*)realloc(s->stack, sizeof(int) * (size_t)s->capstack);
    }
    s->stack[s->nstack++] = e;
}

/* addTriangle, delaunay.cpp:95-107 */
static int sw_add(sweep_t* s, int a, int b, int c, int tab, int tbc, int tca) {
    int e = s->ntri3;
    s->tri[e] = a;
    s->tri[e + 1] = b;
    s->tri[e + 2] = c;
    s->twin[e] = tab;
    s->twin[e + 1] = tbc;
    s->twin[e + 2] = tca;
    if (tab >= 0) s->twin[tab] = e;
    if (tbc >= 0) s->twin[tbc] = e + 1;
    if (tca >= 0) s->twin[tca] = e + 2;
    s->ntri3 += 3;
    return e;
}

static void sw_link(sweep_t* s, int e, int f) {
    s->twin[e] = f;
    if (f >= 0) s->twin[f] = e;
}

static void sw_hull(sweep_t* s, int a, int b) {
    s->hnext[a] = b;
    s->hprev[b] = a;
}

/* visible, delaunay.cpp:116-118: strictly right of the hull edge */
static int sw_visible(const sweep_t* s, int hv, int p) {
    return sw_orient(s, hv, s->hnext[hv], p) < 0;
}

/* buildFan, delaunay.cpp:123-164 */
static void sw_fan(sweep_t* s, const int* line, int k, int apex) {
    long long side = sw_orient(s, line[0], line[1], apex);
    int prev = -1;
    for (int j = 0; j + 1 < k; ++j) {
        if (side > 0) {
            int e = sw_add(s, line[j], line[j + 1], apex, -1, -1, prev);
            if (j == 0) s->hedge[apex] = e + 2;
            s->hedge[line[j]] = e;
            prev = e + 1;
        } else {
            int e = sw_add(s, line[j + 1], line[j], apex, -1, prev, -1);
            if (j == 0) s->hedge[line[0]] = e + 1;
            s->hedge[line[j + 1]] = e;
            prev = e + 2;
        }
    }
    if (side > 0) {
        s->hedge[line[k - 1]] = prev;
        for (int j = 0; j + 1 < k; ++j) sw_hull(s, line[j], line[j + 1]);
        sw_hull(s, line[k - 1], apex);
        sw_hull(s, apex, line[0]);
    } else {
        s->hedge[apex] = prev;
        for (int j = 0; j + 1 < k; ++j) sw_hull(s, line[j + 1], line[j]);
        sw_hull(s, line[0], apex);
        sw_hull(s, apex, line[k - 1]);
    }
    s->last = apex;
}

/* legalizeAll, delaunay.cpp:221-274: LIFO, flip only on strict in-circle */
static void sw_legalize(sweep_t* s) {
    while (s->nstack > 0) {
        int e = s->stack[--s->nstack];
        int f = s->twin[e];
        if (f < 0) continue;
        int e1 = he_next(e), e2 = he_next(e1);
        int f1 = he_next(f), f2 = he_next(f1);
        int a = s->tri[e], b = s->tri[e1], c = s->tri[e2], d = s->tri[f2];
        if (orc_incircle_sign(s->pu[a], s->pv[a], s->pu[b], s->pv[b], s->pu[c], s->pv[c], s->pu[d],
                              s->pv[d]) <= 0)
            continue;
        int te1 = s->twin[e1], te2 = s->twin[e2], tf1 = s->twin[f1], tf2 = s->twin[f2];
        s->tri[e] = a;
        s->tri[e1] = d;
        s->tri[e2] = c;
        s->tri[f] = d;
        s->tri[f1] = b;
        s->tri[f2] = c;
        sw_link(s, e1, f2);
        sw_link(s, e, tf1);
        if (tf1 < 0) s->hedge[a] = e;
        sw_link(s, f, tf2);
        if (tf2 < 0) s->hedge[d] = f;
        sw_link(s, f1, te1);
        if (te1 < 0) s->hedge[b] = f1;
        sw_link(s, e2, te2);
        if (te2 < 0) s->hedge[c] = e2;
        sw_push(s, e);
        sw_push(s, f);
        sw_push(s, f1);
        sw_push(s, e2);
    }
}

/* insert, delaunay.cpp:171-217 */
static int sw_insert(sweep_t* s, int ip) {
    int start = -1, v = s->last;
    do {
        if (sw_visible(s, v, ip)) {
            start = v;
            break;
        }
        v = s->hnext[v];
    } while (v != s->last);
    if (start < 0) return -1;
    int a = start;
    while (s->hprev[a] != start && sw_visible(s, s->hprev[a], ip)) a = s->hprev[a];
    int b = s->hnext[start];
    while (b != start && sw_visible(s, b, ip)) b = s->hnext[b];
    int prev_e1 = -1, first_e0 = -1;
    for (int x = a; x != b;) {
        int xn = s->hnext[x];
        int e = sw_add(s, x, ip, xn, prev_e1, -1, s->hedge[x]);
        if (first_e0 < 0) first_e0 = e;
        prev_e1 = e + 1;
        sw_push(s, e + 2);
        x = xn;
    }
    sw_hull(s, a, ip);
    sw_hull(s, ip, b);
    s->hedge[a] = first_e0;
    s->hedge[ip] = prev_e1;
    s->last = ip;
    sw_legalize(s);
    return 0;
}

typedef struct {
    int u, v, idx;
} lexpt_t;
static int cmp_lex(const void* pa, const void* pb) {
    const lexpt_t* a = (const lexpt_t*)pa;
    const lexpt_t* b = (const lexpt_t*)pb;
    if (a->u != b->u) return a->u < b->u ? -1 : 1;
    if (a->v != b->v) return a->v < b->v ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* delaunayTriangulate, delaunay.cpp:288-325 */
int orc_delaunay(const int* u, const int* v, int n, int* tris) {
    for (int i = 0; i < n; ++i)
        if (abs(u[i]) >= (1 << 20) || abs(v[i]) >= (1 << 20)) return -1;
    if (n < 3) return 0;
    lexpt_t* ord = (lexpt_t*)malloc(sizeof(lexpt_t) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        ord[i].u = u[i];
        ord[i].v = v[i];
        ord[i].idx = i;
    }
    qsort(ord, (size_t)n, sizeof(lexpt_t), cmp_lex);
    int* kept = (int*)malloc(sizeof(int) * (size_t)n);
    int* su = (int*)malloc(sizeof(int) * (size_t)n);
    int* sv = (int*)malloc(sizeof(int) * (size_t)n);
    int m = 0;
    for (int i = 0; i < n; ++i) { /* keep the first of coincident points (:303-311) */
        if (m > 0 && su[m - 1] == ord[i].u && sv[m - 1] == ord[i].v) continue;
        kept[m] = ord[i].idx;
        su[m] = ord[i].u;
        sv[m] = ord[i].v;
        ++m;
    }
    free(ord);
    int result = 0;
    if (m >= 3) {
        sweep_t s;
        memset(&s, 0, sizeof(s));
        s.n = m;
        s.pu = su;
        s.pv = sv;
        s.tri = (int*)malloc(sizeof(int) * (size_t)m * 6);
        s.twin = (int*)malloc(sizeof(int) * (size_t)m * 6);
        s.hnext = (int*)malloc(sizeof(int) * (size_t)m);
        s.hprev = (int*)malloc(sizeof(int) * (size_t)m);
        s.hedge = (int*)malloc(sizeof(int) * (size_t)m);
        for (int i = 0; i < m; ++i) s.hnext[i] = s.hprev[i] = s.hedge[i] = -1;
        s.last = -1;
        /* leading collinear run (build, delaunay.cpp:67-77) */
        int* line = (int*)malloc(sizeof(int) * (size_t)m);
        int k = 1, i = 1;
        line[0] = 0;
        while (i < m && (k < 2 || sw_orient(&s, line[0], line[1], i) == 0)) {
            line[k++] = i;
            ++i;
        }
        if (i < m) {
            sw_fan(&s, line, k, i);
            int ok = 0;
            for (++i; i < m && ok == 0; ++i) ok = sw_insert(&s, i);
            if (ok != 0) {
                result = -2;
            } else {
                result = s.ntri3 / 3;
                for (int e = 0; e < s.ntri3; ++e) tris[e] = kept[s.tri[e]];
            }
        }
        free(line);
        free(s.tri);
        free(s.twin);
        free(s.hnext);
        free(s.hprev);
        free(s.hedge);
        free(s.stack);
    }
    free(kept);
    free(su);
    free(sv);
    return result;
}

/* ---------------------------------------------------------------- mesh.cpp */
/* fitPlane, mesh.cpp:12-26 — source order, no FMA, IEEE division */
int orc_fit_plane(int u1i, int w1i, double d1, int u2i, int w2i, double d2, int u3i, int w3i,
                  double d3, double* abc) {
    const long long u1 = u1i, u2 = u2i, u3 = u3i, w1 = w1i, w2 = w2i, w3 = w3i;
    const long long det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    if (det == 0) return -1;
    const double da = d1 * (double)(w2 - w3) + d2 * (double)(w3 - w1) + d3 * (double)(w1 - w2);
    const double db = (double)u1 * (d2 - d3) + (double)u2 * (d3 - d1) + (double)u3 * (d1 - d2);
    const double dc = d1 * (double)(u2 * w3 - u3 * w2) - d2 * (double)(u1 * w3 - u3 * w1) +
                      d3 * (double)(u1 * w2 - u2 * w1);
    abc[0] = da / (double)det;
    abc[1] = db / (double)det;
    abc[2] = dc / (double)det;
    return 0;
}

/* floorDiv / ceilDiv, mesh.cpp:30-40 */
static long long floor_div(long long a, long long b) {
    long long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}
static long long ceil_div(long long a, long long b) { return -floor_div(-a, b); }

/* DisparityMesh ctor + rasterize, mesh.cpp:44-123 */
int orc_mesh_build(const int* u, const int* v, const double* d, const int* tris, int nt, int w,
                   int h, double* planes, int32_t* lookup) {
    for (size_t i = 0; i < (size_t)w * h; ++i) lookup[i] = -1;
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        if (orc_fit_plane(u[tr[0]], v[tr[0]], d[tr[0]], u[tr[1]], v[tr[1]], d[tr[1]], u[tr[2]],
                          v[tr[2]], d[tr[2]], planes + 3 * t) != 0)
            return -1;
    }
    for (int t = 0; t < nt; ++t) {
        const int* tr = tris + 3 * t;
        int x[3] = {u[tr[0]], u[tr[1]], u[tr[2]]};
        int y[3] = {v[tr[0]], v[tr[1]], v[tr[2]]};
        int vmin = y[0] < y[1] ? y[0] : y[1];
        if (y[2] < vmin) vmin = y[2];
        int vmax = y[0] > y[1] ? y[0] : y[1];
        if (y[2] > vmax) vmax = y[2];
        if (vmin < 0) vmin = 0;
        if (vmax > h - 1) vmax = h - 1;
        long long A[3], bias[3];
        for (int i = 0; i < 3; ++i) {
            int j = (i + 1) % 3;
            A[i] = y[i] - y[j];
            int accept = (y[j] < y[i]) || (y[j] == y[i] && x[j] > x[i]);
            bias[i] = accept ? 0 : 1;
        }
        for (int row = vmin; row <= vmax; ++row) {
            long long lo = 0, hi = w - 1;
            int empty = 0;
            for (int i = 0; i < 3 && !empty; ++i) {
                int j = (i + 1) % 3;
                long long K = (long long)(x[j] - x[i]) * (row - y[i]) + (long long)(y[j] - y[i]) * x[i];
                long long m = bias[i];
                if (A[i] > 0) {
                    long long c = ceil_div(m - K, A[i]);
                    if (c > lo) lo = c;
                } else if (A[i] < 0) {
                    long long f = floor_div(K - m, -A[i]);
                    if (f < hi) hi = f;
                } else if (K < m) {
                    empty = 1;
                }
            }
            if (empty || lo > hi) continue;
            int32_t* line = lookup + (size_t)row * w;
            for (long long c = lo; c <= hi; ++c) line[c] = t;
        }
    }
    /* hull-vertex pinning, mesh.cpp:112-122 */
    for (int t = 0; t < nt; ++t) {
        for (int k = 0; k < 3; ++k) {
            int c = tris[3 * t + k];
            if (u[c] >= 0 && u[c] < w && v[c] >= 0 && v[c] < h) {
                int32_t* cell = lookup + (size_t)v[c] * w + u[c];
                if (*cell == -1) *cell = t;
            }
        }
    }
    return 0;
}

/* interpolate, mesh.cpp:149-182 */
void orc_interpolate(const int32_t* lookup, const double* planes, int w, int h,
                     const uint8_t* mask, float max_disparity, float* value, uint8_t* valid) {
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            size_t i = (size_t)v * w + u;
            value[i] = 0.0f;
            valid[i] = 0;
            if (mask && !mask[i]) continue;
            int t = lookup[i];
            if (t == -1) continue;
            const double* p = planes + 3 * (size_t)t;
            float d = (float)(p[0] * (double)u + p[1] * (double)v + p[2]);
            if (d >= 0.0f && d < max_disparity) {
                value[i] = d;
                valid[i] = 1;
            }
        }
    }
}

/* ---------------------------------------------------------------- pipeline.cpp */
#define SENTINEL_COST 1.0f /* kSentinelCost, pipeline.cpp:15 */

/* costEvaluation, pipeline.cpp:33-54 */
void orc_cost_evaluation(const uint32_t* cl, const uint32_t* cr, int w, int h, const float* value,
                         const uint8_t* valid, const uint8_t* mask, float* cost) {
    for (size_t i = 0; i < (size_t)w * h; ++i) cost[i] = SENTINEL_COST;
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            size_t i = (size_t)v * w + u;
            if (!mask[i] || !valid[i]) continue;
            long d = lroundf(value[i]); /* std::lround: half away from zero */
            long ur = (long)u - d;
            if (d < 0 || ur < CENSUS_R) continue;
            cost[i] = census_cost(cl[i], cr[(size_t)v * w + (size_t)ur]);
        }
    }
}

/* wtaOracle, proj/src/synth.cpp:171-198 */
void orc_wta(const uint8_t* left, const uint8_t* right, int w, int h, const uint8_t* mask, int nd,
             float* disparity, uint8_t* valid, float* cost) {
    const size_t n = (size_t)w * h;
    uint32_t* cl = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* cr = (uint32_t*)malloc(sizeof(uint32_t) * n);
    orc_census(left, w, h, cl);
    orc_census(right, w, h, cr);
    for (size_t i = 0; i < n; ++i) {
        disparity[i] = 0.0f;
        valid[i] = 0;
        cost[i] = 1.0f; /* CostMap(w, h, 1.0f) */
    }
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            const size_t i = (size_t)v * w + u;
            if (!mask[i]) continue; /* mask.points(), row-major */
            const int dmax = nd < u - CENSUS_R ? nd : u - CENSUS_R;
            int best_d = -1;
            float best = 2.0f;
            for (int d = 0; d <= dmax; ++d) {
                const float c = census_cost(cl[i], cr[(size_t)v * w + (size_t)(u - d)]);
                if (c < best) {
                    best = c;
                    best_d = d;
                }
            }
            if (best_d >= 0) {
                disparity[i] = (float)best_d;
                valid[i] = 1;
                cost[i] = best;
            }
        }
    }
    free(cl);
    free(cr);
}

/* writeKittiPng, proj/src/io.cpp:349-368 (the raster it hands to libpng) */
long long orc_encode_kitti16(const float* d, const uint8_t* valid, int w, int h, uint8_t* out) {
    memset(out, 0, (size_t)w * h * 2);
    for (int v = 0; v < h; ++v) {
        uint8_t* row = out + (size_t)v * w * 2;
        for (int u = 0; u < w; ++u) {
            const size_t i = (size_t)v * w + u;
            if (!valid[i]) continue;
            if (d[i] < 0.0f) return (long long)i; /* NegativeDisparity */
            long raw = lround((double)d[i] * 256.0);
            raw = raw < 1L ? 1L : (raw > 65535L ? 65535L : raw); /* raw 0 is reserved */
            row[2 * u] = (uint8_t)(raw >> 8);
            row[2 * u + 1] = (uint8_t)(raw & 0xff);
        }
    }
    return -1;
}

/* writePfm, proj/src/io.cpp:311-329 */
void orc_encode_pfm(const float* d, const uint8_t* valid, int w, int h, float* out) {
    for (int r = 0; r < h; ++r) {
        const int v = h - 1 - r;
        for (int u = 0; u < w; ++u) {
            const size_t i = (size_t)v * w + u;
            out[(size_t)r * w + u] = valid[i] ? d[i] : -1.0f;
        }
    }
}

/* exportPointCloud, proj/src/io.cpp:395-454 (vertex list) */
int orc_point_cloud(const float* d, const uint8_t* valid, const uint8_t* image, int w, int h,
                    const ps_calib* calib, double min_disparity, float* xyz, uint8_t* intensity) {
    if (!(calib->focal > 0.0) || !(calib->baseline > 0.0)) return -1; /* io.cpp:19-26 */
    int n = 0;
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            const size_t i = (size_t)v * w + u;
            if (!valid[i]) continue;
            const double dd = d[i];
            if (dd < min_disparity) continue;
            const double z = calib->focal * calib->baseline / dd;
            const double x = (u - calib->cx) * z / calib->focal;
            const double y = (v - calib->cy) * z / calib->focal;
            xyz[3 * n] = (float)x;
            xyz[3 * n + 1] = (float)y;
            xyz[3 * n + 2] = (float)z;
            intensity[n] = image[i];
            ++n;
        }
    }
    return n;
}

/* accuracyImpl, proj/src/eval.cpp:19-59 */
int orc_accuracy(const float* pred, const uint8_t* pred_valid, const float* gt,
                 const uint8_t* gt_valid, const uint8_t* mask, int w, int h,
                 const double* thresholds, int n_thr, double* fractions, long long* evaluated,
                 double* mean_abs_error) {
    long long n = 0;
    long* hits = (long*)calloc(n_thr > 0 ? n_thr : 1, sizeof(long));
    double err_sum = 0.0;
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            const size_t i = (size_t)v * w + u;
            if (!pred_valid[i] || !gt_valid[i]) continue;
            if (mask && !mask[i]) continue;
            const double err = fabs((double)pred[i] - (double)gt[i]);
            ++n;
            err_sum += err;
            for (int k = 0; k < n_thr; ++k) hits[k] += (err < thresholds[k]);
        }
    }
    *evaluated = n;
    if (n == 0) {
        free(hits);
        return PS_NO_OVERLAP;
    }
    *mean_abs_error = err_sum / (double)n;
    for (int k = 0; k < n_thr; ++k) fractions[k] = (double)hits[k] / (double)n;
    free(hits);
    return PS_OK;
}

static int ceil_div_pos(int a, int b) { return (a + b - 1) / b; }

/* disparityRefinement, pipeline.cpp:56-86 */
void orc_refinement(const float* value, const uint8_t* valid, const float* cost, float* fd,
                    uint8_t* fv, float* fc, const uint8_t* mask, int w, int h, int cell,
                    const ps_config* cfg, ps_cell* confident, ps_cell* invalid) {
    const int cols = ceil_div_pos(w, cell), rows = ceil_div_pos(h, cell);
    for (int i = 0; i < cols * rows; ++i) {
        memset(&confident[i], 0, sizeof(ps_cell));
        memset(&invalid[i], 0, sizeof(ps_cell));
        confident[i].cost = cfg->cost_low;
        invalid[i].cost = cfg->cost_high;
    }
    (void)valid;
    for (int v = 0; v < h; ++v) {
        for (int u = 0; u < w; ++u) {
            size_t i = (size_t)v * w + u;
            if (!mask[i]) continue;
            const float c = cost[i];
            if (c < fc[i]) {
                fd[i] = value[i];
                fv[i] = 1;
                fc[i] = c;
            }
            const int ci = (v / cell) * cols + (u / cell);
            if (c < cfg->cost_low) {
                if (c < confident[ci].cost) {
                    confident[ci].u = u;
                    confident[ci].v = v;
                    confident[ci].disparity = value[i];
                    confident[ci].cost = c;
                    confident[ci].occupied = 1;
                }
            } else if (c > cfg->cost_high) {
                if (c > invalid[ci].cost) {
                    invalid[ci].u = u;
                    invalid[ci].v = v;
                    invalid[ci].disparity = 0.0f;
                    invalid[ci].cost = c;
                    invalid[ci].occupied = 1;
                }
            }
        }
    }
}

/* supportResampling, pipeline.cpp:88-129 */
int orc_support_resampling(const ps_cell* confident, const ps_cell* invalid, int cell,
                           const int* su, const int* sv, const double* sd, int n,
                           const uint32_t* cl, const uint32_t* cr, int w, int h,
                           const ps_config* cfg, int* ou, int* ov, double* od, int cap) {
    const int cols = ceil_div_pos(w, cell), rows = ceil_div_pos(h, cell);
    uint8_t* taken = (uint8_t*)calloc((size_t)w * h, 1);
    int count = 0;
    for (int i = 0; i < n; ++i) {
        ou[count] = su[i];
        ov[count] = sv[i];
        od[count] = sd[i];
        ++count;
        taken[(size_t)sv[i] * w + su[i]] = 1;
    }
    for (int ci = 0; ci < cols * rows; ++ci) {
        const ps_cell* c = &confident[ci];
        if (!c->occupied || (float)c->u - c->disparity < (float)CENSUS_R) continue;
        size_t key = (size_t)c->v * w + c->u;
        if (taken[key]) continue;
        taken[key] = 1;
        if (count < cap) {
            ou[count] = c->u;
            ov[count] = c->v;
            od[count] = (double)c->disparity;
        }
        ++count;
    }
    int nre = 0;
    int* ru = (int*)malloc(sizeof(int) * (size_t)(cols * rows + 1));
    int* rv = (int*)malloc(sizeof(int) * (size_t)(cols * rows + 1));
    for (int ci = 0; ci < cols * rows; ++ci) {
        if (invalid[ci].occupied) {
            ru[nre] = invalid[ci].u;
            rv[nre] = invalid[ci].v;
            ++nre;
        }
    }
    int* mu = (int*)malloc(sizeof(int) * (size_t)(nre + 1));
    int* mv = (int*)malloc(sizeof(int) * (size_t)(nre + 1));
    double* md = (double*)malloc(sizeof(double) * (size_t)(nre + 1));
    int nm = orc_match_epipolar(cl, cr, w, h, ru, rv, nre, cfg, mu, mv, md);
    for (int i = 0; i < nm; ++i) {
        size_t key = (size_t)mv[i] * w + mu[i];
        if (taken[key]) continue;
        taken[key] = 1;
        if (count < cap) {
            ou[count] = mu[i];
            ov[count] = mv[i];
            od[count] = md[i];
        }
        ++count;
    }
    free(ru);
    free(rv);
    free(mu);
    free(mv);
    free(md);
    free(taken);
    return count;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static int is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

/* PipelineConfig::validate, config.cpp:17-49 */
static int validate_config(const ps_config* c) {
    if (c->iterations < 1) return PS_INVALID_CONFIG;
    if (c->max_disparity < 1) return PS_INVALID_CONFIG;
    if (!(c->cost_low > 0.0f && c->cost_low < c->cost_high && c->cost_high <= 1.0f))
        return PS_INVALID_CONFIG;
    if (!is_pow2(c->occupancy_cell_size)) return PS_INVALID_CONFIG;
    if (c->gradient_threshold < 0 || c->corner_threshold < 0) return PS_INVALID_CONFIG;
    if (c->per_bin_cap < 1) return PS_INVALID_CONFIG;
    if (!(c->sparse_accept_cost > 0.0f && c->sparse_accept_cost <= 1.0f)) return PS_INVALID_CONFIG;
    if (!(c->uniqueness_ratio > 0.0f && c->uniqueness_ratio <= 1.0f)) return PS_INVALID_CONFIG;
    if (c->threads < 1) return PS_INVALID_CONFIG;
    return PS_OK;
}

/* run, pipeline.cpp:131-203 (staged; validate optional) */
int orc_run(const uint8_t* left, const uint8_t* right, int w, int h, const ps_config* cfg,
            int validate, float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
            uint8_t* dense_valid, ps_iter_stats* trace, int* sup_u, int* sup_v, double* sup_d,
            int sup_cap, int* sup_count) {
    if (validate) {
        int st = validate_config(cfg);
        if (st != PS_OK) return st;
    }
    if (w < 16 || h < 16) return PS_DIMENSION_TOO_SMALL;
    const size_t P = (size_t)w * h;
    uint8_t* mask = (uint8_t*)malloc(P);
    uint32_t* cl = (uint32_t*)malloc(4 * P);
    uint32_t* cr = (uint32_t*)malloc(4 * P);
    const int M = orc_gradient_mask(left, w, h, cfg->gradient_threshold, mask);
    orc_census(left, w, h, cl);
    orc_census(right, w, h, cr);

    float* fd = (float*)calloc(P, sizeof(float));
    uint8_t* fv = (uint8_t*)calloc(P, 1);
    float* fc = (float*)malloc(P * sizeof(float));
    for (size_t i = 0; i < P; ++i) fc[i] = cfg->cost_high;
    int cell = cfg->occupancy_cell_size;

    const int ccap = 120 * cfg->per_bin_cap;
    int* cu = (int*)malloc(sizeof(int) * (size_t)ccap);
    int* cv = (int*)malloc(sizeof(int) * (size_t)ccap);
    const int nc = orc_detect_candidates(left, w, h, cfg, cu, cv, NULL, ccap);
    size_t scap = P + 16;
    int* su = (int*)malloc(sizeof(int) * scap);
    int* sv = (int*)malloc(sizeof(int) * scap);
    double* sd = (double*)malloc(sizeof(double) * scap);
    int ns = orc_match_epipolar(cl, cr, w, h, cu, cv, nc, cfg, su, sv, sd);
    free(cu);
    free(cv);
    int status = PS_OK;
    if (ns < 3) {
        status = PS_SEEDING_FAILED;
    } else {
        int* tris = (int*)malloc(sizeof(int) * 6 * scap);
        double* planes = (double*)malloc(sizeof(double) * 6 * scap);
        int32_t* lookup = (int32_t*)malloc(sizeof(int32_t) * P);
        float* iv = (float*)malloc(sizeof(float) * P);
        uint8_t* ivalid = (uint8_t*)malloc(P);
        float* ic = (float*)malloc(sizeof(float) * P);
        int* nu = (int*)malloc(sizeof(int) * scap);
        int* nv = (int*)malloc(sizeof(int) * scap);
        double* nd = (double*)malloc(sizeof(double) * scap);
        for (int it = 1; it <= cfg->iterations; ++it) {
            const double tic = now_ms();
            const int nt = orc_delaunay(su, sv, ns, tris);
            if (nt < 0) {
                status = PS_ERROR;
                break;
            }
            if (orc_mesh_build(su, sv, sd, tris, nt, w, h, planes, lookup) != 0) {
                status = PS_DEGENERATE_TRIANGLE;
                break;
            }
            orc_interpolate(lookup, planes, w, h, mask, (float)cfg->max_disparity, iv, ivalid);
            orc_cost_evaluation(cl, cr, w, h, iv, ivalid, mask, ic);
            const int cols = ceil_div_pos(w, cell), rows = ceil_div_pos(h, cell);
            ps_cell* gc = (ps_cell*)malloc(sizeof(ps_cell) * (size_t)cols * rows);
            ps_cell* gi = (ps_cell*)malloc(sizeof(ps_cell) * (size_t)cols * rows);
            orc_refinement(iv, ivalid, ic, fd, fv, fc, mask, w, h, cell, cfg, gc, gi);
            const int used_cell = cell;
            const int used_supports = ns;
            if (it != cfg->iterations) {
                int nn = orc_support_resampling(gc, gi, cell, su, sv, sd, ns, cl, cr, w, h, cfg,
                                                nu, nv, nd, (int)scap);
                memcpy(su, nu, sizeof(int) * (size_t)nn);
                memcpy(sv, nv, sizeof(int) * (size_t)nn);
                memcpy(sd, nd, sizeof(double) * (size_t)nn);
                ns = nn;
                cell = cell / 2 > 1 ? cell / 2 : 1;
            } else {
                if (dense) orc_interpolate(lookup, planes, w, h, NULL, (float)cfg->max_disparity,
                                           dense, dense_valid);
                if (sup_count) {
                    *sup_count = used_supports;
                    for (int i = 0; i < used_supports && i < sup_cap; ++i) {
                        if (sup_u) sup_u[i] = su[i];
                        if (sup_v) sup_v[i] = sv[i];
                        if (sup_d) sup_d[i] = sd[i];
                    }
                }
            }
            free(gc);
            free(gi);
            const double toc = now_ms();
            if (trace) {
                ps_iter_stats* s = &trace[it - 1];
                s->iteration = it;
                s->support_count = used_supports;
                s->triangle_count = nt;
                s->occupancy_cell_size = used_cell;
                double sum = 0.0;
                int valid = 0;
                for (size_t i = 0; i < P; ++i) {
                    if (!mask[i]) continue;
                    sum += fc[i];
                    valid += fc[i] < cfg->cost_high;
                }
                s->mean_cost = M > 0 ? sum / M : 0.0;
                s->valid_count = valid;
                s->millis = toc - tic;
            }
        }
        free(tris);
        free(planes);
        free(lookup);
        free(iv);
        free(ivalid);
        free(ic);
        free(nu);
        free(nv);
        free(nd);
    }
    if (status == PS_OK) {
        if (disparity) memcpy(disparity, fd, P * sizeof(float));
        if (disparity_valid) memcpy(disparity_valid, fv, P);
        if (cost) memcpy(cost, fc, P * sizeof(float));
    }
    free(mask);
    free(cl);
    free(cr);
    free(fd);
    free(fv);
    free(fc);
    free(su);
    free(sv);
    free(sd);
    return status;
}

typedef struct {
    int n, w, h, threads, tid;
    const uint8_t *left, *right;
    const ps_config* cfg;
    float *disparity, *cost, *dense;
    uint8_t *disparity_valid, *dense_valid;
    int* status;
} batch_job_t;

static void* batch_worker(void* arg) {
    batch_job_t* j = (batch_job_t*)arg;
    const size_t P = (size_t)j->w * j->h;
    for (int f = j->tid; f < j->n; f += j->threads) {
        int st = orc_run(j->left + f * P, j->right + f * P, j->w, j->h, j->cfg, 0,
                         j->disparity ? j->disparity + f * P : NULL,
                         j->disparity_valid ? j->disparity_valid + f * P : NULL,
                         j->cost ? j->cost + f * P : NULL, j->dense ? j->dense + f * P : NULL,
                         j->dense_valid ? j->dense_valid + f * P : NULL, NULL, NULL, NULL, NULL, 0,
                         NULL);
        if (j->status) j->status[f] = st;
    }
    return NULL;
}

int orc_run_batch(int n, const uint8_t* left, const uint8_t* right, int w, int h,
                  const ps_config* cfg, int threads, float* disparity, uint8_t* disparity_valid,
                  float* cost, float* dense, uint8_t* dense_valid, int* status) {
    if (threads < 1) threads = 1;
    if (threads > n) threads = n > 0 ? n : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    batch_job_t* jobs = (batch_job_t*)malloc(sizeof(batch_job_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        batch_job_t j = {n, w, h, threads, t, left, right, cfg, disparity, cost, dense,
                         disparity_valid, dense_valid, status};
        jobs[t] = j;
        pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}
