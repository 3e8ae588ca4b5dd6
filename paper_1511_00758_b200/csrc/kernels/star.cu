// star.cu — K4 on the device: per-frame exact Delaunay of the support list
// (star_dt.cuh), hull-vertex pins and rotation checks, for a frame group.
//
// Replaces the host triangulation of every frame-iteration
// (proj/src/delaunay.cpp:288-325 -> DisparityMesh, proj/src/mesh.cpp:44-123):
//   1. a uniform grid of each frame's supports (count, scan, fill), coincident
//      points marked (the reference keeps the first, delaunay.cpp:303-311);
//   2. one thread per support walks its Delaunay star; a triangle is written
//      by its smallest vertex index (slot from a per-frame counter: the
//      order of the list is free, each pixel has one covering triangle and
//      pins are chosen by vertex set); an uncovered hull vertex (open star,
//      mesh.cpp:109-122) whose incident planes give the same binary32 D_it at
//      its pixel is pinned here, otherwise it is listed for the host, which
//      knows the reference sweep's triangle order (SweepOrder);
//   3. one thread per triangle fits the plane in its three rotations
//      (mesh.cpp:12-26, _rn intrinsics in source order); triangles whose
//      rotations round differently are listed for the host (it decides the
//      sweep's stored rotation where some covered pixel would change);
//   4. after the host's fixes are applied, pin bits from the chosen vertex sets.
// Anything a bounded list cannot hold sets the frame's fail flag: the host
// then replays the reference sweep for that frame (exact fallback).
#include <cuda_runtime.h>

#include <cstdio>

#include "launch.hpp"
#include "star_dt.cuh"

namespace ps {

namespace {

constexpr int kT = 128;

__device__ __forceinline__ bool tie_accept(int xi, int yi, int xj, int yj) {
    return (yj < yi) || (yj == yi && xj > xi);  // mesh.cpp:80
}

struct Fit {
    double A, B, C;
    long long det;
};

// fitPlane numerators (mesh.cpp:12-26) in the reference's source order.
__device__ __forceinline__ Fit fit3(const int* __restrict__ su, const int* __restrict__ sv,
                                    const double* __restrict__ sd, int i, int j, int k) {
    const long long u1 = su[i], u2 = su[j], u3 = su[k], w1 = sv[i], w2 = sv[j], w3 = sv[k];
    const double d1 = sd[i], d2 = sd[j], d3 = sd[k];
    Fit f;
    f.det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    f.A = __dadd_rn(__dadd_rn(__dmul_rn(d1, double(w2 - w3)), __dmul_rn(d2, double(w3 - w1))),
                    __dmul_rn(d3, double(w1 - w2)));
    f.B = __dadd_rn(__dadd_rn(__dmul_rn(double(u1), __dsub_rn(d2, d3)), __dmul_rn(double(u2), __dsub_rn(d3, d1))),
                    __dmul_rn(double(u3), __dsub_rn(d1, d2)));
    f.C = __dadd_rn(__dsub_rn(__dmul_rn(d1, double(u2 * w3 - u3 * w2)), __dmul_rn(d2, double(u1 * w3 - u3 * w1))),
                    __dmul_rn(d3, double(u1 * w2 - u2 * w1)));
    return f;
}

__device__ __forceinline__ bool same_bits(const Fit& a, const Fit& b) {
    return __double_as_longlong(a.A) == __double_as_longlong(b.A) &&
           __double_as_longlong(a.B) == __double_as_longlong(b.B) &&
           __double_as_longlong(a.C) == __double_as_longlong(b.C);
}

// D_it bits at (u, v) as the raster stores them (NaN = invalid).
__device__ __forceinline__ unsigned dit_bits(const Fit& f, int u, int v, float nd) {
    if (f.det == 0) return 0x7fc00000u;
    const double a = __ddiv_rn(f.A, double(f.det)), b = __ddiv_rn(f.B, double(f.det)),
                 c = __ddiv_rn(f.C, double(f.det));
    const float d = __double2float_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, double(u)), __dmul_rn(b, double(v))), c));
    if (!(d >= 0.0f && d < nd)) return 0x7fc00000u;
    return __float_as_uint(d);
}

__device__ __forceinline__ void min_first(int& a, int& b, int& c) {  // rotate: smallest first
    if (b < a && b < c) {
        const int t = a;
        a = b;
        b = c;
        c = t;
    } else if (c < a && c < b) {
        const int t = c;
        c = b;
        b = a;
        a = t;
    }
}

__device__ __forceinline__ star::Grid make_grid(const StarArgs& a, int f) {
    const long long sb = (long long)f * a.scap;
    const long long cb = (long long)f * (a.gw * a.gh + 1);
    const int* cols = a.col_idx + 2ll * f * a.W;
    const int* hull = a.hull + 2 * sb;
    return star::Grid{a.su + sb, a.sv + sb, a.dup + sb, a.cell_start + cb, a.cell_items + sb, a.S[f],
                      0, 0, a.W - 1, a.H - 1, a.gs, a.gw, a.gh, cols, cols + a.W, hull, hull + a.scap,
                      a.flags[(long long)f * kStarFlagInts + 4]};
}

__global__ void k_grid_count(StarArgs a) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int cell = (a.sv[sb + i] / a.gs) * a.gw + a.su[sb + i] / a.gs;
    atomicAdd(a.cell_cnt + (long long)f * a.gw * a.gh + cell, 1);
}

// exclusive scan of the frame's cell counts into cell_start; cell_cnt becomes
// the fill cursor
__global__ void k_grid_scan(StarArgs a) {
    const int f = blockIdx.x;
    const int cells = a.gw * a.gh;
    int* cnt = a.cell_cnt + (long long)f * cells;
    int* start = a.cell_start + (long long)f * (cells + 1);
    __shared__ int warp_sum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < cells; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int x = i < cells ? cnt[i] : 0;
        int s = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane == 31) warp_sum[wid] = s;
        __syncthreads();
        if (wid == 0) {
            int w = lane < int(blockDim.x >> 5) ? warp_sum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_sum[lane] = w;
        }
        __syncthreads();
        const int excl = carry + (wid > 0 ? warp_sum[wid - 1] : 0) + s - x;
        if (i < cells) {
            start[i] = excl;
            cnt[i] = excl;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) start[cells] = carry;
}

// column extremes (smallest / largest v; the smallest index on ties, which is
// never a coincident duplicate): candidates for every convex-hull vertex
__global__ void k_col_key(StarArgs a) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int u = a.su[sb + i], v = a.sv[sb + i];
    unsigned long long* key = a.col_key + 2ll * f * a.W;
    atomicMin(key + u, ((unsigned long long)unsigned(v) << 32) | unsigned(i));
    atomicMin(key + a.W + u, ((unsigned long long)unsigned(a.H - 1 - v) << 32) | unsigned(i));
}

__global__ void k_col_decode(StarArgs a) {
    const int f = blockIdx.y;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 2 * a.W) return;
    const unsigned long long k = a.col_key[2ll * f * a.W + c];
    a.col_idx[2ll * f * a.W + c] = k == ~0ull ? -1 : int(k & 0xffffffffu);
}

// The convex hull boundary of each frame, as star_dt.cuh build_hull (the
// same chains, the same candidates in the same order): the block loads the
// column extremes and their rows into shared memory, then one thread runs
// the monotone chains with (u, v, index) stack entries (no dependent global
// loads per step); flags[4] = 1 for a collinear set.
__global__ void k_hull(StarArgs a) {
    const int f = blockIdx.x;
    extern __shared__ int sm[];
    int* s_idx = sm;             // 2W: col_lo then col_hi
    int* s_v = sm + 2 * a.W;     // their rows
    const long long sb = (long long)f * a.scap;
    const int* cols = a.col_idx + 2ll * f * a.W;
    for (int c = threadIdx.x; c < 2 * a.W; c += blockDim.x) {
        const int i = cols[c];
        s_idx[c] = i;
        s_v[c] = i >= 0 ? a.sv[sb + i] : 0;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const star::Grid g = make_grid(a, f);
    const long long ncand = 2ll * a.W + 2ll * a.H + 8;  // column extremes + two whole columns
    int4* lo = reinterpret_cast<int4*>(a.hull_tmp) + 2 * ncand * f;
    int4* hi = lo + ncand;
    int c0 = -1, c1 = -1;
    for (int i = 0; i < a.W; ++i)
        if (s_idx[i] >= 0) {
            if (c0 < 0) c0 = i;
            c1 = i;
        }
    int* hnext = a.hull + 2 * sb;
    int* hprev = hnext + a.scap;
    int* flat = a.flags + (long long)f * kStarFlagInts + 4;
    if (c0 < 0) {
        *flat = 1;
        return;
    }
    int nl = 0, nh = 0;
    auto cross = [](int4 o, int4 b, int x, int y) {
        return (long long)(b.x - o.x) * (y - o.y) - (long long)(b.y - o.y) * (x - o.x);
    };
    auto push = [&](int x, int y, int idx) {
        while (nl >= 2 && cross(lo[nl - 2], lo[nl - 1], x, y) < 0) --nl;
        lo[nl++] = make_int4(x, y, idx, 0);
        while (nh >= 2 && cross(hi[nh - 2], hi[nh - 1], x, y) > 0) --nh;
        hi[nh++] = make_int4(x, y, idx, 0);
    };
    auto whole_column = [&](int x) {  // every point of column x by v (star_dt.cuh)
        const int cx = x / g.gs;
        for (int cy = 0; cy < g.gh; ++cy) {
            const int c = cy * g.gw + cx;
            int last = -2147483647;
            for (;;) {
                int best = -1, bv = 0;
                for (int k = g.cell_start[c]; k < g.cell_start[c + 1]; ++k) {
                    const int s = g.cell_items[k];
                    if (g.u[s] != x || g.dup[s]) continue;
                    const int vs = g.v[s];
                    if (vs <= last) continue;
                    if (best < 0 || vs < bv) {
                        best = s;
                        bv = vs;
                    }
                }
                if (best < 0) break;
                push(x, bv, best);
                last = bv;
            }
        }
    };
    whole_column(c0);
    for (int i = c0 + 1; i < c1; ++i) {
        const int pa = s_idx[i], pb = s_idx[a.W + i];
        if (pa < 0) continue;
        push(i, s_v[i], pa);
        if (pb != pa) push(i, s_v[a.W + i], pb);
    }
    if (c1 != c0) whole_column(c1);
    bool is_flat = nl < 2;
    if (!is_flat) {
        is_flat = true;
        for (int i = 1; i + 1 < nh && is_flat; ++i) is_flat = cross(hi[0], hi[nh - 1], hi[i].x, hi[i].y) == 0;
        for (int i = 1; i + 1 < nl && is_flat; ++i) is_flat = cross(lo[0], lo[nl - 1], lo[i].x, lo[i].y) == 0;
    }
    *flat = is_flat ? 1 : 0;
    if (is_flat) return;
    for (int i = 0; i + 1 < nl; ++i) {
        hnext[lo[i].z] = lo[i + 1].z;
        hprev[lo[i + 1].z] = lo[i].z;
    }
    for (int i = nh - 1; i > 0; --i) {
        hnext[hi[i].z] = hi[i - 1].z;
        hprev[hi[i - 1].z] = hi[i].z;
    }
}

__global__ void k_grid_fill(StarArgs a) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int cell = (a.sv[sb + i] / a.gs) * a.gw + a.su[sb + i] / a.gs;
    const int pos = atomicAdd(a.cell_cnt + (long long)f * a.gw * a.gh + cell, 1);
    a.cell_items[sb + pos] = i;
}

// coincident points: the first occurrence is the vertex; pin choices cleared
__global__ void k_grid_dup(StarArgs a) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int u = a.su[sb + i], v = a.sv[sb + i];
    const int cell = (v / a.gs) * a.gw + u / a.gs;
    const int* start = a.cell_start + (long long)f * (a.gw * a.gh + 1);
    uint8_t d = 0;
    for (int k = start[cell]; k < start[cell + 1]; ++k) {
        const int j = a.cell_items[sb + k];
        if (j < i && a.su[sb + j] == u && a.sv[sb + j] == v) d = 1;
    }
    a.dup[sb + i] = d;
    a.hull[2 * sb + i] = -1;
    a.hull[2 * sb + a.scap + i] = -1;
    int* pt = a.pin_tri + 3 * (sb + i);
    pt[0] = pt[1] = pt[2] = -1;
}

__device__ __forceinline__ void set_fail(const StarArgs& a, int f) { atomicExch(a.flags + (long long)f * kStarFlagInts, 1); }

#ifdef PS_STAR_PROFILE
__device__ unsigned long long g_star_cycles, g_star_max, g_star_n, g_star_hist[24];
__global__ void k_star_report() {
    printf("k_star: %llu points, mean %.0f cycles, max %llu cycles (point %llu)\n", g_star_n,
           double(g_star_cycles) / double(g_star_n > 0 ? g_star_n : 1), g_star_max >> 24, g_star_max & 0xffffff);
    for (int i = 0; i < 24; ++i)
        if (g_star_hist[i]) printf("  2^%d cycles: %llu\n", i, g_star_hist[i]);
    g_star_cycles = g_star_max = g_star_n = 0;
    for (int i = 0; i < 24; ++i) g_star_hist[i] = 0;
}
__device__ void star_clock(long long t0, int p) {
    const unsigned long long c = (unsigned long long)(clock64() - t0);
    atomicAdd(&g_star_cycles, c);
    atomicAdd(&g_star_n, 1ull);
    atomicMax(&g_star_max, (c << 24) | (unsigned long long)(p & 0xffffff));
    int b = 0;
    while (b < 23 && (1ull << (b + 1)) <= c) ++b;
    atomicAdd(&g_star_hist[b], 1ull);
}
#endif

__device__ __forceinline__ void star_body(const StarArgs& a, int f, int p, int radius, int* cand, int cap,
                                          int stride, int* defer_list, int defer_count_slot);

__global__ void __launch_bounds__(kT) k_star(StarArgs a) {
    const int f = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.S[f]) return;
    // threads take the points in grid order: neighbouring threads read the
    // same cells (cache locality) and do similar work (less divergence)
    const int p = a.cell_items[(long long)f * a.scap + t];
    extern __shared__ int s_cand[];
#ifdef PS_STAR_PROFILE
    const long long t0 = clock64();
#endif
    star_body(a, f, p, 2, s_cand, star::kLocalMax, kT, a.hard, 5);
#ifdef PS_STAR_PROFILE
    star_clock(t0, p);
#endif
}

// pass 1b: the points pass 1 deferred, with a 9x9-cell gather (about 100
// candidates); what still needs the grid search goes to the warps
constexpr int kWideT = 64;
constexpr int kWideCap = 160;
__global__ void __launch_bounds__(kWideT) k_star_wide(StarArgs a) {
    const int f = blockIdx.y;
    const int n = min(a.flags[(long long)f * kStarFlagInts + 5], a.scap);
    extern __shared__ int s_cand[];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        star_body(a, f, a.hard[(long long)f * a.scap + t], 4, s_cand, kWideCap, kWideT, a.hard2, 6);
}

// Hull-vertex bookkeeping shared by both passes: whether the vertex pixel is
// covered (tie rule), and whether the incident planes (smallest-first
// rotation) agree on D_it there and are rotation-invariant.
struct HullCheck {
    bool covered = false, agree = true, suspect = false;
    unsigned first_bits = 0;
    int first[3] = {-1, -1, -1};
    int n_inc = 0;
    __device__ void add(const int* su, const int* sv, const double* sd, int hu, int hv, float nd, int t0,
                        int t1, int t2) {
        if (tie_accept(su[t2], sv[t2], hu, hv) && tie_accept(hu, hv, su[t1], sv[t1])) covered = true;
        int x = t0, y = t1, z = t2;
        min_first(x, y, z);
        const Fit f0 = fit3(su, sv, sd, x, y, z);
        const Fit f1 = fit3(su, sv, sd, y, z, x), f2 = fit3(su, sv, sd, z, x, y);
        if (!same_bits(f0, f1) || !same_bits(f0, f2)) suspect = true;
        const unsigned bits = dit_bits(f0, hu, hv, nd);
        if (n_inc == 0) {
            first_bits = bits;
            first[0] = x;
            first[1] = y;
            first[2] = z;
        } else if (bits != first_bits) {
            agree = false;
        }
        ++n_inc;
    }
};

// After a hull vertex's check: pin it here, or list it (and its fan, written
// by `write_fan(out)`) for the host.
template <class W>
__device__ void hull_outcome(const StarArgs& a, int f, int p, const HullCheck& h, W&& write_fan) {
    const long long sb = (long long)f * a.scap;
    const int hu = a.su[sb + p], hv = a.sv[sb + p];
    if (h.covered || h.n_inc == 0 || hu < 0 || hu >= a.W || hv < 0 || hv >= a.H) return;
    if (h.agree && !h.suspect) {
        int s0 = h.first[0], s1 = h.first[1], s2 = h.first[2];
        if (s0 > s1) { const int t = s0; s0 = s1; s1 = t; }
        if (s1 > s2) { const int t = s1; s1 = s2; s2 = t; }
        if (s0 > s1) { const int t = s0; s0 = s1; s1 = t; }
        int* pt = a.pin_tri + 3 * (sb + p);
        pt[0] = s0;
        pt[1] = s1;
        pt[2] = s2;
        return;
    }
    int* fl = a.flags + (long long)f * kStarFlagInts;
    const int need = 2 + 3 * h.n_inc;
    const int at = atomicAdd(fl + 2, need);
    if (kStarFanBase + at + need > kStarFlagInts) {
        set_fail(a, f);
        return;
    }
    atomicAdd(fl + 3, 1);
    int* w = fl + kStarFanBase + at;
    w[0] = p;
    w[1] = h.n_inc;
    write_fan(w + 2);
}

constexpr int kBudget = 8;   // grid searches a thread may do before handing p to a warp
constexpr int kEmitBuf = 12;  // triangles a thread may hold before writing them

__device__ __forceinline__ void star_body(const StarArgs& a, int f, int p, int radius, int* cand, int cap,
                                          int stride, int* defer_list, int defer_count_slot) {
    const star::Grid g = make_grid(a, f);
    const long long sb = (long long)f * a.scap;
    const int* su = a.su + sb;
    const int* sv = a.sv + sb;
    const double* sd = a.sd + sb;
    bool closed;
    // candidates in shared memory, the block's threads interleaved
    star::Local L;
    L.idx = cand + threadIdx.x;
    L.dxy = cand + cap * stride + threadIdx.x;
    L.stride = stride;
    L.cap = cap;
    star::gather(g, p, radius, L);
    // the triangles this point writes (it is their smallest vertex), held
    // until the star is known to be complete within the search budget
    int buf[3 * kEmitBuf];
    int nbuf = 0;
    bool overflow = false;
    const int r = star::walk_star(g, L, p, closed, [&](int t0, int t1, int t2) {
        if (t0 < t1 && t0 < t2) {
            if (nbuf == kEmitBuf) {
                overflow = true;
            } else {
                buf[3 * nbuf] = t0;
                buf[3 * nbuf + 1] = t1;
                buf[3 * nbuf + 2] = t2;
                ++nbuf;
            }
        }
    }, a.budget);
    if (r == -2) {
        set_fail(a, f);
        return;
    }
    HullCheck h;
    bool defer = r == -4 || overflow;
    if (!defer && !closed && r > 0) {
        // a hull vertex: the bookkeeping walk (within the same budget)
        const int hu = su[p], hv = sv[p];
        const int r2 = star::walk_star(g, L, p, closed, [&](int t0, int t1, int t2) {
            h.add(su, sv, sd, hu, hv, a.max_disp, t0, t1, t2);
        }, a.budget);
        defer = r2 == -4;
    }
    if (defer) {  // beyond this pass: a wider gather (k_star_wide), then a warp (k_star_hard)
        int* fl = a.flags + (long long)f * kStarFlagInts;
        const int k = atomicAdd(fl + defer_count_slot, 1);
        if (k < a.scap) defer_list[sb + k] = p;
        return;
    }
    if (nbuf > 0) {
        const int slot = atomicAdd(a.tri_count + f, nbuf);
        int* tris = a.tris + 3 * (long long)f * a.pitch;
        for (int i = 0; i < nbuf; ++i)
            if (slot + i < a.pitch) {
                tris[3 * (long long)(slot + i)] = buf[3 * i];
                tris[3 * (long long)(slot + i) + 1] = buf[3 * i + 1];
                tris[3 * (long long)(slot + i) + 2] = buf[3 * i + 2];
            }
    }
    if (closed || r == 0) return;
    hull_outcome(a, f, p, h, [&](int* out) {
        int k = 0;
        star::walk_star(g, L, p, closed, [&](int t0, int t1, int t2) {
            if (k < h.n_inc) {
                out[3 * k] = t0;
                out[3 * k + 1] = t1;
                out[3 * k + 2] = t2;
            }
            ++k;
        });
    });
}

// ---- pass 2: one warp per deferred point.  The same searches with the
// candidates of a box or a disc spread over the lanes, and the winner chosen
// by a shuffle tournament under the perturbed in-circle order (a strict total
// order on the candidates, so both lanes of a pair pick the same winner).

__device__ __forceinline__ bool w_better(const star::Grid& g, int p, int q, int side, int a, int b) {
    return side > 0 ? star::inside(g, p, q, a, b) : star::inside(g, p, a, q, b);
}

__device__ __forceinline__ int w_reduce(const star::Grid& g, int p, int q, int side, int best) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int other = __shfl_xor_sync(0xffffffffu, best, o);
        if (other >= 0 && (best < 0 || w_better(g, p, q, side, best, other))) best = other;
    }
    return best;
}

__device__ int w_next(const star::Grid& g, int p, int q, int side) {
    // star_dt.cuh next_neighbour with the cells of each ring / row chord
    // spread over the lanes and a tournament after each phase
    if (star::hull_edge(g, p, q, side)) return -1;
    const int lane = threadIdx.x & 31;
    int lbest = -1;
    auto consider = [&](int s) {
        if (s == p || s == q || g.dup[s]) return;
        const long long o = star::orient(g, p, q, s);
        if (side > 0 ? o <= 0 : o >= 0) return;
        if (lbest < 0 || w_better(g, p, q, side, lbest, s)) lbest = s;
    };
    const int pcx = star::cell_x(g, g.u[p]), pcy = star::cell_y(g, g.v[p]);
    const int qcx = star::cell_x(g, g.u[q]), qcy = star::cell_y(g, g.v[q]);
    // rings 0..2 around p and q: a (2k+1)^2 square each, lanes over its cells
    int best = -1;
    for (int o = 0; o < 2; ++o) {
        const int ox = o == 0 ? pcx : qcx, oy = o == 0 ? pcy : qcy;
        for (int c = lane; c < 25; c += 32) {
            const int cx = ox + c % 5 - 2, cy = oy + c / 5 - 2;
            if (cx < 0 || cy < 0 || cx >= g.gw || cy >= g.gh) continue;
            const int cell = cy * g.gw + cx;
            for (int i = g.cell_start[cell]; i < g.cell_start[cell + 1]; ++i) consider(g.cell_items[i]);
        }
    }
    best = w_reduce(g, p, q, side, lbest);
    if (best < 0) {  // a far point from the column extremes
        const int cols = g.maxx - g.minx + 1;
        for (int i = lane; i < cols; i += 32) {
            if (g.col_lo[i] >= 0) consider(g.col_lo[i]);
            if (g.col_hi[i] >= 0) consider(g.col_hi[i]);
        }
        best = w_reduce(g, p, q, side, lbest);
        if (best < 0) return -2;
    }
    lbest = best;
    star::Disc d = side > 0 ? star::disc_of(g, p, q, best) : star::disc_of(g, p, best, q);
    auto read = [&](int cx, int cy) {
        return (cx >= pcx - 2 && cx <= pcx + 2 && cy >= pcy - 2 && cy <= pcy + 2) ||
               (cx >= qcx - 2 && cx <= qcx + 2 && cy >= qcy - 2 && cy <= qcy + 2);
    };
    for (int t = 0;; ++t) {
        bool any = false;
        for (int sgn = 0; sgn < 2; ++sgn) {
            if (t == 0 && sgn == 1) continue;
            const int cy = sgn == 0 ? pcy + t : pcy - t;
            if (cy < 0 || cy >= g.gh) continue;
            const double ya = g.miny + double(cy) * g.gs, yb = ya + g.gs - 1;
            const double dy = d.cy < ya ? ya - d.cy : (d.cy > yb ? d.cy - yb : 0.0);
            if (dy > d.r) continue;
            any = true;
            const double half = sqrt(d.r * d.r - dy * dy);
            const int x0 = star::cell_x(g, d.cx - half), x1 = star::cell_x(g, d.cx + half);
            for (int cx = x0 + lane; cx <= x1; cx += 32) {
                if (read(cx, cy)) continue;
                const int cell = cy * g.gw + cx;
                for (int i = g.cell_start[cell]; i < g.cell_start[cell + 1]; ++i) consider(g.cell_items[i]);
            }
            // a tournament only when some lane found a better point
            if (__any_sync(0xffffffffu, lbest != best)) {
                const int nb = w_reduce(g, p, q, side, lbest);
                if (nb != best) {
                    best = nb;
                    d = side > 0 ? star::disc_of(g, p, q, best) : star::disc_of(g, p, best, q);
                }
                lbest = best;
            }
        }
        const double up = g.miny + double(pcy - t) * g.gs, dn = g.miny + double(pcy + t + 1) * g.gs - 1;
        if (!any && (pcy - t < 0 || up - 1 < d.cy - d.r) && (pcy + t >= g.gh || dn + 1 > d.cy + d.r)) break;
        if (pcy - t < 0 && pcy + t >= g.gh) break;
    }
    return best;
}

__device__ int w_nearest(const star::Grid& g, int p) {
    const int lane = threadIdx.x & 31;
    const int px = star::cell_x(g, g.u[p]), py = star::cell_y(g, g.v[p]);
    unsigned long long best = ~0ull;  // (d2 << 32) | index
    const int maxr = max(g.gw, g.gh);
    for (int k = 0; k <= maxr; ++k) {
        const int side = 2 * k + 1;
        for (int c = lane; c < side * side; c += 32) {
            const int dx = c % side - k, dy = c / side - k;
            if (abs(dx) != k && abs(dy) != k) continue;  // the ring only
            const int cx = px + dx, cy = py + dy;
            if (cx < 0 || cy < 0 || cx >= g.gw || cy >= g.gh) continue;
            const int cell = cy * g.gw + cx;
            for (int i = g.cell_start[cell]; i < g.cell_start[cell + 1]; ++i) {
                const int s = g.cell_items[i];
                if (s == p || g.dup[s]) continue;
                const long long ddx = g.u[s] - g.u[p], ddy = g.v[s] - g.v[p];
                const unsigned long long d2 = (unsigned long long)(ddx * ddx + ddy * ddy);
                if (d2 == 0) continue;
                const unsigned long long key = (d2 << 32) | unsigned(s);
                if (key < best) best = key;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
            best = y < best ? y : best;
        }
        if (best != ~0ull && (unsigned long long)((long long)k * g.gs * k * g.gs) >= (best >> 32)) break;
    }
    return best == ~0ull ? -1 : int(best & 0xffffffffu);
}

template <class F>
__device__ int w_walk(const star::Grid& g, int p, bool& closed, F&& on_tri) {
    closed = false;
    if (g.dup[p]) return 0;
    const int q0 = w_nearest(g, p);
    if (q0 < 0) return 0;
    int count = 0, cur = q0;
    for (int guard = 0; guard <= g.n; ++guard) {
        const int r = w_next(g, p, cur, +1);
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
    for (int guard = 0; guard <= g.n; ++guard) {
        const int r = w_next(g, p, cur, -1);
        if (r == -2) return -2;
        if (r < 0) break;
        on_tri(p, r, cur);
        ++count;
        cur = r;
    }
    return count;
}

__global__ void k_star_hard(StarArgs a) {
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int nhard = min(a.flags[(long long)f * kStarFlagInts + 6], a.scap);
    const int warps = gridDim.x * (blockDim.x >> 5);
    const star::Grid g = make_grid(a, f);
    const long long sb = (long long)f * a.scap;
    const int* su = a.su + sb;
    const int* sv = a.sv + sb;
    const double* sd = a.sd + sb;
    int* tris = a.tris + 3 * (long long)f * a.pitch;
    for (int h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); h < nhard; h += warps) {
        const int p = a.hard2[sb + h];
        bool closed;
        HullCheck hc;  // kept on the fly: one walk serves both purposes
        const int hu = su[p], hv = sv[p];
        const int r = w_walk(g, p, closed, [&](int t0, int t1, int t2) {
            if (lane == 0 && t0 < t1 && t0 < t2) {
                const int slot = atomicAdd(a.tri_count + f, 1);
                if (slot < a.pitch) {
                    tris[3 * (long long)slot] = t0;
                    tris[3 * (long long)slot + 1] = t1;
                    tris[3 * (long long)slot + 2] = t2;
                }
            }
            hc.add(su, sv, sd, hu, hv, a.max_disp, t0, t1, t2);
        });
        if (r == -2) {
            if (lane == 0) set_fail(a, f);
            continue;
        }
        if (closed || r == 0) continue;
        // the fan, if needed, is written by a third walk (rare)
        bool need_fan = !hc.covered && !(hc.agree && !hc.suspect) && hc.n_inc > 0 && hu >= 0 && hu < a.W &&
                        hv >= 0 && hv < a.H;
        int* fan = nullptr;
        if (lane == 0) {
            hull_outcome(a, f, p, hc, [&](int* out) { fan = out; });
        }
        if (need_fan) {
            fan = (int*)__shfl_sync(0xffffffffu, (unsigned long long)fan, 0);
            int k = 0;
            w_walk(g, p, closed, [&](int t0, int t1, int t2) {
                if (lane == 0 && fan && k < hc.n_inc) {
                    fan[3 * k] = t0;
                    fan[3 * k + 1] = t1;
                    fan[3 * k + 2] = t2;
                }
                ++k;
            });
        }
    }
}

// rotation check: a triangle whose three rotations fit different planes is
// listed (index + vertices) for the host
__global__ void k_tri_check(StarArgs a) {
    const int f = blockIdx.y;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = min(a.tri_count[f], int(a.pitch));
    if (t >= n) return;
    const long long sb = (long long)f * a.scap;
    const int* tr = a.tris + 3 * ((long long)f * a.pitch + t);
    const int i = tr[0], j = tr[1], k = tr[2];
    const int* su = a.su + sb;
    const int* sv = a.sv + sb;
    const double* sd = a.sd + sb;
    const double d1 = sd[i], d2 = sd[j], d3 = sd[k];
    // integer disparities: every product and sum is exact, any rotation
    if (d1 == floor(d1) && d2 == floor(d2) && d3 == floor(d3)) return;
    const Fit f0 = fit3(su, sv, sd, i, j, k), f1 = fit3(su, sv, sd, j, k, i), f2 = fit3(su, sv, sd, k, i, j);
    if (same_bits(f0, f1) && same_bits(f0, f2)) return;
    int* fl = a.flags + (long long)f * kStarFlagInts;
    const int s = atomicAdd(fl + 1, 1);
    if (s >= kStarMaxSuspect) {
        set_fail(a, f);
        return;
    }
    int* w = fl + kStarSuspectBase + 4 * s;
    w[0] = int(t);
    w[1] = i;
    w[2] = j;
    w[3] = k;
}

// host fixes: rotation overrides (triangle index -> vertex order) and pin
// choices (vertex -> vertex set); fix = {frame, kind, a, b, c, d}
__global__ void k_apply_fixes(StarArgs a, const int* fixes, int n_fix) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_fix) return;
    const int* x = fixes + 6 * i;
    const int f = x[0];
    if (x[1] == 0) {  // rotation: triangle x[2] stored as (x[3], x[4], x[5])
        int* tr = a.tris + 3 * ((long long)f * a.pitch + x[2]);
        tr[0] = x[3];
        tr[1] = x[4];
        tr[2] = x[5];
    } else {  // pin: vertex x[2] pinned to the triangle with vertex set {x[3], x[4], x[5]} (sorted)
        int* pt = a.pin_tri + 3 * ((long long)f * a.scap + x[2]);
        pt[0] = x[3];
        pt[1] = x[4];
        pt[2] = x[5];
    }
}

__global__ void k_pin_bits(StarArgs a) {
    const int f = blockIdx.y;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = min(a.tri_count[f], int(a.pitch));
    if (t >= n) return;
    const long long sb = (long long)f * a.scap;
    const int* tr = a.tris + 3 * ((long long)f * a.pitch + t);
    int v[3] = {tr[0], tr[1], tr[2]};
    int s0 = v[0], s1 = v[1], s2 = v[2];
    if (s0 > s1) { const int q = s0; s0 = s1; s1 = q; }
    if (s1 > s2) { const int q = s1; s1 = s2; s2 = q; }
    if (s0 > s1) { const int q = s0; s0 = s1; s1 = q; }
    unsigned bits = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int* pt = a.pin_tri + 3 * (sb + v[k]);
        if (pt[0] == s0 && pt[1] == s1 && pt[2] == s2) bits |= 1u << k;
    }
    a.pins[(long long)f * a.pitch + t] = uint8_t(bits);
}

}  // namespace

#ifdef PS_STAR_SYNC_DEBUG
#define STAR_CHECK(name)                                                                        \
    do {                                                                                        \
        cudaError_t e_ = cudaStreamSynchronize(st);                                             \
        if (e_ == cudaSuccess) e_ = cudaGetLastError();                                         \
        if (e_ != cudaSuccess) printf("star: %s failed: %s\n", name, cudaGetErrorString(e_));   \
    } while (0)
#else
#define STAR_CHECK(name)
#endif

int launch_star_mesh(const StarArgs& a, int max_points, cudaStream_t st) {
    const long long cells = (long long)a.gw * a.gh;
    cudaMemsetAsync(a.cell_cnt, 0, sizeof(int) * cells * a.frames, st);
    cudaMemsetAsync(a.tri_count, 0, sizeof(int) * a.frames, st);
    cudaMemset2DAsync(a.flags, sizeof(int) * kStarFlagInts, 0, sizeof(int) * kStarFanBase, a.frames, st);
    if (max_points <= 0) return 0;
    const dim3 grid((max_points + 255) / 256, a.frames);
    k_grid_count<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_count");
    k_grid_scan<<<a.frames, 1024, 0, st>>>(a); STAR_CHECK("k_grid_scan");
    k_grid_fill<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_fill");
    k_grid_dup<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_dup");
    cudaMemsetAsync(a.col_key, 0xff, sizeof(unsigned long long) * 2 * a.W * a.frames, st);
    k_col_key<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_col_key");
    k_col_decode<<<dim3((2 * a.W + 255) / 256, a.frames), 256, 0, st>>>(a);
    {
        const int hsm = 4 * a.W * int(sizeof(int));
        cudaFuncSetAttribute(k_hull, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
        k_hull<<<a.frames, 256, hsm, st>>>(a);
    } STAR_CHECK("k_hull");
    const int smem = 2 * star::kLocalMax * kT * int(sizeof(int));
    cudaFuncSetAttribute(k_star, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_star<<<dim3((max_points + kT - 1) / kT, a.frames), kT, smem, st>>>(a);
    {
        const int wsm = 2 * kWideCap * kWideT * int(sizeof(int));
        cudaFuncSetAttribute(k_star_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, wsm);
        // deferred points are a few percent: size the grid for 1/8 of them
        k_star_wide<<<dim3((max_points / 8 + kWideT - 1) / kWideT + 1, a.frames), kWideT, wsm, st>>>(a);
    }
    STAR_CHECK("k_star");
    k_star_hard<<<dim3(128, a.frames), 128, 0, st>>>(a); STAR_CHECK("k_star_hard");
#ifdef PS_STAR_PROFILE
    k_star_report<<<1, 1, 0, st>>>();
#endif
    return 9;
}

int launch_star_check(const StarArgs& a, long long max_tris, cudaStream_t st) {
    if (max_tris <= 0) return 0;
    k_tri_check<<<dim3(unsigned((max_tris + 255) / 256), a.frames), 256, 0, st>>>(a);
    return 1;
}

int launch_star_finish(const StarArgs& a, const int* fixes, int n_fix, long long max_tris, cudaStream_t st) {
    int n = 0;
    if (n_fix > 0) {
        k_apply_fixes<<<(n_fix + 255) / 256, 256, 0, st>>>(a, fixes, n_fix);
        ++n;
    }
    if (max_tris > 0) {
        k_pin_bits<<<dim3(unsigned((max_tris + 255) / 256), a.frames), 256, 0, st>>>(a);
        ++n;
    }
    return n;
}

}  // namespace ps
