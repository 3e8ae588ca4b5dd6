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

#include <algorithm>
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
                      a.flags[(long long)f * a.flag_ints + 4], 1.0 / a.gs};
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
// column extremes and their rows into shared memory, then thread 0 runs the
// lower monotone chain and thread 1 the upper one, each over (u, v, index)
// stack entries in shared memory when they fit (no dependent global loads
// per step); flags[4] = 1 for a collinear set.
__device__ __forceinline__ int w_scan(int x) {  // inclusive prefix sum over the warp
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__host__ __device__ inline int hull_stack_entries(int W, int H) { return 2 * W + 2 * H + 8; }
inline size_t hull_smem_bytes(int W, int H, bool stacks) {
    return size_t(4) * W * sizeof(int) + size_t(2) * H * sizeof(int2) +
           (stacks ? size_t(3) * hull_stack_entries(W, H) * sizeof(int2) : 0) + 16;
}

__global__ void k_hull(StarArgs a, int stacks_in_smem) {
    const int f = blockIdx.x;
    extern __shared__ int sm[];
    int* s_idx = sm;                                        // 2W: col_lo then col_hi
    int* s_v = sm + 2 * a.W;                                // their rows
    int2* s_col = reinterpret_cast<int2*>(sm + 4 * a.W);    // 2H: the first / last column's points (v, index)
    __shared__ int s_n[2], s_c[2], s_cnt[2];
    const long long sb = (long long)f * a.scap;
    const int* cols = a.col_idx + 2ll * f * a.W;
    if (threadIdx.x == 0) {
        s_c[0] = 0x7fffffff;
        s_c[1] = -1;
        s_cnt[0] = s_cnt[1] = 0;
    }
    __syncthreads();
    int lo_c = 0x7fffffff, hi_c = -1;
    for (int c = threadIdx.x; c < 2 * a.W; c += blockDim.x) {
        const int i = cols[c];
        s_idx[c] = i;
        s_v[c] = i >= 0 ? a.sv[sb + i] : 0;
        if (c < a.W && i >= 0) {
            lo_c = min(lo_c, c);
            hi_c = max(hi_c, c);
        }
    }
    atomicMin(&s_c[0], lo_c);
    atomicMax(&s_c[1], hi_c);
    __syncthreads();
    const int c0 = s_c[0] == 0x7fffffff ? -1 : s_c[0], c1 = s_c[1];
    const star::Grid g = make_grid(a, f);
    // every point of the first and last columns, by v (star_dt.cuh build_hull):
    // a thread per cell of the column collects its points, sorted within the
    // cell (a column's cells are in v order), then a scan places the cells
    if (c0 >= 0) {
        for (int e = 0; e < (c1 != c0 ? 2 : 1); ++e) {
            const int x = e == 0 ? c0 : c1, cx = x / g.gs;
            // pass 1: counts; pass 2: positions (cells in order, block-strided)
            for (int base = 0; base < g.gh; base += blockDim.x) {
                const int cy = base + threadIdx.x;
                int n = 0;
                int start = 0, stop = 0;
                if (cy < g.gh) {
                    start = g.cell_start[cy * g.gw + cx];
                    stop = g.cell_start[cy * g.gw + cx + 1];
                    for (int k = start; k < stop; ++k) {
                        const int s2 = g.cell_items[k];
                        n += g.u[s2] == x && !g.dup[s2];
                    }
                }
                // block-wide exclusive scan of n (in cell order)
                __shared__ int s_warp[32];
                const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
                int incl = w_scan(n);
                if (lane == 31) s_warp[w] = incl;
                __syncthreads();
                if (w == 0) {
                    int t = lane < int(blockDim.x >> 5) ? s_warp[lane] : 0;
                    t = w_scan(t);
                    s_warp[lane] = t;
                }
                __syncthreads();
                const int off = s_cnt[e] + (w > 0 ? s_warp[w - 1] : 0) + incl - n;
                int2* out = s_col + e * a.H + off;
                int m = 0;
                for (int k = start; k < stop; ++k) {
                    const int s2 = g.cell_items[k];
                    if (g.u[s2] != x || g.dup[s2]) continue;
                    // insertion by v
                    const int vs = g.v[s2];
                    int j = m++;
                    while (j > 0 && out[j - 1].x > vs) {
                        out[j] = out[j - 1];
                        --j;
                    }
                    out[j] = make_int2(vs, s2);
                }
                __syncthreads();
                if (threadIdx.x == 0) s_cnt[e] += s_warp[(blockDim.x >> 5) - 1];
                __syncthreads();
            }
        }
    }
    const long long ncand = hull_stack_entries(a.W, a.H);  // column extremes + two whole columns
    int2* stk = stacks_in_smem ? s_col + 2 * a.H : reinterpret_cast<int2*>(a.hull_tmp) + 4 * ncand * f;
    int2* lo = stk;  // entries ((v << 16) | u, index)
    int2* hi = stk + ncand;
    int2* cand = stk + 2 * ncand;  // the candidates in chain order
    int* hnext = a.hull + 2 * sb;
    int* hprev = hnext + a.scap;
    int* flat = a.flags + (long long)f * a.flag_ints + 4;
    // (1) the candidates in the chains' order: the first column by v, each
    // middle column's low then high extreme (one if they coincide), the last
    // column by v; middle columns placed by a block scan of their counts
    __shared__ int s_base;
    int n_c = 0;
    if (c0 >= 0) {
        const int n0 = s_cnt[0];
        for (int k = threadIdx.x; k < n0; k += blockDim.x)
            cand[k] = make_int2((s_col[k].x << 16) | c0, s_col[k].y);
        if (threadIdx.x == 0) s_base = n0;
        __syncthreads();
        __shared__ int s_wsum[32];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int base = c0 + 1; base < c1; base += blockDim.x) {
            const int i = base + threadIdx.x;
            int pa = -1, pb = -1, cnt = 0;
            if (i < c1) {
                pa = s_idx[i];
                pb = s_idx[a.W + i];
                cnt = pa < 0 ? 0 : (pb != pa ? 2 : 1);
            }
            const int incl = w_scan(cnt);
            if (lane == 31) s_wsum[w] = incl;
            __syncthreads();
            if (w == 0) {
                int t = lane < nw ? s_wsum[lane] : 0;
                t = w_scan(t);
                s_wsum[lane] = t;
            }
            __syncthreads();
            const int at = s_base + (w > 0 ? s_wsum[w - 1] : 0) + incl - cnt;
            if (cnt >= 1) cand[at] = make_int2((s_v[i] << 16) | i, pa);
            if (cnt == 2) cand[at + 1] = make_int2((s_v[a.W + i] << 16) | i, pb);
            __syncthreads();
            if (threadIdx.x == 0) s_base += s_wsum[nw - 1];
            __syncthreads();
        }
        const int n1 = c1 != c0 ? s_cnt[1] : 0;
        const int b1 = s_base;
        for (int k = threadIdx.x; k < n1; k += blockDim.x)
            cand[b1 + k] = make_int2((s_col[a.H + k].x << 16) | c1, s_col[a.H + k].y);
        n_c = b1 + n1;
    }
    __syncthreads();
    // (2) Andrew's chains, chunk-parallel: warp 0 the lower chain, warp 1 the
    // upper; each lane runs the chain over its chunk of the candidates (in
    // place), then lane 0 runs it over the concatenated chunk chains.  A
    // candidate a chunk pops lies strictly inside a segment of two other
    // candidates, so it is off the whole set's chain too: the result is the
    // chain of all candidates.
    if (threadIdx.x < 64 && n_c > 0) {
        const int lane = threadIdx.x & 31;
        const bool upper = threadIdx.x >= 32;
        int2* st = upper ? hi : lo;
        auto cross = [](int2 o, int2 b, int2 c) {
            const int ox = o.x & 0xffff, oy = o.x >> 16, bx = b.x & 0xffff, by = b.x >> 16;
            const int x = c.x & 0xffff, y = c.x >> 16;
            return (long long)(bx - ox) * (y - oy) - (long long)(by - oy) * (x - ox);
        };
        auto pops = [upper](long long c) { return upper ? c > 0 : c < 0; };  // lower: right turn
        const int k0 = int((long long)n_c * lane / 32), k1 = int((long long)n_c * (lane + 1) / 32);
        int n = 0;
        for (int k = k0; k < k1; ++k) {
            const int2 e = cand[k];
            while (n >= 2 && pops(cross(st[k0 + n - 2], st[k0 + n - 1], e))) --n;
            st[k0 + n++] = e;
        }
        const int my_len = n;
        __syncwarp();
        // chunk chain lengths through shared memory
        __shared__ int s_len[2][32];
        s_len[upper ? 1 : 0][lane] = my_len;
        __syncwarp();
        if (lane == 0) {
            int m = 0;
            for (int l = 0; l < 32; ++l) {
                const int l0 = int((long long)n_c * l / 32), ln = s_len[upper ? 1 : 0][l];
                for (int k = 0; k < ln; ++k) {
                    const int2 e = st[l0 + k];  // read position >= write position m
                    while (m >= 2 && pops(cross(st[m - 2], st[m - 1], e))) --m;
                    st[m++] = e;
                }
            }
            s_n[upper ? 1 : 0] = m;
        }
    } else if (threadIdx.x < 2) {
        s_n[threadIdx.x] = 0;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (c0 < 0) {
        *flat = 1;
        return;
    }
    const int nl = s_n[0], nh = s_n[1];
    auto cross = [](int2 o, int2 b, int2 c) {
        const int ox = o.x & 0xffff, oy = o.x >> 16, bx = b.x & 0xffff, by = b.x >> 16;
        const int x = c.x & 0xffff, y = c.x >> 16;
        return (long long)(bx - ox) * (y - oy) - (long long)(by - oy) * (x - ox);
    };
    bool is_flat = nl < 2;
    if (!is_flat) {
        is_flat = true;
        for (int i = 1; i + 1 < nh && is_flat; ++i) is_flat = cross(hi[0], hi[nh - 1], hi[i]) == 0;
        for (int i = 1; i + 1 < nl && is_flat; ++i) is_flat = cross(lo[0], lo[nl - 1], lo[i]) == 0;
    }
    *flat = is_flat ? 1 : 0;
    if (is_flat) return;
    for (int i = 0; i + 1 < nl; ++i) {
        hnext[lo[i].y] = lo[i + 1].y;
        hprev[lo[i + 1].y] = lo[i].y;
    }
    for (int i = nh - 1; i > 0; --i) {
        hnext[hi[i].y] = hi[i - 1].y;
        hprev[hi[i - 1].y] = hi[i].y;
    }
}

__global__ void k_grid_fill(StarArgs a) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int cell = (a.sv[sb + i] / a.gs) * a.gw + a.su[sb + i] / a.gs;
    PS_CHECK(cell >= 0 && cell < a.gw * a.gh);
    const int pos = atomicAdd(a.cell_cnt + (long long)f * a.gw * a.gh + cell, 1);
    PS_CHECK(pos >= 0 && pos < a.S[f]);
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
    if (a.ring) a.ring[(sb + i) * kRingInts] = -1;
    a.hull[2 * sb + a.scap + i] = -1;
    int* pt = a.pin_tri + 3 * (sb + i);
    pt[0] = pt[1] = pt[2] = -1;
}

// the points of each cell run packed for the tiled pass (duplicates -1)
__global__ void k_grid_pack(StarArgs a) {
    const int f = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.S[f]) return;
    const long long sb = (long long)f * a.scap;
    const int s = a.cell_items[sb + k];
    a.cell_xy[sb + k] = a.dup[sb + s] ? -1 : (a.sv[sb + s] << 16) | a.su[sb + s];
}

// flags[0] = 1 sends the frame to the host replay; flags[6] ORs the causes
// (1 fan record full, 2 search failed, 4 star above kFarTris, 8 suspects full)
__device__ __forceinline__ void set_fail(const StarArgs& a, int f, int why) {
    atomicExch(a.flags + (long long)f * a.flag_ints, 1);
    atomicOr(a.flags + (long long)f * a.flag_ints + 6, why);
}

#ifdef PS_STAR_PROFILE
__device__ unsigned long long g_star_cycles, g_star_max, g_star_n, g_star_hist[24];
// pass 2: [0] points [1] gather cycles [2] local steps [3] local cycles [4] row searches
// [5] row cycles [6] rows visited [7] column searches [8] column cycles [9] nearest cycles [10] total cycles
__device__ unsigned long long g_far[12];
__device__ unsigned long long g_far_pt[1 << 16][16];  // per warp slot: this point's counters
#define FAR_PT(i, v) do { if ((threadIdx.x & 31) == 0) g_far_pt[far_slot()][i] += (unsigned long long)(v); } while (0)
__device__ __forceinline__ int far_slot() {
    return int(((blockIdx.y * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) & 0xffff);
}
#define FAR_ADD(i, v) do { if ((threadIdx.x & 31) == 0) { atomicAdd(&g_far[i], (unsigned long long)(v)); g_far_pt[far_slot()][i] += (unsigned long long)(v); } } while (0)
#define FAR_CLOCK() clock64()
__global__ void k_star_report() {
    printf("k_star_far: %llu points, gather %llu cyc, local %llu steps %llu cyc, rows %llu searches %llu cyc %llu rows, cols %llu %llu cyc, nearest %llu cyc, total %llu cyc\n",
           g_far[0], g_far[1], g_far[2], g_far[3], g_far[4], g_far[5], g_far[6], g_far[7], g_far[8], g_far[9], g_far[10]);
    for (int i = 0; i < 12; ++i) g_far[i] = 0;
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
#else
#define FAR_ADD(i, v) do { } while (0)
#define FAR_PT(i, v) do { } while (0)
#define FAR_CLOCK() 0ll
#endif

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
    int* fl = a.flags + (long long)f * a.flag_ints;
    const int need = 2 + 3 * h.n_inc;
    const int at = atomicAdd(fl + 2, need);
    if (a.fan_base + at + need > a.flag_ints) {
        set_fail(a, f, 1);
        return;
    }
    atomicAdd(fl + 3, 1);
    int* w = fl + a.fan_base + at;
    w[0] = p;
    w[1] = h.n_inc;
    write_fan(w + 2);
}


constexpr int kStarTris = 16;  // triangles of one star a pass-1 thread may hold
constexpr int kTileT = 128;
constexpr int kTileCap = 1024;  // points of a tile's region (more: its points go to pass 2)
constexpr int kRegionCells = star::kTileRegion * star::kTileRegion;
static_assert(kRegionCells == 2 * kTileT, "two region cells per thread");

__device__ __forceinline__ void defer_point(const StarArgs& a, int f, int p) {
    const int k = atomicAdd(a.flags + (long long)f * a.flag_ints + 5, 1);
    if (k < a.scap) a.hard[(long long)f * a.scap + k] = p;
}

// p's pass-1 star kept for pass 2: a deferred point walking past p reads
// its next neighbour here instead of searching
__device__ __forceinline__ void keep_star(const StarArgs& a, int f, int p, const int* tb, int nt) {
    if (!a.ring || nt > (kRingInts - 1) / 2) return;
    int* rg = a.ring + ((long long)f * a.scap + p) * kRingInts;
    for (int j = 0; j < 2 * nt; ++j) rg[1 + j] = tb[j];
    rg[0] = nt;
}

// the triangles of p's star that p writes (it is their smallest vertex)
__device__ __forceinline__ void emit_star(const StarArgs& a, int f, int p, const int* tb, int nt) {
    int ne = 0;
    for (int j = 0; j < nt; ++j) ne += p < tb[2 * j] && p < tb[2 * j + 1];
    if (ne == 0) return;
    int slot = atomicAdd(a.tri_count + f, ne);
    PS_CHECK(nt >= 0 && nt <= kStarTris && p >= 0 && p < a.S[f]);
    int* tris = a.tris + 3 * (long long)f * a.pitch;
    for (int j = 0; j < nt; ++j)
        if (p < tb[2 * j] && p < tb[2 * j + 1]) {
            if (slot < a.pitch) {
                tris[3 * (long long)slot] = p;
                tris[3 * (long long)slot + 1] = tb[2 * j];
                tris[3 * (long long)slot + 2] = tb[2 * j + 1];
            }
            ++slot;
        }
}

// a star's outcome: deferred to pass 2 (nt < 0), else its triangles, its
// ring entry and, for a hull vertex, the hull bookkeeping
__device__ __noinline__ void finish_star(const StarArgs& a, int f, int p, int pu, int pv, const int* tb, int nt,
                                         bool closed) {
    if (nt < 0) {
        defer_point(a, f, p);
        return;
    }
    emit_star(a, f, p, tb, nt);
    keep_star(a, f, p, tb, nt);
    if (closed || nt == 0) return;
    const long long sb = (long long)f * a.scap;
    const int* su = a.su + sb;
    const int* sv = a.sv + sb;
    const double* sd = a.sd + sb;
    HullCheck h;
    for (int j = 0; j < nt; ++j) h.add(su, sv, sd, pu, pv, a.max_disp, p, tb[2 * j], tb[2 * j + 1]);
    hull_outcome(a, f, p, h, [&](int* out) {
        for (int j = 0; j < nt; ++j) {
            out[3 * j] = p;
            out[3 * j + 1] = tb[2 * j];
            out[3 * j + 2] = tb[2 * j + 1];
        }
    });
}

// Pass 1, one block per tile of kTileCells^2 cells: the tile's region
// (star_dt.cuh Tile: the tile plus a kTileHalo-cell halo) is staged in
// shared memory, then one thread per point of the tile walks its star from
// it (radius 2, else 4) into a buffer; the triangles it writes, its hull
// bookkeeping and, rarely, its fan all come from that buffer.  A point whose
// star needs a wider search (about 1% at BASELINE config 2's last iteration:
// next to holes and along the hull) or has more than kStarTris triangles is
// listed for pass 2.
#ifndef PS_KSTAR_MINB
#define PS_KSTAR_MINB 6  // resident blocks per SM (80 registers; 8 / 64: +7% time)
#endif
__global__ void __launch_bounds__(kTileT, PS_KSTAR_MINB) k_star(StarArgs a) {
    __shared__ int s_start[kRegionCells + 1];
    __shared__ int s_xy[kTileCap], s_id[kTileCap];
    __shared__ int s_warp[kTileT / 32];
    __shared__ int s_list[kTileT], s_nlist;
    __shared__ int s_near[star::kNearCap * kTileT];  // each thread's near set (star_dt.cuh), strided
    const int f = blockIdx.y;
    const int tw = (a.gw + star::kTileCells - 1) / star::kTileCells;
    const int cx0 = (blockIdx.x % tw) * star::kTileCells - star::kTileHalo;
    const int cy0 = (blockIdx.x / tw) * star::kTileCells - star::kTileHalo;
    const long long sb = (long long)f * a.scap;
    const int* cs = a.cell_start + (long long)f * (a.gw * a.gh + 1);
    const int* cxy = a.cell_xy + sb;
    const int* ci = a.cell_items + sb;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // region cells 2t and 2t + 1: their non-duplicate points
    int r0[2], r1[2], cnt[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int c = 2 * threadIdx.x + k;
        const int gx = cx0 + c % star::kTileRegion, gy = cy0 + c / star::kTileRegion;
        r0[k] = r1[k] = cnt[k] = 0;
        if (gx >= 0 && gy >= 0 && gx < a.gw && gy < a.gh) {
            r0[k] = cs[gy * a.gw + gx];
            r1[k] = cs[gy * a.gw + gx + 1];
            for (int i = r0[k]; i < r1[k]; ++i) cnt[k] += cxy[i] != -1;
        }
    }
    const int mine = cnt[0] + cnt[1];
    int incl = w_scan(mine);
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    for (int w = 0; w < wid; ++w) incl += s_warp[w];
    const int total = s_warp[0] + s_warp[1] + s_warp[2] + s_warp[3];
    int at = incl - mine;
    s_start[2 * threadIdx.x] = at;
    s_start[2 * threadIdx.x + 1] = at + cnt[0];
    if (threadIdx.x == 0) {
        s_start[kRegionCells] = total;
        s_nlist = 0;
    }
    if (total <= kTileCap) {
        const int ox = cx0 * a.gs, oy = cy0 * a.gs;
#pragma unroll
        for (int k = 0; k < 2; ++k)
            for (int i = r0[k]; i < r1[k]; ++i) {
                const int w = cxy[i];
                if (w == -1) continue;
                s_xy[at] = (((w >> 16) - oy) << 16) | ((w & 0xffff) - ox);
                s_id[at] = ci[i];
                ++at;
            }
    }
    __syncthreads();
    const star::Grid g = make_grid(a, f);
    const star::Tile T{s_start, s_xy, s_id, cx0, cy0};
    // the tile's points: row y's entries from row_at[y], row_len[y] of them
    int n_inner = 0;
    int row_at[star::kTileCells], row_len[star::kTileCells];
#pragma unroll
    for (int y = 0; y < star::kTileCells; ++y) {
        const int c = (star::kTileHalo + y) * star::kTileRegion + star::kTileHalo;
        row_at[y] = s_start[c];
        row_len[y] = s_start[c + star::kTileCells] - row_at[y];
        n_inner += row_len[y];
    }
    // the region's entry i as p's walk state
    auto point_at = [&](int i) {
        star::TilePoint P;
        const int w = s_xy[i];
        P.p = s_id[i];
        P.pxr = w & 0xffff;
        P.pyr = w >> 16;
        P.pcx = cx0 + P.pxr / a.gs;
        P.pcy = cy0 + P.pyr / a.gs;
        P.pu = cx0 * a.gs + P.pxr;
        P.pv = cy0 * a.gs + P.pyr;
        P.hprev = g.hprev[P.p];
        P.hnext = g.hnext[P.p];
        return P;
    };
    // phase 1: radius 2; the points needing more, and the hull vertices
    // (their bookkeeping is heavy), are listed for phase 2 so a warp's
    // threads stay on the common path together
    for (int k = threadIdx.x; k < n_inner; k += kTileT) {
        int y = 0, kk = k;
        while (kk >= row_len[y]) kk -= row_len[y++];
        const int i = row_at[y] + kk;
        if (total > kTileCap) {  // an overfull region: the tile's points go to pass 2
            // (entries were not written: find the kk-th non-duplicate point of the row)
            const int gy = cy0 + star::kTileHalo + y;
            int left = kk;
            for (int gx = cx0 + star::kTileHalo; gx < cx0 + star::kTileHalo + star::kTileCells && gx < a.gw; ++gx)
                for (int j = cs[gy * a.gw + gx]; j < cs[gy * a.gw + gx + 1]; ++j)
                    if (cxy[j] != -1 && left-- == 0) defer_point(a, f, ci[j]);
            continue;
        }
        const star::TilePoint P = point_at(i);
        int tb[2 * kStarTris];  // (b, c) of each triangle (p, b, c), walk order
        bool closed;
        star::Near N{s_near + threadIdx.x, kTileT, -1, 0};
        if (a.near && !star::near_build(g, T, P, N)) N.n = -1;
        const int nt = star::tile_walk_near(g, T, P, N, closed, tb, kStarTris);
        if (nt == -4 && a.phase2 == 2) {  // radius 4 right away (PS_STAR_PHASE2=2)
            const int nt4 = star::tile_walk(g, T, P, 4, closed, tb, kStarTris);
            finish_star(a, f, P.p, P.pu, P.pv, tb, nt4, closed);
            continue;
        }
        if (nt == -4 || (a.hull_late && nt > 0 && !closed)) {
            // radius 4 / hull bookkeeping: in this block (phase 2, a thread per
            // point) or, PS_STAR_PHASE2=0, in pass 2 (a warp per point)
            if (a.phase2) {
                const int at2 = atomicAdd(&s_nlist, 1);
                if (at2 < kTileT) s_list[at2] = i;
                else defer_point(a, f, P.p);
            } else {
                defer_point(a, f, P.p);
            }
            continue;
        }
        finish_star(a, f, P.p, P.pu, P.pv, tb, nt, closed);
    }
    __syncthreads();
    // phase 2: radius 4, hull bookkeeping
    const int nl = min(s_nlist, kTileT);
    for (int k = threadIdx.x; k < nl; k += kTileT) {
        const star::TilePoint P = point_at(s_list[k]);
        int tb[2 * kStarTris];
        bool closed;
        const int nt = star::tile_walk(g, T, P, 4, closed, tb, kStarTris);
        finish_star(a, f, P.p, P.pu, P.pv, tb, nt, closed);
    }
}

// ---- pass 2: one warp per deferred point.  The warp gathers the 9x9 cells
// around p into shared memory (about 100 points, three or four per lane);
// each search is a lane-parallel scan of them under the pencil order
// (star_dt.cuh Pencil) and a shuffle tournament, certified like pass 1's.
// Only a winner whose circle leaves the gathered box continues on the grid:
// the rows of its circle on the search side of p -> q, outside the box.

constexpr int kFarT = 128;      // 4 warps per block
constexpr int kFarR = 4;        // gather radius in cells
constexpr int kFarCap = 256;    // gathered points per warp
constexpr int kFarTris = 640;   // triangles of one star (more: the frame is replayed on the host)

struct WLocal {
    const unsigned long long* ckey;  // the frame's column-extreme keys (k_col_key): lo [0, W), hi [W, 2W)
    const int* ring;                 // the frame's pass-1 stars (StarArgs::ring), nullptr: none
    int n;
    bool complete;
    star::Box box;
    int* idx;
    int* dxy;  // (dy << 16) | (dx & 0xffff) relative to p; 0 for p and duplicates
};


__device__ void w_gather(const star::Grid& g, int p, WLocal& L) {
    const int lane = threadIdx.x & 31;
    const int px = star::cell_x(g, g.u[p]), py = star::cell_y(g, g.v[p]);
    L.box = star::Box{max(px - kFarR, 0), max(py - kFarR, 0), min(px + kFarR, g.gw - 1), min(py + kFarR, g.gh - 1)};
    const int bw = L.box.x1 - L.box.x0 + 1, cells = bw * (L.box.y1 - L.box.y0 + 1);
    // lane l takes cells l, l + 32, l + 64 (<= 81)
    int cnt[3], first[3];
    int total = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int c = lane + 32 * k;
        cnt[k] = 0;
        first[k] = 0;
        if (c < cells) {
            const int cell = (L.box.y0 + c / bw) * g.gw + L.box.x0 + c % bw;
            first[k] = g.cell_start[cell];
            cnt[k] = g.cell_start[cell + 1] - first[k];
        }
        total += cnt[k];
    }
    const int incl = w_scan(total);
    L.n = __shfl_sync(0xffffffffu, incl, 31);
    L.complete = L.n <= kFarCap && g.maxx - g.minx < 4096 && g.maxy - g.miny < 4096;
    if (!L.complete) return;
    int at = incl - total;
    const int pu = g.u[p], pv = g.v[p];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int i = 0; i < cnt[k]; ++i, ++at) {
            const int s = g.cell_items[first[k] + i];
            L.idx[at] = s;
            L.dxy[at] = g.dup[s] ? 0 : ((g.v[s] - pv) << 16) | ((g.u[s] - pu) & 0xffff);
        }
    __syncwarp();
}

// the shuffle tournament over (position, num, den) under the pencil order;
// ties (cocircular) by the exact perturbed rule on the point indices
__device__ __forceinline__ int w_tournament(const star::Grid& g, const WLocal& L, int p, int q, int side, int bi,
                                            int bnum, int bden) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int on = __shfl_xor_sync(0xffffffffu, bnum, o);
        const int od = __shfl_xor_sync(0xffffffffu, bden, o);
        if (oi < 0 || oi == bi) continue;
        bool take = bi < 0;
        if (!take) {
            const long long l = (long long)on * bden, r = (long long)bnum * od;
            if (l == r) {
                const int s = L.idx[oi], b = L.idx[bi];
                take = side > 0 ? star::inside(g, p, q, b, s) : star::inside(g, p, b, q, s);
            } else {
                take = side > 0 ? l < r : l > r;
            }
        }
        if (take) {
            bi = oi;
            bnum = on;
            bden = od;
        }
    }
    return bi;
}

// Local next neighbour over the warp: the winner if certified, -1 hull edge,
// -3 otherwise with `start` = the local winner (or -1: none on that side).
__device__ int w_next_local(const star::Grid& g, const WLocal& L, int p, int q, int side, int& start) {
    start = -1;
    if (star::hull_edge(g, p, q, side)) return -1;
    if (!L.complete) return -3;
    const int lane = threadIdx.x & 31;
    const int qx = g.u[q] - g.u[p], qy = g.v[q] - g.v[p];
    int bi = -1, bnum = 0, bden = 0;
    for (int i = lane; i < L.n; i += 32) {
        const int w = L.dxy[i];
        const int sx = int(short(w & 0xffff)), sy = w >> 16;
        const int den = qx * sy - qy * sx;
        if (side > 0 ? den <= 0 : den >= 0) continue;
        const int num = sx * (sx - qx) + sy * (sy - qy);
        if (bi >= 0) {
            const long long l = (long long)num * bden, r = (long long)bnum * den;
            if (l == r) {
                const int s = L.idx[i], b = L.idx[bi];
                if (!(side > 0 ? star::inside(g, p, q, b, s) : star::inside(g, p, b, q, s))) continue;
            } else if (side > 0 ? l > r : l < r) {
                continue;
            }
        }
        bi = i;
        bnum = num;
        bden = den;
    }
    bi = w_tournament(g, L, p, q, side, bi, bnum, bden);
    if (bi < 0) return -3;
    const int w = L.dxy[bi];
    const double bx = int(short(w & 0xffff)), by = w >> 16;
    const star::Box need = side > 0 ? star::circle_box_rel(g, p, double(qx), double(qy), bx, by)
                                    : star::circle_box_rel(g, p, bx, by, double(qx), double(qy));
    if (star::covers(L.box, need)) return L.idx[bi];
    start = L.idx[bi];
    return -3;
}

__device__ __forceinline__ bool w_better(const star::Grid& g, int p, int q, int side, int b, int s) {
    return side > 0 ? star::inside(g, p, q, b, s) : star::inside(g, p, b, q, s);
}

// the tournament over point indices with their pencil keys (ties: inside())
__device__ __forceinline__ int w_reduce(const star::Grid& g, int p, int q, int side, int best, star::Pencil k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int other = __shfl_xor_sync(0xffffffffu, best, o);
        const long long on = __shfl_xor_sync(0xffffffffu, k.num, o);
        const long long od = __shfl_xor_sync(0xffffffffu, k.den, o);
        if (other < 0 || other == best) continue;
        bool take = best < 0;
        if (!take) {
            const int c = star::pencil_cmp(star::Pencil{on, od}, k, side);
            take = c > 0 || (c == 0 && w_better(g, p, q, side, best, other));
        }
        if (take) {
            best = other;
            k = star::Pencil{on, od};
        }
    }
    return best;
}

// The grid search from a first candidate `best` (one on the search side):
// the cell rows of the search region (star_dt.cuh search_region) outward
// from p's row, 32 rows at a time, one row per lane, each read over the
// chord of the winner's circle at the start of its batch and only on the
// search side of p -> q, the cells of `skip` excluded (already scanned).
// A tournament after each batch; the region only shrinks as the winner
// improves (circles through p and q form a pencil), so the rows read with
// an older circle cover everything a newer one could need.
__device__ __noinline__ int w_rows(const star::Grid& g, int p, int q, int side, int best, const star::Box& skip) {
    const int lane = threadIdx.x & 31;
    const long long qx = (long long)g.u[q] - g.u[p], qy = (long long)g.v[q] - g.v[p];
    auto key = [&](int s) { return star::pencil(qx, qy, (long long)g.u[s] - g.u[p], (long long)g.v[s] - g.v[p]); };
    star::Pencil bk = key(best);
    star::Disc d = side > 0 ? star::disc_of(g, p, q, best) : star::disc_of(g, p, best, q);
    star::Region reg = star::search_region(g, p, q, side, d);
    const int pcy = star::cell_y(g, g.v[p]);
    // batch b reads rows pcy + t for t in [-16 b - 15, -16 b] and [16 b + 1, 16 b + 16] (b = 0: pcy - 15 .. pcy + 16)
    for (int b = 0;; ++b) {
        const int t = lane < 16 ? -16 * b - lane : 16 * b + lane - 15;
        const int cy = pcy + t;
        int lbest = best;
        star::Pencil lk = bk;
        // this lane's row: the item range of its cells over the chord (one
        // contiguous range: a row's cells are consecutive in cell_items);
        // the skip box's cells are filtered per point below
        int i0 = 0, cnt = 0;
        bool in_rows = false;
        const double ya = g.miny + double(cy) * g.gs, yb = ya + g.gs - 1;
        if (cy >= 0 && cy < g.gh && yb >= reg.y0 && ya <= reg.y1) {
            const double dy = d.cy < ya ? ya - d.cy : (d.cy > yb ? d.cy - yb : 0.0);
            if (dy <= d.r) {
                const double half = sqrt(d.r * d.r - dy * dy);
                int x0 = star::cell_x(g, d.cx - half > reg.x0 ? d.cx - half : reg.x0);
                int x1 = star::cell_x(g, d.cx + half < reg.x1 ? d.cx + half : reg.x1);
                if (star::clip_side(g, p, q, side, ya, yb, x0, x1)) {
                    in_rows = cy >= skip.y0 && cy <= skip.y1 && skip.x0 <= skip.x1;
                    i0 = g.cell_start[cy * g.gw + x0];
                    cnt = g.cell_start[cy * g.gw + x1 + 1] - i0;
                }
            }
        }
        // the batch's points over the whole warp (a wide, flat region -- the
        // thin segment along a hull edge -- is one long row: one lane per
        // row would walk it alone)
        const int incl = w_scan(cnt);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int base = 0; base < total; base += 32) {
            const int k = base + lane;
            int owner = 0;  // the lane whose range holds item k: #lanes with incl <= k
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= k) owner += step;
            }
            const int oi0 = __shfl_sync(0xffffffffu, i0, owner & 31);
            const int oex = __shfl_sync(0xffffffffu, incl - cnt, owner & 31);
            const bool orows = __shfl_sync(0xffffffffu, in_rows, owner & 31);
            if (k >= total) continue;
            const int s = g.cell_items[oi0 + (k - oex)];
            if (s == p || s == q || g.dup[s]) continue;
            if (orows) {
                const int cx = (g.u[s] - g.minx) / g.gs;  // the cell k_grid_fill put it in
                if (cx >= skip.x0 && cx <= skip.x1) continue;
            }
            const star::Pencil ps = key(s);
            if (side > 0 ? ps.den <= 0 : ps.den >= 0) continue;
            const int c = star::pencil_cmp(ps, lk, side);
            if (c < 0 || (c == 0 && !w_better(g, p, q, side, lbest, s))) continue;
            lbest = s;
            lk = ps;
        }
        FAR_ADD(6, 1);
        if (__any_sync(0xffffffffu, lbest != best)) {
            const int nb = w_reduce(g, p, q, side, lbest, lk);
            if (nb != best) {
                best = nb;
                bk = key(best);
                d = side > 0 ? star::disc_of(g, p, q, best) : star::disc_of(g, p, best, q);
                reg = star::search_region(g, p, q, side, d);
            }
        }
        // done when the next batch's rows both ways lie outside the region
        const int up = pcy - 16 * b - 16, dn = pcy + 16 * b + 17;  // nearest rows of batch b + 1
        const bool up_out = up < 0 || g.miny + double(up + 1) * g.gs - 1 < reg.y0;
        const bool dn_out = dn >= g.gh || g.miny + double(dn) * g.gs > reg.y1;
        if (up_out && dn_out) break;
    }
    return best;
}

// No candidate in the gathered box on the search side: a first one from the
// column extremes (nearest columns first), then w_rows.  -2 if none exists.
__device__ int w_next_far(const star::Grid& g, const unsigned long long* ckey, int p, int q, int side,
                           const star::Box& skip) {
    const int lane = threadIdx.x & 31;
    {  // the 5x5 cells around q: in a fan along the hull the next neighbour is
       // next to q.  The seed is the best of them in the pencil order (not
       // just any point on the search side): along a sliver fan its circle is
       // then the thin one through the true neighbour, and the row search
       // below reads a few rows instead of the disc of a far seed.
        const int qcx = star::cell_x(g, g.u[q]), qcy = star::cell_y(g, g.v[q]);
        const long long qx = (long long)g.u[q] - g.u[p], qy = (long long)g.v[q] - g.v[p];
        int lbest = -1;
        star::Pencil lk{0, 0};
        if (lane < 25) {
            const int cx = qcx + lane % 5 - 2, cy = qcy + lane / 5 - 2;
            if (cx >= 0 && cy >= 0 && cx < g.gw && cy < g.gh) {
                const int cell = cy * g.gw + cx;
                for (int i = g.cell_start[cell]; i < g.cell_start[cell + 1]; ++i) {
                    const int s2 = g.cell_items[i];
                    if (s2 == p || s2 == q || g.dup[s2]) continue;
                    const star::Pencil ps =
                        star::pencil(qx, qy, (long long)g.u[s2] - g.u[p], (long long)g.v[s2] - g.v[p]);
                    if (side > 0 ? ps.den <= 0 : ps.den >= 0) continue;
                    if (lbest >= 0) {
                        const int c = star::pencil_cmp(ps, lk, side);
                        if (c < 0 || (c == 0 && !w_better(g, p, q, side, lbest, s2))) continue;
                    }
                    lbest = s2;
                    lk = ps;
                }
            }
        }
        if (__any_sync(0xffffffffu, lbest >= 0)) {
            const int seed = w_reduce(g, p, q, side, lbest, lk);
            FAR_PT(11, 1);
            const long long tr = FAR_CLOCK();
            const int r = w_rows(g, p, q, side, seed, skip);
            FAR_PT(12, FAR_CLOCK() - tr);
            return r;
        }
    }
    // Column extremes nearest first: lanes 0..15 take columns c0 - k, lanes
    // 16..31 c0 + k, four rounds of 16 per side per pass with all their
    // (v, index) keys loaded up front (one memory round trip per 64 columns
    // a side; the keys hold the row, so no dependent coordinate loads).  The
    // seed is the first hit in round order, then lane order, low extreme
    // first -- the same seed as a one-round-at-a-time scan.
    const int cols = g.maxx - g.minx + 1, c0 = g.u[p] - g.minx;
    const int pu = g.u[p], pv = g.v[p];
    const long long qx = g.u[q] - pu, qy = g.v[q] - pv;
    for (int base = 0; base < cols; base += 64) {
        unsigned long long kk[4][2];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int k = base + 16 * r + (lane & 15);
            const int i = lane < 16 ? c0 - k : c0 + k;
            const bool in = i >= 0 && i < cols;
            kk[r][0] = in ? ckey[i] : ~0ull;
            kk[r][1] = in ? ckey[cols + i] : ~0ull;
        }
        int found = -1, fr = 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int k = base + 16 * r + (lane & 15);
            const int i = lane < 16 ? c0 - k : c0 + k;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const unsigned long long key = kk[r][e];
                if (found >= 0 || key == ~0ull) continue;
                const int s = int(key & 0xffffffffu);
                if (s == p || s == q) continue;
                const int sv = e == 0 ? g.miny + int(key >> 32) : g.maxy - int(key >> 32);
                const long long o = qx * (sv - pv) - qy * (g.minx + i - pu);
                if (side > 0 ? o > 0 : o < 0) {
                    found = s;
                    fr = r;
                }
            }
        }
        const int mr = __reduce_min_sync(0xffffffffu, fr);
        FAR_PT(13, 1);
        if (mr < 4) {
            const unsigned m = __ballot_sync(0xffffffffu, fr == mr);
            const int first = __shfl_sync(0xffffffffu, found, __ffs(m) - 1);
            const long long tr = FAR_CLOCK();
            const int r = w_rows(g, p, q, side, first, star::Box{1, 1, 0, 0});
            FAR_PT(14, FAR_CLOCK() - tr);
            return r;
        }
        if (base + 48 >= c0 && base + 48 >= cols - c0) break;
    }
    return -2;
}

__device__ int w_nearest_local(const star::Grid& g, const WLocal& L, int p) {
    if (!L.complete) return -3;
    const int lane = threadIdx.x & 31;
    unsigned long long best = ~0ull;  // (d2 << 32) | index
    for (int i = lane; i < L.n; i += 32) {
        const int w = L.dxy[i];
        const int sx = int(short(w & 0xffff)), sy = w >> 16;
        const unsigned long long d2 = (unsigned long long)(sx * sx + sy * sy);
        if (d2 == 0) continue;
        const unsigned long long key = (d2 << 32) | unsigned(L.idx[i]);
        best = key < best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
    }
    const long long px = g.u[p] - g.minx, py = g.v[p] - g.miny;
    long long m = 1ll << 40;
    if (L.box.x0 > 0) m = min(m, px - (long long)L.box.x0 * g.gs + 1);
    if (L.box.y0 > 0) m = min(m, py - (long long)L.box.y0 * g.gs + 1);
    if (L.box.x1 < g.gw - 1) m = min(m, (long long)(L.box.x1 + 1) * g.gs - px);
    if (L.box.y1 < g.gh - 1) m = min(m, (long long)(L.box.y1 + 1) * g.gs - py);
    if (best == ~0ull) return m >= (1ll << 40) ? -1 : -3;
    return (long long)(best >> 32) < m * m ? int(best & 0xffffffffu) : -3;
}

__device__ __noinline__ int w_nearest(const star::Grid& g, int p) {
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

__device__ __noinline__ int w_step(const star::Grid& g, const WLocal& L, int p, int q, int side) {
    if (L.ring) {
        // q's star from pass 1 holds the triangle after p -> q: (q, r, p)
        // counter-clockwise for side > 0, (q, p, r) for side < 0
        const int* rg = L.ring + (long long)q * kRingInts;
        const int n = rg[0];
        if (n > 0) {
            const int lane = threadIdx.x & 31;
            int r = -1;
            if (lane < n) {
                const int b = rg[1 + 2 * lane], c = rg[2 + 2 * lane];
                if (side > 0 ? c == p : b == p) r = side > 0 ? b : c;
            }
            const unsigned m = __ballot_sync(0xffffffffu, r >= 0);
            FAR_ADD(9, 0);
            if (m) return __shfl_sync(0xffffffffu, r, __ffs(m) - 1);
        }
    }
    int start;
    long long t0 = FAR_CLOCK();
    const int r = w_next_local(g, L, p, q, side, start);
    FAR_ADD(2, 1);
    FAR_ADD(3, FAR_CLOCK() - t0);
    if (r != -3) return r;
    t0 = FAR_CLOCK();
    if (start >= 0) {
        const int x = w_rows(g, p, q, side, start, L.box);
        FAR_ADD(4, 1);
        FAR_ADD(5, FAR_CLOCK() - t0);
        return x;
    }
    const int x = w_next_far(g, L.ckey, p, q, side, L.complete ? L.box : star::Box{1, 1, 0, 0});
    FAR_ADD(7, 1);
    FAR_ADD(8, FAR_CLOCK() - t0);
    return x;
}

// The star of p into tb ((b, c) per triangle (p, b, c): counter-clockwise
// from p's nearest neighbour, then clockwise for a hull vertex).  Returns
// the triangle count, -2 on a failed search, -4 past kFarTris triangles.
__device__ __noinline__ int w_walk(const star::Grid& g, const WLocal& L, int p, bool& closed, int* tb) {
    const int lane = threadIdx.x & 31;
    closed = false;
    if (g.dup[p]) return 0;
    const long long t0 = FAR_CLOCK();
    int q0 = w_nearest_local(g, L, p);
    if (q0 == -3) q0 = w_nearest(g, p);
    FAR_ADD(9, FAR_CLOCK() - t0);
    if (q0 < 0) return 0;
    int count = 0;
    for (int dir = 0; dir < 2; ++dir) {
        const int side = dir == 0 ? +1 : -1;
        int cur = q0;
        for (int guard = 0; guard <= g.n; ++guard) {
            const int r = w_step(g, L, p, cur, side);
            if (r == -2) return -2;
            if (r < 0) break;
            if (count == kFarTris) return -4;
            if (lane == 0) {
                tb[2 * count] = side > 0 ? cur : r;
                tb[2 * count + 1] = side > 0 ? r : cur;
            }
            ++count;
            if (side > 0 && r == q0) {
                closed = true;
                return count;
            }
            cur = r;
        }
    }
    return count;
}

__global__ void __launch_bounds__(kFarT) k_star_far(StarArgs a) {
    __shared__ int s_idx[kFarT / 32][kFarCap], s_dxy[kFarT / 32][kFarCap];
    __shared__ int s_tri[kFarT / 32][2 * kFarTris];  // (b, c) of each triangle (p, b, c), walk order
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n = min(a.flags[(long long)f * a.flag_ints + 5], a.scap);
    const int warps = gridDim.x * (kFarT >> 5);
    const star::Grid g = make_grid(a, f);
    const long long sb = (long long)f * a.scap;
    int* tris = a.tris + 3 * (long long)f * a.pitch;
    WLocal L;
    L.ckey = a.col_key + 2ll * f * a.W;
    L.ring = a.ring ? a.ring + (long long)f * a.scap * kRingInts : nullptr;
    L.idx = s_idx[wid];
    L.dxy = s_dxy[wid];
    int* tb = s_tri[wid];
    for (int h = blockIdx.x * (kFarT >> 5) + wid; h < n; h += warps) {
        const int p = a.hard[sb + h];
        __syncwarp();
#ifdef PS_STAR_PROFILE
        if (lane == 0)
            for (int i = 0; i < 16; ++i) g_far_pt[far_slot()][i] = 0;
#endif
        const long long tg = FAR_CLOCK();
        w_gather(g, p, L);
        FAR_ADD(0, 1);
        FAR_ADD(1, FAR_CLOCK() - tg);
        bool closed;
        const int nt = w_walk(g, L, p, closed, tb);
        FAR_ADD(10, FAR_CLOCK() - tg);
#ifdef PS_STAR_PROFILE
        {
            const long long cyc = FAR_CLOCK() - tg;
            if (lane == 0) {
                atomicMax(&g_star_max, ((unsigned long long)cyc << 24) | (unsigned long long)(p & 0xffffff));
                int b = 0;
                while (b < 23 && (1ll << (b + 1)) <= cyc) ++b;
                atomicAdd(&g_star_hist[b], 1ull);
                if (cyc > 2000000 && atomicAdd(&g_far[11], 1ull) < 40) {
                    const unsigned long long* c = g_far_pt[far_slot()];
                    printf("slow far point f %d p %d (%d,%d) cycles %lld nt %d closed %d gathered %d complete %d hull %d/%d | "
                           "local %llu/%llu cyc rows %llu/%llu cyc (%llu rows) cols %llu/%llu cyc nearest %llu | qfound %llu rows %llu cyc; col rounds %llu rows %llu cyc\n",
                           f, p, g.u[p], g.v[p], cyc, nt, int(closed), L.n, int(L.complete), g.hnext[p], g.hprev[p],
                           c[2], c[3], c[4], c[5], c[6], c[7], c[8], c[9], c[11], c[12], c[13], c[14]);
                }
            }
        }
#endif
        if (nt < 0) {  // a failed search, or more than kFarTris triangles
            if (lane == 0) set_fail(a, f, nt == -4 ? 4 : 2);
            continue;
        }
        __syncwarp();
        // the triangles p writes (it is their smallest vertex): one slot range
        int ne = 0;
        for (int i = lane; i < nt; i += 32) ne += p < tb[2 * i] && p < tb[2 * i + 1];
        const int incl = w_scan(ne);
        int slot = 0;
        if (lane == 31 && incl > 0) slot = atomicAdd(a.tri_count + f, incl);
        slot = __shfl_sync(0xffffffffu, slot, 31) + incl - ne;
        for (int i = lane; i < nt; i += 32)
            if (p < tb[2 * i] && p < tb[2 * i + 1]) {
                if (slot < a.pitch) {
                    tris[3 * (long long)slot] = p;
                    tris[3 * (long long)slot + 1] = tb[2 * i];
                    tris[3 * (long long)slot + 2] = tb[2 * i + 1];
                }
                ++slot;
            }
        if (closed || nt == 0 || lane != 0) continue;
        // a hull vertex: its bookkeeping (lane 0)
        const int* su = a.su + sb;
        const int* sv = a.sv + sb;
        const double* sd = a.sd + sb;
        HullCheck hc;
        for (int i = 0; i < nt; ++i) hc.add(su, sv, sd, su[p], sv[p], a.max_disp, p, tb[2 * i], tb[2 * i + 1]);
        hull_outcome(a, f, p, hc, [&](int* out) {
            for (int i = 0; i < nt; ++i) {
                out[3 * i] = p;
                out[3 * i + 1] = tb[2 * i];
                out[3 * i + 2] = tb[2 * i + 1];
            }
        });
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
    int* fl = a.flags + (long long)f * a.flag_ints;
    const int s = atomicAdd(fl + 1, 1);
    if (s >= a.max_suspect) {
        set_fail(a, f, 8);
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
    cudaMemset2DAsync(a.flags, sizeof(int) * a.flag_ints, 0, sizeof(int) * a.fan_base, a.frames, st);
    if (max_points <= 0) return 0;
    const dim3 grid((max_points + 255) / 256, a.frames);
    k_grid_count<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_count");
    k_grid_scan<<<a.frames, 1024, 0, st>>>(a); STAR_CHECK("k_grid_scan");
    k_grid_fill<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_fill");
    k_grid_dup<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_dup");
    k_grid_pack<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_grid_pack");
    cudaMemsetAsync(a.col_key, 0xff, sizeof(unsigned long long) * 2 * a.W * a.frames, st);
    k_col_key<<<grid, 256, 0, st>>>(a); STAR_CHECK("k_col_key");
    k_col_decode<<<dim3((2 * a.W + 255) / 256, a.frames), 256, 0, st>>>(a);
    {
        // the chains' stacks in shared memory up to 160 KB (VGA: 46 KB)
        const bool stacks = hull_smem_bytes(a.W, a.H, true) <= 160 * 1024;
        const int hsm = int(hull_smem_bytes(a.W, a.H, stacks));
        cudaFuncSetAttribute(k_hull, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
        k_hull<<<a.frames, 256, hsm, st>>>(a, stacks ? 1 : 0);
    } STAR_CHECK("k_hull");
    {
        const int tiles = ((a.gw + star::kTileCells - 1) / star::kTileCells) * ((a.gh + star::kTileCells - 1) / star::kTileCells);
        k_star<<<dim3(tiles, a.frames), kTileT, 0, st>>>(a);
    }
    STAR_CHECK("k_star");
    // deferred points are a few percent: a warp each, the grid strided
    // (the grid strides over the deferred list: ~1-8% of the points, so a
    // warp per 32 points would leave most blocks empty; a warp per ~1k points
    // of the frame, at least 48 blocks, keeps a point per warp at VGA)
    {
        const int per_frame = std::min((max_points / 32 + 3) / 4 + 1, std::max(48, max_points / 1024));
        k_star_far<<<dim3(per_frame, a.frames), kFarT, 0, st>>>(a);
    }
    STAR_CHECK("k_star_far");
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
