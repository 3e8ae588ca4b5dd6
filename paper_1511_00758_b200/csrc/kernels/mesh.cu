// mesh.cu — K5+K6: per-triangle plane fit and exact rasterisation into the
// pixel -> triangle lookup, with hull-vertex pinning.
//
// Replaces the DisparityMesh constructor (proj/src/mesh.cpp:44-56), fitPlane
// (:12-26) and rasterize (:58-123).  One thread per triangle (flat over all
// frames of the batch; a triangle finds its frame by binary search of the
// per-frame offsets):
//   * the thread solves its plane in binary64 in the reference's source order
//     with _rn intrinsics (no FMA);
//   * small triangles (the vast majority after the first iteration: median
//     2x area 3-15 px): the warp deals its 32 triangles' rows to
//     its lanes, 32 rows at a time, each lane computing the exact integer
//     span [lo, hi] of its row with the top-left tie bias (mesh.cpp:75-106),
//     then deals the pixels of those spans, 32 at a time — every lane busy
//     whatever the shapes of the 32 triangles;
//   * large ones are handed to the whole warp, which computes 32 row spans at
//     once (one per lane) and fills each row with coalesced stores; when the
//     mean triangle of a launch covers >= 64 px (the first iteration's mesh)
//     the launch runs one warp per triangle.
// Pinning (mesh.cpp:109-122): an uncovered vertex pixel takes its first
// incident triangle; which (triangle, corner) pairs pin is decided on the host
// from the exact tie rule (pins.cpp) and passed as 3 bits per triangle, so the
// pin is a plain store here (no other triangle writes an uncovered pixel).
// Lookup entries are flat triangle ids, so the per-pixel kernels index the
// flat plane array directly.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

constexpr int kThreads = 256;

// floorDiv / ceilDiv of mesh.cpp:30-40, for 32- or 64-bit operands.
template <class T>
__device__ __forceinline__ T floor_div(T a, T b) {
    T q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}
template <class T>
__device__ __forceinline__ T ceil_div(T a, T b) { return -floor_div<T>(-a, b); }

__device__ __forceinline__ int frame_of(const int* __restrict__ tri_off, int frames, long long t) {
    int lo = 0, hi = frames - 1;  // largest f with tri_off[f] <= t
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(tri_off + mid) <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Exact covered span of row v (mesh.cpp:84-103); false if the row is empty.
template <class Int>
__device__ __forceinline__ bool row_span(const int* x, const int* y, int v, int W, Int& lo, Int& hi) {
    lo = 0;
    hi = W - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3;
        const Int A = Int(y[i] - y[j]);
        const Int bias = ((y[j] < y[i]) || (y[j] == y[i] && x[j] > x[i])) ? 0 : 1;
        const Int K = Int(x[j] - x[i]) * Int(v - y[i]) + Int(y[j] - y[i]) * Int(x[i]);
        if (A > 0) {
            lo = max(lo, ceil_div<Int>(bias - K, A));
        } else if (A < 0) {
            hi = min(hi, floor_div<Int>(K - bias, -A));
        } else if (K < bias) {
            return false;
        }
    }
    return lo <= hi;
}

// floor(m / d) for d > 0 (C division truncates toward zero).
template <class Int>
__device__ __forceinline__ Int floor_div_pos(Int m, Int d) {
    const Int q = m / d;
    return (m - q * d < 0) ? q - 1 : q;
}

// Per-edge constants of the row-span rule (mesh.cpp:84-103) for edge i -> j:
// the edge value at (u, v) is A*u + K(v) with K(v) = dx*v + C, and the pixel
// is covered iff A*u + K >= bias.  With m(v) = K(v) - bias = dx*v + cb and
// F = floor(m / |A|): A > 0 bounds u >= ceil((bias - K) / A) = -F, A < 0
// bounds u <= floor((K - bias) / -A) = F, and A == 0 empties the row iff
// m < 0 — one division per edge and row, no branches on the edge kind.
template <class Int>
struct EdgeConst {
    Int a, dx, cb;
    double rd;  // 1 / max(|a|, 1): floor(m / |a|) by one multiply (32-bit operands)
    __device__ __forceinline__ void init(int xi, int yi, int xj, int yj) {
        a = Int(yi - yj);
        const Int bias = ((yj < yi) || (yj == yi && xj > xi)) ? 0 : 1;
        dx = Int(xj - xi);
        cb = Int(yj - yi) * Int(xi) - dx * Int(yi) - bias;
        const Int d = a > 0 ? a : (a < 0 ? -a : Int(1));
        rd = __drcp_rn(double(d));
    }
};

// floor(m / d), d > 0.  For 32-bit operands (|m| < 2^31, d < 2^14) the double
// product m * RN(1/d) is within 2^-21 of m / d, so its floor is off by at most
// one, only next to an exact quotient; one remainder test corrects it.
template <class Int>
__device__ __forceinline__ Int floor_div_rcp(Int m, Int d, double rd) {
    if constexpr (sizeof(Int) == 4) {
        Int q = Int(floor(double(m) * rd));
        const Int r = m - q * d;
        q += (r >= d) ? 1 : 0;
        q -= (r < 0) ? 1 : 0;
        return q;
    } else {
        return floor_div_pos<Int>(m, d);
    }
}

template <class Int>
__device__ __forceinline__ bool row_span_const(const EdgeConst<Int>* e, int v, int W, Int& lo, Int& hi) {
    lo = 0;
    hi = W - 1;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const Int a = e[i].a;
        const Int m = e[i].dx * Int(v) + e[i].cb;
        const Int d = a > 0 ? a : (a < 0 ? -a : Int(1));
        const Int F = floor_div_rcp<Int>(m, d, e[i].rd);
        if (a > 0) lo = max(lo, -F);
        if (a < 0) hi = min(hi, F);
        if (a == 0 && m < 0) ok = false;
    }
    return ok && lo <= hi;
}

// Output of the raster: the triangle id (DisparityMesh::lookup, the stage
// API) or, for the pipeline, the interpolated disparity itself
// (interpolate(), mesh.cpp:149-164: binary32 plane value if 0 <= d < ND,
// NaN for "invalid or outside the hull"), so the per-pixel kernel reads one
// word per pixel and never gathers planes.
struct RasterOut {
    int32_t* lookup;  // mode lookup
    float* dit;       // mode disparity
    float max_disp;
};

__device__ __forceinline__ void put(const RasterOut& o, long long frame_base, long long idx,
                                    int32_t t, double a, double b, double c, int u, int v) {
    PS_CHECK(u >= 0 && v >= 0 && idx >= 0 && frame_base >= 0);
    if (o.lookup) {
        o.lookup[frame_base + idx] = t;
    } else {
        const double s = __dadd_rn(__dmul_rn(a, double(u)), __dmul_rn(b, double(v)));
        const float d = __double2float_rn(__dadd_rn(s, c));
        o.dit[frame_base + idx] = (d >= 0.0f && d < o.max_disp) ? d : __int_as_float(0x7fffffff);
    }
}

// Int = int when every edge-function value fits in 32 bits (W, H < 2^14),
// long long otherwise; the results are identical, 32-bit division is faster.
template <class Int>
__global__ void __launch_bounds__(kThreads) k_raster(
    const int* __restrict__ tris, const int* __restrict__ tri_off, int frames, long long total,
    const int* __restrict__ su, const int* __restrict__ sv, const double* __restrict__ sd, int scap,
    FrameGeom g, const uint8_t* __restrict__ pin_bits, double* __restrict__ planes, RasterOut out,
    int* __restrict__ err, long long tri_pitch, bool warp_per_tri) {
    // one thread per triangle, or (large triangles, e.g. the first
    // iteration's mesh) one warp per triangle: lane 0 owns it, the warp fills it
    const int lane = threadIdx.x & 31;
    const long long gtid = (long long)blockIdx.x * kThreads + threadIdx.x;
    const long long t = warp_per_tri ? gtid >> 5 : gtid;
    const long long t_block = warp_per_tri ? (long long)blockIdx.x * (kThreads / 32)
                                           : (long long)blockIdx.x * kThreads;
    const bool active = t < total && (!warp_per_tri || lane == 0);
    const int W = g.width, H = g.height;
    PS_CHECK(total > 0 && frames > 0);
    int x[3] = {0, 0, 0}, y[3] = {0, 0, 0};
    int f = 0, vmin = 0, vmax = -1;
    double pa = 0.0, pb = 0.0, pc = 0.0;
    bool big = false, small = false;
    // frame of the block's first triangle (uniform), then a short local scan
    const int fblk = frame_of(tri_off, frames, t_block < total ? t_block : total - 1);
    if (active) {
        f = fblk;
        while (f + 1 < frames && __ldg(tri_off + f + 1) <= t) ++f;
        const long long sb = (long long)f * scap;
        // slot of the triangle in the (flat or per-frame pitched) input arrays
        const long long ts = tri_pitch > 0 ? (long long)f * tri_pitch + (t - __ldg(tri_off + f)) : t;
        const int i0 = __ldg(tris + 3 * ts), i1 = __ldg(tris + 3 * ts + 1), i2 = __ldg(tris + 3 * ts + 2);
        x[0] = __ldg(su + sb + i0); x[1] = __ldg(su + sb + i1); x[2] = __ldg(su + sb + i2);
        y[0] = __ldg(sv + sb + i0); y[1] = __ldg(sv + sb + i1); y[2] = __ldg(sv + sb + i2);
        // fitPlane, mesh.cpp:12-26 (integer det exact; doubles in source order)
        const long long u1 = x[0], u2 = x[1], u3 = x[2], w1 = y[0], w2 = y[1], w3 = y[2];
        const long long det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
        double* pl = planes ? planes + 3 * t : nullptr;
        if (det == 0) {
            atomicExch(err, 1);
            if (pl) pl[0] = pl[1] = pl[2] = 0.0;
        } else {
            const double d1 = __ldg(sd + sb + i0), d2 = __ldg(sd + sb + i1), d3 = __ldg(sd + sb + i2);
            const double dA = __dadd_rn(__dadd_rn(__dmul_rn(d1, double(w2 - w3)),
                                                  __dmul_rn(d2, double(w3 - w1))),
                                        __dmul_rn(d3, double(w1 - w2)));
            const double dB = __dadd_rn(__dadd_rn(__dmul_rn(double(u1), __dsub_rn(d2, d3)),
                                                  __dmul_rn(double(u2), __dsub_rn(d3, d1))),
                                        __dmul_rn(double(u3), __dsub_rn(d1, d2)));
            const double dC = __dadd_rn(__dsub_rn(__dmul_rn(d1, double(u2 * w3 - u3 * w2)),
                                                  __dmul_rn(d2, double(u1 * w3 - u3 * w1))),
                                        __dmul_rn(d3, double(u1 * w2 - u2 * w1)));
            pa = __ddiv_rn(dA, double(det));
            pb = __ddiv_rn(dB, double(det));
            pc = __ddiv_rn(dC, double(det));
            if (planes) {
                pl[0] = pa;
                pl[1] = pb;
                pl[2] = pc;
            }
        }
        const long long fb = f * g.pixels;
        if (pin_bits) {
            const unsigned bits = __ldg(pin_bits + ts);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if ((bits >> k) & 1u)
                    put(out, fb, (long long)y[k] * W + x[k], int32_t(t), pa, pb, pc, x[k], y[k]);
        }
        vmin = max(0, min(y[0], min(y[1], y[2])));
        vmax = min(H - 1, max(y[0], max(y[1], y[2])));
        const int xmin = min(x[0], min(x[1], x[2])), xmax = max(x[0], max(x[1], x[2]));
        // warp-cooperative only when the bounding box is large (many pixels
        // or many rows); slivers and small triangles stay on their thread
        big = warp_per_tri || (long long)(vmax - vmin + 1) * (xmax - xmin + 1) > 512 || (vmax - vmin) >= 64;
        small = !big && vmin <= vmax;
    }
    // Small triangles, flattened twice so that every lane stays busy: the
    // warp's (triangle, row) pairs are dealt 32 at a time, one row per lane
    // (exact span by row_span), then the pixels of those 32 spans are dealt
    // 32 at a time (span found by binary search of the span prefix sums).
    {
        __shared__ EdgeConst<Int> s_e[3 * kThreads];
        __shared__ double s_pa[kThreads], s_pb[kThreads], s_pc[kThreads];
        __shared__ long long s_fb[kThreads], s_row[kThreads];
        __shared__ int s_vmin[kThreads], s_tid[kThreads], s_rpre[kThreads];
        __shared__ int s_pre[kThreads], s_lo[kThreads], s_k[kThreads], s_v[kThreads];
        const int me = threadIdx.x, wb = me & ~31;
#pragma unroll
        for (int k = 0; k < 3; ++k) s_e[3 * me + k].init(x[k], y[k], x[(k + 1) % 3], y[(k + 1) % 3]);
        s_pa[me] = pa;
        s_pb[me] = pb;
        s_pc[me] = pc;
        s_fb[me] = (long long)f * g.pixels;
        s_vmin[me] = vmin;
        s_tid[me] = int32_t(t);
        const int nrows = small ? vmax - vmin + 1 : 0;
        int rincl = nrows;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y2 = __shfl_up_sync(0xffffffffu, rincl, o);
            if (lane >= o) rincl += y2;
        }
        s_rpre[me] = rincl - nrows;
        const int total_rows = __shfl_sync(0xffffffffu, rincl, 31);
        __syncwarp();
        for (int r0 = 0; r0 < total_rows; r0 += 32) {
            const int r = r0 + lane;
            int len = 0, lo32 = 0, k = wb, v = 0;
            if (r < total_rows) {
                int sp = 0;  // the last triangle whose row prefix is <= r
#pragma unroll
                for (int step = 16; step; step >>= 1)
                    if (s_rpre[wb + sp + step] <= r) sp += step;
                k = wb + sp;
                v = s_vmin[k] + (r - s_rpre[k]);
                Int lo, hi;
                if (row_span_const<Int>(s_e + 3 * k, v, W, lo, hi)) {
                    len = int(hi - lo) + 1;
                    lo32 = int(lo);
                }
            }
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y2 = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y2;
            }
            const int total_px = __shfl_sync(0xffffffffu, incl, 31);
            s_pre[me] = incl - len;
            s_lo[me] = lo32;
            s_k[me] = k;
            s_v[me] = v;
            s_row[me] = s_fb[k] + (long long)v * W;
            __syncwarp();
            for (int j = lane; j < total_px; j += 32) {
                int sp = 0;  // the last span whose pixel prefix is <= j
#pragma unroll
                for (int step = 16; step; step >>= 1)
                    if (s_pre[wb + sp + step] <= j) sp += step;
                const int q = wb + sp;
                const int kt = s_k[q];
                const int u = s_lo[q] + (j - s_pre[q]);
                put(out, s_row[q], u, s_tid[kt], s_pa[kt], s_pb[kt], s_pc[kt], u, s_v[q]);
            }
            __syncwarp();
        }
    }
    // Large triangles: the whole warp, 32 rows at a time.
    __shared__ int s_bpre[kThreads], s_blo[kThreads];
    unsigned bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {
        const int src = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        int bx[3], by[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            bx[k] = __shfl_sync(0xffffffffu, x[k], src);
            by[k] = __shfl_sync(0xffffffffu, y[k], src);
        }
        const int bf = __shfl_sync(0xffffffffu, f, src);
        const int b0 = __shfl_sync(0xffffffffu, vmin, src);
        const int b1 = __shfl_sync(0xffffffffu, vmax, src);
        const int32_t bt = int32_t(__shfl_sync(0xffffffffu, (long long)t, src));
        const double ba = __shfl_sync(0xffffffffu, pa, src);
        const double bb = __shfl_sync(0xffffffffu, pb, src);
        const double bc = __shfl_sync(0xffffffffu, pc, src);
        const long long fb = bf * g.pixels;
        // 32 rows at a time, one per lane; then the pixels of those 32 spans
        // are dealt 32 at a time (span by binary search of the prefix sums),
        // so a long sliver (1-2 px per row) costs ~rows/32 steps, not ~rows
        for (int r0 = b0; r0 <= b1; r0 += 32) {
            const int v = r0 + lane;
            Int lo = 0, hi = -1;
            const bool ok = v <= b1 && row_span<Int>(bx, by, v, W, lo, hi);
            const int len = ok ? int(hi - lo) + 1 : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y2 = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y2;
            }
            const int total_px = __shfl_sync(0xffffffffu, incl, 31);
            s_bpre[threadIdx.x] = incl - len;
            s_blo[threadIdx.x] = int(lo);
            __syncwarp();
            const int wb = threadIdx.x & ~31;
            for (int j = lane; j < total_px; j += 32) {
                int sp = 0;  // the last row whose pixel prefix is <= j
#pragma unroll
                for (int step = 16; step; step >>= 1)
                    if (s_bpre[wb + sp + step] <= j) sp += step;
                const int u = s_blo[wb + sp] + (j - s_bpre[wb + sp]);
                put(out, fb, (long long)(r0 + sp) * W + u, bt, ba, bb, bc, u, r0 + sp);
            }
            __syncwarp();
        }
    }
}

template <class Int>
void launch_raster(const int* tris, const int* tri_off, int frames, long long total, const int* su,
                   const int* sv, const double* sd, int scap, FrameGeom g, const uint8_t* pin_bits,
                   double* planes, RasterOut out, int* err, cudaStream_t st, long long tri_pitch = 0) {
    // warp per triangle when the mean triangle covers >= 64 px: a thread per
    // triangle would leave too few warps, each looping over 32 large triangles
    const bool warp_per_tri = double(g.pixels) * frames >= 64.0 * double(total);
    const long long threads = warp_per_tri ? 32 * total : total;
    const unsigned blocks = unsigned((threads + kThreads - 1) / kThreads);
    k_raster<Int><<<blocks, kThreads, 0, st>>>(tris, tri_off, frames, total, su, sv, sd, scap, g,
                                               pin_bits, planes, out, err, tri_pitch, warp_per_tri);
}

}  // namespace

int launch_mesh(const int* tris, const int* tri_off, int frames, long long total_tris,
                const int* su, const int* sv, const double* sd, int scap, FrameGeom g,
                const uint8_t* pin_bits, double* planes, int32_t* lookup, int* err_flag,
                cudaStream_t st) {
    if (total_tris <= 0) return 0;
    const RasterOut out{lookup, nullptr, 0.0f};
    if (g.width < (1 << 14) && g.height < (1 << 14))
        launch_raster<int>(tris, tri_off, frames, total_tris, su, sv, sd, scap, g, pin_bits, planes,
                           out, err_flag, st);
    else
        launch_raster<long long>(tris, tri_off, frames, total_tris, su, sv, sd, scap, g, pin_bits,
                                 planes, out, err_flag, st);
    return 1;
}

int launch_mesh_disparity(const int* tris, const int* tri_off, int frames, long long total_tris,
                          const int* su, const int* sv, const double* sd, int scap, FrameGeom g,
                          const uint8_t* pin_bits, float max_disp, float* dit, int* err_flag,
                          cudaStream_t st, long long tri_pitch) {
    if (total_tris <= 0) return 0;
    const RasterOut out{nullptr, dit, max_disp};
    if (g.width < (1 << 14) && g.height < (1 << 14))
        launch_raster<int>(tris, tri_off, frames, total_tris, su, sv, sd, scap, g, pin_bits,
                           nullptr, out, err_flag, st, tri_pitch);
    else
        launch_raster<long long>(tris, tri_off, frames, total_tris, su, sv, sd, scap, g, pin_bits,
                                 nullptr, out, err_flag, st, tri_pitch);
    return 1;
}

}  // namespace ps
