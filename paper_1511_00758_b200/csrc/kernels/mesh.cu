// mesh.cu — K5+K6: per-triangle plane fit and exact rasterisation into the
// pixel -> triangle lookup, then hull-vertex pinning.
//
// Replaces the DisparityMesh constructor (proj/src/mesh.cpp:44-56), fitPlane
// (:12-26) and rasterize (:58-123).  One warp per triangle (flat over all
// frames of the batch; a triangle finds its frame by binary search of the
// per-frame offsets).  Lane 0 solves the plane in binary64 in the reference's
// source order with _rn intrinsics (no FMA); the warp then walks the rows of
// the triangle's bounding box, every lane computing the exact integer span
// [lo, hi] of the row with the top-left tie bias (mesh.cpp:75-106), and fills
// the span with coalesced 4-byte stores.  Lookup entries are flat triangle
// ids, so the per-pixel kernels index the flat plane array directly.
//
// Pinning (mesh.cpp:109-122): vertex pixels left uncovered by the tie rule get
// their first incident triangle.  Done with atomicMin on an encoded value
// (INT_MIN + t, always < -1) over the uncovered vertex pixels, then decoded.
#include <climits>
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

constexpr int kWarpsPerBlock = 8;

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

// Int = int when every edge-function value fits in 32 bits (W, H < 2^14),
// long long otherwise; the results are identical, 32-bit division is faster.
template <class Int>
__global__ void __launch_bounds__(256) k_raster(const int* __restrict__ tris,
                                                const int* __restrict__ tri_off, int frames,
                                                long long total, const int* __restrict__ su,
                                                const int* __restrict__ sv,
                                                const double* __restrict__ sd, int scap,
                                                FrameGeom g, double* __restrict__ planes,
                                                int32_t* __restrict__ lookup,
                                                int* __restrict__ err) {
    const long long t = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (t >= total) return;
    const int lane = threadIdx.x & 31;
    const int f = frame_of(tri_off, frames, t);
    const long long sb = (long long)f * scap;
    const int i0 = __ldg(tris + 3 * t), i1 = __ldg(tris + 3 * t + 1), i2 = __ldg(tris + 3 * t + 2);
    const int x[3] = {__ldg(su + sb + i0), __ldg(su + sb + i1), __ldg(su + sb + i2)};
    const int y[3] = {__ldg(sv + sb + i0), __ldg(sv + sb + i1), __ldg(sv + sb + i2)};

    if (lane == 0) {
        // fitPlane, mesh.cpp:12-26 (integer det exact; doubles in source order)
        const long long u1 = x[0], u2 = x[1], u3 = x[2], w1 = y[0], w2 = y[1], w3 = y[2];
        const long long det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
        double* pl = planes + 3 * t;
        if (det == 0) {
            atomicExch(err, 1);
            pl[0] = pl[1] = pl[2] = 0.0;
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
            pl[0] = __ddiv_rn(dA, double(det));
            pl[1] = __ddiv_rn(dB, double(det));
            pl[2] = __ddiv_rn(dC, double(det));
        }
    }

    const int W = g.width, H = g.height;
    const int vmin = max(0, min(y[0], min(y[1], y[2])));
    const int vmax = min(H - 1, max(y[0], max(y[1], y[2])));
    Int A[3], bias[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3;
        A[i] = y[i] - y[j];
        bias[i] = ((y[j] < y[i]) || (y[j] == y[i] && x[j] > x[i])) ? 0 : 1;
    }
    int32_t* lk = lookup + f * g.pixels;
    // 32 rows at a time: lane r computes the exact span of row r0 + r
    // (mesh.cpp:84-103), then the warp fills each non-empty row with
    // coalesced stores.
    for (int r0 = vmin; r0 <= vmax; r0 += 32) {
        const int v = r0 + lane;
        Int lo = 0, hi = W - 1;
        bool empty = v > vmax;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            const Int K = Int(x[j] - x[i]) * Int(v - y[i]) + Int(y[j] - y[i]) * Int(x[i]);
            if (A[i] > 0) {
                lo = max(lo, ceil_div(bias[i] - K, A[i]));
            } else if (A[i] < 0) {
                hi = min(hi, floor_div(K - bias[i], -A[i]));
            } else if (K < bias[i]) {
                empty = true;
            }
        }
        unsigned rows = __ballot_sync(0xffffffffu, !empty && lo <= hi);
        const int lo32 = int(lo), hi32 = int(hi);
        while (rows) {
            const int r = __ffs(rows) - 1;
            rows &= rows - 1;
            const int l = __shfl_sync(0xffffffffu, lo32, r);
            const int h = __shfl_sync(0xffffffffu, hi32, r);
            int32_t* row = lk + (long long)(r0 + r) * W;
            for (int u = l + lane; u <= h; u += 32) row[u] = int32_t(t);
        }
    }
}

__global__ void k_pin(const int* __restrict__ tris, const int* __restrict__ tri_off, int frames,
                      long long total, const int* __restrict__ su, const int* __restrict__ sv,
                      int scap, FrameGeom g, int32_t* __restrict__ lookup, int decode) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 3 * total) return;
    const long long t = c / 3;
    const int f = frame_of(tri_off, frames, t);
    const int idx = __ldg(tris + c);
    const int u = __ldg(su + (long long)f * scap + idx), v = __ldg(sv + (long long)f * scap + idx);
    if (u < 0 || u >= g.width || v < 0 || v >= g.height) return;
    int32_t* cell = lookup + f * g.pixels + (long long)v * g.width + u;
    if (!decode) {
        if (*cell < 0) atomicMin(cell, int32_t(INT_MIN + t));
    } else {
        const int32_t x = *cell;
        if (x < -1) *cell = int32_t((long long)x - INT_MIN);
    }
}

}  // namespace

int launch_mesh(const int* tris, const int* tri_off, int frames, long long total_tris,
                const int* su, const int* sv, const double* sd, int scap, FrameGeom g,
                double* planes, int32_t* lookup, int* err_flag, cudaStream_t st) {
    if (total_tris <= 0) return 0;
    const long long blocks = (total_tris + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (g.width < (1 << 14) && g.height < (1 << 14)) {
        k_raster<int><<<unsigned(blocks), 32 * kWarpsPerBlock, 0, st>>>(
            tris, tri_off, frames, total_tris, su, sv, sd, scap, g, planes, lookup, err_flag);
    } else {
        k_raster<long long><<<unsigned(blocks), 32 * kWarpsPerBlock, 0, st>>>(
            tris, tri_off, frames, total_tris, su, sv, sd, scap, g, planes, lookup, err_flag);
    }
    const long long corners = 3 * total_tris;
    const unsigned pb = unsigned((corners + 255) / 256);
    k_pin<<<pb, 256, 0, st>>>(tris, tri_off, frames, total_tris, su, sv, scap, g, lookup, 0);
    k_pin<<<pb, 256, 0, st>>>(tris, tri_off, frames, total_tris, su, sv, scap, g, lookup, 1);
    return 3;
}

}  // namespace ps
