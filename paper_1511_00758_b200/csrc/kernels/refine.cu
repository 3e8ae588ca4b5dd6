// refine.cu — K7 (+K9): the graded per-pixel kernel.
//
// One pass over the frame fuses, per gradient-mask pixel:
//   interpolate   (proj/src/mesh.cpp:149-164): D_it is read as written by the
//                 raster (launch_mesh_disparity): binary32 plane value, NaN
//                 when invalid or outside the hull;
//   costEvaluation (proj/src/pipeline.cpp:33-54): k = popcount(cL(u) ^ cR(u-d)),
//                 d = lround(D_it), sentinel k = 24 (cost 1.0) when unusable;
//   disparityRefinement (pipeline.cpp:56-86): C_f/D_f fold, and the two
//                 occupancy grids as packed 64-bit keys reduced with atomicMin:
//                   confident: (k << 32 | v*W+u)        min k, first row-major
//                   invalid  : ((24-k) << 32 | v*W+u)   max k, first row-major
//                 which is exactly the sequential strict-compare update order
//                 (SURVEY App. A.6);
//   trace (pipeline.cpp:183-191): sum of C_f over the mask in 2^-36 fixed
//                 point (exact for every k/24 float) and the valid count.
// In the last iteration the same pass also writes the full-image dense
// interpolation (mesh.cpp:166-182, K9).
//
// Layout: a warp owns a 128-pixel chunk of one frame; slot j of lane l is
// pixel chunk + 32*j + l, so every load/store instruction of the warp covers
// 32 consecutive pixels (coalesced), the four first-level loads of all slots
// (mask, D_it, cL, C_f) are issued before any use (memory-level parallelism),
// and pixels of one occupancy cell are contiguous lanes of a slot: the grid
// keys of a cell are min-reduced across the warp (__match_any_sync +
// __reduce_min_sync on the two key words) before ONE atomicMin per cell and
// slot.  Algorithmic traffic P + 29*M bytes per frame.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

constexpr int kSlots = 4;
constexpr int kChunk = 32 * kSlots;

constexpr unsigned kIdxBits = 27;  // 32-bit warp keys (k << 27 | idx) need P <= 2^27
constexpr unsigned kIdxMask = (1u << kIdxBits) - 1;

__device__ __forceinline__ unsigned long long widen(unsigned key32) {
    // (k << 27 | idx) -> the grid's (k << 32 | idx): same order
    return (unsigned long long)(key32 >> kIdxBits) << 32 | (key32 & kIdxMask);
}

__device__ __forceinline__ int div_small(int n, int d, float inv) {
    // n / d for 0 <= n < 2^24 via a float reciprocal and one exact correction
    int q = __float2int_rz(__int2float_rn(n) * inv);
    if (q * d > n) --q;
    else if ((q + 1) * d <= n) ++q;
    return q;
}

template <bool LAST, bool KEY32>
__global__ void __launch_bounds__(256) k_refine(RefineArgs a, CostTables tab, float inv_cell,
                                                float inv_w) {
    const int f = blockIdx.y;
    const long long P = a.g.pixels;
    const int W = a.g.width;
    const int lane = threadIdx.x & 31;
    const long long chunk = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kChunk;
    unsigned long long tsum = 0;
    unsigned tvalid = 0;
    if (chunk < P) {  // warp-uniform
        const long long fb = (long long)f * P;
        uint8_t m[kSlots];
        float d[kSlots], cf[kSlots];
        uint32_t cl[kSlots];
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            const long long i = chunk + 32 * j + lane;
            const bool in = i < P;
            m[j] = in ? __ldg(a.mask + fb + i) : 0;
            d[j] = in ? __ldg(a.dit + fb + i) : __int_as_float(0x7fffffff);
            cl[j] = in ? __ldg(a.cl + fb + i) : 0u;
            cf[j] = in ? a.Cf[fb + i] : 0.0f;
        }
        int u[kSlots], v[kSlots], k[kSlots];
        uint32_t crv[kSlots];
        const long long v0 = chunk / W;  // one 64-bit division per warp
        const int r0 = int(chunk - v0 * W);
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            const int r = r0 + 32 * j + lane;  // < W + 128 < 2^24
            const int dv = W >= kChunk ? (r >= W ? 1 : 0) : div_small(r, W, inv_w);
            v[j] = int(v0) + dv;
            u[j] = r - dv * W;
            k[j] = kCensusBits;  // sentinel cost 1.0 (pipeline.cpp:15,35)
            crv[j] = 0;
            if (m[j] && d[j] == d[j]) {  // mask pixel with a valid D_it
                const int dr = lround_away(d[j]);
                const int ur = u[j] - dr;
                if (dr >= 0 && ur >= 2) {
                    k[j] = 0;
                    crv[j] = __ldg(a.cr + fb + (long long)v[j] * W + ur);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            const long long i = chunk + 32 * j + lane;
            const bool valid = d[j] == d[j];
            if (LAST && i < P) {
                a.dense[fb + i] = valid ? d[j] : 0.0f;
                a.dense_valid[fb + i] = valid ? 1 : 0;
            }
            if (k[j] == 0) k[j] = __popc(cl[j] ^ crv[j]);
            bool qg = false, qb = false;
            unsigned long long keyg = 0, keyb = 0;
            int cell = -1;
            if (m[j]) {
                const float c = tab.cost[k[j]];
                if (c < cf[j]) {  // pipeline.cpp:68-71
                    cf[j] = c;
                    a.Cf[fb + i] = c;
                    a.Df[fb + i] = d[j];
                    a.Dv[fb + i] = 1;
                }
                const unsigned long long idx = (unsigned long long)i;
                qg = (tab.low_mask >> k[j]) & 1u;
                qb = !qg && ((tab.high_mask >> k[j]) & 1u);
                keyg = (unsigned long long)k[j] << 32 | idx;
                keyb = (unsigned long long)(kCensusBits - k[j]) << 32 | idx;
                tsum += __double2ull_rn(__dmul_rn(double(cf[j]), 68719476736.0));  // * 2^36
                tvalid += cf[j] < tab.cost_high ? 1u : 0u;
            }
            if (i < P) {
                cell = div_small(v[j], a.cell, inv_cell) * a.cols + div_small(u[j], a.cell, inv_cell);
            }
            unsigned long long* cg = a.Cg + (long long)f * a.cell_stride + (cell < 0 ? 0 : cell);
            unsigned long long* cb = a.Cb + (long long)f * a.cell_stride + (cell < 0 ? 0 : cell);
            if (!KEY32) {
                if (qg) atomicMin(cg, keyg);
                if (qb) atomicMin(cb, keyb);
                continue;
            }
            // One atomic per (cell, slot): the pixels of a cell are contiguous
            // lanes, so a segmented shuffle min (doubling, with a same-cell
            // check) leaves each run's minimum key in its first lane.
            if (__ballot_sync(0xffffffffu, qg | qb) == 0u) continue;
            unsigned kg = qg ? ((unsigned)k[j] << kIdxBits) | unsigned(i) : 0xffffffffu;
            unsigned kb = qb ? ((unsigned)(kCensusBits - k[j]) << kIdxBits) | unsigned(i) : 0xffffffffu;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int c2 = __shfl_down_sync(0xffffffffu, cell, o);
                const unsigned g2 = __shfl_down_sync(0xffffffffu, kg, o);
                const unsigned b2 = __shfl_down_sync(0xffffffffu, kb, o);
                if (lane + o < 32 && c2 == cell) {
                    kg = min(kg, g2);
                    kb = min(kb, b2);
                }
            }
            const int cprev = __shfl_up_sync(0xffffffffu, cell, 1);
            if (lane == 0 || cprev != cell) {
                if (kg != 0xffffffffu) atomicMin(cg, widen(kg));
                if (kb != 0xffffffffu) atomicMin(cb, widen(kb));
            }
        }
    }
    // trace reduction: warp, then one atomic per warp
    tsum = __shfl_xor_sync(0xffffffffu, tsum, 16) + tsum;
    tsum = __shfl_xor_sync(0xffffffffu, tsum, 8) + tsum;
    tsum = __shfl_xor_sync(0xffffffffu, tsum, 4) + tsum;
    tsum = __shfl_xor_sync(0xffffffffu, tsum, 2) + tsum;
    tsum = __shfl_xor_sync(0xffffffffu, tsum, 1) + tsum;
    tvalid = __reduce_add_sync(0xffffffffu, tvalid);
    if (lane == 0 && (tsum | tvalid)) {
        atomicAdd(a.trace_sum + (long long)f * a.trace_stride, tsum);
        atomicAdd(a.trace_valid + (long long)f * a.trace_stride, tvalid);
    }
}

__global__ void k_interpolate(const int32_t* __restrict__ lookup, const double* __restrict__ planes,
                              FrameGeom g, const uint8_t* __restrict__ mask, float max_disp,
                              float* __restrict__ value, uint8_t* __restrict__ valid) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.pixels) return;
    float out = 0.0f;
    uint8_t ok = 0;
    if (!mask || mask[i]) {
        const int t = lookup[i];
        if (t >= 0) {
            const int v = int(i / g.width), u = int(i - (long long)v * g.width);
            const float d = plane_eval(planes + 3ll * t, u, v);
            if (d >= 0.0f && d < max_disp) {
                out = d;
                ok = 1;
            }
        }
    }
    value[i] = out;
    valid[i] = ok;
}

__global__ void k_cost_eval(const uint32_t* __restrict__ cl, const uint32_t* __restrict__ cr,
                            FrameGeom g, const float* __restrict__ value,
                            const uint8_t* __restrict__ valid, const uint8_t* __restrict__ mask,
                            CostTables tab, float* __restrict__ cost) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.pixels) return;
    float c = tab.cost[kCensusBits];
    if (mask[i] && valid[i]) {
        const int v = int(i / g.width), u = int(i - (long long)v * g.width);
        const int d = lround_away(value[i]);
        const int ur = u - d;
        if (d >= 0 && ur >= 2) c = tab.cost[__popc(cl[i] ^ cr[(long long)v * g.width + ur])];
    }
    cost[i] = c;
}

__global__ void k_fill_f32(float* __restrict__ p, long long n, float x) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n && (reinterpret_cast<uintptr_t>(p + i) & 15) == 0) {
        *reinterpret_cast<float4*>(p + i) = make_float4(x, x, x, x);
    } else {
        for (long long j = i; j < i + 4 && j < n; ++j) p[j] = x;
    }
}

}  // namespace

int launch_refine(const RefineArgs& a, const CostTables& tab, bool last, cudaStream_t st) {
    const long long chunks = (a.g.pixels + kChunk - 1) / kChunk;
    dim3 grid(unsigned((chunks + 7) / 8), a.frames);
    // reciprocals for the exact small-integer divisions (div_small corrects them)
    const float inv_cell = 1.0f / float(a.cell), inv_w = 1.0f / float(a.g.width);
    const bool key32 = a.g.pixels <= (1ll << kIdxBits);
    if (last) {
        if (key32) k_refine<true, true><<<grid, 256, 0, st>>>(a, tab, inv_cell, inv_w);
        else k_refine<true, false><<<grid, 256, 0, st>>>(a, tab, inv_cell, inv_w);
    } else {
        if (key32) k_refine<false, true><<<grid, 256, 0, st>>>(a, tab, inv_cell, inv_w);
        else k_refine<false, false><<<grid, 256, 0, st>>>(a, tab, inv_cell, inv_w);
    }
    return 1;
}

int launch_interpolate(const int32_t* lookup, const double* planes, FrameGeom g,
                       const uint8_t* mask, float max_disp, float* value, uint8_t* valid,
                       cudaStream_t st) {
    k_interpolate<<<unsigned((g.pixels + 255) / 256), 256, 0, st>>>(lookup, planes, g, mask,
                                                                     max_disp, value, valid);
    return 1;
}

int launch_cost_eval(const uint32_t* cl, const uint32_t* cr, FrameGeom g, const float* value,
                     const uint8_t* valid, const uint8_t* mask, const CostTables& tab, float* cost,
                     cudaStream_t st) {
    k_cost_eval<<<unsigned((g.pixels + 255) / 256), 256, 0, st>>>(cl, cr, g, value, valid, mask, tab,
                                                                   cost);
    return 1;
}

int launch_fill_f32(float* p, long long n, float x, cudaStream_t st) {
    if (n <= 0) return 0;
    const long long groups = (n + 3) / 4;
    k_fill_f32<<<unsigned((groups + 255) / 256), 256, 0, st>>>(p, n, x);
    return 1;
}

}  // namespace ps
