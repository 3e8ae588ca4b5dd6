// refine.cu — K7 (+K9): the graded per-pixel kernel.
//
// One pass over the frame fuses, per gradient-mask pixel:
//   interpolate   (proj/src/mesh.cpp:149-164): lookup -> plane -> binary32 D_it,
//                 valid iff 0 <= D_it < ND;
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
// interpolation (mesh.cpp:166-182, K9), reusing the lookup read.
//
// Each thread owns 4 consecutive pixels of a frame (uchar4 mask, int4 lookup,
// uint4 census, float4 C_f/D_f when the frame stride allows 16-B alignment).
// Algorithmic traffic P + 29*M bytes per frame; planes and the
// census gather of the right view are L2-resident.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

struct CellAcc {
    int cell = -1;
    unsigned long long key = kEmptyCell;
};

__device__ __forceinline__ void acc_push(CellAcc& a, unsigned long long* __restrict__ grid, int cell,
                                         unsigned long long key) {
    if (cell != a.cell) {
        if (a.cell >= 0) atomicMin(grid + a.cell, a.key);
        a.cell = cell;
        a.key = key;
    } else if (key < a.key) {
        a.key = key;
    }
}

template <bool VEC, bool LAST>
__global__ void __launch_bounds__(256) k_refine(RefineArgs a, CostTables tab) {
    const int f = blockIdx.y;
    const long long P = a.g.pixels;
    const int W = a.g.width;
    const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;  // per-frame index (P < 2^31)
    unsigned long long tsum = 0;
    unsigned tvalid = 0;
    if (i0 < P) {
        const long long fb = (long long)f * P;
        uint8_t m[4];
        int32_t lk[4];
        if (VEC) {
            const uchar4 mv = *reinterpret_cast<const uchar4*>(a.mask + fb + i0);
            m[0] = mv.x; m[1] = mv.y; m[2] = mv.z; m[3] = mv.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) m[j] = (i0 + j < P) ? a.mask[fb + i0 + j] : 0;
        }
        const bool any_mask = (m[0] | m[1] | m[2] | m[3]) != 0;
        if (LAST || any_mask) {
            if (VEC) {
                const int4 l4 = *reinterpret_cast<const int4*>(a.lookup + fb + i0);
                lk[0] = l4.x; lk[1] = l4.y; lk[2] = l4.z; lk[3] = l4.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) lk[j] = (i0 + j < P) ? a.lookup[fb + i0 + j] : -1;
            }
        }
        const int v = i0 / W;
        const int u = i0 - v * W;
        float dit[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ok[j] = false;
            dit[j] = 0.0f;
            const int uj = u + j;
            const int vj = v + (uj >= W ? 1 : 0);  // W >= 16, so at most one wrap
            const int uu = uj >= W ? uj - W : uj;
            if ((LAST || m[j]) && (i0 + j < P) && lk[j] >= 0) {
                const float d = plane_eval(a.planes + 3ll * lk[j], uu, vj);
                dit[j] = d;
                ok[j] = d >= 0.0f && d < a.max_disp;
            }
        }
        if (LAST) {
            float dv[4];
            uint8_t dvv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                dv[j] = ok[j] ? dit[j] : 0.0f;
                dvv[j] = ok[j] ? 1 : 0;
            }
            if (VEC) {
                *reinterpret_cast<float4*>(a.dense + fb + i0) = make_float4(dv[0], dv[1], dv[2], dv[3]);
                *reinterpret_cast<uchar4*>(a.dense_valid + fb + i0) =
                    make_uchar4(dvv[0], dvv[1], dvv[2], dvv[3]);
            } else {
                for (int j = 0; j < 4 && i0 + j < P; ++j) {
                    a.dense[fb + i0 + j] = dv[j];
                    a.dense_valid[fb + i0 + j] = dvv[j];
                }
            }
        }
        if (any_mask) {
            uint32_t cl4[4];
            float cf[4], df[4];
            uint8_t dvalid[4];
            if (VEC) {
                const uint4 c = *reinterpret_cast<const uint4*>(a.cl + fb + i0);
                cl4[0] = c.x; cl4[1] = c.y; cl4[2] = c.z; cl4[3] = c.w;
                const float4 c2 = *reinterpret_cast<const float4*>(a.Cf + fb + i0);
                cf[0] = c2.x; cf[1] = c2.y; cf[2] = c2.z; cf[3] = c2.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    cl4[j] = (i0 + j < P) ? a.cl[fb + i0 + j] : 0u;
                    cf[j] = (i0 + j < P) ? a.Cf[fb + i0 + j] : 0.0f;
                }
            }
            bool upd[4];
            CellAcc accg, accb;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                upd[j] = false;
                df[j] = 0.0f;
                dvalid[j] = 0;
                if (!m[j]) continue;
                const int uj = u + j;
                const int vj = v + (uj >= W ? 1 : 0);
                const int uu = uj >= W ? uj - W : uj;
                int k = kCensusBits;  // sentinel cost 1.0 (pipeline.cpp:15,35)
                if (ok[j]) {
                    const int d = lround_away(dit[j]);
                    const int ur = uu - d;
                    if (d >= 0 && ur >= 2)
                        k = __popc(cl4[j] ^ __ldg(a.cr + fb + (long long)vj * W + ur));
                }
                const float c = tab.cost[k];
                if (c < cf[j]) {  // pipeline.cpp:68-71
                    upd[j] = true;
                    cf[j] = c;
                    df[j] = dit[j];
                    dvalid[j] = 1;
                }
                const int cell = (vj / a.cell) * a.cols + (uu / a.cell);
                const unsigned long long idx = (unsigned long long)vj * W + uu;
                if ((tab.low_mask >> k) & 1u) {
                    acc_push(accg, a.Cg + (long long)f * a.cell_stride, cell,
                             (unsigned long long)k << 32 | idx);
                } else if ((tab.high_mask >> k) & 1u) {
                    acc_push(accb, a.Cb + (long long)f * a.cell_stride, cell,
                             (unsigned long long)(kCensusBits - k) << 32 | idx);
                }
                tsum += __double2ull_rn(__dmul_rn(double(cf[j]), 68719476736.0));  // * 2^36
                tvalid += cf[j] < tab.cost_high ? 1u : 0u;
            }
            if (accg.cell >= 0) atomicMin(a.Cg + (long long)f * a.cell_stride + accg.cell, accg.key);
            if (accb.cell >= 0) atomicMin(a.Cb + (long long)f * a.cell_stride + accb.cell, accb.key);
            const bool any_upd = upd[0] | upd[1] | upd[2] | upd[3];
            if (any_upd) {
                if (VEC && upd[0] && upd[1] && upd[2] && upd[3]) {
                    *reinterpret_cast<float4*>(a.Cf + fb + i0) = make_float4(cf[0], cf[1], cf[2], cf[3]);
                    *reinterpret_cast<float4*>(a.Df + fb + i0) = make_float4(df[0], df[1], df[2], df[3]);
                    *reinterpret_cast<uchar4*>(a.Dv + fb + i0) = make_uchar4(1, 1, 1, 1);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (!upd[j]) continue;
                        a.Cf[fb + i0 + j] = cf[j];
                        a.Df[fb + i0 + j] = df[j];
                        a.Dv[fb + i0 + j] = 1;
                    }
                }
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
    if ((threadIdx.x & 31) == 0 && (tsum | tvalid)) {
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

}  // namespace

int launch_refine(const RefineArgs& a, const CostTables& tab, bool last, cudaStream_t st) {
    const long long groups = (a.g.pixels + 3) / 4;
    dim3 grid(unsigned((groups + 255) / 256), a.frames);
    const bool vec = (a.g.pixels % 4) == 0;
    if (vec) {
        if (last) k_refine<true, true><<<grid, 256, 0, st>>>(a, tab);
        else k_refine<true, false><<<grid, 256, 0, st>>>(a, tab);
    } else {
        if (last) k_refine<false, true><<<grid, 256, 0, st>>>(a, tab);
        else k_refine<false, false><<<grid, 256, 0, st>>>(a, tab);
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

}  // namespace ps

namespace ps {
namespace {
__global__ void k_fill_f32(float* __restrict__ p, long long n, float x) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n && (reinterpret_cast<uintptr_t>(p + i) & 15) == 0) {
        *reinterpret_cast<float4*>(p + i) = make_float4(x, x, x, x);
    } else {
        for (long long j = i; j < i + 4 && j < n; ++j) p[j] = x;
    }
}
}  // namespace

int launch_fill_f32(float* p, long long n, float x, cudaStream_t st) {
    if (n <= 0) return 0;
    const long long groups = (n + 3) / 4;
    k_fill_f32<<<unsigned((groups + 255) / 256), 256, 0, st>>>(p, n, x);
    return 1;
}
}  // namespace ps
