// wta.cu — the exhaustive winner-take-all census matcher.
//
// Replaces planestereo::wtaOracle (proj/src/synth.cpp:171-198): for every
// gradient-mask pixel the cost-minimal integer disparity in
// [0, min(maxDisparity, u - 2)] (maxDisparity INCLUSIVE, unlike
// matchEpipolar), ties toward the smaller d (strict `c < bestCost` scanning d
// upward), cost = census cost (k/24); pixels outside the mask keep cost 1.0
// and no disparity.  It is the dense lower bound the pipeline's final costs
// are checked against (proj/tests/test_pipeline.cpp:255-268).
//
// Block = 128 pixels of one row of one frame; the cR row span the block can
// reach, [u0 - nd, u0 + 128), is staged in shared memory, so the d loop is
// LDS + LOP3 + POPC + IMNMX on a packed (k << 16 | d) key — the minimum key
// is the reference's first minimum because cost is increasing in k.
#include <cuda_runtime.h>

#include <algorithm>

#include "launch.hpp"

namespace ps {

namespace {

constexpr int kWtaBlock = 128;

__global__ void __launch_bounds__(kWtaBlock) k_wta(const uint32_t* __restrict__ cl,
                                                   const uint32_t* __restrict__ cr,
                                                   const uint8_t* __restrict__ mask, FrameGeom g,
                                                   int nd, CostTables tab,
                                                   float* __restrict__ disparity,
                                                   uint8_t* __restrict__ valid,
                                                   float* __restrict__ cost) {
    extern __shared__ uint32_t s_cr[];
    __shared__ float s_cost[32];
    const int W = g.width;
    const int v = blockIdx.y, f = blockIdx.z;
    const int u0 = blockIdx.x * kWtaBlock;
    const int reach = min(nd, W);  // d never exceeds u - 2 < W
    const int seg0 = max(0, u0 - reach), seg1 = min(W, u0 + kWtaBlock);
    const long long row = (long long)f * g.pixels + (long long)v * W;
    for (int j = threadIdx.x; j < seg1 - seg0; j += kWtaBlock) s_cr[j] = __ldg(cr + row + seg0 + j);
    if (threadIdx.x <= kCensusBits) s_cost[threadIdx.x] = tab.cost[threadIdx.x];
    __syncthreads();
    const int u = u0 + threadIdx.x;
    if (u >= W) return;
    const long long i = row + u;
    float d_out = 0.0f, c_out = 1.0f;  // CostMap(w, h, 1.0f); DisparityMap invalid
    uint8_t ok = 0;
    if (__ldg(mask + i) && u >= kCensusRadius) {
        const uint32_t a = __ldg(cl + i);
        const int dmax = min(nd, u - kCensusRadius);
        const uint32_t* s = s_cr + (u - seg0);  // s[-d] = cR(u - d)
        unsigned best = 0xffffffffu;
#pragma unroll 4
        for (int d = 0; d <= dmax; ++d) best = min(best, unsigned(__popc(a ^ s[-d])) << 16 | unsigned(d));
        d_out = float(best & 0xffffu);
        c_out = s_cost[best >> 16];
        ok = 1;
    }
    disparity[i] = d_out;
    valid[i] = ok;
    cost[i] = c_out;
}

}  // namespace

int launch_wta(const uint32_t* cl, const uint32_t* cr, const uint8_t* mask, FrameGeom g, int frames,
               int max_disparity, const CostTables& tab, float* disparity, uint8_t* valid,
               float* cost, cudaStream_t st) {
    const int reach = std::min(max_disparity, g.width);
    const size_t smem = sizeof(uint32_t) * size_t(kWtaBlock + reach);
    if (smem > 48 * 1024)  // per-device function attribute: set on every launch
        cudaFuncSetAttribute(k_wta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid((g.width + kWtaBlock - 1) / kWtaBlock, g.height, frames);
    k_wta<<<grid, kWtaBlock, smem, st>>>(cl, cr, mask, g, max_disparity, tab, disparity, valid, cost);
    return 1;
}

}  // namespace ps
