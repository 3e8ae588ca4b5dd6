// stage.cu — kernels behind the single-frame stage entry points whose inputs
// are arbitrary user maps rather than pipeline state:
//   disparityRefinement (proj/src/pipeline.cpp:56-86) over a float CostMap,
//   the confident / invalid candidate extraction of supportResampling
//   (pipeline.cpp:102-122) over user OccupancyGrids.
// Costs here are arbitrary binary32 values, so the cell keys order the float
// itself: a monotone uint32 image of the float in the high word, the
// row-major pixel index in the low word; min = smallest cost, first pixel.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

__device__ __forceinline__ unsigned float_order(float x) {
    const unsigned b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float order_float(unsigned o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void k_stage_refine(FrameGeom g, const float* __restrict__ interp,
                               const uint8_t* __restrict__ interp_valid,
                               const float* __restrict__ cost, const uint8_t* __restrict__ mask,
                               float* __restrict__ fd, uint8_t* __restrict__ fv,
                               float* __restrict__ fc, int cell, int cols, float cost_low,
                               float cost_high, unsigned long long* __restrict__ kg,
                               unsigned long long* __restrict__ kb) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.pixels || !mask[i]) return;
    const float c = cost[i];
    if (c < fc[i]) {  // pipeline.cpp:68-71
        fd[i] = interp_valid[i] ? interp[i] : 0.0f;
        fv[i] = 1;
        fc[i] = c;
    }
    const int v = int(i / g.width), u = int(i - (long long)v * g.width);
    const int ci = (v / cell) * cols + (u / cell);
    if (c < cost_low) {  // pipeline.cpp:73-77
        atomicMin(kg + ci, (unsigned long long)float_order(c) << 32 | (unsigned long long)i);
    } else if (c > cost_high) {  // pipeline.cpp:78-82
        atomicMin(kb + ci, (unsigned long long)(~float_order(c)) << 32 | (unsigned long long)i);
    }
}

__global__ void k_stage_cells(FrameGeom g, const unsigned long long* __restrict__ kg,
                              const unsigned long long* __restrict__ kb, int cells,
                              const float* __restrict__ interp,
                              const uint8_t* __restrict__ interp_valid, float cost_low,
                              float cost_high, StageCell* __restrict__ out_conf,
                              StageCell* __restrict__ out_inv) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const unsigned long long a = kg[c], b = kb[c];
    StageCell conf{0, 0, 0.0f, cost_low, 0}, inv{0, 0, 0.0f, cost_high, 0};  // OccupancyGrid init
    if (a != kEmptyCell) {
        const long long idx = (long long)(a & 0xffffffffull);
        const int v = int(idx / g.width), u = int(idx - (long long)v * g.width);
        const float d = interp_valid[idx] ? interp[idx] : 0.0f;  // interpolated.at(u, v)
        conf = StageCell{u, v, d, order_float(unsigned(a >> 32)), 1};
    }
    if (b != kEmptyCell) {
        const long long idx = (long long)(b & 0xffffffffull);
        const int v = int(idx / g.width), u = int(idx - (long long)v * g.width);
        inv = StageCell{u, v, 0.0f, order_float(~unsigned(b >> 32)), 1};
    }
    out_conf[c] = conf;
    out_inv[c] = inv;
}

}  // namespace

int launch_stage_refine(FrameGeom g, const float* interp, const uint8_t* interp_valid,
                        const float* cost, const uint8_t* mask, float* fd, uint8_t* fv, float* fc,
                        int cell, float cost_low, float cost_high, unsigned long long* kg,
                        unsigned long long* kb, StageCell* out_conf, StageCell* out_inv,
                        cudaStream_t st) {
    const int cols = (g.width + cell - 1) / cell;
    const int cells = cols * ((g.height + cell - 1) / cell);
    cudaMemsetAsync(kg, 0xff, sizeof(unsigned long long) * cells, st);
    cudaMemsetAsync(kb, 0xff, sizeof(unsigned long long) * cells, st);
    k_stage_refine<<<unsigned((g.pixels + 255) / 256), 256, 0, st>>>(
        g, interp, interp_valid, cost, mask, fd, fv, fc, cell, cols, cost_low, cost_high, kg, kb);
    k_stage_cells<<<(cells + 255) / 256, 256, 0, st>>>(g, kg, kb, cells, interp, interp_valid,
                                                       cost_low, cost_high, out_conf, out_inv);
    return 2;
}

}  // namespace ps
