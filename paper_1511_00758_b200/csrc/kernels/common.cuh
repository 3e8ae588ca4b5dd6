// common.cuh — shared device-side definitions for the sm_100a kernels.
//
// Parity-critical arithmetic lives here:
//   * census cost k/24 is carried as the integer k (0..24); every float
//     comparison the reference makes on costs is pre-evaluated on the host in
//     binary32 into the tables of CostTables, so no device float rounding can
//     differ from the reference;
//   * plane evaluation is ((a*u)+(b*v))+c in binary64 with explicit _rn
//     intrinsics (no FMA contraction, mesh.hpp:19 as compiled without
//     -march), then rounded to binary32 with __double2float_rn.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace ps {

// Device-side bounds checks of the checked build (make CHECKED=1, or
// -DPS_CHECKED): a failing check prints its site and traps, so the launch
// fails and the run returns PS_CUDA_ERROR.  The stand-in for
// compute-sanitizer, which this GPU pool does not allow.
#ifdef PS_CHECKED
#define PS_CHECK(cond)                                                                             \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("PS_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,   \
                   int(blockIdx.x), int(threadIdx.x));                                             \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define PS_CHECK(cond) \
    do {               \
    } while (0)
#endif

constexpr int kCensusBits = 24;
constexpr int kCensusRadius = 2;  // CensusField::kRadius (census.hpp:19)
constexpr int kNoKey = 25;  // "no second-best" marker (BestMatch init 2.0f, sparse.cpp:38-42)
constexpr unsigned long long kEmptyCell = ~0ull;
constexpr unsigned char kCodeOff = 0xFF;  // C_f code of a pixel outside the gradient mask

// Host-built lookup tables derived from the PipelineConfig floats.
struct CostTables {
    float cost[kCensusBits + 1];        // float(k)/24.0f, census.hpp:45-47
    unsigned low_mask;                  // bit k: cost[k] <  costLow   (pipeline.cpp:73)
    unsigned high_mask;                 // bit k: cost[k] >  costHigh  (pipeline.cpp:78)
    unsigned accept_mask;               // bit k: !(cost[k] > sparseAcceptCost)   (sparse.cpp:169)
    unsigned uniq_reject[kCensusBits + 1];  // bit k2 of [k1]: cost[k1] > ratio*cost[k2] (sparse.cpp:172)
    // C_f as a byte code: c < code_high is cost[c], code_high is costHigh
    // (the initial value), kCodeOff marks a pixel outside the gradient mask.
    // Every C_f value the reference can hold is one of these: C_f starts at
    // costHigh and only takes cost[k] < C_f (pipeline.cpp:68-71), so
    // cost[k] < C_f  <=>  k < code, and C_f < costHigh  <=>  code < code_high.
    unsigned long long fixed[kCensusBits + 2];  // C_f*2^36 per code (trace)
    int code_high;                              // #{k : cost[k] < costHigh}
    float cost_high;
};

// Launch parameters shared by the per-frame kernels of one batch.
struct FrameGeom {
    int width;
    int height;
    long long pixels;  // P = width*height, frame stride of image-shaped buffers
};

#ifdef __CUDACC__
__device__ __forceinline__ float plane_eval(const double* __restrict__ pl, int u, int v) {
    // DisparityPlane::at (mesh.hpp:19) evaluated as the reference binary does:
    // mulsd, mulsd, addsd, addsd, cvtsd2ss.
    const double a = __ldg(pl), b = __ldg(pl + 1), c = __ldg(pl + 2);
    const double s = __dadd_rn(__dmul_rn(a, double(u)), __dmul_rn(b, double(v)));
    return __double2float_rn(__dadd_rn(s, c));
}

__device__ __forceinline__ int lround_away(float x) {
    // std::lround(float): half away from zero (pipeline.cpp:44, App. A.3).
    return int(roundf(x));
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
        x = y < x ? y : x;
    }
    return x;
}

__device__ __forceinline__ unsigned warp_min_u32(unsigned x) {
    return __reduce_min_sync(0xffffffffu, x);
}
#endif  // __CUDACC__

}  // namespace ps
