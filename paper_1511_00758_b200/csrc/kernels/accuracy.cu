// accuracy.cu — on-device evaluation of disparity maps against ground truth
// (SURVEY 8(f) item 3): planestereo::accuracy (proj/src/eval.cpp:19-70).
//
// Per frame: over the pixels valid in both maps (and inside the mask when one
// is given), evaluated = count, hits[k] = #{err < thresholds[k]} (strict),
// errSum = the binary64 sum of err = |double(pred) - double(gt)| IN ROW-MAJOR
// ORDER — the reference accumulates sequentially, and floating-point addition
// does not reassociate, so the sum is folded in that order: one warp per
// frame, lanes compute 32 consecutive errors, then every lane folds them in
// lane order (shuffles, `__dadd_rn`).  meanAbsError = errSum / evaluated and
// the fractions are formed on the host in binary64, as in the reference.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

__global__ void __launch_bounds__(256) k_accuracy(
    const float* __restrict__ pred, const uint8_t* __restrict__ pred_valid,
    const float* __restrict__ gt, const uint8_t* __restrict__ gt_valid,
    const uint8_t* __restrict__ mask, long long P, int frames, const double* __restrict__ thr,
    int n_thr, unsigned long long* __restrict__ counts /* [frames][1 + n_thr] */,
    double* __restrict__ err_sum) {
    const int lane = threadIdx.x & 31;
    const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (f >= frames) return;
    const long long b = (long long)f * P;
    unsigned long long n = 0;
    unsigned long long hits[16] = {};
    double sum = 0.0;
    constexpr int U = 8;  // 256 pixels per step: 8 independent load groups in flight
    for (long long i0 = 0; i0 < P; i0 += 32 * U) {
        double err[U];
        unsigned flags[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const long long i = i0 + 32 * q + lane;
            bool ok = false;
            err[q] = 0.0;
            if (i < P) {
                ok = pred_valid[b + i] && gt_valid[b + i] && (!mask || mask[b + i]);
                if (ok) err[q] = fabs(__dsub_rn(double(pred[b + i]), double(gt[b + i])));
            }
            if (ok) {
                ++n;
                for (int k = 0; k < n_thr && k < 16; ++k) hits[k] += err[q] < thr[k];
            }
            flags[q] = __ballot_sync(0xffffffffu, ok);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            if (!flags[q]) continue;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {  // the reference's sequential order
                const double x = __shfl_sync(0xffffffffu, err[q], j);
                if ((flags[q] >> j) & 1u) sum = __dadd_rn(sum, x);
            }
        }
    }
    // counts are order-free: warp sums
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    for (int k = 0; k < n_thr && k < 16; ++k)
        for (int o = 16; o; o >>= 1) hits[k] += __shfl_xor_sync(0xffffffffu, hits[k], o);
    if (lane == 0) {
        unsigned long long* c = counts + (long long)f * (1 + n_thr);
        c[0] = n;
        for (int k = 0; k < n_thr && k < 16; ++k) c[1 + k] = hits[k];
        err_sum[f] = sum;
    }
}

}  // namespace

int launch_accuracy(const float* pred, const uint8_t* pred_valid, const float* gt,
                    const uint8_t* gt_valid, const uint8_t* mask, long long P, int frames,
                    const double* thresholds, int n_thr, unsigned long long* counts,
                    double* err_sum, cudaStream_t st) {
    k_accuracy<<<unsigned((frames + 7) / 8), 256, 0, st>>>(pred, pred_valid, gt, gt_valid, mask, P,
                                                          frames, thresholds, n_thr, counts,
                                                          err_sum);
    return 1;
}

}  // namespace ps
