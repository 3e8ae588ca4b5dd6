// resample.cu — K8: support resampling from the two occupancy grids.
//
// Replaces supportResampling (proj/src/pipeline.cpp:88-129):
//   result = old supports
//          ++ confident cells in row-major cell order with u - d >= 2 (binary32)
//             whose pixel is not yet a support            -> {u, v, double(d)}
//          ++ matchEpipolar(occupied invalid cells, row-major) not yet taken.
// Cells hold packed keys written by K7; the winner pixel is the low word and
// its stored disparity is D_it at that pixel, recomputed here from the same
// lookup + plane (bit-identical to the value K7 saw).  A per-frame taken
// bitmap (1 bit/pixel, persistent across iterations) replaces the
// reference's unordered_set; confident and invalid winners are disjoint
// pixels (a cost cannot be both < costLow and > costHigh), so every
// compaction is a stable warp-ballot/scan pass (compact.cuh).
#include <cuda_runtime.h>

#include "compact.cuh"
#include "launch.hpp"

namespace ps {

namespace {

struct ConfidentOp {
    const unsigned long long* Cg;
    int cells;
    int stride;
    FrameGeom g;
    const float* dit;
    uint32_t* taken;
    int* su;
    int* sv;
    double* sd;
    int scap;

    __device__ int items(int) const { return cells; }
    __device__ bool winner(int f, int c, int& u, int& v, float& d) const {
        const unsigned long long key = Cg[(long long)f * stride + c];
        if (key == kEmptyCell) return false;  // !cell.occupied
        const long long idx = (long long)(key & 0xffffffffull);
        v = int(idx / g.width);
        u = int(idx - (long long)v * g.width);
        d = dit[(long long)f * g.pixels + idx];  // the winner's D_it (valid: its cost < costLow)
        return true;
    }
    __device__ bool test(int f, int c) const {
        int u, v;
        float d;
        if (!winner(f, c, u, v, d)) return false;
        // cell.u - cell.disparity < kRadius, evaluated in binary32 (pipeline.cpp:105)
        if (__fsub_rn(float(u), d) < 2.0f) return false;
        const long long pix = (long long)v * g.width + u;
        const long long words = (g.pixels + 31) >> 5;
        return !((taken[f * words + (pix >> 5)] >> (pix & 31)) & 1u);
    }
    __device__ void emit(int f, int c, int pos) const {
        int u, v;
        float d;
        winner(f, c, u, v, d);
        const long long s = (long long)f * scap + pos;
        PS_CHECK(pos >= 0 && pos < scap && u >= 0 && u < g.width && v >= 0 && v < g.height);
        su[s] = u;
        sv[s] = v;
        sd[s] = double(d);
        const long long pix = (long long)v * g.width + u;
        const long long words = (g.pixels + 31) >> 5;
        atomicOr(taken + f * words + (pix >> 5), 1u << (pix & 31));
    }
};

struct InvalidOp {
    const unsigned long long* Cb;
    int cells;
    int stride;
    FrameGeom g;
    int* ru;
    int* rv;
    int rstride;

    __device__ int items(int) const { return cells; }
    __device__ bool test(int f, int c) const { return Cb[(long long)f * stride + c] != kEmptyCell; }
    __device__ void emit(int f, int c, int pos) const {
        const long long idx = (long long)(Cb[(long long)f * stride + c] & 0xffffffffull);
        const int v = int(idx / g.width);
        PS_CHECK(pos >= 0 && pos < rstride && v >= 0 && v < g.height);
        ru[(long long)f * rstride + pos] = int(idx - (long long)v * g.width);
        rv[(long long)f * rstride + pos] = v;
    }
};

__global__ void k_add_counts(int* S, const int* a, const int* b, int frames) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < frames) S[f] += (a ? a[f] : 0) + (b ? b[f] : 0);
}

__global__ void k_pack_new(const int* __restrict__ su, const int* __restrict__ sv,
                           const double* __restrict__ sd, int scap,
                           const int* __restrict__ S_prev, const int* __restrict__ S_now,
                           const int* __restrict__ off, int2* __restrict__ out,
                           double* __restrict__ out_d) {
    const int f = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = S_now[f] - S_prev[f];
    if (i >= n) return;
    const long long s = (long long)f * scap + S_prev[f] + i;
    out[off[f] + i] = make_int2(su[s], sv[s]);
    if (out_d) out_d[off[f] + i] = sd[s];
}

}  // namespace

int launch_resample_confident(const unsigned long long* Cg, int cells_per_frame, int cell_stride,
                              FrameGeom g, int frames, const float* dit, uint32_t* taken, int* su,
                              int* sv, double* sd, int scap, const int* S_old, int* conf_count,
                              int* chunk_buf, cudaStream_t st) {
    ConfidentOp op{Cg, cells_per_frame, cell_stride, g, dit, taken, su, sv, sd, scap};
    return run_compaction(op, frames, cells_per_frame, chunk_buf, conf_count, S_old, nullptr,
                          nullptr, st);
}

int launch_resample_invalid(const unsigned long long* Cb, int cells_per_frame, int cell_stride,
                            FrameGeom g, int frames, int* rem_u, int* rem_v, int rem_stride,
                            int* rem_count, int* chunk_buf, cudaStream_t st) {
    InvalidOp op{Cb, cells_per_frame, cell_stride, g, rem_u, rem_v, rem_stride};
    return run_compaction(op, frames, cells_per_frame, chunk_buf, rem_count, nullptr, nullptr,
                          nullptr, st);
}

int launch_add_counts(int* S, const int* a, const int* b, int frames, cudaStream_t st) {
    k_add_counts<<<(frames + 255) / 256, 256, 0, st>>>(S, a, b, frames);
    return 1;
}

int launch_pack_new_supports(const int* su, const int* sv, const double* sd, int scap,
                             const int* S_prev, const int* S_now, const int* off, int frames,
                             int max_new, int2* out, double* out_d, cudaStream_t st) {
    if (max_new <= 0) return 0;
    dim3 grid((max_new + 255) / 256, frames);
    k_pack_new<<<grid, 256, 0, st>>>(su, sv, sd, scap, S_prev, S_now, off, out, out_d);
    return 1;
}

}  // namespace ps
