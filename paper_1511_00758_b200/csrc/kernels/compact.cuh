// compact.cuh — stable per-frame stream compaction used by seeding and
// resampling (the reference appends in candidate / row-major cell order,
// proj/src/sparse.cpp:183-192 and proj/src/pipeline.cpp:102-127, so every
// compaction here must preserve item order).
//
// Three launches per compaction, all frames at once (frame = blockIdx.y):
//   count : chunk of 1024 items per block -> flag count per chunk;
//   scan  : one block per frame, exclusive scan of its chunk counts (+ base);
//   emit  : re-evaluates the flags, warp-ballot + block scan, and calls
//           op.emit(f, item, position) for every kept item, in order.
// The flag predicate is evaluated twice (it is cheap and side-effect free for
// the items of other chunks), which avoids storing per-item flags.
#pragma once

#include <cuda_runtime.h>

namespace ps {

constexpr int kChunkItems = 1024;  // 256 threads x 4 items
constexpr int kMaxChunks = 1 << 16;

template <class Op>
__global__ void __launch_bounds__(256) k_compact_count(Op op, int* __restrict__ chunk_cnt,
                                                       int chunks_per_frame) {
    __shared__ int wsum[8];
    const int f = blockIdx.y;
    const int n = op.items(f);
    const int base = blockIdx.x * kChunkItems;
    if (base >= n) {
        if (threadIdx.x == 0) chunk_cnt[f * chunks_per_frame + blockIdx.x] = 0;
        return;
    }
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = base + threadIdx.x * 4 + j;
        if (i < n && op.test(f, i)) ++c;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < 8; ++w) s += wsum[w];
        chunk_cnt[f * chunks_per_frame + blockIdx.x] = s;
    }
}

// In place: chunk_cnt[f][c] -> exclusive offset; total[f] = sum (optional);
// out_total[f] (optional) = base0[f] + base1[f] + sum.
template <int kUnused = 0>
__global__ void __launch_bounds__(1024) k_compact_scan(int* __restrict__ chunk_cnt,
                                                       int chunks_per_frame,
                                                       int* __restrict__ total,
                                                       const int* __restrict__ base0,
                                                       const int* __restrict__ base1,
                                                       int* __restrict__ out_total) {
    __shared__ int wsum[32];
    __shared__ int carry;
    const int f = blockIdx.x;
    int* c = chunk_cnt + (long long)f * chunks_per_frame;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t0 = 0; t0 < chunks_per_frame; t0 += 1024) {
        const int i = t0 + threadIdx.x;
        const int x = i < chunks_per_frame ? c[i] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            int s = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const int excl = carry + (w > 0 ? wsum[w - 1] : 0) + incl - x;
        if (i < chunks_per_frame) c[i] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (total) total[f] = carry;
        if (out_total) out_total[f] = carry + (base0 ? base0[f] : 0) + (base1 ? base1[f] : 0);
    }
}

template <class Op>
__global__ void __launch_bounds__(256) k_compact_emit(Op op, const int* __restrict__ chunk_off,
                                                      int chunks_per_frame,
                                                      const int* __restrict__ base0,
                                                      const int* __restrict__ base1) {
    __shared__ int wsum[8];
    const int f = blockIdx.y;
    const int n = op.items(f);
    const int base = blockIdx.x * kChunkItems;
    if (base >= n) return;
    bool flag[4];
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = base + threadIdx.x * 4 + j;
        flag[j] = i < n && op.test(f, i);
        c += flag[j];
    }
    // inclusive warp scan of per-thread counts
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    int wofs = 0;
    for (int k = 0; k < w; ++k) wofs += wsum[k];
    int pos = chunk_off[f * chunks_per_frame + blockIdx.x] + wofs + incl - c;
    if (base0) pos += base0[f];
    if (base1) pos += base1[f];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (flag[j]) op.emit(f, base + threadIdx.x * 4 + j, pos++);
    }
}

// Host helper: count + scan + emit over `max_items` per frame.
template <class Op>
inline int run_compaction(const Op& op, int frames, int max_items, int* chunk_buf,
                          int* total, const int* base0, const int* base1, int* out_total,
                          cudaStream_t st) {
    const int chunks = max_items > 0 ? (max_items + kChunkItems - 1) / kChunkItems : 0;
    dim3 grid(chunks, frames);
    if (chunks > 0) k_compact_count<Op><<<grid, 256, 0, st>>>(op, chunk_buf, chunks);
    k_compact_scan<<<frames, 1024, 0, st>>>(chunk_buf, chunks, total, base0, base1, out_total);
    if (chunks > 0) k_compact_emit<Op><<<grid, 256, 0, st>>>(op, chunk_buf, chunks, base0, base1);
    return chunks > 0 ? 3 : 1;
}

}  // namespace ps
