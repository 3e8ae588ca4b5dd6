// match.cu — K3: epipolar census matching, one warp per candidate.
//
// Replaces searchLeftToRight / searchRightToLeft / matchEpipolar
// (proj/src/sparse.cpp:44-80, 148-195).  Lanes stride the disparity range;
// the first minimum is a warp min over the packed key (k << 16 | d), which
// reproduces the reference's strict `<` scan in increasing d (first-min tie
// rule); the second-best over |d - d*| > 1 is a second warp min.  Accept and
// uniqueness decisions index host-built binary32 tables (CostTables), so the
// float expressions of sparse.cpp:169,172 are evaluated exactly as the
// reference evaluates them.  Census rows stay in L1/L2:
// at most 2*ND words per candidate.
#include <cuda_runtime.h>

#include "compact.cuh"
#include "launch.hpp"

namespace ps {

namespace {

constexpr int kWarpsPerBlock = 8;

__global__ void __launch_bounds__(256) k_match(const uint32_t* __restrict__ cl,
                                               const uint32_t* __restrict__ cr, FrameGeom g,
                                               int nd, CostTables tab,
                                               const int* __restrict__ cand_u,
                                               const int* __restrict__ cand_v,
                                               const int* __restrict__ cand_count,
                                               int cand_stride, uint8_t* __restrict__ ok,
                                               int* __restrict__ disp,
                                               int* __restrict__ costk) {
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (i >= cand_count[f]) return;
    const long long o = (long long)f * cand_stride + i;
    const int W = g.width, H = g.height;
    const int u = cand_u[o], v = cand_v[o];
    bool accept = false;
    int dbest = -1, kbest = kNoKey;
    // left.valid(u, v) and dMax >= 0 (sparse.cpp:160-166)
    const int dmax = min(nd - 1, u - 2);
    if (u >= 2 && u < W - 2 && v >= 2 && v < H - 2 && dmax >= 0) {
        const long long row = f * g.pixels + (long long)v * W;
        const uint32_t ref = __ldg(cl + row + u);
        unsigned best = 0xffffffffu;
        for (int d = lane; d <= dmax; d += 32) {
            const unsigned k = __popc(ref ^ __ldg(cr + row + u - d));
            const unsigned key = (k << 16) | unsigned(d);
            best = key < best ? key : best;
        }
        best = warp_min_u32(best);
        dbest = int(best & 0xffffu);
        kbest = int(best >> 16);
        unsigned second = kNoKey;
        for (int d = lane; d <= dmax; d += 32) {
            if (abs(d - dbest) <= 1) continue;
            const unsigned k = __popc(ref ^ __ldg(cr + row + u - d));
            second = k < second ? k : second;
        }
        second = warp_min_u32(second);
        accept = (tab.accept_mask >> kbest) & 1u;
        if (accept && second != unsigned(kNoKey) && ((tab.uniq_reject[kbest] >> second) & 1u))
            accept = false;
        if (accept) {
            // R->L consistency (sparse.cpp:176-181)
            const int ur = u - dbest;
            const int bmax = min(nd - 1, W - 1 - 2 - ur);
            const uint32_t rref = __ldg(cr + row + ur);
            unsigned bb = 0xffffffffu;
            for (int d = lane; d <= bmax; d += 32) {
                const unsigned k = __popc(rref ^ __ldg(cl + row + ur + d));
                const unsigned key = (k << 16) | unsigned(d);
                bb = key < bb ? key : bb;
            }
            bb = warp_min_u32(bb);
            const int back = bmax >= 0 ? int(bb & 0xffffu) : 0;
            if (abs(ur + back - u) > 1) accept = false;
        }
    }
    if (lane == 0) {
        ok[o] = accept ? 1 : 0;
        disp[o] = dbest;
        if (costk) costk[o] = kbest;
    }
}

struct MatchEmitOp {
    const int* cand_u;
    const int* cand_v;
    const int* cand_count;
    int cand_stride;
    const uint8_t* ok;
    const int* disp;
    FrameGeom g;
    uint32_t* taken;
    int* su;
    int* sv;
    double* sd;
    int scap;

    __device__ int items(int f) const { return cand_count[f]; }
    __device__ bool test(int f, int i) const {
        const long long o = (long long)f * cand_stride + i;
        if (!ok[o]) return false;
        const long long pix = (long long)cand_v[o] * g.width + cand_u[o];
        const long long words = (g.pixels + 31) >> 5;
        return !((taken[f * words + (pix >> 5)] >> (pix & 31)) & 1u);
    }
    __device__ void emit(int f, int i, int pos) const {
        const long long o = (long long)f * cand_stride + i;
        const long long s = (long long)f * scap + pos;
        const int u = cand_u[o], v = cand_v[o];
        PS_CHECK(pos >= 0 && pos < scap && u >= 0 && u < g.width && v >= 0 && v < g.height);
        su[s] = u;
        sv[s] = v;
        sd[s] = double(disp[o]);  // SupportPoint{u, v, double(match.disparity)}, sparse.cpp:187
        const long long pix = (long long)v * g.width + u;
        const long long words = (g.pixels + 31) >> 5;
        atomicOr(taken + f * words + (pix >> 5), 1u << (pix & 31));
    }
};

}  // namespace

int launch_match(const uint32_t* cl, const uint32_t* cr, FrameGeom g, int frames, int max_disp,
                 const CostTables& tab, const int* cand_u, const int* cand_v,
                 const int* cand_count, int cand_stride, int max_candidates, uint8_t* ok,
                 int* disp, int* costk, cudaStream_t st) {
    if (max_candidates <= 0 || frames <= 0) return 0;
    dim3 grid((max_candidates + kWarpsPerBlock - 1) / kWarpsPerBlock, frames);
    k_match<<<grid, 32 * kWarpsPerBlock, 0, st>>>(cl, cr, g, max_disp, tab, cand_u, cand_v,
                                                   cand_count, cand_stride, ok, disp, costk);
    return 1;
}

int launch_emit_matches(const int* cand_u, const int* cand_v, const int* cand_count,
                        int cand_stride, int max_candidates, const uint8_t* ok, const int* disp,
                        FrameGeom g, int frames, uint32_t* taken, int* su, int* sv, double* sd,
                        int scap, const int* base, const int* base2, int* out_count,
                        int* chunk_buf, cudaStream_t st) {
    MatchEmitOp op{cand_u, cand_v, cand_count, cand_stride, ok, disp, g, taken, su, sv, sd, scap};
    return run_compaction(op, frames, max_candidates, chunk_buf, nullptr, base, base2, out_count,
                          st);
}

}  // namespace ps
