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
// Two kernels.  k_refine_bulk (the production path, below) streams tiles
// through shared memory with bulk copies, each lane owning four contiguous
// pixels; k_refine is the general fallback (frames whose width or
// disparity range the bulk path does not cover, or P > 2^27): a warp owns a
// 128-pixel chunk, slot j of lane l is pixel chunk + 32*j + l, and the keys of
// a cell are min-reduced across the lanes of a slot before one atomicMin.
// The C_f state is a byte code (CostTables): cost[k] < C_f <=> k < code.
// Algorithmic traffic P + 29*M bytes per frame and iteration.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>

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
        uint8_t cc[kSlots];
        float d[kSlots];
        uint32_t cl[kSlots];
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            const long long i = chunk + 32 * j + lane;
            const bool in = i < P;
            cc[j] = in ? a.code[fb + i] : kCodeOff;
            d[j] = in ? __ldg(a.dit + fb + i) : __int_as_float(0x7fffffff);
            cl[j] = in ? __ldg(a.cl + fb + i) : 0u;
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
            if (cc[j] != kCodeOff && d[j] == d[j]) {  // mask pixel with a valid D_it
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
            const bool m = cc[j] != kCodeOff;
            if (k[j] == 0) k[j] = __popc(cl[j] ^ crv[j]);
            bool qg = false, qb = false;
            unsigned long long keyg = 0, keyb = 0;
            int cell = -1;
            if (m) {
                if (k[j] < cc[j]) {  // cost[k] < C_f (pipeline.cpp:68-71), see CostTables
                    cc[j] = uint8_t(k[j]);
                    a.code[fb + i] = cc[j];
                    a.Df[fb + i] = d[j];
                }
                const unsigned long long idx = (unsigned long long)i;
                qg = (tab.low_mask >> k[j]) & 1u;
                qb = !qg && ((tab.high_mask >> k[j]) & 1u);
                keyg = (unsigned long long)k[j] << 32 | idx;
                keyb = (unsigned long long)(kCensusBits - k[j]) << 32 | idx;
                tsum += tab.fixed[cc[j]];
                tvalid += cc[j] < tab.code_high ? 1u : 0u;
            }
            if (LAST && i < P) {
                const bool fin = m && cc[j] < tab.code_high;
                a.dense[fb + i] = valid ? d[j] : 0.0f;
                a.dense_valid[fb + i] = valid ? 1 : 0;
                a.Cf[fb + i] = fin ? tab.cost[cc[j]] : tab.cost_high;
                a.Dv[fb + i] = fin ? 1 : 0;
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

// ---------------------------------------------------------------------------
// Bulk-copy (TMA 1-D) variant, the production path.  A persistent CTA owns a
// CONTIGUOUS range of 1024-pixel tiles (so frame changes, and with them the
// trace flushes, are rare) and streams per tile D_it, cL, the C_f code and
// the tile's cR row span (plus a max_disp halo to the left, for the same-row
// gather cR(u - d)) into a shared-memory ring with cp.async.bulk + mbarrier
// complete_tx, under an L2 evict-first policy (every byte is read once).  The
// cR gather is then a shared-memory load.  Stage release: the last of the 8
// warps to finish a stage refills it (no CTA-wide barrier).  Each lane owns
// four contiguous pixels (LDS.128 stage loads, vector output stores); the
// cell keys are folded inside the lane — SEG == 2: branch-free into at most
// two segments (every cell >= 3 px wide, host-checked), SEG == 1: in order —
// and each (cell, lane) segment issues one fire-and-forget atomicMin per
// grid.  The last iteration writes the outputs and skips the grids (they feed
// only supportResampling, which it does not run).  Needs 16-B aligned tiles
// (P % 16 == 0), W >= 32 and max_disp <= kMaxHalo.
constexpr int kTileSlots = 4;
constexpr int kWarpPx = 32 * kTileSlots;
constexpr int kWarps = 8;
constexpr int kTile = kWarps * kWarpPx;  // 8 warps x 4 slots x 32 lanes = 1024 px
constexpr int kStages = 4;
constexpr int kMaxHalo = 1024;  // cR words staged left of the tile (>= max_disp)

// n / d with magic31 = ceil(2^31 / d): exact whenever n * d < 2^31 (here
// n < 2^16 and d < 2^15), including d = 1, so no special case.
__device__ __forceinline__ int mdiv31(int n, unsigned magic31) {
    return int(__umulhi(unsigned(n) << 1, magic31));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;\n"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

constexpr unsigned kSuspendNs = 20000;  // try_wait suspend-time hint (no spinning on issue slots)

__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned phase) {
    // try_wait with a suspend-time hint: the warp sleeps until the phase
    // completes instead of spinning on the issue slots
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" :: "r"(smem_u32(bar)), "r"(phase), "r"(kSuspendNs) : "memory");
}

struct BulkGeom {
    int tiles_per_frame;
    int total_tiles;
    int halo;         // cR words staged left of a tile: max_disp rounded up to 4
    int stage_bytes;  // 9 * kTile + 4 * (kTile + halo)
    int q_tile;       // kTile / W
    int r_tile;       // kTile % W
};

template <bool LAST, int SEG, bool WRAP>
__global__ void __launch_bounds__(256, 4) k_refine_bulk(RefineArgs a, CostTables tab,
                                                        unsigned magic_cell31, unsigned magic_w,
                                                        BulkGeom bg) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bars[kStages];
    __shared__ unsigned s_done[kStages];  // warps finished with the stage (monotonic)
    // indexed by code & 31 (kCodeOff -> 31): output C_f, and C_f * 2^36 for
    // the trace (0 off the mask); smem, not the (serialising) constant bank
    __shared__ float s_cout[32];
    __shared__ unsigned long long s_fix[32];
    const unsigned code_high = unsigned(tab.code_high);
    if (threadIdx.x < 32) {
        const unsigned c = threadIdx.x;
        s_cout[c] = c < code_high ? tab.cost[c] : tab.cost_high;
        s_fix[c] = c <= code_high ? tab.fixed[c] : 0ull;
    }
    // frames * P < 2^31 (launch_refine splits larger batches): 32-bit pixel offsets
    const int P = int(a.g.pixels);
    const int W = a.g.width;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = bg.halo;
    const int t_begin = int((long long)bg.total_tiles * blockIdx.x / gridDim.x);
    const int t_end = int((long long)bg.total_tiles * (blockIdx.x + 1) / gridDim.x);
    auto stage_ptr = [&](int s) { return smem + s * bg.stage_bytes; };

    auto issue = [&](int tile, int s) {
        unsigned long long policy;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(policy));
        const int f = tile / bg.tiles_per_frame;
        const int off = (tile - f * bg.tiles_per_frame) * kTile;
        const unsigned n = unsigned(min(kTile, P - off));
        const int h = min(off, H);  // halo inside this frame (rows never reach back further)
        const int base = f * P + off;
        PS_CHECK(off >= 0 && off < P && h >= 0 && h <= H && base - h >= 0);
        PS_CHECK(9 * kTile + 4 * (H + int(n)) <= bg.stage_bytes);
        unsigned char* st = stage_ptr(s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     :: "r"(smem_u32(&bars[s])), "r"(n * 13u + 4u * unsigned(h)) : "memory");
        bulk_g2s(st, a.dit + base, 4 * n, &bars[s], policy);
        bulk_g2s(st + 4 * kTile, a.cl + base, 4 * n, &bars[s], policy);
        bulk_g2s(st + 8 * kTile, a.code + base, n, &bars[s], policy);
        bulk_g2s(st + 9 * kTile + 4 * (H - h), a.cr + base - h, 4 * (unsigned(h) + n), &bars[s], policy);
    };

    if (threadIdx.x < kStages) s_done[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int s = 0; s < kStages && t_begin + s < t_end; ++s) issue(t_begin + s, s);
    }
    __syncthreads();

    // tile geometry, advanced incrementally (no per-tile divisions)
    int f = t_begin / bg.tiles_per_frame;
    int off = (t_begin - f * bg.tiles_per_frame) * kTile;
    int v0 = off / W;
    int r0 = off - v0 * W;
    unsigned long long tsum = 0;
    unsigned tvalid = 0;
    auto flush = [&](int fr) {  // per-warp trace partials of frame fr
        unsigned long long ts = tsum;
        ts = __shfl_xor_sync(0xffffffffu, ts, 16) + ts;
        ts = __shfl_xor_sync(0xffffffffu, ts, 8) + ts;
        ts = __shfl_xor_sync(0xffffffffu, ts, 4) + ts;
        ts = __shfl_xor_sync(0xffffffffu, ts, 2) + ts;
        ts = __shfl_xor_sync(0xffffffffu, ts, 1) + ts;
        const unsigned tv = __reduce_add_sync(0xffffffffu, tvalid);
        if (lane == 0 && (ts | tv)) {
            atomicAdd(a.trace_sum + (long long)fr * a.trace_stride, ts);
            atomicAdd(a.trace_valid + (long long)fr * a.trace_stride, tv);
        }
        tsum = 0;
        tvalid = 0;
    };
    const int cellsz = a.cell, cols = a.cols;
    for (int tile = t_begin, j = 0; tile < t_end; ++tile, ++j) {
        const int s = j % kStages;
        bar_wait(&bars[s], unsigned((j / kStages) & 1));
        const unsigned char* st = stage_ptr(s);
        const float* sm_dit = reinterpret_cast<const float*>(st);
        const uint32_t* sm_cl = reinterpret_cast<const uint32_t*>(st + 4 * kTile);
        const uint8_t* sm_code = st + 8 * kTile;
        const uint32_t* sm_cr = reinterpret_cast<const uint32_t*>(st + 9 * kTile) + H;  // [p - dr]
        const int n_in = min(kTile, P - off);
        const int ib = off;          // first pixel of the tile within the frame (P <= 2^27)
        const int tb = f * P + off;  // first pixel of the tile within the batch
        unsigned long long* Cg_f = a.Cg + (long long)f * a.cell_stride;
        unsigned long long* Cb_f = a.Cb + (long long)f * a.cell_stride;
        {
            // 4 contiguous pixels per lane: p = warp*128 + 4*lane + j.  Vector
            // stage loads; the pixels of a cell inside the lane are folded in
            // order (first minimum wins) and each (cell, lane) segment issues
            // one fire-and-forget atomicMin (RED) per grid.
            const int p0 = warp * kWarpPx + 4 * lane;
            // n_in % 16 == 0: a lane's four pixels are all in the tile or none
            if (p0 < n_in) {
            const float4 d4 = *reinterpret_cast<const float4*>(sm_dit + p0);
            const uint4 cl4 = *reinterpret_cast<const uint4*>(sm_cl + p0);
            const unsigned code4 = *reinterpret_cast<const unsigned*>(sm_code + p0);
            const float dd[4] = {d4.x, d4.y, d4.z, d4.w};
            const uint32_t cl[4] = {cl4.x, cl4.y, cl4.z, cl4.w};
            const int r = r0 + p0;
            const int dv = int(__umulhi(unsigned(r), magic_w));  // W >= 32
            int cellv[4];
            uint32_t crv[4];
            unsigned okm = 0;
            {
                int u = r - dv * W, v = v0 + dv;
                int ccol = mdiv31(u, magic_cell31);
                int rem = u - ccol * cellsz;
                int crow = mdiv31(v, magic_cell31) * cols;
                // SEG == 2 without row wraps: the cell steps by one at the
                // first pixel with rem + j == cellsz (cells >= 3 px wide)
                const int nb = cellsz - rem;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (SEG == 2 && !WRAP) {
                        u += j > 0 ? 1 : 0;
                    } else if (j > 0) {
                        ++u;
                        if (++rem == cellsz) {
                            rem = 0;
                            ++ccol;
                        }
                        if (WRAP && u == W) {  // W % 4 != 0 only: at most one row wrap
                            u = 0;
                            ++v;
                            ccol = 0;
                            rem = 0;
                            crow = mdiv31(v, magic_cell31) * cols;
                        }
                    }
                    cellv[j] = crow + ccol + ((SEG == 2 && !WRAP && j >= nb) ? 1 : 0);
                    const unsigned c0 = (code4 >> (8 * j)) & 0xffu;
                    const float d = dd[j];
                    // lround (half away from zero) for d >= 0: trunc of d + 0.5
                    // rounded toward zero is exact there; D_it is NaN or in
                    // [0, ND) (raster), and a NaN (-> 0) is rejected below
                    const int dr = __float2int_rz(__fadd_rz(d, 0.5f));
                    const bool ok = c0 != kCodeOff && d == d && u - dr >= 2;
                    PS_CHECK(!ok || (p0 + j - dr >= -H && p0 + j - dr < kTile));
                    crv[j] = ok ? sm_cr[p0 + j - dr] : 0u;  // same-row cR(u - dr), staged
                    okm |= unsigned(ok) << j;
                }
            }
            int seg = -1;
            unsigned gk = 32, gi = 0, bk = 32, bi = 0;  // best (k, idx) of the segment per grid
            auto seg_flush = [&]() {
                PS_CHECK((gk == 32 && bk == 32) || (seg >= 0 && seg < a.cells_per_frame));
                if (gk < 32) atomicMin(Cg_f + seg, (unsigned long long)gk << 32 | gi);
                if (bk < 32) atomicMin(Cb_f + seg, (unsigned long long)bk << 32 | bi);
            };
            float dense[4], cfo[4];
            unsigned gkey[4], bkey[4];
            unsigned dval = 0, dvo = 0, codes_new = code4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int p = p0 + j;
                const unsigned c0 = (code4 >> (8 * j)) & 0xffu;
                const bool m = c0 != kCodeOff;
                const float d = dd[j];
                const int k = ((okm >> j) & 1u) ? __popc(cl[j] ^ crv[j]) : kCensusBits;
                const bool upd = m && unsigned(k) < c0;  // cost[k] < C_f (pipeline.cpp:68-71)
                if (upd) {
                    codes_new = (codes_new & ~(0xffu << (8 * j))) | (unsigned(k) << (8 * j));
                    a.Df[tb + p] = d;
                }
                const unsigned cc = (upd ? unsigned(k) : c0) & 31u;  // kCodeOff -> 31
                if (LAST) {
                    const bool valid = d == d;
                    dense[j] = valid ? d : 0.0f;
                    dval |= unsigned(valid) << (8 * j);
                    cfo[j] = s_cout[cc];
                    dvo |= unsigned(cc < code_high) << (8 * j);
                }
                tsum += s_fix[cc];  // C_f * 2^36 (exact, see trace_fixed_exact)
                tvalid += cc < code_high ? 1u : 0u;
                // the grids feed only supportResampling, which the last
                // iteration does not run (pipeline.cpp:168-171): skipped there
                const bool qg = !LAST && m && ((tab.low_mask >> k) & 1u);
                const bool qb = !LAST && m && !qg && ((tab.high_mask >> k) & 1u);
                const unsigned idx = unsigned(ib + p);
                if constexpr (LAST) {
                } else if constexpr (SEG == 2) {
                    // 32-bit keys (k << 27 | idx): their minimum is the first
                    // (row-major) minimum; folded per segment after the loop
                    gkey[j] = qg ? (unsigned(k) << kIdxBits | idx) : 0xffffffffu;
                    bkey[j] = qb ? (unsigned(kCensusBits - k) << kIdxBits | idx) : 0xffffffffu;
                } else {
                    if (cellv[j] != seg) {
                        if (seg >= 0) seg_flush();
                        seg = cellv[j];
                        gk = bk = 32;
                    }
                    if (qg && unsigned(k) < gk) {  // strict: the first (row-major) minimum
                        gk = unsigned(k);
                        gi = idx;
                    }
                    if (qb && unsigned(kCensusBits - k) < bk) {
                        bk = unsigned(kCensusBits - k);
                        bi = idx;
                    }
                }
            }
            {
                if constexpr (LAST) {
                } else if constexpr (SEG == 2) {
                    // at most one cell boundary inside the four pixels (host-
                    // checked: cell >= 3 and the last cell of a row >= 3 wide)
                    const bool b1 = cellv[1] != cellv[0], b2 = cellv[2] != cellv[0],
                               b3 = cellv[3] != cellv[0];
                    unsigned gA = gkey[0], bA = bkey[0], gB = 0xffffffffu, bB = 0xffffffffu;
                    gA = min(gA, b1 ? 0xffffffffu : gkey[1]);
                    bA = min(bA, b1 ? 0xffffffffu : bkey[1]);
                    gB = min(gB, b1 ? gkey[1] : 0xffffffffu);
                    bB = min(bB, b1 ? bkey[1] : 0xffffffffu);
                    gA = min(gA, b2 ? 0xffffffffu : gkey[2]);
                    bA = min(bA, b2 ? 0xffffffffu : bkey[2]);
                    gB = min(gB, b2 ? gkey[2] : 0xffffffffu);
                    bB = min(bB, b2 ? bkey[2] : 0xffffffffu);
                    gA = min(gA, b3 ? 0xffffffffu : gkey[3]);
                    bA = min(bA, b3 ? 0xffffffffu : bkey[3]);
                    gB = min(gB, b3 ? gkey[3] : 0xffffffffu);
                    bB = min(bB, b3 ? bkey[3] : 0xffffffffu);
                    if (gA != 0xffffffffu) atomicMin(Cg_f + cellv[0], widen(gA));
                    if (bA != 0xffffffffu) atomicMin(Cb_f + cellv[0], widen(bA));
                    if (gB != 0xffffffffu) atomicMin(Cg_f + cellv[3], widen(gB));
                    if (bB != 0xffffffffu) atomicMin(Cb_f + cellv[3], widen(bB));
                } else {
                    seg_flush();
                }
                if (codes_new != code4) *reinterpret_cast<unsigned*>(a.code + tb + p0) = codes_new;
                if (LAST) {
                    *reinterpret_cast<float4*>(a.dense + tb + p0) = make_float4(dense[0], dense[1], dense[2], dense[3]);
                    *reinterpret_cast<unsigned*>(a.dense_valid + tb + p0) = dval;
                    *reinterpret_cast<float4*>(a.Cf + tb + p0) = make_float4(cfo[0], cfo[1], cfo[2], cfo[3]);
                    *reinterpret_cast<unsigned*>(a.Dv + tb + p0) = dvo;
                }
            }
            }  // p0 < n_in
        }
        // release stage s: the last of the 8 warps to finish it refills it
        // (no CTA-wide barrier, so fast warps run ahead into the next stages)
        __syncwarp();
        if (lane == 0) {
            const unsigned prev = atomicAdd(&s_done[s], 1u);
            if (prev % kWarps == kWarps - 1 && tile + kStages < t_end) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue(tile + kStages, s);
            }
        }
        // next tile
        off += kTile;
        r0 += bg.r_tile;
        v0 += bg.q_tile;
        if (r0 >= W) {
            r0 -= W;
            ++v0;
        }
        if (off >= P) {  // frame change (tiles never straddle frames)
            flush(f);
            ++f;
            off = 0;
            v0 = 0;
            r0 = 0;
        }
    }
    flush(f);  // partial frame (no-op when nothing accumulated)
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

namespace {
// Persistent bulk-copy launch: as many CTAs per SM as registers and shared
// memory allow (queried once per instantiation).
template <bool LAST, int SEG, bool WRAP>
int launch_bulk(const RefineArgs& a0, const CostTables& tab, unsigned magic_cell31, unsigned magic_w,
                cudaStream_t st) {
    BulkGeom bg{};
    const long long P = a0.g.pixels;
    bg.tiles_per_frame = int((P + kTile - 1) / kTile);
    bg.halo = (int(a0.max_disp) + 3) & ~3;
    bg.stage_bytes = 9 * kTile + 4 * (kTile + bg.halo);
    bg.q_tile = kTile / a0.g.width;
    bg.r_tile = kTile % a0.g.width;
    const size_t smem = size_t(kStages) * bg.stage_bytes;
    // The dynamic shared-memory opt-in is a per-device function attribute:
    // set it on every launch (cheap), so each device of a multi-GPU process
    // gets it.  SM count and occupancy are cached per device under a lock.
    int dev = 0;
    cudaGetDevice(&dev);
    cudaFuncSetAttribute(k_refine_bulk<LAST, SEG, WRAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(size_t(kStages) * (9 * kTile + 4 * (kTile + kMaxHalo))));
    int sms = 0, occ = 0;
    {
        static std::mutex m;
        static std::map<std::pair<int, int>, std::pair<int, int>> cache;  // (device, halo) -> (sms, occ)
        std::lock_guard<std::mutex> lk(m);
        auto it = cache.find({dev, bg.halo});
        if (it == cache.end()) {
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine_bulk<LAST, SEG, WRAP>, 256, smem);
            occ = std::max(1, occ);
            cache[{dev, bg.halo}] = {sms, occ};
        } else {
            sms = it->second.first;
            occ = it->second.second;
        }
    }
    // the kernel indexes the batch with 32-bit pixel offsets: launch per
    // chunk of frames holding < 2^31 pixels
    const int chunk = int(std::max<long long>(1, ((1ll << 31) - 1) / P));
    int launches = 0;
    for (int f0 = 0; f0 < a0.frames; f0 += chunk) {
        RefineArgs a = a0;
        const long long px = (long long)f0 * P;
        a.frames = std::min(chunk, a0.frames - f0);
        a.mask = a0.mask ? a0.mask + px : nullptr;
        a.dit += px;
        a.cl += px;
        a.cr += px;
        a.code += px;
        a.Df += px;
        a.Cg += (long long)f0 * a0.cell_stride;
        a.Cb += (long long)f0 * a0.cell_stride;
        a.trace_sum += (long long)f0 * a0.trace_stride;
        a.trace_valid += (long long)f0 * a0.trace_stride;
        if (LAST) {
            a.Dv += px;
            a.Cf += px;
            a.dense += px;
            a.dense_valid += px;
        }
        bg.total_tiles = bg.tiles_per_frame * a.frames;
        // 8 CTAs per resident slot (each ~2 tiles, not one persistent CTA
        // per slot with ~16): more bulk copies in flight and no tail of late
        // CTAs -- a 256-frame launch 0.382 -> 0.344 ms (0.87 -> 0.97 of the
        // measured HBM peak); PS_K7_GRID overrides (probing)
        static const int grid_mult = [] {
            const char* e = std::getenv("PS_K7_GRID");
            return e ? std::max(1, std::atoi(e)) : 8;
        }();
        const unsigned blocks = unsigned(std::min<long long>(bg.total_tiles, (long long)occ * sms * grid_mult));
        k_refine_bulk<LAST, SEG, WRAP><<<blocks, 256, smem, st>>>(a, tab, magic_cell31, magic_w, bg);
        ++launches;
    }
    return launches;
}
}  // namespace

int launch_refine(const RefineArgs& a, const CostTables& tab, bool last, cudaStream_t st) {
    const long long chunks = (a.g.pixels + kChunk - 1) / kChunk;
    dim3 grid(unsigned((chunks + 7) / 8), a.frames);
    // reciprocals for the exact small-integer divisions (div_small corrects them)
    const float inv_cell = 1.0f / float(a.cell), inv_w = 1.0f / float(a.g.width);
    const bool key32 = a.g.pixels <= (1ll << kIdxBits);
    if (a.g.pixels % 16 == 0 && key32 && a.g.width >= 32 && a.g.width + kTile < (1 << 16) &&
        a.g.height < (1 << 16) && a.cell < (1 << 15) && a.max_disp >= 0.0f &&
        a.max_disp <= float(kMaxHalo)) {
        // exact 16-bit magic reciprocals for the row / cell divisions (mdiv)
        const unsigned magic_w = unsigned((0x100000000ull + a.g.width - 1) / a.g.width);
        const unsigned magic_cell = unsigned((0x80000000ull + a.cell - 1) / a.cell);  // 2^31 / cell
        // at most one cell boundary in any four consecutive pixels
        const int tail = a.g.width % a.cell;
        const bool seg2 = a.cell >= 3 && (tail == 0 || tail >= 3);
        // a lane's four pixels cross a row end only when W % 4 != 0
        if (a.g.width % 4 == 0) {
            if (seg2)
                return last ? launch_bulk<true, 2, false>(a, tab, magic_cell, magic_w, st)
                            : launch_bulk<false, 2, false>(a, tab, magic_cell, magic_w, st);
            return last ? launch_bulk<true, 1, false>(a, tab, magic_cell, magic_w, st)
                        : launch_bulk<false, 1, false>(a, tab, magic_cell, magic_w, st);
        }
        if (seg2)
            return last ? launch_bulk<true, 2, true>(a, tab, magic_cell, magic_w, st)
                        : launch_bulk<false, 2, true>(a, tab, magic_cell, magic_w, st);
        return last ? launch_bulk<true, 1, true>(a, tab, magic_cell, magic_w, st)
                    : launch_bulk<false, 1, true>(a, tab, magic_cell, magic_w, st);
    }
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
