// frontend.cu — K1 (gradient mask + both census fields) and K2 (segment-test
// corners, per-bin top-k, global candidate sort).
//
// K1 replaces gradientMask (proj/src/image.cpp:43-60) and censusTransform
// (proj/src/census.cpp:10-41).  One 256-thread block stages a 128x8 tile of L
// and R plus a 2-px halo in shared memory (coalesced byte rows), each thread
// produces 4 horizontally adjacent pixels and writes them as one uint4 census
// word group and one uchar4 mask group when the row segment is 16-B aligned.
// HBM traffic is the algorithmic 11 B/px.
//
// K2 replaces detectCandidates (proj/src/sparse.cpp:84-146).  One block per
// (bin, frame): every thread keeps a sorted register top-k of packed keys
//   key = (4095 - score) << 40 | v << 20 | u
// (ascending key = score desc, v asc, u asc = byScoreThenRowMajor, :130-134),
// then the block merges the per-thread lists by repeated block-min.  A second
// kernel sorts the <= 120*cap survivors of each frame with a shared-memory
// bitonic sort.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ps {

namespace {

// K1 layout.  A block covers a 128 x 32 tile of the frame.  Shared memory
// holds the tile plus a 2-px halo as 32-bit words in a column-INTERLEAVED
// order: word (r, j) packs the bytes of tile columns j-2, j+30, j+62 and j+94
// (byte q = column j-2+32q) of tile row r-2.  Lane c of a warp then owns the
// four pixels c, c+32, c+64, c+96 of a row, and the 5x5 census window of all
// four is the 5x5 block of words (rows r-2..r+2, words c..c+4): one aligned
// 32-bit shared load per neighbour and no byte extraction.  The 24 census
// comparisons run four pixels per instruction group (SWAR, below), the
// outputs of a lane are warp-contiguous per q (coalesced 128-B census stores).
constexpr int kK1W = 128;             // tile columns (4 x 32)
constexpr int kK1H = 32;              // tile rows (8 warps x 4 rows)
constexpr int kK1Rows = kK1H + 4;     // staged rows (2-px halo above and below)
constexpr int kK1Words = 36;          // interleaved words per staged row (32 + halo)
constexpr int kK1RowsPerWarp = kK1H / 8;

// Byte-wise a < b flags in bit 7 of each byte (SWAR, no carries across
// bytes): d7 = [a_lo7 < b_lo7] from (b & 0x7f) + (~a & 0x7f); then
// a < b <=> (!a7 & b7) | (a7 == b7 & d7).  na = ~a & 0x7f7f7f7f and
// cb = b & 0x7f7f7f7f are computed once per word.
__device__ __forceinline__ uint32_t lt_flags(uint32_t a, uint32_t na, uint32_t b, uint32_t cb, uint32_t one) {
    // the add as an IMAD by a runtime 1: it issues on the FMA pipe, the LOP3s
    // on the ALU pipe
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(na), "r"(one), "r"(cb));
    uint32_t t;
    // f(a, b, d) = (~a & b) | (~(a ^ b) & d): truth table over (a, b, d) = (0xF0, 0xCC, 0xAA)
    asm("lop3.b32 %0, %1, %2, %3, 0x8e;" : "=r"(t) : "r"(a), "r"(b), "r"(d));
    return t;
}

// Census of the four interleaved pixels of the centre word w[2][2] of a 5x5
// word window: three accumulators hold bits 0-7, 8-15, 16-23 of the four
// descriptors, byte q for pixel q (bit k = k-th neighbour in row-major order,
// centre skipped, set when strictly darker: census.cpp:22-35).  Each
// comparison shifts its accumulator right by one and ORs its flags into bit 7,
// so after eight the first is in bit 0.  Per comparison and four pixels: two
// ALU-pipe LOP3s and two FMA-pipe IMADs (the two pipes issue in parallel).
__device__ __forceinline__ void census4(const uint32_t (&w)[5][5], const uint32_t (&nw)[5][5], uint32_t one,
                                        uint32_t& a0, uint32_t& a1, uint32_t& a2) {
    const uint32_t b = w[2][2], cb = b & 0x7f7f7f7fu;
    uint32_t acc[3] = {0u, 0u, 0u};
    int k = 0;
#pragma unroll
    for (int dv = 0; dv < 5; ++dv) {
#pragma unroll
        for (int du = 0; du < 5; ++du) {
            if (dv == 2 && du == 2) continue;
            const uint32_t t = lt_flags(w[dv][du], nw[dv][du], b, cb, one);
            // acc >> 1 as the high word of acc * 2^31 (FMA pipe; no carries
            // cross bytes: a byte holds at most 7 flags before this shift)
            acc[k >> 3] = __umulhi(acc[k >> 3], 0x80000000u) | (t & 0x80808080u);
            ++k;
        }
    }
    a0 = acc[0];
    a1 = acc[1];
    a2 = acc[2];
}

// descriptor of interleaved pixel q from the three accumulators
__device__ __forceinline__ uint32_t census_of(uint32_t a0, uint32_t a1, uint32_t a2, int q) {
    const uint32_t lo = __byte_perm(a0, a1, uint32_t(q) | uint32_t(4 + q) << 4);
    return __byte_perm(lo, a2, 0x0010u | uint32_t(4 + q) << 8) & 0x00ffffffu;
}

// Stage rows [v0-2, v0+kK1H+2) x columns [u0-2, u0+130) of both images into
// the interleaved words (zeros outside the image; those bytes only feed
// border pixels, whose census and mask are 0).  Thread i builds word
// (r, j) = i from its four bytes (columns j-2+32q: for each q the warp's
// lanes read consecutive bytes); all of a thread's loads are issued before
// its first shared store.
constexpr int kK1Src = kK1Rows * kK1Words;          // interleaved words per image
constexpr int kK1SrcIt = (kK1Src + 255) / 256;      // per thread

__device__ __forceinline__ uint32_t k1_word(const uint8_t* __restrict__ img, int W, int H, int u0, int v0,
                                            int i) {
    const int r = i / kK1Words, j = i - r * kK1Words;
    const int gv = v0 - 2 + r, gu = u0 + j - 2;
    uint32_t x = 0;
    if (i < kK1Src && gv >= 0 && gv < H) {
        const uint8_t* row = img + (long long)gv * W;
        if (gu >= 0 && gu + 96 < W) {  // all four columns inside (most words)
            const uint8_t* q = row + gu;
            x = __byte_perm(__byte_perm(uint32_t(__ldg(q)), uint32_t(__ldg(q + 32)), 0x0040u),
                            __byte_perm(uint32_t(__ldg(q + 64)), uint32_t(__ldg(q + 96)), 0x0040u), 0x5410u);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int u = gu + 32 * q;
                if (u >= 0 && u < W) x |= uint32_t(__ldg(row + u)) << (8 * q);
            }
        }
    }
    return x;
}

__global__ void __launch_bounds__(256, 4) k_frontend(const uint8_t* __restrict__ left,
                                                  const uint8_t* __restrict__ right, FrameGeom g,
                                                  int thr, uint8_t* __restrict__ mask,
                                                  uint32_t* __restrict__ cl,
                                                  uint32_t* __restrict__ cr,
                                                  int* __restrict__ mask_count,
                                                  uint8_t* __restrict__ code, uint8_t code_high) {
    __shared__ uint32_t sl[kK1Rows][kK1Words];
    __shared__ uint32_t sr[kK1Rows][kK1Words];
    __shared__ int warp_cnt[8];
    const int f = blockIdx.z;
    const int W = g.width, H = g.height;
    const int u0 = blockIdx.x * kK1W;
    const int v0 = blockIdx.y * kK1H;
    const uint8_t* L = left + f * g.pixels;
    const uint8_t* R = right ? right + f * g.pixels : nullptr;
    {
        const int tid = threadIdx.y * 32 + threadIdx.x;
        uint32_t xl[kK1SrcIt], xr[kK1SrcIt];
#pragma unroll
        for (int it = 0; it < kK1SrcIt; ++it) {
            xl[it] = k1_word(L, W, H, u0, v0, tid + 256 * it);
            xr[it] = R ? k1_word(R, W, H, u0, v0, tid + 256 * it) : 0u;
        }
        uint32_t* fl = &sl[0][0];
        uint32_t* fr = &sr[0][0];
#pragma unroll
        for (int it = 0; it < kK1SrcIt; ++it) {
            const int i = tid + 256 * it;
            if (i < kK1Src) {
                fl[i] = xl[it];
                if (R) fr[i] = xr[it];
            }
        }
    }
    __syncthreads();

    const int c = threadIdx.x, wy = threadIdx.y;
    const uint32_t one = W != 0 ? 1u : 0u;  // 1, opaque to the compiler (see lt_flags)
    // gradient threshold in 16-bit lanes: grad in [0, 510]
    const int tc = thr < 0 ? 0 : (thr > 511 ? 511 : thr);
    const uint32_t tbias = uint32_t(0x8000 - tc) * 0x00010001u;
    // interior test per pixel (u in [2, W-2)) and in-frame test (u < W) of the
    // lane's four columns
    uint32_t colok = 0, colin = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int u = u0 + c + 32 * q;
        colok |= uint32_t(u >= 2 && u < W - 2) << q;
        colin |= uint32_t(u < W) << q;
    }
    int cnt = 0;
    const int y0 = wy * kK1RowsPerWarp;  // first tile row of this warp
    const long long fb = f * g.pixels + u0 + c;
    const bool want_mask = mask || code || mask_count;
    // one view at a time (half the live window registers): L with the
    // gradient mask and code, then R; the rows fully unrolled (a row past the
    // frame only stores nothing), so the window slides by renaming
#pragma unroll 1
    for (int view = 0; view < (R ? 2 : 1); ++view) {
        const uint32_t(*sw)[kK1Words] = view ? sr : sl;
        uint32_t* cen = view ? cr : cl;
        uint32_t w[5][5], nw[5][5];
#pragma unroll
        for (int dv = 0; dv < 4; ++dv)
#pragma unroll
            for (int du = 0; du < 5; ++du) {
                w[dv + 1][du] = sw[y0 + dv][c + du];
                nw[dv + 1][du] = ~w[dv + 1][du] & 0x7f7f7f7fu;
            }
#pragma unroll
        for (int i = 0; i < kK1RowsPerWarp; ++i) {
            // slide the window one row down: staged rows y0+i .. y0+i+4
#pragma unroll
            for (int dv = 0; dv < 4; ++dv)
#pragma unroll
                for (int du = 0; du < 5; ++du) {
                    w[dv][du] = w[dv + 1][du];
                    nw[dv][du] = nw[dv + 1][du];
                }
#pragma unroll
            for (int du = 0; du < 5; ++du) {
                w[4][du] = sw[y0 + i + 4][c + du];
                nw[4][du] = ~w[4][du] & 0x7f7f7f7fu;
            }
            const int v = v0 + y0 + i;
            const bool row_ok = v < H;  // warp-uniform
            const uint32_t ok = (v >= 2 && v < H - 2) ? colok : 0u;
            const uint32_t st = row_ok ? colin : 0u;
            const long long rb = fb + (long long)v * W;
            if (cen && st) {
                uint32_t a0, a1, a2;
                census4(w, nw, one, a0, a1, a2);
                uint32_t* crow = cen + rb;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if ((st >> q) & 1u) crow[32 * q] = ((ok >> q) & 1u) ? census_of(a0, a1, a2, q) : 0u;
            }
            if (view == 0 && want_mask && st) {
                // |L(u+1)-L(u-1)| + |L(v+1)-L(v-1)| >= threshold (image.cpp:43-60), 16-bit lanes
                const uint32_t gh = __vabsdiffu4(w[2][3], w[2][1]);
                const uint32_t gv = __vabsdiffu4(w[3][2], w[1][2]);
                const uint32_t ge = (gh & 0x00ff00ffu) + (gv & 0x00ff00ffu) + tbias;                // pixels 0, 2
                const uint32_t go = ((gh >> 8) & 0x00ff00ffu) + ((gv >> 8) & 0x00ff00ffu) + tbias;  // 1, 3
                const uint32_t mk =
                    (((ge >> 15) & 1u) | ((go >> 14) & 2u) | ((ge >> 29) & 4u) | ((go >> 28) & 8u)) & ok;
                cnt += __popc(mk);
                uint8_t* mrow = mask ? mask + rb : nullptr;
                uint8_t* crow8 = code ? code + rb : nullptr;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!((st >> q) & 1u)) continue;
                    const bool m = (mk >> q) & 1u;
                    if (mrow) mrow[32 * q] = m ? 1 : 0;
                    if (crow8) crow8[32 * q] = m ? code_high : kCodeOff;
                }
            }
        }
    }
    if (mask_count) {
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (threadIdx.x == 0) warp_cnt[threadIdx.y] = cnt;
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0) {
            int s = 0;
            for (int i = 0; i < 8; ++i) s += warp_cnt[i];
            if (s) atomicAdd(mask_count + f, s);
        }
    }
}

// ---------------------------------------------------------------- K2

// Bresenham circle of radius 3, clockwise from 12 o'clock (sparse.cpp:12-15).
__constant__ int8_t c_ring_u[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
__constant__ int8_t c_ring_v[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

__device__ __forceinline__ bool arc9(unsigned m16) {
    // contiguous run >= 9 on the 16-ring (sparse.cpp:22-36): x has a run of
    // length >= 9 iff the 9-fold AND of its rotations is non-zero.
    unsigned r = m16 | (m16 << 16);
    unsigned a = r;
#pragma unroll
    for (int s = 1; s < 9; ++s) a &= r >> s;
    return (a & 0xffffu) != 0;
}

// Segment test at (u, v) (sparse.cpp:94-122) on a shared-memory tile,
// p(k) = s[base + off[k]]; returns the score (> 0, >= 9 for any accepted
// corner) or 0.  The four compass pixels first, so a rejected pixel (the vast
// majority) costs five shared loads.
__device__ __forceinline__ int corner_score_s(const uint8_t* __restrict__ s, int base,
                                              const int (&off)[16], int t) {
    const int c = s[base];
    const int hi = c + t, lo = c - t;
    const int p0 = s[base + off[0]], p4 = s[base + off[4]], p8 = s[base + off[8]],
              p12 = s[base + off[12]];
    const int nb = (p0 > hi) + (p4 > hi) + (p8 > hi) + (p12 > hi);
    const int nd = (p0 < lo) + (p4 < lo) + (p8 < lo) + (p12 < lo);
    if (nb < 2 && nd < 2) return 0;
    unsigned bright = 0, dark = 0;
    int score = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int p = s[base + off[k]];
        bright |= unsigned(p > hi) << k;
        dark |= unsigned(p < lo) << k;
        score += max(0, abs(p - c) - t);
    }
    if (!arc9(bright) && !arc9(dark)) return 0;
    return score;
}

// Stage the bin [ulo, uhi) x [vlo, vhi) plus the 3-pixel ring halo into
// shared memory (row stride sw) and set up the ring offsets.  Rows vlo-3 ..
// vhi+2 and columns ulo-3 .. uhi+2 are inside the image (bin_range keeps a
// 3-pixel margin).
__device__ __forceinline__ void stage_bin(const uint8_t* __restrict__ L, int W, int ulo, int uhi,
                                          int vlo, int vhi, uint8_t* __restrict__ s, int sw,
                                          int (&off)[16]) {
    const int tw = uhi - ulo + 6, th = vhi - vlo + 6;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r < th; r += nw) {
        const uint8_t* src = L + (long long)(vlo - 3 + r) * W + (ulo - 3);
        for (int c = lane; c < tw; c += 32) s[r * sw + c] = __ldg(src + c);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) off[k] = c_ring_v[k] * sw + c_ring_u[k];
    __syncthreads();
}

__device__ __forceinline__ unsigned long long corner_key(int score, int u, int v) {
    return (unsigned long long)(4095 - score) << 40 | (unsigned long long)v << 20 |
           (unsigned long long)u;
}

// Pixel range [lo, hi) of bin b among nb bins over an axis of n pixels,
// intersected with [3, n-3): bin(x) = min(nb-1, x*nb/n) (sparse.cpp:124-125).
__device__ __forceinline__ void bin_range(int b, int nb, int n, int& lo, int& hi) {
    lo = (b * n + nb - 1) / nb;
    hi = (b == nb - 1) ? n : ((b + 1) * n + nb - 1) / nb;
    lo = max(lo, 3);
    hi = min(hi, n - 3);
}

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long x,
                                                            unsigned long long* red) {
    x = warp_min_u64(x);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long y = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : kEmptyCell;
        y = warp_min_u64(y);
        if (threadIdx.x == 0) red[32] = y;
    }
    __syncthreads();
    return red[32];
}

template <int LK>
__global__ void __launch_bounds__(256) k_corner_bins(const uint8_t* __restrict__ left, FrameGeom g,
                                                     int t, int cap,
                                                     unsigned long long* __restrict__ bin_keys,
                                                     int* __restrict__ bin_count) {
    __shared__ unsigned long long lists[256][LK];
    __shared__ unsigned long long red[33];
    extern __shared__ uint8_t s_tile[];
    const int f = blockIdx.y, bin = blockIdx.x;
    const int bu = bin % 12, bv = bin / 12;
    int ulo, uhi, vlo, vhi;
    bin_range(bu, 12, g.width, ulo, uhi);
    bin_range(bv, 10, g.height, vlo, vhi);
    const uint8_t* L = left + f * g.pixels;
    unsigned long long best[LK];
#pragma unroll
    for (int k = 0; k < LK; ++k) best[k] = kEmptyCell;
    const int bw = uhi - ulo, bh = vhi - vlo;
    if (bw > 0 && bh > 0) {  // block-uniform
        const int sw = bw + 6;
        int off[16];
        stage_bin(L, g.width, ulo, uhi, vlo, vhi, s_tile, sw, off);
        const int n = bw * bh;
        // (u, v) of pixel i = tid + 256 j, advanced without divisions
        int cu = int(threadIdx.x) % bw, cv = int(threadIdx.x) / bw;
        const int su = int(blockDim.x) % bw, sv = int(blockDim.x) / bw;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int u = ulo + cu, v = vlo + cv;
            const int s = corner_score_s(s_tile, (cv + 3) * sw + cu + 3, off, t);
            cu += su;
            cv += sv;
            if (cu >= bw) {
                cu -= bw;
                ++cv;
            }
            if (s == 0) continue;
            unsigned long long key = corner_key(s, u, v);
            if (key >= best[LK - 1]) continue;
#pragma unroll
            for (int k = 0; k < LK; ++k) {  // sorted insertion
                const unsigned long long lo = key < best[k] ? key : best[k];
                const unsigned long long hi = key < best[k] ? best[k] : key;
                best[k] = lo;
                key = hi;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < LK; ++k) lists[threadIdx.x][k] = best[k];
    int head = 0;
    int out = 0;
    for (; out < cap; ++out) {
        const unsigned long long mine = head < LK ? lists[threadIdx.x][head] : kEmptyCell;
        const unsigned long long m = block_min_u64(mine, red);
        if (m == kEmptyCell) break;
        if (mine == m) ++head;  // keys are unique pixels: exactly one owner
        if (threadIdx.x == 0) bin_keys[((long long)f * 120 + bin) * cap + out] = m;
    }
    if (threadIdx.x == 0) bin_count[f * 120 + bin] = out;
}

// Generic per-bin selection for caps above the register top-k width: all
// corner keys of the bin go to global scratch, then `cap` block-min rounds.
__global__ void __launch_bounds__(256) k_corner_bins_generic(
    const uint8_t* __restrict__ left, FrameGeom g, int t, int cap,
    unsigned long long* __restrict__ scratch, long long scratch_stride,
    unsigned long long* __restrict__ bin_keys, int* __restrict__ bin_count) {
    __shared__ unsigned long long red[33];
    __shared__ int n_keys;
    extern __shared__ uint8_t s_tile[];
    const int f = blockIdx.y, bin = blockIdx.x;
    const int bu = bin % 12, bv = bin / 12;
    int ulo, uhi, vlo, vhi;
    bin_range(bu, 12, g.width, ulo, uhi);
    bin_range(bv, 10, g.height, vlo, vhi);
    const uint8_t* L = left + f * g.pixels;
    unsigned long long* sc = scratch + ((long long)f * 120 + bin) * scratch_stride;
    if (threadIdx.x == 0) n_keys = 0;
    __syncthreads();
    const int bw = uhi - ulo, bh = vhi - vlo;
    if (bw > 0 && bh > 0) {  // block-uniform
        const int sw = bw + 6;
        int off[16];
        stage_bin(L, g.width, ulo, uhi, vlo, vhi, s_tile, sw, off);
        const int n = bw * bh;
        int cu = int(threadIdx.x) % bw, cv = int(threadIdx.x) / bw;
        const int su = int(blockDim.x) % bw, sv = int(blockDim.x) / bw;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int u = ulo + cu, v = vlo + cv;
            const int s = corner_score_s(s_tile, (cv + 3) * sw + cu + 3, off, t);
            cu += su;
            cv += sv;
            if (cu >= bw) {
                cu -= bw;
                ++cv;
            }
            if (s == 0) continue;
            sc[atomicAdd(&n_keys, 1)] = corner_key(s, u, v);
        }
    }
    __syncthreads();
    const int nk = n_keys;
    unsigned long long last = 0;
    int out = 0;
    for (; out < cap && out < nk; ++out) {
        unsigned long long mine = kEmptyCell;
        for (int i = threadIdx.x; i < nk; i += blockDim.x) {
            const unsigned long long k = sc[i];
            if ((out == 0 || k > last) && k < mine) mine = k;
        }
        const unsigned long long m = block_min_u64(mine, red);
        if (m == kEmptyCell) break;
        last = m;
        if (threadIdx.x == 0) bin_keys[((long long)f * 120 + bin) * cap + out] = m;
    }
    if (threadIdx.x == 0) bin_count[f * 120 + bin] = out;
}

// Bitonic sort of n (power of two) keys by one block; data in shared or global memory.
__device__ void bitonic_sort(unsigned long long* d, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = d[i], b = d[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        d[i] = b;
                        d[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(1024) k_candidate_sort(
    const unsigned long long* __restrict__ bin_keys, const int* __restrict__ bin_count, int cap,
    int n_pow2, unsigned long long* __restrict__ global_buf, int* __restrict__ cand_u,
    int* __restrict__ cand_v, float* __restrict__ cand_score, int* __restrict__ cand_count,
    int cand_stride) {
    extern __shared__ unsigned long long sm_keys[];
    __shared__ int offs[121];
    const int f = blockIdx.x;
    unsigned long long* keys = global_buf ? global_buf + (long long)f * n_pow2 : sm_keys;
    if (threadIdx.x == 0) {
        int s = 0;
        for (int b = 0; b < 120; ++b) {
            offs[b] = s;
            s += bin_count[f * 120 + b];
        }
        offs[120] = s;
    }
    __syncthreads();
    const int n = offs[120];
    for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) keys[i] = kEmptyCell;
    __syncthreads();
    for (int b = 0; b < 120; ++b) {
        const int c = offs[b + 1] - offs[b];
        for (int i = threadIdx.x; i < c; i += blockDim.x)
            keys[offs[b] + i] = bin_keys[((long long)f * 120 + b) * cap + i];
    }
    __syncthreads();
    bitonic_sort(keys, n_pow2);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long k = keys[i];
        const long long o = (long long)f * cand_stride + i;
        cand_u[o] = int(k & 0xfffff);
        cand_v[o] = int((k >> 20) & 0xfffff);
        if (cand_score) cand_score[o] = float(4095 - int(k >> 40));
    }
    if (threadIdx.x == 0) cand_count[f] = n;
}

}  // namespace

int launch_frontend(const uint8_t* left, const uint8_t* right, FrameGeom g, int frames,
                    int grad_threshold, uint8_t* mask, uint32_t* cl, uint32_t* cr,
                    int* mask_count, cudaStream_t st, uint8_t* code, int code_high) {
    dim3 grid((g.width + kK1W - 1) / kK1W, (g.height + kK1H - 1) / kK1H, frames);
    k_frontend<<<grid, dim3(32, 8), 0, st>>>(left, right, g, grad_threshold, mask, cl, cr,
                                             mask_count, code, uint8_t(code_high));
    return 1;
}

long long candidate_scratch_stride(FrameGeom g) {
    const long long bw = (g.width + 11) / 12 + 1, bh = (g.height + 9) / 10 + 1;
    return bw * bh;
}

int launch_candidates(const uint8_t* left, FrameGeom g, int frames, int corner_threshold, int cap,
                      unsigned long long* bin_keys, int* bin_count, unsigned long long* scratch,
                      long long scratch_stride, int* cand_u, int* cand_v, float* cand_score,
                      int* cand_count, int cand_stride, cudaStream_t st) {
    dim3 grid(120, frames);
    // bin tile + ring halo (bins are at most ceil(n/nb) + 1 wide, bin_range)
    const size_t tile = size_t((g.width + 11) / 12 + 1 + 6) * size_t((g.height + 9) / 10 + 1 + 6);
    // per-device function attribute: set before every launch that needs it
    auto allow = [&](const void* fn, int, size_t static_bytes) {
        if (tile + static_bytes > 48 * 1024)
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tile));
    };
    if (cap <= 4) {
        allow((const void*)k_corner_bins<4>, 0, 256 * 4 * 8 + 264);
        k_corner_bins<4><<<grid, 256, tile, st>>>(left, g, corner_threshold, cap, bin_keys, bin_count);
    } else if (cap == 5) {  // the default perBinCap (config.hpp): a top-5 per thread
        allow((const void*)k_corner_bins<5>, 0, 256 * 5 * 8 + 264);
        k_corner_bins<5><<<grid, 256, tile, st>>>(left, g, corner_threshold, cap, bin_keys, bin_count);
    } else if (cap <= 8) {
        allow((const void*)k_corner_bins<8>, 1, 256 * 8 * 8 + 264);
        k_corner_bins<8><<<grid, 256, tile, st>>>(left, g, corner_threshold, cap, bin_keys, bin_count);
    } else {
        allow((const void*)k_corner_bins_generic, 2, 272);
        k_corner_bins_generic<<<grid, 256, tile, st>>>(left, g, corner_threshold, cap, scratch,
                                                       scratch_stride, bin_keys, bin_count);
    }
    const int n = 120 * cap;
    int n_pow2 = 1;
    while (n_pow2 < n) n_pow2 <<= 1;
    const bool in_smem = n_pow2 <= 8192;
    const size_t smem = in_smem ? size_t(n_pow2) * 8 : 0;
    if (in_smem && smem > 48 * 1024) {
        cudaFuncSetAttribute(k_candidate_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
    }
    // Large caps sort in global memory: reuse the corner scratch (>= n_pow2 keys per frame).
    k_candidate_sort<<<frames, 1024, smem, st>>>(bin_keys, bin_count, cap, n_pow2,
                                                 in_smem ? nullptr : scratch, cand_u, cand_v,
                                                 cand_score, cand_count, cand_stride);
    return 2;
}

}  // namespace ps
