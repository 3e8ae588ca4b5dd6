// synth.cpp — seeded BASELINE-style stereo pair generator.
//
// Bench/test fixture only; it is not on the hot path.  BASELINE.json's
// configs describe KITTI-like synthetic scenes; no dataset exists in this
// image, so this generator stands in for them:
//   * disparity map: a piecewise-constant background of 4x3 blocks, an
//     optional ground region whose disparity rises linearly with the row,
//     then `n_planes` random rectangular planar patches with base disparity
//     in [0, ND-1] and slopes U(-0.05, 0.05) px/px (clamped to [0, ND-1]);
//   * left view: 3x3 box filter of uniform bytes;
//   * right view: the left forward-warped by lround(d), the nearest (largest
//     d) source winning each right pixel; unfilled pixels keep fresh uniform
//     bytes; then + N(0, sigma), rounded and clamped to uint8.
// Only raw std::mt19937 32-bit draws are used (a standardised engine), with an
// explicit Box-Muller transform, so the stream does not depend on the
// standard library's distribution implementations.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "planestereo_c.h"

namespace {

struct Rng {
    explicit Rng(uint32_t seed) : eng(seed) {}
    uint32_t next() { return uint32_t(eng()); }
    double uniform() { return next() * (1.0 / 4294967296.0); }          // [0,1)
    int range(int lo, int hi) { return lo + int(next() % uint32_t(hi - lo + 1)); }
    double gaussian() {  // Box-Muller, one draw per call
        const double u1 = (double(next()) + 1.0) * (1.0 / 4294967297.0);  // (0,1)
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
    std::mt19937 eng;
};

}  // namespace

extern "C" ps_status ps_synth_pair(const ps_synth_params* p, uint8_t* left, uint8_t* right,
                                   float* gt) {
    if (!p || !left || !right) return PS_ERROR;
    const int w = p->width, h = p->height, nd = std::max(1, p->max_disparity);
    if (w < 16 || h < 16) return PS_DIMENSION_TOO_SMALL;
    const std::size_t P = std::size_t(w) * h;
    Rng rng(p->seed);
    std::vector<float> disp(P);

    // Background: 4x3 blocks of constant disparity in the far range.
    const int bw = (w + 3) / 4, bh = (h + 2) / 3;
    float block[12];
    for (float& b : block) b = float(rng.range(0, std::max(0, (nd - 1) / 3)));
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) disp[std::size_t(v) * w + u] = block[(v / bh) * 4 + (u / bw)];

    // Ground: bottom 40% of the rows, disparity rising linearly to ~0.9*(ND-1).
    if (p->ground) {
        const int v0 = int(0.6 * h);
        const double d0 = double((nd - 1) / 4);
        const double d1 = 0.9 * (nd - 1);
        for (int v = v0; v < h; ++v) {
            const float d = float(d0 + (d1 - d0) * double(v - v0) / double(std::max(1, h - 1 - v0)));
            for (int u = 0; u < w; ++u) disp[std::size_t(v) * w + u] = d;
        }
    }

    // Random planar patches, painted in order.
    for (int k = 0; k < p->n_planes; ++k) {
        const int pw = rng.range(std::max(2, w / 16), std::max(3, w / 4));
        const int ph = rng.range(std::max(2, h / 16), std::max(3, h / 4));
        const int u0 = rng.range(0, w - 1), v0 = rng.range(0, h - 1);
        const double base = double(rng.range(0, nd - 1));
        const double gu = (rng.uniform() - 0.5) * 0.1;
        const double gv = (rng.uniform() - 0.5) * 0.1;
        const double cu = u0 + 0.5 * pw, cv = v0 + 0.5 * ph;
        for (int v = v0; v < std::min(h, v0 + ph); ++v)
            for (int u = u0; u < std::min(w, u0 + pw); ++u) {
                double d = base + gu * (u - cu) + gv * (v - cv);
                d = std::min(std::max(d, 0.0), double(nd - 1));
                disp[std::size_t(v) * w + u] = float(d);
            }
    }

    // Left view: 3x3 box filter (clipped at the border) of uniform bytes.
    std::vector<uint8_t> raw(P);
    for (auto& x : raw) x = uint8_t(rng.next() & 0xffu);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            int sum = 0, n = 0;
            for (int dv = -1; dv <= 1; ++dv) {
                const int vv = v + dv;
                if (vv < 0 || vv >= h) continue;
                for (int du = -1; du <= 1; ++du) {
                    const int uu = u + du;
                    if (uu < 0 || uu >= w) continue;
                    sum += raw[std::size_t(vv) * w + uu];
                    ++n;
                }
            }
            left[std::size_t(v) * w + u] = uint8_t(sum / n);
        }

    // Right view: fresh noise, overwritten by the forward warp (nearest wins).
    for (std::size_t i = 0; i < P; ++i) right[i] = uint8_t(rng.next() & 0xffu);
    std::vector<float> best(w);
    std::vector<int> src(w);
    for (int v = 0; v < h; ++v) {
        std::fill(best.begin(), best.end(), -1.0f);
        std::fill(src.begin(), src.end(), -1);
        const float* drow = disp.data() + std::size_t(v) * w;
        for (int u = 0; u < w; ++u) {
            const int ur = int(std::lround(double(u) - drow[u]));
            if (ur < 0 || ur >= w) continue;
            if (drow[u] > best[ur] || (drow[u] == best[ur] && u > src[ur])) {
                best[ur] = drow[u];
                src[ur] = u;
            }
        }
        for (int ur = 0; ur < w; ++ur)
            if (src[ur] >= 0) right[std::size_t(v) * w + ur] = left[std::size_t(v) * w + src[ur]];
    }
    if (p->noise_sigma > 0.0f) {
        for (std::size_t i = 0; i < P; ++i) {
            const double x = double(right[i]) + double(p->noise_sigma) * rng.gaussian();
            right[i] = uint8_t(std::min(255.0, std::max(0.0, std::nearbyint(x))));
        }
    }
    if (gt) std::copy(disp.begin(), disp.end(), gt);
    return PS_OK;
}

extern "C" ps_status ps_synth_batch(const ps_synth_params* p, int n_frames, int threads,
                                    uint8_t* left, uint8_t* right) {
    if (!p || n_frames < 0) return PS_ERROR;
    const std::size_t P = std::size_t(p->width) * p->height;
    threads = std::max(1, std::min(threads, std::max(1, n_frames)));
    std::vector<std::thread> pool;
    std::vector<ps_status> st(threads, PS_OK);
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            for (int f = t; f < n_frames; f += threads) {
                ps_synth_params q = *p;
                q.seed = p->seed + uint32_t(f);
                const ps_status s = ps_synth_pair(&q, left + f * P, right + f * P, nullptr);
                if (s != PS_OK) st[t] = s;
            }
        });
    }
    for (auto& th : pool) th.join();
    for (ps_status s : st)
        if (s != PS_OK) return s;
    return PS_OK;
}
