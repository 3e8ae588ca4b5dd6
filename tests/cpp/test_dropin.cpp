// test_dropin.cpp — the reference's own unit tests (proj/tests/test_*.cpp),
// re-expressed against the drop-in C++ API (include/planestereo/*.hpp) and
// run on the GPU.  Includes only the reference's header names, as a user of
// the reference would.  Built by __graft_entry__.build() (tests/cpp/Makefile),
// run by tests/test_gpu_dropin.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "planestereo/census.hpp"
#include "planestereo/config.hpp"
#include "planestereo/delaunay.hpp"
#include "planestereo/eval.hpp"
#include "planestereo/image.hpp"
#include "planestereo/mesh.hpp"
#include "planestereo/pipeline.hpp"
#include "planestereo/sparse.hpp"
#include "planestereo/synth.hpp"
#include "planestereo_c.h"

using namespace planestereo;

namespace {

struct Case {
    const char* name;
    std::function<void()> fn;
};
std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
int g_fail = 0;
const char* g_case = "";
#define TEST(name) \
    static void name(); \
    static Reg reg_##name(#name, name); \
    static void name()
#define CHECK(cond)                                                                   \
    do {                                                                              \
        if (!(cond)) {                                                                \
            ++g_fail;                                                                 \
            std::printf("FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_case, #cond); \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, Ex)              \
    do {                                       \
        bool thrown = false;                   \
        try {                                  \
            (void)(expr);                      \
        } catch (const Ex&) {                  \
            thrown = true;                     \
        } catch (...) {                        \
        }                                      \
        CHECK(thrown && #Ex);                  \
    } while (0)

// testutil::randomImage (proj/tests/testutil.hpp:10-17)
GrayImage randomImage(int w, int h, std::uint32_t seed) {
    std::mt19937 rng(seed);
    std::vector<std::uint8_t> px(std::size_t(w) * h);
    for (auto& p : px) p = std::uint8_t(rng() & 0xffu);
    return GrayImage(w, h, std::move(px));
}

GrayImage shiftLeftBy(const GrayImage& img, int shift, std::uint32_t seed) {
    GrayImage out = randomImage(img.width(), img.height(), seed);
    for (int v = 0; v < img.height(); ++v)
        for (int u = 0; u + shift < img.width(); ++u) out.at(u, v) = img.at(u + shift, v);
    return out;
}

std::pair<GrayImage, GrayImage> synthPair(int w, int h, int planes, int nd, std::uint32_t seed) {
    ps_synth_params p{w, h, planes, nd, 0, 2.0f, seed};
    std::vector<std::uint8_t> L(std::size_t(w) * h), R(std::size_t(w) * h);
    ps_synth_pair(&p, L.data(), R.data(), nullptr);
    return {GrayImage(w, h, L), GrayImage(w, h, R)};
}

DisparityMap constantMap(int w, int h, float d) {
    DisparityMap m(w, h);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) m.set(u, v, d);
    return m;
}

double inCircleDet(const Pixel& a, const Pixel& b, const Pixel& c, const Pixel& d) {
    const double adx = a.u - d.u, ady = a.v - d.v, bdx = b.u - d.u, bdy = b.v - d.v;
    const double cdx = c.u - d.u, cdy = c.v - d.v;
    const double aq = adx * adx + ady * ady, bq = bdx * bdx + bdy * bdy, cq = cdx * cdx + cdy * cdy;
    return adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) + aq * (bdx * cdy - cdx * bdy);
}

}  // namespace

// ----------------------------------------------------------- test_core.cpp
TEST(image_minimum_size) {
    CHECK_THROWS_AS(GrayImage(15, 64), DimensionTooSmall);
    CHECK_THROWS_AS(GrayImage(64, 15), DimensionTooSmall);
    CHECK_THROWS_AS(GrayImage(16, 16, std::vector<std::uint8_t>(10)), DimensionMismatch);
    GrayImage ok(16, 16, 7);
    CHECK(ok.at(3, 5) == 7);
}

TEST(gradient_mask_cases) {
    CHECK(gradientMask(GrayImage(32, 32, 100), 1).count() == 0);
    const GradientMask all = gradientMask(randomImage(20, 18, 99), 0);
    CHECK(all.count() == (20 - 4) * (18 - 4));
    for (const Pixel& p : all.points()) CHECK(p.u >= 2 && p.v >= 2 && p.u < 18 && p.v < 16);
    GrayImage step(16, 16, 50);
    for (int v = 0; v < 16; ++v)
        for (int u = 8; u < 16; ++u) step.at(u, v) = 150;
    const GradientMask m = gradientMask(step, 20);
    CHECK(m.count() == 24);
    for (const Pixel& p : m.points()) CHECK(p.u == 7 || p.u == 8);
    const GrayImage img = randomImage(48, 40, 7);
    const GradientMask loose = gradientMask(img, 10), tight = gradientMask(img, 35);
    CHECK(tight.count() <= loose.count());
    for (const Pixel& p : tight.points()) CHECK(loose.contains(p.u, p.v));
}

TEST(census_known_answers) {
    const CensusField flat = censusTransform(GrayImage(16, 16, 77));
    for (int v = 2; v < 14; ++v)
        for (int u = 2; u < 14; ++u) CHECK(flat.at(u, v) == 0);
    CHECK(!flat.valid(1, 8));
    CHECK(!flat.valid(8, 14));
    GrayImage dot(16, 16, 50);
    dot.at(8, 8) = 100;
    CHECK(censusTransform(dot).at(8, 8) == 0x00ffffffu);
    GrayImage ramp(16, 16, 0);
    for (int v = 0; v < 16; ++v)
        for (int u = 0; u < 16; ++u) ramp.at(u, v) = std::uint8_t(10 * (u + 1));
    std::uint32_t expected = 0;
    int bit = 0;
    for (int dv = -2; dv <= 2; ++dv)
        for (int du = -2; du <= 2; ++du) {
            if (dv == 0 && du == 0) continue;
            if (ramp.at(4 + du, 4 + dv) < ramp.at(4, 4)) expected |= 1u << bit;
            ++bit;
        }
    CHECK(censusTransform(ramp).at(4, 4) == expected);
    CHECK(censusCost(0x123456u, 0x123456u) == 0.0f);
    CHECK(censusCost(0x00ffffffu, 0x0u) == 1.0f);
}

TEST(census_translation_covariance) {
    const GrayImage img = randomImage(40, 32, 5);
    GrayImage shifted(40, 32, 0);
    for (int v = 0; v < 32; ++v)
        for (int u = 0; u < 40; ++u)
            if (u - 3 >= 0 && v - 2 >= 0) shifted.at(u, v) = img.at(u - 3, v - 2);
    const CensusField a = censusTransform(img), b = censusTransform(shifted);
    for (int v = 4; v < 30; ++v)
        for (int u = 5; u < 38; ++u) CHECK(a.at(u - 3, v - 2) == b.at(u, v));
}

TEST(config_validation) {
    PipelineConfig cfg;
    cfg.validate();
    PipelineConfig bad = cfg;
    bad.iterations = 0;
    CHECK_THROWS_AS(bad.validate(), InvalidConfig);
    bad = cfg;
    bad.costLow = 0.6f;
    CHECK_THROWS_AS(bad.validate(), InvalidConfig);
    bad = cfg;
    bad.occupancyCellSize = 24;
    CHECK_THROWS_AS(bad.validate(), InvalidConfig);
    bad = cfg;
    bad.maxDisparity = 0;
    CHECK_THROWS_AS(bad.validate(), InvalidConfig);
}

// ----------------------------------------------------------- test_sparse.cpp
TEST(corner_candidates) {
    PipelineConfig cfg;
    CHECK(detectCandidates(GrayImage(64, 48, 120), cfg).empty());
    GrayImage dot(16, 16, 0);
    dot.at(8, 8) = 255;
    const auto c = detectCandidates(dot, cfg);
    CHECK(c.size() == 1);
    if (!c.empty()) CHECK(c[0].u == 8 && c[0].v == 8 && c[0].score > 0.0f);
    const auto cand = detectCandidates(randomImage(64, 64, 9), cfg);
    for (std::size_t i = 1; i < cand.size(); ++i) {
        const auto& a = cand[i - 1];
        const auto& b = cand[i];
        CHECK(a.score > b.score || (a.score == b.score && (a.v < b.v || (a.v == b.v && a.u < b.u))));
    }
}

TEST(matching_properties) {
    PipelineConfig cfg;
    const GrayImage img = randomImage(80, 64, 12);
    const auto self = matchEpipolar(img, img, detectCandidates(img, cfg), cfg);
    CHECK(!self.empty());
    for (const auto& s : self) CHECK(s.d == 0.0);
    const GrayImage left = randomImage(64, 48, 5);
    const GrayImage right = shiftLeftBy(left, 9, 77);
    std::vector<CandidatePixel> border{{3, 20, 1.0f}, {3, 30, 1.0f}, {3, 40, 1.0f}};
    for (const auto& s : matchEpipolar(left, right, border, cfg)) CHECK(s.d <= 1.0);
    for (std::uint32_t seed = 0; seed < 10; ++seed) {
        const GrayImage l = randomImage(72, 56, seed), r = randomImage(72, 56, seed + 50);
        for (const auto& s : matchEpipolar(l, r, detectCandidates(l, cfg), cfg)) {
            CHECK(s.d >= 0.0 && s.d < cfg.maxDisparity && s.u - s.d >= 2.0);
            CHECK(s.u >= 2 && s.u < 70 && s.v >= 2 && s.v < 54);
        }
    }
    const GrayImage l1 = randomImage(80, 60, 1), r1 = shiftLeftBy(l1, 4, 2);
    const auto cand = detectCandidates(l1, cfg);
    CHECK(matchEpipolar(l1, r1, cand, cfg) == matchEpipolar(l1, r1, cand, cfg));
    const GrayImage l2 = randomImage(64, 48, 3);
    std::vector<CandidatePixel> twice{{20, 20, 1.0f}, {20, 20, 2.0f}, {30, 25, 1.0f}};
    int at = 0;
    for (const auto& s : matchEpipolar(l2, l2, twice, cfg)) at += (s.u == 20 && s.v == 20);
    CHECK(at <= 1);
}

// ----------------------------------------------------------- test_delaunay.cpp
TEST(delaunay_cases) {
    CHECK(orient2d({0, 0}, {4, 0}, {0, 4}) > 0);
    CHECK(orient2d({0, 0}, {0, 4}, {4, 0}) < 0);
    CHECK(orient2d({0, 0}, {4, 4}, {8, 8}) == 0);
    CHECK(inCircleSign({0, 0}, {4, 0}, {0, 4}, {1, 1}) > 0);
    CHECK(inCircleSign({0, 0}, {4, 0}, {0, 4}, {9, 9}) < 0);
    CHECK(inCircleSign({0, 0}, {4, 0}, {0, 4}, {4, 4}) == 0);
    CHECK(delaunayTriangulate({}).empty());
    CHECK(delaunayTriangulate({{0, 0}, {4, 2}, {8, 4}, {12, 6}, {16, 8}}).empty());
    CHECK(delaunayTriangulate({{0, 0}, {10, 0}, {4, 8}}).size() == 1);
    const std::vector<Pixel> square{{0, 0}, {8, 0}, {0, 8}, {8, 8}};
    const auto two = delaunayTriangulate(square);
    CHECK(two.size() == 2);
    const auto dup = delaunayTriangulate({{0, 0}, {8, 0}, {4, 6}, {8, 0}, {0, 0}});
    CHECK(dup.size() == 1);
    for (const auto& t : dup)
        for (int i : t) CHECK(i <= 2);
    std::vector<Pixel> grid;
    for (int v = 0; v < 7; ++v)
        for (int u = 0; u < 7; ++u) grid.push_back({4 * u, 4 * v});
    const auto tris = delaunayTriangulate(grid);
    CHECK(tris.size() == 72);
    for (const auto& t : tris)
        for (const Pixel& p : grid) CHECK(inCircleDet(grid[t[0]], grid[t[1]], grid[t[2]], p) <= 1e-9);
    std::mt19937 rng(42);
    std::set<std::pair<int, int>> seen;
    std::vector<Pixel> pts;
    while (pts.size() < 40) {
        Pixel p{int(rng() % 64), int(rng() % 64)};
        if (std::find(pts.begin(), pts.end(), p) == pts.end()) pts.push_back(p);
    }
    for (const auto& t : delaunayTriangulate(pts))
        for (int i = 0; i < 3; ++i) CHECK(seen.insert({t[i], t[(i + 1) % 3]}).second);
}

// ----------------------------------------------------------- test_mesh.cpp
TEST(mesh_cases) {
    const DisparityPlane flat = fitPlane({0, 0, 10}, {10, 0, 10}, {0, 10, 10});
    CHECK(std::abs(flat.a) < 1e-12 && std::abs(flat.b) < 1e-12 && std::abs(flat.c - 10.0) < 1e-12);
    const DisparityPlane slope = fitPlane({0, 0, 0}, {16, 0, 8}, {0, 16, 0});
    CHECK(std::abs(slope.a - 0.5) < 1e-12);
    CHECK_THROWS_AS(fitPlane({0, 0, 5}, {8, 0, 5}, {16, 0, 5}), DegenerateTriangle);
    CHECK_THROWS_AS(triangulate({{2, 2, 1}, {10, 2, 1}}, 32, 32), FewerThanThreePoints);
    const DisparityMesh line = triangulate({{2, 2, 1}, {6, 6, 1}, {10, 10, 1}, {14, 14, 1}}, 32, 32);
    CHECK(line.triangles().empty());
    for (int v = 0; v < 32; ++v)
        for (int u = 0; u < 32; ++u) CHECK(line.triangleAt(u, v) == DisparityMesh::kOutside);
    const DisparityMesh mesh = triangulate({{0, 0, 0}, {16, 0, 8}, {0, 16, 0}}, 32, 32);
    const DisparityMap full = interpolate(mesh, 128.0f);
    CHECK(full.valid(8, 4) && std::abs(full.at(8, 4) - 4.0f) < 1e-6f);
    CHECK(!full.valid(30, 30));
    const DisparityMap capped = interpolate(mesh, 4.0f);
    CHECK(!capped.valid(10, 2) && capped.valid(4, 4));
    const DisparityMesh two = triangulate({{2, 2, 4}, {22, 2, 8}, {2, 22, 4}, {22, 22, 8}}, 32, 32);
    CHECK(two.triangles().size() == 2);
    const DisparityMap full2 = interpolate(two, 128.0f);
    for (const SupportPoint& p : two.vertices())
        CHECK(full2.valid(p.u, p.v) && std::abs(full2.at(p.u, p.v) - p.d) < 1e-6);
    std::ostringstream off;
    triangulate({{2, 2, 5}, {20, 2, 5}, {10, 18, 5}}, 32, 32).writeOff(off);
    CHECK(off.str().rfind("OFF\n3 1 0\n", 0) == 0);
}

// ----------------------------------------------------------- test_pipeline.cpp
TEST(cost_evaluation_cases) {
    const GrayImage img = randomImage(64, 48, 4);
    const GradientMask mask = gradientMask(img, 20);
    const CensusField census = censusTransform(img);
    const CostMap zero = costEvaluation(census, census, constantMap(64, 48, 0.0f), mask);
    CHECK(mask.count() > 0);
    for (const Pixel& p : mask.points()) CHECK(zero.at(p.u, p.v) == 0.0f);
    DisparityMap tooFar(64, 48);
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u) tooFar.set(u, v, float(u + 5));
    const CostMap far = costEvaluation(census, census, tooFar, mask);
    for (const Pixel& p : mask.points()) CHECK(far.at(p.u, p.v) == 1.0f);
    const CostMap inv = costEvaluation(census, census, DisparityMap(64, 48), mask);
    for (const Pixel& p : mask.points()) CHECK(inv.at(p.u, p.v) == 1.0f);
}

TEST(refinement_known_answer) {
    PipelineConfig cfg;
    GradientMask mask(32, 32);
    mask.add(10, 10);
    mask.add(11, 10);
    mask.add(20, 12);
    DisparityMap interpolated(32, 32);
    interpolated.set(10, 10, 6.0f);
    interpolated.set(11, 10, 6.5f);
    interpolated.set(20, 12, 9.0f);
    CostMap costs(32, 32, 1.0f);
    costs.set(10, 10, 0.10f);
    costs.set(11, 10, 0.05f);
    costs.set(20, 12, 0.30f);
    DisparityMap fd(32, 32);
    CostMap fc(32, 32, cfg.costHigh);
    const RefinementGrids g = disparityRefinement(interpolated, costs, fd, fc, mask, 32, cfg);
    CHECK(fd.at(10, 10) == 6.0f && fc.at(10, 10) == 0.10f);
    CHECK(fd.at(20, 12) == 9.0f && fc.at(20, 12) == 0.30f);
    const OccupancyCell& c = g.confident.cellForPixel(10, 10);
    CHECK(c.occupied && c.u == 11 && c.v == 10 && c.cost == 0.05f && c.disparity == 6.5f);
    CHECK(!g.invalid.cellForPixel(20, 12).occupied);
    GradientMask mask2(32, 32);
    mask2.add(5, 5);
    mask2.add(6, 5);
    CostMap costs2(32, 32, 1.0f);
    costs2.set(5, 5, 0.8f);
    costs2.set(6, 5, 0.9f);
    DisparityMap interp2(32, 32);
    interp2.set(5, 5, 1.0f);
    interp2.set(6, 5, 1.0f);
    const RefinementGrids g2 = disparityRefinement(interp2, costs2, fd, fc, mask2, 32, cfg);
    const OccupancyCell& bad = g2.invalid.cellForPixel(5, 5);
    CHECK(bad.occupied && bad.u == 6 && bad.cost == 0.9f);
    const OccupancyGrid grid(100, 70, 32, 0.5f);
    CHECK(grid.cols() == 4 && grid.rows() == 3);
}

TEST(resampling_known_answer) {
    const CensusField census = censusTransform(randomImage(64, 48, 10));
    PipelineConfig cfg;
    const std::vector<SupportPoint> supports{{10, 10, 3.0}, {40, 30, 5.0}};
    OccupancyGrid empty(64, 48, 32, cfg.costLow), emptyBad(64, 48, 32, cfg.costHigh);
    CHECK(supportResampling(empty, emptyBad, supports, census, census, cfg) == supports);
    OccupancyGrid confident(64, 48, 32, cfg.costLow);
    confident.cell(1, 1) = {40, 40, 12.3f, 0.08f, true};
    const auto grown = supportResampling(confident, emptyBad, supports, census, census, cfg);
    CHECK(grown.size() == 3);
    if (grown.size() == 3) CHECK(grown[2].u == 40 && grown[2].v == 40 && std::abs(grown[2].d - 12.3) < 1e-5);
    OccupancyGrid duplicate(64, 48, 32, cfg.costLow);
    duplicate.cell(0, 0) = {10, 10, 9.0f, 0.01f, true};
    const auto same = supportResampling(duplicate, emptyBad, supports, census, census, cfg);
    CHECK(same.size() == 2 && same[0].d == 3.0);
}

TEST(run_contract) {
    const auto [L, R] = synthPair(128, 96, 4, 32, 5);
    PipelineConfig cfg;
    cfg.iterations = 7;
    cfg.maxDisparity = 32;
    const StereoResult r = run(L, R, cfg);
    const std::vector<int> cells{32, 16, 8, 4, 2, 1, 1};
    CHECK(r.trace.size() == 7);
    for (int i = 0; i < 7 && i < int(r.trace.size()); ++i) CHECK(r.trace[i].occupancyCellSize == cells[i]);
    for (std::size_t i = 1; i < r.trace.size(); ++i) {
        CHECK(r.trace[i].supportCount >= r.trace[i - 1].supportCount);
        CHECK(r.trace[i].meanCost <= r.trace[i - 1].meanCost + 1e-9);
    }
    for (int v = 0; v < 96; ++v)
        for (int u = 0; u < 128; ++u) CHECK(r.disparity.valid(u, v) == (r.costs.at(u, v) < cfg.costHigh));
    std::vector<std::vector<float>> hist;
    cfg.iterations = 4;
    run(L, R, cfg, [&](int, const DisparityMap&, const CostMap& c) { hist.push_back(c.values()); });
    CHECK(hist.size() == 4);
    for (std::size_t it = 1; it < hist.size(); ++it)
        for (std::size_t i = 0; i < hist[it].size(); ++i) CHECK(hist[it][i] <= hist[it - 1][i]);
    const StereoResult a = run(L, R, cfg), b = run(L, R, cfg);
    CHECK(a.disparity.values() == b.disparity.values() && a.costs.values() == b.costs.values());
    CHECK(a.dense.values() == b.dense.values());
    const auto batch = runBatch({L, L}, {R, R}, cfg);
    CHECK(batch.size() == 2 && batch[1].costs.values() == a.costs.values());
}

TEST(run_errors) {
    PipelineConfig cfg;
    const GrayImage flat(64, 48, 128);
    CHECK_THROWS_AS(run(flat, flat, cfg), SeedingFailed);
    CHECK_THROWS_AS(run(GrayImage(64, 48, 0), GrayImage(48, 64, 0), cfg), DimensionMismatch);
    PipelineConfig bad;
    bad.iterations = 0;
    CHECK_THROWS_AS(run(flat, flat, bad), InvalidConfig);
    PipelineConfig grid10;
    grid10.occupancyCellSize = 10;
    CHECK_THROWS_AS(run(flat, flat, grid10), InvalidConfig);
    const auto [L, R] = synthPair(96, 72, 4, 32, 9);
    grid10.maxDisparity = 32;
    grid10.iterations = 2;
    const StereoResult r = runUnchecked(L, R, grid10);
    CHECK(r.trace.size() == 2 && r.trace[1].occupancyCellSize == 5);
}

// ----------------------------------------------------------- test_synth.cpp
TEST(wta_oracle_cases) {
    // identical images: d = 0 and cost 0 on every mask pixel (test_synth.cpp:82-91)
    const GrayImage img = randomImage(64, 48, 5);
    const GradientMask mask = gradientMask(img, 20);
    const auto [disparity, costs] = wtaOracle(img, img, mask, 128);
    for (const Pixel& p : mask.points()) {
        CHECK(disparity.valid(p.u, p.v));
        CHECK(disparity.at(p.u, p.v) == 0.0f);
        CHECK(costs.at(p.u, p.v) == 0.0f);
    }
    // a pure shift of 7 (right = left moved left by 7) is found wherever the
    // true match is in range and unique; off-mask pixels keep cost 1.0
    const GrayImage R = shiftLeftBy(img, 7, 6);
    const auto [d7, c7] = wtaOracle(img, R, mask, 16);
    int exact = 0, n = 0;
    for (const Pixel& p : mask.points())
        if (p.u >= 16 + 2 && p.u + 2 < 64 - 7) {
            ++n;
            exact += d7.at(p.u, p.v) == 7.0f;
        }
    CHECK(n > 100 && exact * 10 >= n * 9);
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u)
            if (!mask.contains(u, v)) CHECK(c7.at(u, v) == 1.0f && !d7.valid(u, v));
    CHECK_THROWS_AS(wtaOracle(img, GrayImage(32, 48, 0), mask, 8), DimensionMismatch);
}

TEST(render_scene_cases) {
    // fronto-parallel plane: the right view is the left shifted by d, nothing
    // occluded, truth d everywhere and valid iff u >= d (test_synth.cpp:10-28)
    const RenderedScene flat = renderScene(PlanarScene::flat(20.0, 64, 48));
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u + 20 < 64; ++u) CHECK(flat.right.at(u, v) == flat.left.at(u + 20, v));
    int occluded = 0;
    for (std::uint8_t o : flat.occlusion) occluded += o;
    CHECK(occluded == 0);
    // (test_synth.cpp:22-27 expects the value 20 at every pixel, but the
    // reference's renderScene invalidates out-of-view pixels with
    // DisparityMap::invalidate, which zeroes the value (disparity.hpp:22-25);
    // this build follows the implementation, bit for bit)
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u) {
            CHECK(flat.groundTruth.at(u, v) == (u >= 20 ? 20.0f : 0.0f));
            CHECK(flat.groundTruth.valid(u, v) == (u >= 20));
        }
    // a slanted plane's truth is the plane itself where valid (test_synth.cpp:30-38;
    // occluded and out-of-view pixels are zeroed as above)
    const RenderedScene slant = renderScene(PlanarScene::slanted(0.25, 0.0, 4.0, 64, 48));
    CHECK(slant.groundTruth.at(32, 10) == 12.0f);
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u)
            CHECK(slant.groundTruth.valid(u, v) ? slant.groundTruth.at(u, v) == float(0.25 * u + 4.0)
                                                 : slant.groundTruth.at(u, v) == 0.0f);
    // near right half over a far left half: 20 occluded px per row, all in
    // [w/2 - 20, w/2) and invalid (test_synth.cpp:40-58)
    const RenderedScene st = renderScene(PlanarScene::steps(10.0, 30.0, 64, 48));
    for (int v = 0; v < 48; ++v) {
        int row = 0;
        for (int u = 0; u < 64; ++u)
            if (st.occlusion[std::size_t(v) * 64 + u]) {
                ++row;
                CHECK(u >= 32 - 20 && u < 32);
                CHECK(!st.groundTruth.valid(u, v));
            }
        CHECK(row == 20);
    }
    // planes leaving [0, maxDisparity) are rejected (test_synth.cpp:60-65)
    CHECK_THROWS_AS(renderScene(PlanarScene::flat(-1.0, 64, 48)), InvalidPlane);
    CHECK_THROWS_AS(renderScene(PlanarScene::flat(130.0, 64, 48)), InvalidPlane);
    CHECK_THROWS_AS(renderScene(PlanarScene::slanted(2.0, 0.0, 10.0, 64, 48)), InvalidPlane);
    // deterministic for a seed; textured enough for the default gradient mask
    const RenderedScene a = renderScene(PlanarScene::flat(12.0, 64, 48, 99));
    const RenderedScene b = renderScene(PlanarScene::flat(12.0, 64, 48, 99));
    CHECK(a.left.data() == b.left.data() && a.right.data() == b.right.data());
    CHECK(a.groundTruth.values() == b.groundTruth.values());
    CHECK(gradientMask(renderScene(PlanarScene::flat(5.0, 64, 48)).left, 20).count() > (64 - 4) * (48 - 4) / 2);
    // the WTA oracle recovers a rendered constant shift (test_synth.cpp:92-108)
    const RenderedScene s7 = renderScene(PlanarScene::flat(7.0, 96, 64));
    const GradientMask m7 = gradientMask(s7.left, 20);
    const auto [d7, c7] = wtaOracle(s7.left, s7.right, m7, 128);
    int evaluated = 0, exact = 0;
    for (const Pixel& p : m7.points()) {
        if (!s7.groundTruth.valid(p.u, p.v) || !d7.valid(p.u, p.v)) continue;
        ++evaluated;
        exact += d7.at(p.u, p.v) == 7.0f;
    }
    // (test_synth.cpp:107 asks for 99%; the reference implementation itself
    // reaches 96.5% on this scene — tests/test_oracle.py pins the exact rate)
    CHECK(evaluated > 500 && exact >= 0.96 * evaluated);
}

// ----------------------------------------------------------- test_eval.cpp
TEST(accuracy_cases) {
    const DisparityMap gt = renderScene(PlanarScene::flat(15.0, 64, 48)).groundTruth;
    // identical maps: every fraction 1, zero error (test_eval.cpp:28-36)
    const AccuracyReport same = accuracy(gt, gt, {2.0, 3.0, 4.0, 5.0});
    CHECK(same.evaluated > 0 && same.meanAbsError == 0.0);
    for (double f : same.fractions) CHECK(f == 1.0);
    // a constant +5 px offset: strict thresholds 3 and 5 fail, 6 passes
    DisparityMap shifted(64, 48);
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u)
            if (gt.valid(u, v)) shifted.set(u, v, gt.at(u, v) + 5.0f);
    const AccuracyReport off = accuracy(shifted, gt, {3.0, 5.0, 6.0});
    CHECK(off.fractions[0] == 0.0 && off.fractions[1] == 0.0 && off.fractions[2] == 1.0);
    CHECK(std::fabs(off.meanAbsError - 5.0) < 1e-12);
    // symmetric in its arguments and monotone in the threshold
    const RenderedScene sl = renderScene(PlanarScene::slanted(0.1, 0.05, 8.0, 64, 48));
    DisparityMap noisy(64, 48);
    std::mt19937 rng(5);
    for (int v = 0; v < 48; ++v)
        for (int u = 0; u < 64; ++u)
            if (sl.groundTruth.valid(u, v)) noisy.set(u, v, sl.groundTruth.at(u, v) + float(int(rng() % 7)) - 3.0f);
    const std::vector<double> th{1.0, 2.0, 3.0, 4.0};
    const AccuracyReport ab = accuracy(noisy, sl.groundTruth, th), ba = accuracy(sl.groundTruth, noisy, th);
    for (std::size_t i = 0; i < th.size(); ++i) {
        CHECK(ab.fractions[i] == ba.fractions[i]);
        if (i) CHECK(ab.fractions[i] >= ab.fractions[i - 1]);
    }
    // the evaluated set is prediction-valid AND truth-valid AND in the mask
    DisparityMap p1(64, 48), g1(64, 48);
    GradientMask mk(64, 48);
    p1.set(10, 10, 5.0f);
    p1.set(20, 20, 5.0f);
    g1.set(10, 10, 5.0f);
    g1.set(30, 30, 5.0f);
    mk.add(10, 10);
    mk.add(21, 20);
    CHECK(accuracy(p1, g1, mk, {1.0}).evaluated == 1);
    // more thresholds than one device call takes
    std::vector<double> many;
    for (int i = 1; i <= 40; ++i) many.push_back(0.25 * i);
    const AccuracyReport big = accuracy(noisy, sl.groundTruth, many);
    CHECK(big.fractions.size() == 40 && big.fractions[3] == ab.fractions[0] && big.fractions[39] == 1.0);
    // disjoint maps raise NoOverlap; sizes must agree (test_eval.cpp:85-94)
    DisparityMap a(32, 32), b(32, 32), c(16, 32);
    a.set(2, 2, 1.0f);
    b.set(3, 3, 1.0f);
    CHECK_THROWS_AS(accuracy(a, b, {1.0}), NoOverlap);
    CHECK_THROWS_AS(accuracy(a, c, {1.0}), DimensionMismatch);
}

int main() {
    for (const Case& c : cases()) {
        g_case = c.name;
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL [%s] unexpected exception: %s\n", c.name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", c.name);
    }
    std::printf("%zu cases, %d failed checks\n", cases().size(), g_fail);
    return g_fail == 0 ? 0 : 1;
}
