// planestereo.cpp — the drop-in C++ API (include/planestereo/planestereo.hpp)
// implemented over the C ABI (include/planestereo_c.h).
//
// Value types and list bookkeeping live here (host); every per-pixel or
// per-candidate computation goes through a ps_* entry point, i.e. the sm_100a
// kernels.  Scalar geometry helpers (orient2d, inCircleSign, fitPlane) are
// evaluated inline with the reference's exact arithmetic (delaunay.cpp:11-41,
// mesh.cpp:12-26); DisparityMesh's planes and lookup come from the device.
#include <algorithm>
#include <cstdlib>
#include <ostream>
#include <string>

#include "planestereo/planestereo.hpp"
#include "planestereo_c.h"

namespace planestereo {

namespace {

[[noreturn]] void raise(ps_status s, const char* fallback = nullptr) {
    const char* m = ps_last_error(nullptr);
    const std::string msg = (m && *m) ? m : (fallback ? fallback : "planestereo error");
    switch (s) {
        case PS_INVALID_CONFIG: throw InvalidConfig(msg);
        case PS_DIMENSION_TOO_SMALL: throw DimensionTooSmall(msg);
        case PS_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case PS_FEWER_THAN_THREE_POINTS: throw FewerThanThreePoints(msg);
        case PS_DEGENERATE_TRIANGLE: throw DegenerateTriangle(msg);
        case PS_SEEDING_FAILED: throw SeedingFailed(msg);
        case PS_NEGATIVE_DISPARITY: throw NegativeDisparity(msg);
        case PS_EMPTY_CLOUD: throw EmptyCloud(msg);
        case PS_NO_OVERLAP: throw NoOverlap(msg);
        case PS_INVALID_PLANE: throw InvalidPlane(msg);
        default: throw Error(msg);
    }
}

void check(ps_status s) {
    if (s != PS_OK) raise(s);
}

struct ThreadContext {
    int device = 0;
    ps_ctx* ctx = nullptr;
    ~ThreadContext() {
        if (ctx) ps_ctx_destroy(ctx);
    }
    ps_ctx* get() {
        if (!ctx) check(ps_ctx_create(device, &ctx));
        return ctx;
    }
};

thread_local ThreadContext t_ctx;

ps_ctx* ctx() { return t_ctx.get(); }

ps_config to_c(const PipelineConfig& c) {
    return ps_config{c.iterations,        c.maxDisparity,     c.costLow,         c.costHigh,
                     c.gradientThreshold, c.occupancyCellSize, c.cornerThreshold, c.perBinCap,
                     c.sparseAcceptCost,  c.uniquenessRatio,  c.threads};
}

StereoResult run_impl(const GrayImage& left, const GrayImage& right, const PipelineConfig& config,
                      const IterationObserver& observer, unsigned flags) {
    // precedence of run(): InvalidConfig, then DimensionMismatch (pipeline.cpp:133-136)
    const ps_config c = to_c(config);
    check(ps_config_validate(&c, flags));
    if (!left.sameSize(right)) throw DimensionMismatch("stereo pair dimensions differ");
    const int w = left.width(), h = left.height();
    StereoResult r{DisparityMap(w, h), CostMap(w, h, config.costHigh), DisparityMap(w, h), {}};
    std::vector<ps_iter_stats> trace(config.iterations);
    struct Obs {
        const IterationObserver* fn;
    } obs{&observer};
    auto tramp = [](int it, const float* fd, const uint8_t* fv, const float* fc, int ww, int hh,
                    void* user) {
        const Obs* o = static_cast<const Obs*>(user);
        DisparityMap d(ww, hh);
        CostMap cm(ww, hh, 0.0f);
        const std::size_t n = std::size_t(ww) * hh;
        std::copy(fd, fd + n, d.mutableValues().begin());
        std::copy(fv, fv + n, d.mutableValidity().begin());
        std::copy(fc, fc + n, cm.mutableValues().begin());
        (*o->fn)(it, d, cm);
    };
    check(ps_run(ctx(), left.data().data(), right.data().data(), w, h, &c, flags,
                 r.disparity.mutableValues().data(), r.disparity.mutableValidity().data(),
                 r.costs.mutableValues().data(), r.dense.mutableValues().data(),
                 r.dense.mutableValidity().data(), trace.data(), observer ? +tramp : nullptr,
                 &obs));
    for (const ps_iter_stats& s : trace)
        r.trace.push_back({s.iteration, s.support_count, s.triangle_count, s.occupancy_cell_size,
                           s.mean_cost, s.valid_count, s.millis});
    return r;
}

}  // namespace

// ------------------------------------------------------------------ config
void PipelineConfig::validate() const {
    const ps_config c = to_c(*this);
    check(ps_config_validate(&c, 0));
}

// ------------------------------------------------------------------ images
GrayImage::GrayImage(int width, int height, std::uint8_t fill)
    : w_(width), h_(height) {
    if (width < kMinDimension || height < kMinDimension)
        throw DimensionTooSmall("image must be at least 16x16, got " + std::to_string(width) +
                                "x" + std::to_string(height));
    px_.assign(std::size_t(width) * height, fill);
}

GrayImage::GrayImage(int width, int height, std::vector<std::uint8_t> data)
    : w_(width), h_(height), px_(std::move(data)) {
    if (width < kMinDimension || height < kMinDimension)
        throw DimensionTooSmall("image must be at least 16x16, got " + std::to_string(width) +
                                "x" + std::to_string(height));
    if (px_.size() != std::size_t(width) * height)
        throw DimensionMismatch("pixel buffer size does not match image dimensions");
}

GradientMask::GradientMask(int width, int height)
    : w_(width), h_(height), in_(std::size_t(width) * height, 0) {}

void GradientMask::add(int u, int v) {
    std::uint8_t& m = in_[std::size_t(v) * w_ + u];
    if (!m) {
        m = 1;
        pts_.push_back({u, v});
    }
}

GradientMask gradientMask(const GrayImage& image, int threshold) {
    const int w = image.width(), h = image.height();
    std::vector<std::uint8_t> member(std::size_t(w) * h);
    int count = 0;
    check(ps_gradient_mask(ctx(), image.data().data(), w, h, threshold, member.data(), &count));
    GradientMask m(w, h);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u)
            if (member[std::size_t(v) * w + u]) m.add(u, v);
    return m;
}

DisparityMap::DisparityMap(int width, int height)
    : w_(width), h_(height), val_(std::size_t(width) * height, 0.0f),
      ok_(std::size_t(width) * height, 0) {}

int DisparityMap::validCount() const {
    int n = 0;
    for (std::uint8_t b : ok_) n += b == 1;
    return n;
}

CostMap::CostMap(int width, int height, float fill)
    : w_(width), h_(height), c_(std::size_t(width) * height, fill) {}

CensusField::CensusField(int width, int height)
    : w_(width), h_(height), d_(std::size_t(width) * height, 0) {}

CensusField censusTransform(const GrayImage& image, int /*threads: the GPU grid*/) {
    CensusField f(image.width(), image.height());
    check(ps_census(ctx(), image.data().data(), image.width(), image.height(),
                    f.mutableWords().data()));
    return f;
}

// ------------------------------------------------------------------ sparse
std::vector<CandidatePixel> detectCandidates(const GrayImage& image, const PipelineConfig& config) {
    const ps_config c = to_c(config);
    const int cap = 120 * std::max(1, config.perBinCap);
    std::vector<int> u(cap), v(cap);
    std::vector<float> s(cap);
    int n = 0;
    check(ps_detect_candidates(ctx(), image.data().data(), image.width(), image.height(), &c,
                               u.data(), v.data(), s.data(), cap, &n));
    std::vector<CandidatePixel> out(n);
    for (int i = 0; i < n; ++i) out[i] = {u[i], v[i], s[i]};
    return out;
}

std::vector<SupportPoint> matchEpipolar(const CensusField& left, const CensusField& right,
                                        const std::vector<CandidatePixel>& candidates,
                                        const PipelineConfig& config) {
    const ps_config c = to_c(config);
    const int n = int(candidates.size());
    std::vector<int> cu(n), cv(n);
    for (int i = 0; i < n; ++i) {
        cu[i] = candidates[i].u;
        cv[i] = candidates[i].v;
    }
    std::vector<int> u(n + 1), v(n + 1);
    std::vector<double> d(n + 1);
    int m = 0;
    check(ps_match_epipolar(ctx(), left.words().data(), right.words().data(), left.width(),
                            left.height(), cu.data(), cv.data(), n, &c, u.data(), v.data(),
                            d.data(), n + 1, &m));
    std::vector<SupportPoint> out(m);
    for (int i = 0; i < m; ++i) out[i] = {u[i], v[i], d[i]};
    return out;
}

std::vector<SupportPoint> matchEpipolar(const GrayImage& left, const GrayImage& right,
                                        const std::vector<CandidatePixel>& candidates,
                                        const PipelineConfig& config) {
    return matchEpipolar(censusTransform(left, config.threads),
                         censusTransform(right, config.threads), candidates, config);
}

// ------------------------------------------------------------------ delaunay
long long orient2d(const Pixel& a, const Pixel& b, const Pixel& c) {
    return ((long long)b.u - a.u) * ((long long)c.v - a.v) -
           ((long long)b.v - a.v) * ((long long)c.u - a.u);
}

int inCircleSign(const Pixel& a, const Pixel& b, const Pixel& c, const Pixel& d) {
    const long long adx = (long long)a.u - d.u, ady = (long long)a.v - d.v;
    const long long bdx = (long long)b.u - d.u, bdy = (long long)b.v - d.v;
    const long long cdx = (long long)c.u - d.u, cdy = (long long)c.v - d.v;
    const long long aq = adx * adx + ady * ady, bq = bdx * bdx + bdy * bdy,
                    cq = cdx * cdx + cdy * cdy;
    using W = __int128;
    const W det = W(adx) * (W(bdy) * cq - W(cdy) * bq) - W(ady) * (W(bdx) * cq - W(cdx) * bq) +
                  W(aq) * (W(bdx) * cdy - W(cdx) * bdy);
    return (det > 0) - (det < 0);
}

std::vector<std::array<int, 3>> delaunayTriangulate(const std::vector<Pixel>& points) {
    const int n = int(points.size());
    std::vector<int> u(n), v(n);
    for (int i = 0; i < n; ++i) {
        u[i] = points[i].u;
        v[i] = points[i].v;
    }
    std::vector<int> tris(6 * std::size_t(n) + 6);
    int nt = 0;
    check(ps_delaunay(u.data(), v.data(), n, tris.data(), 2 * n + 2, &nt));
    std::vector<std::array<int, 3>> out(nt);
    for (int t = 0; t < nt; ++t) out[t] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    return out;
}

// ------------------------------------------------------------------ mesh
DisparityPlane fitPlane(const SupportPoint& p1, const SupportPoint& p2, const SupportPoint& p3) {
    // mesh.cpp:12-26 (this file is compiled with -ffp-contract=off)
    const long long u1 = p1.u, u2 = p2.u, u3 = p3.u, w1 = p1.v, w2 = p2.v, w3 = p3.v;
    const long long det = u1 * (w2 - w3) + u2 * (w3 - w1) + u3 * (w1 - w2);
    if (det == 0)
        throw DegenerateTriangle("collinear vertices at (" + std::to_string(p1.u) + "," +
                                 std::to_string(p1.v) + ")");
    const double d1 = p1.d, d2 = p2.d, d3 = p3.d;
    const double dA = d1 * double(w2 - w3) + d2 * double(w3 - w1) + d3 * double(w1 - w2);
    const double dB = double(u1) * (d2 - d3) + double(u2) * (d3 - d1) + double(u3) * (d1 - d2);
    const double dC = d1 * double(u2 * w3 - u3 * w2) - d2 * double(u1 * w3 - u3 * w1) +
                      d3 * double(u1 * w2 - u2 * w1);
    return {dA / double(det), dB / double(det), dC / double(det)};
}

DisparityMesh::DisparityMesh(std::vector<SupportPoint> vertices,
                             std::vector<std::array<int, 3>> triangles, int width, int height)
    : verts_(std::move(vertices)), tris_(std::move(triangles)),
      lookup_(std::size_t(width) * height, kOutside), w_(width), h_(height) {
    const int n = int(verts_.size()), nt = int(tris_.size());
    std::vector<int> u(n), v(n), t(3 * std::size_t(nt));
    std::vector<double> d(n);
    for (int i = 0; i < n; ++i) {
        u[i] = verts_[i].u;
        v[i] = verts_[i].v;
        d[i] = verts_[i].d;
    }
    for (int i = 0; i < nt; ++i)
        for (int k = 0; k < 3; ++k) t[3 * i + k] = tris_[i][k];
    std::vector<double> pl(3 * std::size_t(nt) + 3);
    check(ps_mesh_build(ctx(), u.data(), v.data(), d.data(), n, t.data(), nt, width, height,
                        pl.data(), lookup_.data()));
    planes_.resize(nt);
    for (int i = 0; i < nt; ++i) planes_[i] = {pl[3 * i], pl[3 * i + 1], pl[3 * i + 2]};
}

void DisparityMesh::writeOff(std::ostream& out) const {
    out << "OFF\n" << verts_.size() << ' ' << tris_.size() << " 0\n";
    for (const SupportPoint& p : verts_) out << p.u << ' ' << p.v << ' ' << p.d << '\n';
    for (const auto& t : tris_) out << "3 " << t[0] << ' ' << t[1] << ' ' << t[2] << '\n';
}

DisparityMesh triangulate(const std::vector<SupportPoint>& points, int width, int height) {
    if (points.size() < 3)
        throw FewerThanThreePoints("triangulation needs at least 3 support points, got " +
                                   std::to_string(points.size()));
    std::vector<Pixel> px(points.size());
    for (std::size_t i = 0; i < points.size(); ++i) px[i] = {points[i].u, points[i].v};
    return DisparityMesh(points, delaunayTriangulate(px), width, height);
}

static DisparityMap interpolate_impl(const DisparityMesh& mesh, const std::uint8_t* mask,
                                     float maxDisparity) {
    const int w = mesh.width(), h = mesh.height();
    DisparityMap map(w, h);
    const auto& planes = mesh.planes();
    std::vector<double> pl(3 * planes.size() + 3);
    for (std::size_t i = 0; i < planes.size(); ++i) {
        pl[3 * i] = planes[i].a;
        pl[3 * i + 1] = planes[i].b;
        pl[3 * i + 2] = planes[i].c;
    }
    check(ps_interpolate(ctx(), mesh.lookup().data(), pl.data(), int(planes.size()), w, h, mask,
                         maxDisparity, map.mutableValues().data(), map.mutableValidity().data()));
    return map;
}

DisparityMap interpolate(const DisparityMesh& mesh, const GradientMask& domain, float maxDisparity) {
    return interpolate_impl(mesh, domain.membership().data(), maxDisparity);
}

DisparityMap interpolate(const DisparityMesh& mesh, float maxDisparity) {
    return interpolate_impl(mesh, nullptr, maxDisparity);
}

// ------------------------------------------------------------------ pipeline
OccupancyGrid::OccupancyGrid(int imageWidth, int imageHeight, int cellSize, float initialCost)
    : size_(cellSize), cols_((imageWidth + cellSize - 1) / cellSize),
      rows_((imageHeight + cellSize - 1) / cellSize) {
    cells_.resize(std::size_t(cols_) * rows_);
    for (auto& c : cells_) c.cost = initialCost;
}

CostMap costEvaluation(const CensusField& left, const CensusField& right,
                       const DisparityMap& interpolated, const GradientMask& mask, int) {
    CostMap costs(left.width(), left.height(), 1.0f);
    check(ps_cost_evaluation(ctx(), left.words().data(), right.words().data(), left.width(),
                             left.height(), interpolated.values().data(),
                             interpolated.validity().data(), mask.membership().data(),
                             costs.mutableValues().data()));
    return costs;
}

std::pair<DisparityMap, CostMap> wtaOracle(const GrayImage& left, const GrayImage& right,
                                           const GradientMask& mask, int maxDisparity) {
    if (left.width() != right.width() || left.height() != right.height() ||
        mask.width() != left.width() || mask.height() != left.height())
        throw DimensionMismatch("wtaOracle inputs differ in size");
    DisparityMap disparity(left.width(), left.height());
    CostMap costs(left.width(), left.height(), 1.0f);
    check(ps_wta_oracle(ctx(), left.data().data(), right.data().data(), left.width(),
                        left.height(), mask.membership().data(), maxDisparity,
                        disparity.mutableValues().data(), disparity.mutableValidity().data(),
                        costs.mutableValues().data()));
    return {std::move(disparity), std::move(costs)};
}

namespace {
AccuracyReport accuracy_impl(const DisparityMap& prediction, const DisparityMap& groundTruth,
                             const GradientMask* mask, const std::vector<double>& thresholds) {
    const int w = prediction.width(), h = prediction.height();
    if (groundTruth.width() != w || groundTruth.height() != h ||
        (mask && (mask->width() != w || mask->height() != h)))
        throw DimensionMismatch("accuracy inputs differ in size");
    AccuracyReport r;
    r.thresholds = thresholds;
    r.fractions.assign(thresholds.size(), 0.0);
    long long evaluated = 0;
    double mae = 0.0;
    // the device kernel takes up to 16 thresholds per call; counts and the
    // error sum do not depend on them
    std::size_t k0 = 0;
    do {
        const int k = int(std::min<std::size_t>(16, thresholds.size() - k0));
        check(ps_accuracy(ctx(), 1, prediction.values().data(), prediction.validity().data(),
                          groundTruth.values().data(), groundTruth.validity().data(),
                          mask ? mask->membership().data() : nullptr, w, h,
                          k ? thresholds.data() + k0 : nullptr, k,
                          k ? r.fractions.data() + k0 : nullptr, &evaluated, &mae));
        k0 += std::size_t(k);
    } while (k0 < thresholds.size());
    r.evaluated = long(evaluated);
    r.meanAbsError = mae;
    return r;
}
}  // namespace

AccuracyReport accuracy(const DisparityMap& prediction, const DisparityMap& groundTruth,
                        const GradientMask& mask, const std::vector<double>& thresholds) {
    return accuracy_impl(prediction, groundTruth, &mask, thresholds);
}

AccuracyReport accuracy(const DisparityMap& prediction, const DisparityMap& groundTruth,
                        const std::vector<double>& thresholds) {
    return accuracy_impl(prediction, groundTruth, nullptr, thresholds);
}

PlanarScene PlanarScene::flat(double d, int width, int height, std::uint32_t seed) {
    return slanted(0.0, 0.0, d, width, height, seed);
}

PlanarScene PlanarScene::slanted(double a, double b, double c, int width, int height,
                                 std::uint32_t seed) {
    PlanarScene s;
    s.width = width;
    s.height = height;
    s.seed = seed;
    s.regions.push_back({0, 0, width, height, {a, b, c}});
    return s;
}

PlanarScene PlanarScene::steps(double dLeft, double dRight, int width, int height,
                               std::uint32_t seed) {
    PlanarScene s;
    s.width = width;
    s.height = height;
    s.seed = seed;
    const int mid = width / 2;
    s.regions.push_back({0, 0, mid, height, {0.0, 0.0, dLeft}});
    s.regions.push_back({mid, 0, width, height, {0.0, 0.0, dRight}});
    return s;
}

RenderedScene renderScene(const PlanarScene& scene) {
    const int w = scene.width, h = scene.height;
    std::vector<ps_scene_region> regs;
    regs.reserve(scene.regions.size());
    for (const SceneRegion& r : scene.regions)
        regs.push_back({r.u0, r.v0, r.u1, r.v1, r.plane.a, r.plane.b, r.plane.c});
    const std::size_t P = std::size_t(std::max(w, 0)) * std::size_t(std::max(h, 0));
    std::vector<std::uint8_t> left(P), right(P), gtv(P), occ(P);
    std::vector<float> gt(P);
    check(ps_render_scene(ctx(), w, h, scene.maxDisparity, scene.seed, regs.data(), int(regs.size()),
                          left.data(), right.data(), gt.data(), gtv.data(), occ.data()));
    RenderedScene out{GrayImage(w, h, std::move(left)), GrayImage(w, h, std::move(right)),
                      DisparityMap(w, h), std::move(occ)};
    out.groundTruth.mutableValues() = std::move(gt);
    out.groundTruth.mutableValidity() = std::move(gtv);
    return out;
}

RefinementGrids disparityRefinement(const DisparityMap& interpolated, const CostMap& costs,
                                    DisparityMap& finalDisparity, CostMap& finalCost,
                                    const GradientMask& mask, int cellSize,
                                    const PipelineConfig& config) {
    const int w = costs.width(), h = costs.height();
    RefinementGrids g{OccupancyGrid(w, h, cellSize, config.costLow),
                      OccupancyGrid(w, h, cellSize, config.costHigh)};
    const int cells = g.confident.cols() * g.confident.rows();
    std::vector<ps_cell> conf(cells), inv(cells);
    const ps_config c = to_c(config);
    check(ps_refinement(ctx(), interpolated.values().data(), interpolated.validity().data(),
                        costs.values().data(), finalDisparity.mutableValues().data(),
                        finalDisparity.mutableValidity().data(), finalCost.mutableValues().data(),
                        mask.membership().data(), w, h, cellSize, &c, conf.data(), inv.data()));
    for (int cv = 0; cv < g.confident.rows(); ++cv)
        for (int cu = 0; cu < g.confident.cols(); ++cu) {
            const ps_cell& a = conf[std::size_t(cv) * g.confident.cols() + cu];
            const ps_cell& b = inv[std::size_t(cv) * g.confident.cols() + cu];
            g.confident.cell(cu, cv) = {a.u, a.v, a.disparity, a.cost, a.occupied != 0};
            g.invalid.cell(cu, cv) = {b.u, b.v, b.disparity, b.cost, b.occupied != 0};
        }
    return g;
}

std::vector<SupportPoint> supportResampling(const OccupancyGrid& confident,
                                            const OccupancyGrid& invalid,
                                            const std::vector<SupportPoint>& supports,
                                            const CensusField& left, const CensusField& right,
                                            const PipelineConfig& config) {
    const int cells = confident.cols() * confident.rows();
    std::vector<ps_cell> conf(cells), inv(cells);
    for (int cv = 0; cv < confident.rows(); ++cv)
        for (int cu = 0; cu < confident.cols(); ++cu) {
            const OccupancyCell& a = confident.cell(cu, cv);
            const OccupancyCell& b = invalid.cell(cu, cv);
            conf[std::size_t(cv) * confident.cols() + cu] = {a.u, a.v, a.disparity, a.cost, a.occupied};
            inv[std::size_t(cv) * confident.cols() + cu] = {b.u, b.v, b.disparity, b.cost, b.occupied};
        }
    const int n = int(supports.size());
    std::vector<int> su(n), sv(n);
    std::vector<double> sd(n);
    for (int i = 0; i < n; ++i) {
        su[i] = supports[i].u;
        sv[i] = supports[i].v;
        sd[i] = supports[i].d;
    }
    const int cap = n + 2 * cells + 1;
    std::vector<int> u(cap), v(cap);
    std::vector<double> d(cap);
    int m = 0;
    const ps_config c = to_c(config);
    check(ps_support_resampling(ctx(), conf.data(), inv.data(), confident.cellSize(), su.data(),
                                sv.data(), sd.data(), n, left.words().data(), right.words().data(),
                                left.width(), left.height(), &c, u.data(), v.data(), d.data(), cap,
                                &m));
    std::vector<SupportPoint> out(m);
    for (int i = 0; i < m; ++i) out[i] = {u[i], v[i], d[i]};
    return out;
}

StereoResult run(const GrayImage& left, const GrayImage& right, const PipelineConfig& config,
                 const IterationObserver& observer) {
    return run_impl(left, right, config, observer, 0);
}

StereoResult runUnchecked(const GrayImage& left, const GrayImage& right,
                          const PipelineConfig& config, const IterationObserver& observer) {
    return run_impl(left, right, config, observer, PS_RUN_UNCHECKED_CELL);
}

std::vector<StereoResult> runBatch(const std::vector<GrayImage>& left,
                                   const std::vector<GrayImage>& right,
                                   const PipelineConfig& config, bool uncheckedCell,
                                   std::vector<std::string>* errors) {
    const unsigned flags = uncheckedCell ? PS_RUN_UNCHECKED_CELL : 0u;
    const ps_config c = to_c(config);
    check(ps_config_validate(&c, flags));
    const int n = int(left.size());
    if (n == 0) return {};
    if (int(right.size()) != n) throw DimensionMismatch("left and right batches differ in length");
    const int w = left[0].width(), h = left[0].height();
    const std::size_t P = std::size_t(w) * h;
    std::vector<std::uint8_t> L(P * n), R(P * n);
    for (int i = 0; i < n; ++i) {
        if (!left[i].sameSize(left[0]) || !right[i].sameSize(left[0]))
            throw DimensionMismatch("all pairs of a batch must share one size");
        std::copy(left[i].data().begin(), left[i].data().end(), L.begin() + i * P);
        std::copy(right[i].data().begin(), right[i].data().end(), R.begin() + i * P);
    }
    std::vector<float> disp(P * n), cost(P * n), dense(P * n);
    std::vector<std::uint8_t> dv(P * n), denv(P * n);
    std::vector<ps_iter_stats> trace(std::size_t(n) * config.iterations);
    std::vector<int> status(n);
    const ps_status s = ps_run_batch(ctx(), n, L.data(), R.data(), w, h, &c, flags, disp.data(),
                                     dv.data(), cost.data(), dense.data(), denv.data(),
                                     trace.data(), status.data());
    if (s != PS_OK && s != PS_SEEDING_FAILED) raise(s);
    std::vector<StereoResult> out;
    out.reserve(n);
    if (errors) errors->assign(n, std::string());
    for (int i = 0; i < n; ++i) {
        StereoResult r{DisparityMap(w, h), CostMap(w, h, config.costHigh), DisparityMap(w, h), {}};
        if (status[i] == PS_OK) {
            std::copy(disp.begin() + i * P, disp.begin() + (i + 1) * P, r.disparity.mutableValues().begin());
            std::copy(dv.begin() + i * P, dv.begin() + (i + 1) * P, r.disparity.mutableValidity().begin());
            std::copy(cost.begin() + i * P, cost.begin() + (i + 1) * P, r.costs.mutableValues().begin());
            std::copy(dense.begin() + i * P, dense.begin() + (i + 1) * P, r.dense.mutableValues().begin());
            std::copy(denv.begin() + i * P, denv.begin() + (i + 1) * P, r.dense.mutableValidity().begin());
            for (int it = 0; it < config.iterations; ++it) {
                const ps_iter_stats& t = trace[std::size_t(i) * config.iterations + it];
                r.trace.push_back({t.iteration, t.support_count, t.triangle_count,
                                   t.occupancy_cell_size, t.mean_cost, t.valid_count, t.millis});
            }
        } else if (errors) {
            (*errors)[i] = "seeding failed";
        }
        out.push_back(std::move(r));
    }
    return out;
}

void setDevice(int device) {
    if (t_ctx.ctx && t_ctx.device != device) {
        ps_ctx_destroy(t_ctx.ctx);
        t_ctx.ctx = nullptr;
    }
    t_ctx.device = device;
}

}  // namespace planestereo
