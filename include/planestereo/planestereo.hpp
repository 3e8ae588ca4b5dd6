// planestereo.hpp — drop-in C++ API of the B200 hot path.
//
// Declares, in namespace planestereo, every type and function of the
// reference's public header API (proj/include/planestereo/{error,config,
// image,disparity,census,sparse,delaunay,mesh,pipeline,synth}.hpp and accuracy() of eval.hpp) with the same
// names, signatures, value semantics and exceptions, so code written against
// the reference recompiles unchanged (the per-name headers next to this one
// just include it).  The implementation (paper_1511_00758_b200/csrc/cpp_api)
// forwards to the C ABI of include/planestereo_c.h: the per-pixel and
// per-candidate work runs on the B200 kernels, the Delaunay triangulation and
// the list bookkeeping on the host.  A thread-local ps_ctx on device 0 backs
// the free functions; planestereo::setDevice() selects another GPU.
#pragma once

#include <array>
#include <bit>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace planestereo {

// ------------------------------------------------------------------ errors
// (reference error.hpp:9-72)
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
#define PLANESTEREO_ERROR_CLASS(Name) \
    class Name : public Error {       \
    public:                           \
        using Error::Error;           \
    }
PLANESTEREO_ERROR_CLASS(InvalidConfig);
PLANESTEREO_ERROR_CLASS(DimensionTooSmall);
PLANESTEREO_ERROR_CLASS(DimensionMismatch);
PLANESTEREO_ERROR_CLASS(FewerThanThreePoints);
PLANESTEREO_ERROR_CLASS(DegenerateTriangle);
PLANESTEREO_ERROR_CLASS(SeedingFailed);
PLANESTEREO_ERROR_CLASS(UnsupportedFormat);
PLANESTEREO_ERROR_CLASS(CorruptFile);
PLANESTEREO_ERROR_CLASS(NegativeDisparity);
PLANESTEREO_ERROR_CLASS(EmptyCloud);
PLANESTEREO_ERROR_CLASS(NoOverlap);
PLANESTEREO_ERROR_CLASS(InvalidPlane);
#undef PLANESTEREO_ERROR_CLASS

// ------------------------------------------------------------------ config
// Field order, types and defaults of the reference (config.hpp:8-34); the
// layout is that of ps_config.
struct PipelineConfig {
    int iterations = 1;
    int maxDisparity = 128;
    float costLow = 0.25f;
    float costHigh = 0.5f;
    int gradientThreshold = 20;
    int occupancyCellSize = 32;
    int cornerThreshold = 20;
    int perBinCap = 5;
    float sparseAcceptCost = 0.25f;
    float uniquenessRatio = 0.9f;
    int threads = 1;

    void validate() const;  // throws InvalidConfig (config.cpp:17-49)
};

// ------------------------------------------------------------------ images
struct Pixel {
    int u = 0;
    int v = 0;
    friend bool operator==(const Pixel&, const Pixel&) = default;
};

class GrayImage {
public:
    static constexpr int kMinDimension = 16;
    GrayImage(int width, int height, std::uint8_t fill = 0);
    GrayImage(int width, int height, std::vector<std::uint8_t> data);
    int width() const { return w_; }
    int height() const { return h_; }
    std::uint8_t at(int u, int v) const { return px_[std::size_t(v) * w_ + u]; }
    std::uint8_t& at(int u, int v) { return px_[std::size_t(v) * w_ + u]; }
    const std::uint8_t* row(int v) const { return px_.data() + std::size_t(v) * w_; }
    std::uint8_t* row(int v) { return px_.data() + std::size_t(v) * w_; }
    const std::vector<std::uint8_t>& data() const { return px_; }
    bool sameSize(const GrayImage& o) const { return w_ == o.w_ && h_ == o.h_; }

private:
    int w_;
    int h_;
    std::vector<std::uint8_t> px_;
};

class GradientMask {
public:
    static constexpr int kMargin = 2;
    GradientMask(int width, int height);
    int width() const { return w_; }
    int height() const { return h_; }
    int count() const { return int(pts_.size()); }
    bool contains(int u, int v) const { return in_[std::size_t(v) * w_ + u] != 0; }
    const std::vector<Pixel>& points() const { return pts_; }  // row-major
    void add(int u, int v);
    const std::vector<std::uint8_t>& membership() const { return in_; }  // extension

private:
    int w_;
    int h_;
    std::vector<std::uint8_t> in_;
    std::vector<Pixel> pts_;
};

GradientMask gradientMask(const GrayImage& image, int threshold);

// ------------------------------------------------------------------ maps
class DisparityMap {
public:
    DisparityMap(int width, int height);
    int width() const { return w_; }
    int height() const { return h_; }
    float at(int u, int v) const { return val_[idx(u, v)]; }
    bool valid(int u, int v) const { return ok_[idx(u, v)] != 0; }
    void set(int u, int v, float d) {
        val_[idx(u, v)] = d;
        ok_[idx(u, v)] = 1;
    }
    void invalidate(int u, int v) {
        val_[idx(u, v)] = 0.0f;
        ok_[idx(u, v)] = 0;
    }
    int validCount() const;
    const std::vector<float>& values() const { return val_; }
    const std::vector<std::uint8_t>& validity() const { return ok_; }
    std::vector<float>& mutableValues() { return val_; }          // extension (bulk fill)
    std::vector<std::uint8_t>& mutableValidity() { return ok_; }  // extension (bulk fill)

private:
    std::size_t idx(int u, int v) const { return std::size_t(v) * w_ + u; }
    int w_;
    int h_;
    std::vector<float> val_;
    std::vector<std::uint8_t> ok_;
};

class CostMap {
public:
    CostMap(int width, int height, float fill);
    int width() const { return w_; }
    int height() const { return h_; }
    float at(int u, int v) const { return c_[std::size_t(v) * w_ + u]; }
    void set(int u, int v, float cost) { c_[std::size_t(v) * w_ + u] = cost; }
    const std::vector<float>& values() const { return c_; }
    std::vector<float>& mutableValues() { return c_; }  // extension (bulk fill)

private:
    int w_;
    int h_;
    std::vector<float> c_;
};

// ------------------------------------------------------------------ census
class CensusField {
public:
    static constexpr int kRadius = 2;
    static constexpr int kBits = 24;
    CensusField(int width, int height);
    int width() const { return w_; }
    int height() const { return h_; }
    bool valid(int u, int v) const {
        return u >= kRadius && u < w_ - kRadius && v >= kRadius && v < h_ - kRadius;
    }
    std::uint32_t at(int u, int v) const { return d_[std::size_t(v) * w_ + u]; }
    std::uint32_t& at(int u, int v) { return d_[std::size_t(v) * w_ + u]; }
    const std::uint32_t* row(int v) const { return d_.data() + std::size_t(v) * w_; }
    const std::vector<std::uint32_t>& words() const { return d_; }  // extension
    std::vector<std::uint32_t>& mutableWords() { return d_; }        // extension

private:
    int w_;
    int h_;
    std::vector<std::uint32_t> d_;
};

CensusField censusTransform(const GrayImage& image, int threads = 1);

inline float censusCost(std::uint32_t a, std::uint32_t b) {
    return float(std::popcount(a ^ b)) / float(CensusField::kBits);
}

// ------------------------------------------------------------------ sparse
struct SupportPoint {
    int u = 0;
    int v = 0;
    double d = 0.0;
    friend bool operator==(const SupportPoint&, const SupportPoint&) = default;
};

struct CandidatePixel {
    int u = 0;
    int v = 0;
    float score = 0.0f;
};

std::vector<CandidatePixel> detectCandidates(const GrayImage& image, const PipelineConfig& config);
std::vector<SupportPoint> matchEpipolar(const GrayImage& left, const GrayImage& right,
                                        const std::vector<CandidatePixel>& candidates,
                                        const PipelineConfig& config);
std::vector<SupportPoint> matchEpipolar(const CensusField& left, const CensusField& right,
                                        const std::vector<CandidatePixel>& candidates,
                                        const PipelineConfig& config);

// ------------------------------------------------------------------ delaunay
long long orient2d(const Pixel& a, const Pixel& b, const Pixel& c);
int inCircleSign(const Pixel& a, const Pixel& b, const Pixel& c, const Pixel& d);
std::vector<std::array<int, 3>> delaunayTriangulate(const std::vector<Pixel>& points);

// ------------------------------------------------------------------ mesh
struct DisparityPlane {
    double a = 0.0;
    double b = 0.0;
    double c = 0.0;
    double at(double u, double v) const { return a * u + b * v + c; }
};

DisparityPlane fitPlane(const SupportPoint& v1, const SupportPoint& v2, const SupportPoint& v3);

class DisparityMesh {
public:
    static constexpr int kOutside = -1;
    DisparityMesh(std::vector<SupportPoint> vertices, std::vector<std::array<int, 3>> triangles,
                  int width, int height);
    int width() const { return w_; }
    int height() const { return h_; }
    const std::vector<SupportPoint>& vertices() const { return verts_; }
    const std::vector<std::array<int, 3>>& triangles() const { return tris_; }
    const std::vector<DisparityPlane>& planes() const { return planes_; }
    int triangleAt(int u, int v) const { return lookup_[std::size_t(v) * w_ + u]; }
    const std::vector<std::int32_t>& lookup() const { return lookup_; }
    void writeOff(std::ostream& out) const;

private:
    std::vector<SupportPoint> verts_;
    std::vector<std::array<int, 3>> tris_;
    std::vector<DisparityPlane> planes_;
    std::vector<std::int32_t> lookup_;
    int w_;
    int h_;
};

DisparityMesh triangulate(const std::vector<SupportPoint>& points, int width, int height);
DisparityMap interpolate(const DisparityMesh& mesh, const GradientMask& domain, float maxDisparity);
DisparityMap interpolate(const DisparityMesh& mesh, float maxDisparity);

// ------------------------------------------------------------------ pipeline
struct OccupancyCell {
    int u = 0;
    int v = 0;
    float disparity = 0.0f;
    float cost = 0.0f;
    bool occupied = false;
};

class OccupancyGrid {
public:
    OccupancyGrid(int imageWidth, int imageHeight, int cellSize, float initialCost);
    int cellSize() const { return size_; }
    int cols() const { return cols_; }
    int rows() const { return rows_; }
    const OccupancyCell& cell(int cu, int cv) const { return cells_[std::size_t(cv) * cols_ + cu]; }
    OccupancyCell& cell(int cu, int cv) { return cells_[std::size_t(cv) * cols_ + cu]; }
    const OccupancyCell& cellForPixel(int u, int v) const { return cell(u / size_, v / size_); }
    OccupancyCell& cellForPixel(int u, int v) { return cell(u / size_, v / size_); }

private:
    int size_;
    int cols_;
    int rows_;
    std::vector<OccupancyCell> cells_;
};

struct IterationStats {
    int iteration = 0;
    int supportCount = 0;
    int triangleCount = 0;
    int occupancyCellSize = 0;
    double meanCost = 0.0;
    int validCount = 0;
    double millis = 0.0;
};

using IterationTrace = std::vector<IterationStats>;

struct StereoResult {
    DisparityMap disparity;
    CostMap costs;
    DisparityMap dense;
    IterationTrace trace;
};

CostMap costEvaluation(const CensusField& left, const CensusField& right,
                       const DisparityMap& interpolated, const GradientMask& mask, int threads = 1);

struct RefinementGrids {
    OccupancyGrid confident;
    OccupancyGrid invalid;
};

RefinementGrids disparityRefinement(const DisparityMap& interpolated, const CostMap& costs,
                                    DisparityMap& finalDisparity, CostMap& finalCost,
                                    const GradientMask& mask, int cellSize,
                                    const PipelineConfig& config);

std::vector<SupportPoint> supportResampling(const OccupancyGrid& confident,
                                            const OccupancyGrid& invalid,
                                            const std::vector<SupportPoint>& supports,
                                            const CensusField& left, const CensusField& right,
                                            const PipelineConfig& config);

using IterationObserver =
    std::function<void(int iteration, const DisparityMap& finalDisparity, const CostMap& finalCost)>;

StereoResult run(const GrayImage& left, const GrayImage& right, const PipelineConfig& config,
                 const IterationObserver& observer = {});

// (reference synth.hpp:52-56) Exhaustive winner-take-all census matcher: per
// mask pixel the cost-minimal integer disparity in [0, min(maxDisparity, u-2)],
// ties toward smaller d.  Runs on the GPU (wta.cu).
std::pair<DisparityMap, CostMap> wtaOracle(const GrayImage& left, const GrayImage& right,
                                           const GradientMask& mask, int maxDisparity);

// ------------------------------------------------------------------ eval
// (reference eval.hpp:15-29) Fractions of the pixels valid in both maps (and
// inside the mask) whose absolute error is strictly below each threshold, and
// the mean absolute error (binary64, row-major sum).  Throws NoOverlap when
// no pixel qualifies.  Runs on the GPU (accuracy.cu).  The table / CSV / JSON
// writers and the timing harness of eval.hpp are not part of this build.
struct AccuracyReport {
    std::vector<double> thresholds;
    std::vector<double> fractions;
    long evaluated = 0;
    double meanAbsError = 0.0;
};
AccuracyReport accuracy(const DisparityMap& prediction, const DisparityMap& groundTruth,
                        const GradientMask& mask, const std::vector<double>& thresholds);
AccuracyReport accuracy(const DisparityMap& prediction, const DisparityMap& groundTruth,
                        const std::vector<double>& thresholds);

// ------------------------------------------------------------------ synth
// (reference synth.hpp:14-50) Piecewise-planar test scenes rendered on the GPU
// (synth.cu: renderScene's texture, contrast stretch, forward warp with
// occlusion), bit for bit the reference's images and ground truth.
struct SceneRegion {  // [u0, u1) x [v0, v1) carrying one disparity plane
    int u0 = 0;
    int v0 = 0;
    int u1 = 0;
    int v1 = 0;
    DisparityPlane plane;
};

struct PlanarScene {  // regions must partition the image
    int width = 640;
    int height = 480;
    float maxDisparity = 128.0f;
    std::uint32_t seed = 1234;
    std::vector<SceneRegion> regions;

    static PlanarScene flat(double d, int width = 640, int height = 480, std::uint32_t seed = 1234);
    static PlanarScene slanted(double a, double b, double c, int width = 640, int height = 480,
                               std::uint32_t seed = 1234);
    static PlanarScene steps(double dLeft, double dRight, int width = 640, int height = 480,
                             std::uint32_t seed = 1234);  // left half at dLeft, right at dRight
};

struct RenderedScene {
    GrayImage left;
    GrayImage right;
    DisparityMap groundTruth;             // invalid where occluded or out of the right view
    std::vector<std::uint8_t> occlusion;  // 1 where a nearer surface hides the pixel
};

// Throws InvalidPlane when a region's plane leaves [0, maxDisparity) inside it.
RenderedScene renderScene(const PlanarScene& scene);

// ------------------------------------------------------------------ extensions
// GPU selection for the calling thread's default context (device 0 otherwise).
void setDevice(int device);
// run() without the power-of-two cell rule of validate() (SURVEY App. B:
// the BASELINE grids 10 and 6); every other check is identical.
StereoResult runUnchecked(const GrayImage& left, const GrayImage& right,
                          const PipelineConfig& config, const IterationObserver& observer = {});
// Many independent pairs of one size on the current GPU in one batch; a pair
// whose seeding fails yields an empty result and SeedingFailed in `errors`.
std::vector<StereoResult> runBatch(const std::vector<GrayImage>& left,
                                   const std::vector<GrayImage>& right,
                                   const PipelineConfig& config, bool uncheckedCell = false,
                                   std::vector<std::string>* errors = nullptr);

}  // namespace planestereo
