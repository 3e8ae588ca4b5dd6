// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the REFERENCE library itself, compiled by
// oracle/Makefile from the unmodified sources under /root/reference/proj/src
// into oracle/_ref/libps_ref.so.  Same signatures as ps_oracle.h with a
// `ref_` prefix, so tests can diff the C restatement (ps_oracle.c) and the
// CUDA product against the reference's own code on identical inputs.
//
// ref_run mirrors planestereo::run (proj/src/pipeline.cpp:131-203) stage by
// stage through the public stage functions, with validate() optional: the
// BASELINE grids 10 and 6 fail the power-of-two rule.  With
// validate=2 it calls planestereo::run itself (for checking the staged loop).
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "planestereo/census.hpp"
#include "planestereo/delaunay.hpp"
#include "planestereo/eval.hpp"
#include "planestereo/mesh.hpp"
#include "planestereo/pipeline.hpp"
#include "planestereo/sparse.hpp"
#include "planestereo/synth.hpp"
#include "planestereo_c.h"

using namespace planestereo;

namespace {

PipelineConfig toConfig(const ps_config* c) {
    PipelineConfig p;
    p.iterations = c->iterations;
    p.maxDisparity = c->max_disparity;
    p.costLow = c->cost_low;
    p.costHigh = c->cost_high;
    p.gradientThreshold = c->gradient_threshold;
    p.occupancyCellSize = c->occupancy_cell_size;
    p.cornerThreshold = c->corner_threshold;
    p.perBinCap = c->per_bin_cap;
    p.sparseAcceptCost = c->sparse_accept_cost;
    p.uniquenessRatio = c->uniqueness_ratio;
    p.threads = c->threads;
    return p;
}

GrayImage toImage(const uint8_t* px, int w, int h) {
    return GrayImage(w, h, std::vector<std::uint8_t>(px, px + std::size_t(w) * h));
}

CensusField toCensus(const uint32_t* c, int w, int h) {
    CensusField f(w, h);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) f.at(u, v) = c[std::size_t(v) * w + u];
    return f;
}

GradientMask toMask(const uint8_t* m, int w, int h) {
    GradientMask mask(w, h);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u)
            if (m[std::size_t(v) * w + u]) mask.add(u, v);
    return mask;
}

int statusOf(const std::exception& e) {
    if (dynamic_cast<const InvalidConfig*>(&e)) return PS_INVALID_CONFIG;
    if (dynamic_cast<const DimensionTooSmall*>(&e)) return PS_DIMENSION_TOO_SMALL;
    if (dynamic_cast<const DimensionMismatch*>(&e)) return PS_DIMENSION_MISMATCH;
    if (dynamic_cast<const FewerThanThreePoints*>(&e)) return PS_FEWER_THAN_THREE_POINTS;
    if (dynamic_cast<const DegenerateTriangle*>(&e)) return PS_DEGENERATE_TRIANGLE;
    if (dynamic_cast<const SeedingFailed*>(&e)) return PS_SEEDING_FAILED;
    if (dynamic_cast<const NoOverlap*>(&e)) return PS_NO_OVERLAP;
    if (dynamic_cast<const InvalidPlane*>(&e)) return PS_INVALID_PLANE;
    return PS_ERROR;
}

void copyMap(const DisparityMap& m, float* val, uint8_t* valid) {
    if (val) std::memcpy(val, m.values().data(), m.values().size() * sizeof(float));
    if (valid) std::memcpy(valid, m.validity().data(), m.validity().size());
}

}  // namespace

extern "C" {

int ref_gradient_mask(const uint8_t* img, int w, int h, int threshold, uint8_t* member) {
    GradientMask m = gradientMask(toImage(img, w, h), threshold);
    std::memset(member, 0, std::size_t(w) * h);
    for (const Pixel& p : m.points()) member[std::size_t(p.v) * w + p.u] = 1;
    return m.count();
}

void ref_census(const uint8_t* img, int w, int h, uint32_t* out) {
    CensusField f = censusTransform(toImage(img, w, h));
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) out[std::size_t(v) * w + u] = f.at(u, v);
}

int ref_detect_candidates(const uint8_t* img, int w, int h, const ps_config* cfg, int* u, int* v,
                          float* score, int cap) {
    auto c = detectCandidates(toImage(img, w, h), toConfig(cfg));
    int n = 0;
    for (; n < int(c.size()) && n < cap; ++n) {
        u[n] = c[n].u;
        v[n] = c[n].v;
        if (score) score[n] = c[n].score;
    }
    return n;
}

int ref_match_epipolar(const uint32_t* cl, const uint32_t* cr, int w, int h, const int* cu,
                       const int* cv, int n, const ps_config* cfg, int* su, int* sv, double* sd) {
    std::vector<CandidatePixel> cand(n);
    for (int i = 0; i < n; ++i) cand[i] = {cu[i], cv[i], 0.0f};
    auto s = matchEpipolar(toCensus(cl, w, h), toCensus(cr, w, h), cand, toConfig(cfg));
    for (std::size_t i = 0; i < s.size(); ++i) {
        su[i] = s[i].u;
        sv[i] = s[i].v;
        sd[i] = s[i].d;
    }
    return int(s.size());
}

long long ref_orient2d(int au, int av, int bu, int bv, int cu, int cv) {
    return orient2d({au, av}, {bu, bv}, {cu, cv});
}

int ref_incircle_sign(int au, int av, int bu, int bv, int cu, int cv, int du, int dv) {
    return inCircleSign({au, av}, {bu, bv}, {cu, cv}, {du, dv});
}

int ref_delaunay(const int* u, const int* v, int n, int* tris) {
    std::vector<Pixel> pts(n);
    for (int i = 0; i < n; ++i) pts[i] = {u[i], v[i]};
    try {
        auto t = delaunayTriangulate(pts);
        for (std::size_t i = 0; i < t.size(); ++i)
            for (int k = 0; k < 3; ++k) tris[3 * i + k] = t[i][k];
        return int(t.size());
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_fit_plane(int u1, int v1, double d1, int u2, int v2, double d2, int u3, int v3, double d3,
                  double* abc) {
    try {
        DisparityPlane p = fitPlane({u1, v1, d1}, {u2, v2, d2}, {u3, v3, d3});
        abc[0] = p.a;
        abc[1] = p.b;
        abc[2] = p.c;
        return 0;
    } catch (const DegenerateTriangle&) {
        return -1;
    }
}

int ref_mesh_build(const int* u, const int* v, const double* d, const int* tris, int nt, int w,
                   int h, double* planes, int32_t* lookup) {
    int nv = 0;
    for (int i = 0; i < 3 * nt; ++i) nv = std::max(nv, tris[i] + 1);
    std::vector<SupportPoint> verts(nv);
    for (int i = 0; i < nv; ++i) verts[i] = {u[i], v[i], d[i]};
    std::vector<std::array<int, 3>> tr(nt);
    for (int i = 0; i < nt; ++i) tr[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    try {
        DisparityMesh mesh(verts, tr, w, h);
        for (int i = 0; i < nt; ++i) {
            planes[3 * i] = mesh.planes()[i].a;
            planes[3 * i + 1] = mesh.planes()[i].b;
            planes[3 * i + 2] = mesh.planes()[i].c;
        }
        std::memcpy(lookup, mesh.lookup().data(), sizeof(int32_t) * std::size_t(w) * h);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Full DisparityMesh path from a support list: triangulate + mesh, as used by run().
int ref_triangulate(const int* u, const int* v, const double* d, int n, int w, int h, int* tris,
                    double* planes, int32_t* lookup) {
    std::vector<SupportPoint> pts(n);
    for (int i = 0; i < n; ++i) pts[i] = {u[i], v[i], d[i]};
    try {
        DisparityMesh mesh = triangulate(pts, w, h);
        const int nt = int(mesh.triangles().size());
        for (int i = 0; i < nt; ++i) {
            for (int k = 0; k < 3; ++k) tris[3 * i + k] = mesh.triangles()[i][k];
            planes[3 * i] = mesh.planes()[i].a;
            planes[3 * i + 1] = mesh.planes()[i].b;
            planes[3 * i + 2] = mesh.planes()[i].c;
        }
        std::memcpy(lookup, mesh.lookup().data(), sizeof(int32_t) * std::size_t(w) * h);
        return nt;
    } catch (const std::exception& e) {
        return -statusOf(e);
    }
}

void ref_interpolate_mesh(const int* u, const int* v, const double* d, int n, const int* tris,
                          int nt, int w, int h, const uint8_t* mask, float max_disparity,
                          float* value, uint8_t* valid) {
    std::vector<SupportPoint> verts(n);
    for (int i = 0; i < n; ++i) verts[i] = {u[i], v[i], d[i]};
    std::vector<std::array<int, 3>> tr(nt);
    for (int i = 0; i < nt; ++i) tr[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    DisparityMesh mesh(verts, tr, w, h);
    if (mask) {
        copyMap(interpolate(mesh, toMask(mask, w, h), max_disparity), value, valid);
    } else {
        copyMap(interpolate(mesh, max_disparity), value, valid);
    }
}

void ref_cost_evaluation(const uint32_t* cl, const uint32_t* cr, int w, int h, const float* value,
                         const uint8_t* valid, const uint8_t* mask, float* cost) {
    DisparityMap interp(w, h);
    for (int vv = 0; vv < h; ++vv)
        for (int uu = 0; uu < w; ++uu) {
            std::size_t i = std::size_t(vv) * w + uu;
            if (valid[i]) interp.set(uu, vv, value[i]);
        }
    CostMap c = costEvaluation(toCensus(cl, w, h), toCensus(cr, w, h), interp, toMask(mask, w, h));
    std::memcpy(cost, c.values().data(), sizeof(float) * std::size_t(w) * h);
}

void ref_refinement(const float* value, const uint8_t* valid, const float* cost, float* fd,
                    uint8_t* fv, float* fc, const uint8_t* mask, int w, int h, int cell,
                    const ps_config* cfg, ps_cell* confident, ps_cell* invalid) {
    DisparityMap interp(w, h), fdm(w, h);
    CostMap costs(w, h, 1.0f), fcm(w, h, 0.0f);
    for (int vv = 0; vv < h; ++vv)
        for (int uu = 0; uu < w; ++uu) {
            std::size_t i = std::size_t(vv) * w + uu;
            if (valid[i]) interp.set(uu, vv, value[i]);
            costs.set(uu, vv, cost[i]);
            if (fv[i]) fdm.set(uu, vv, fd[i]);
            fcm.set(uu, vv, fc[i]);
        }
    RefinementGrids g =
        disparityRefinement(interp, costs, fdm, fcm, toMask(mask, w, h), cell, toConfig(cfg));
    copyMap(fdm, fd, fv);
    std::memcpy(fc, fcm.values().data(), sizeof(float) * std::size_t(w) * h);
    for (int cv = 0; cv < g.confident.rows(); ++cv)
        for (int cu = 0; cu < g.confident.cols(); ++cu) {
            const int i = cv * g.confident.cols() + cu;
            const OccupancyCell& a = g.confident.cell(cu, cv);
            const OccupancyCell& b = g.invalid.cell(cu, cv);
            confident[i] = {a.u, a.v, a.disparity, a.cost, a.occupied ? 1 : 0};
            invalid[i] = {b.u, b.v, b.disparity, b.cost, b.occupied ? 1 : 0};
        }
}

int ref_support_resampling(const ps_cell* confident, const ps_cell* invalid, int cell,
                           const int* su, const int* sv, const double* sd, int n,
                           const uint32_t* cl, const uint32_t* cr, int w, int h,
                           const ps_config* cfg, int* ou, int* ov, double* od, int cap) {
    OccupancyGrid gc(w, h, cell, cfg->cost_low), gi(w, h, cell, cfg->cost_high);
    for (int cv = 0; cv < gc.rows(); ++cv)
        for (int cu = 0; cu < gc.cols(); ++cu) {
            const int i = cv * gc.cols() + cu;
            gc.cell(cu, cv) = {confident[i].u, confident[i].v, confident[i].disparity,
                               confident[i].cost, confident[i].occupied != 0};
            gi.cell(cu, cv) = {invalid[i].u, invalid[i].v, invalid[i].disparity, invalid[i].cost,
                               invalid[i].occupied != 0};
        }
    std::vector<SupportPoint> s(n);
    for (int i = 0; i < n; ++i) s[i] = {su[i], sv[i], sd[i]};
    auto r = supportResampling(gc, gi, s, toCensus(cl, w, h), toCensus(cr, w, h), toConfig(cfg));
    for (std::size_t i = 0; i < r.size() && int(i) < cap; ++i) {
        ou[i] = r[i].u;
        ov[i] = r[i].v;
        od[i] = r[i].d;
    }
    return int(r.size());
}

int ref_run(const uint8_t* left, const uint8_t* right, int w, int h, const ps_config* cfg,
            int validate, float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
            uint8_t* dense_valid, ps_iter_stats* trace, int* sup_u, int* sup_v, double* sup_d,
            int sup_cap, int* sup_count) {
    try {
        const PipelineConfig config = toConfig(cfg);
        const GrayImage L = toImage(left, w, h);
        const GrayImage R = toImage(right, w, h);
        if (validate == 2) {
            StereoResult r = run(L, R, config);
            copyMap(r.disparity, disparity, disparity_valid);
            if (cost) std::memcpy(cost, r.costs.values().data(), sizeof(float) * std::size_t(w) * h);
            copyMap(r.dense, dense, dense_valid);
            for (std::size_t i = 0; trace && i < r.trace.size(); ++i) {
                const IterationStats& s = r.trace[i];
                trace[i] = {s.iteration, s.supportCount, s.triangleCount, s.occupancyCellSize,
                            s.meanCost, s.validCount, s.millis};
            }
            return PS_OK;
        }
        if (validate) config.validate();
        // Staged mirror of run(), pipeline.cpp:141-202.
        const GradientMask mask = gradientMask(L, config.gradientThreshold);
        const CensusField cL = censusTransform(L, config.threads);
        const CensusField cR = censusTransform(R, config.threads);
        DisparityMap finalDisparity(w, h);
        CostMap finalCost(w, h, config.costHigh);
        int cellSize = config.occupancyCellSize;
        std::vector<SupportPoint> supports =
            matchEpipolar(cL, cR, detectCandidates(L, config), config);
        if (supports.size() < 3) throw SeedingFailed("seeding failed");
        DisparityMap denseMap(w, h);
        for (int it = 1; it <= config.iterations; ++it) {
            const auto tic = std::chrono::steady_clock::now();
            const DisparityMesh mesh = triangulate(supports, w, h);
            const DisparityMap interp = interpolate(mesh, mask, float(config.maxDisparity));
            const CostMap costs = costEvaluation(cL, cR, interp, mask, config.threads);
            const RefinementGrids grids = disparityRefinement(interp, costs, finalDisparity,
                                                              finalCost, mask, cellSize, config);
            const int usedSupports = int(mesh.vertices().size());
            if (it != config.iterations) {
                supports = supportResampling(grids.confident, grids.invalid, supports, cL, cR, config);
                cellSize = std::max(1, cellSize / 2);
            } else {
                denseMap = interpolate(mesh, float(config.maxDisparity));
                if (sup_count) {
                    *sup_count = usedSupports;
                    for (int i = 0; i < usedSupports && i < sup_cap; ++i) {
                        if (sup_u) sup_u[i] = mesh.vertices()[i].u;
                        if (sup_v) sup_v[i] = mesh.vertices()[i].v;
                        if (sup_d) sup_d[i] = mesh.vertices()[i].d;
                    }
                }
            }
            const auto toc = std::chrono::steady_clock::now();
            if (trace) {
                double sum = 0.0;
                int valid = 0;
                for (const Pixel& p : mask.points()) {
                    const float c = finalCost.at(p.u, p.v);
                    sum += c;
                    valid += (c < config.costHigh);
                }
                trace[it - 1] = {it,
                                 usedSupports,
                                 int(mesh.triangles().size()),
                                 grids.confident.cellSize(),
                                 mask.count() > 0 ? sum / mask.count() : 0.0,
                                 valid,
                                 std::chrono::duration<double, std::milli>(toc - tic).count()};
            }
        }
        copyMap(finalDisparity, disparity, disparity_valid);
        if (cost) std::memcpy(cost, finalCost.values().data(), sizeof(float) * std::size_t(w) * h);
        copyMap(denseMap, dense, dense_valid);
        return PS_OK;
    } catch (const std::exception& e) {
        return statusOf(e);
    }
}

// One frame per host thread (BASELINE.md §3 throughput plan), threads=1 per frame.
int ref_run_batch(int n, const uint8_t* left, const uint8_t* right, int w, int h,
                  const ps_config* cfg, int threads, float* disparity, uint8_t* disparity_valid,
                  float* cost, float* dense, uint8_t* dense_valid, int* status) {
    if (threads < 1) threads = 1;
    if (threads > n) threads = std::max(1, n);
    const std::size_t P = std::size_t(w) * h;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([=] {
            for (int f = t; f < n; f += threads) {
                int st = ref_run(left + f * P, right + f * P, w, h, cfg, 0,
                                 disparity ? disparity + f * P : nullptr,
                                 disparity_valid ? disparity_valid + f * P : nullptr,
                                 cost ? cost + f * P : nullptr, dense ? dense + f * P : nullptr,
                                 dense_valid ? dense_valid + f * P : nullptr, nullptr, nullptr,
                                 nullptr, nullptr, 0, nullptr);
                if (status) status[f] = st;
            }
        });
    }
    for (auto& th : pool) th.join();
    return 0;
}

// renderScene (proj/src/synth.cpp:148-227) for the fixture generator:
// kind 0 = flat(p0), 1 = slanted(p0, p1, p2), 2 = steps(p0, p1).
int ref_render_scene(int kind, double p0, double p1, double p2, int w, int h, uint32_t seed,
                     float max_disparity, uint8_t* left, uint8_t* right, float* gt,
                     uint8_t* gt_valid) {
    try {
        PlanarScene s = kind == 0   ? PlanarScene::flat(p0, w, h, seed)
                        : kind == 1 ? PlanarScene::slanted(p0, p1, p2, w, h, seed)
                                    : PlanarScene::steps(p0, p1, w, h, seed);
        s.maxDisparity = max_disparity;
        RenderedScene r = renderScene(s);
        std::memcpy(left, r.left.data().data(), std::size_t(w) * h);
        std::memcpy(right, r.right.data().data(), std::size_t(w) * h);
        copyMap(r.groundTruth, gt, gt_valid);
        return PS_OK;
    } catch (const std::exception& e) {
        return statusOf(e);
    }
}

// renderScene over arbitrary regions (proj/src/synth.cpp:88-169), with the
// occlusion map: the known answers for ps_render_scene.
int ref_render_regions(int w, int h, float max_disparity, uint32_t seed, const int* box,
                       const double* plane, int n, uint8_t* left, uint8_t* right, float* gt,
                       uint8_t* gt_valid, uint8_t* occluded) {
    try {
        PlanarScene s;
        s.width = w;
        s.height = h;
        s.maxDisparity = max_disparity;
        s.seed = seed;
        for (int k = 0; k < n; ++k)
            s.regions.push_back({box[4 * k], box[4 * k + 1], box[4 * k + 2], box[4 * k + 3],
                                 {plane[3 * k], plane[3 * k + 1], plane[3 * k + 2]}});
        RenderedScene r = renderScene(s);
        std::memcpy(left, r.left.data().data(), std::size_t(w) * h);
        std::memcpy(right, r.right.data().data(), std::size_t(w) * h);
        copyMap(r.groundTruth, gt, gt_valid);
        std::memcpy(occluded, r.occlusion.data(), std::size_t(w) * h);
        return PS_OK;
    } catch (const std::exception& e) {
        return statusOf(e);
    }
}

// wtaOracle (proj/src/synth.cpp:229-256): exhaustive census WTA lower bound.
void ref_wta(const uint8_t* left, const uint8_t* right, int w, int h, const uint8_t* mask,
             int max_disparity, float* disp, uint8_t* valid, float* cost) {
    auto r = wtaOracle(toImage(left, w, h), toImage(right, w, h), toMask(mask, w, h), max_disparity);
    copyMap(r.first, disp, valid);
    std::memcpy(cost, r.second.values().data(), sizeof(float) * std::size_t(w) * h);
}

// accuracy (proj/src/eval.cpp:19-70); mask may be null (the maskless overload).
int ref_accuracy(const float* pred, const uint8_t* pred_valid, const float* gt,
                 const uint8_t* gt_valid, const uint8_t* mask, int w, int h,
                 const double* thresholds, int n_thr, double* fractions, long long* evaluated,
                 double* mean_abs_error) {
    try {
        DisparityMap p(w, h), g(w, h);
        for (int v = 0; v < h; ++v)
            for (int u = 0; u < w; ++u) {
                const std::size_t i = std::size_t(v) * w + u;
                if (pred_valid[i]) p.set(u, v, pred[i]);
                if (gt_valid[i]) g.set(u, v, gt[i]);
            }
        const std::vector<double> th(thresholds, thresholds + n_thr);
        const AccuracyReport r =
            mask ? accuracy(p, g, toMask(mask, w, h), th) : accuracy(p, g, th);
        for (int i = 0; i < n_thr; ++i) fractions[i] = r.fractions[i];
        *evaluated = r.evaluated;
        *mean_abs_error = r.meanAbsError;
        return PS_OK;
    } catch (const std::exception& e) {
        return statusOf(e);
    }
}

// The reference's own timing harness (proj/src/eval.cpp:144-177): pinned
// core, one warm-up, sorted samples; returns the median ms of `repeats` runs.
double ref_benchmark_run(const uint8_t* left, const uint8_t* right, int w, int h,
                         const ps_config* cfg, int repeats) {
    TimingReport r = benchmark(
        [&] {
            ref_run(left, right, w, h, cfg, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, nullptr, nullptr, 0, nullptr);
        },
        repeats, true, "ref_run");
    return r.medianMs;
}

// Inputs for the reference arm: the repo's seeded generator (synth.cpp,
// compiled into this library), frame f seeded with seed + f.
ps_status ps_synth_batch(const ps_synth_params* p, int n_frames, int threads, uint8_t* left,
                         uint8_t* right);
int ref_synth_batch(int width, int height, int n_planes, int max_disparity, int ground,
                    float sigma, unsigned seed, int n_frames, int threads, uint8_t* left,
                    uint8_t* right) {
    ps_synth_params p{width, height, n_planes, max_disparity, ground, sigma, seed};
    return ps_synth_batch(&p, n_frames, threads, left, right);
}

}  // extern "C"
