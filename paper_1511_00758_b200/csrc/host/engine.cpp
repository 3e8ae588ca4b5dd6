// engine.cpp — batched B200 pipeline (see engine.hpp).
//
// Stage order per batch mirrors planestereo::run (proj/src/pipeline.cpp:131-203):
//   K1 frontend -> K2 candidates -> K3 seed match -> seed compaction     (all frames)
//   for it in 1..iterations:  for each frame group g (own stream):
//       supports delta D2H -> host Delaunay per frame (thread pool) -> triangles H2D
//       K5/K6 mesh (planes + lookup) -> K7 refine (+K9 dense on the last iteration)
//       if not last: K8 resample (confident append, invalid cells -> K3 re-match -> append)
//   trace reduction D2H.
// The device stages of group g are enqueued asynchronously, so they run while
// the host triangulates group g+1 (a software pipeline over groups).
#include "engine.hpp"

#include <algorithm>
#ifdef __SSE2__
#include <emmintrin.h>
#endif
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <sys/resource.h>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include <sched.h>

#include "../kernels/launch.hpp"
#include "frame_mesh.hpp"

namespace ps {

namespace {

int ceil_div(int a, int b) { return (a + b - 1) / b; }

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

// PipelineConfig::validate (proj/src/config.cpp:17-49); messages match.
ps_status validate_config(const ps_config& c, unsigned flags, std::string& msg) {
    if (c.iterations < 1) {
        msg = "iterations must be >= 1, got " + std::to_string(c.iterations);
        return PS_INVALID_CONFIG;
    }
    if (c.max_disparity < 1) {
        msg = "max disparity must be >= 1, got " + std::to_string(c.max_disparity);
        return PS_INVALID_CONFIG;
    }
    if (!(c.cost_low > 0.0f && c.cost_low < c.cost_high && c.cost_high <= 1.0f)) {
        msg = "cost thresholds must satisfy 0 < low < high <= 1";
        return PS_INVALID_CONFIG;
    }
    const bool cell_ok = (flags & PS_RUN_UNCHECKED_CELL) ? c.occupancy_cell_size >= 1
                                                          : is_pow2(c.occupancy_cell_size);
    if (!cell_ok) {
        msg = "occupancy cell size must be a power of two, got " +
              std::to_string(c.occupancy_cell_size);
        return PS_INVALID_CONFIG;
    }
    if (c.gradient_threshold < 0) {
        msg = "gradient threshold must be non-negative";
        return PS_INVALID_CONFIG;
    }
    if (c.corner_threshold < 0) {
        msg = "corner threshold must be non-negative";
        return PS_INVALID_CONFIG;
    }
    if (c.per_bin_cap < 1) {
        msg = "per-bin cap must be >= 1";
        return PS_INVALID_CONFIG;
    }
    if (!(c.sparse_accept_cost > 0.0f && c.sparse_accept_cost <= 1.0f)) {
        msg = "sparse accept cost must lie in (0, 1]";
        return PS_INVALID_CONFIG;
    }
    if (!(c.uniqueness_ratio > 0.0f && c.uniqueness_ratio <= 1.0f)) {
        msg = "uniqueness ratio must lie in (0, 1]";
        return PS_INVALID_CONFIG;
    }
    if (c.threads < 1) {
        msg = "threads must be >= 1";
        return PS_INVALID_CONFIG;
    }
    if (c.max_disparity > 65535) {  // packed (k << 16 | d) warp keys in K3
        msg = "max disparity above 65535 is not supported by this build";
        return PS_INVALID_CONFIG;
    }
    return PS_OK;
}

// Host-evaluated binary32 decision tables (this file is built with
// -ffp-contract=off; x86-64 SSE evaluates float in binary32 exactly as the
// reference does).
CostTables make_tables(const ps_config& c) {
    CostTables t{};
    volatile float ratio = c.uniqueness_ratio;
    for (int k = 0; k <= kCensusBits; ++k) t.cost[k] = float(k) / float(kCensusBits);
    for (int k = 0; k <= kCensusBits; ++k) {
        if (t.cost[k] < c.cost_low) t.low_mask |= 1u << k;
        if (t.cost[k] > c.cost_high) t.high_mask |= 1u << k;
        if (!(t.cost[k] > c.sparse_accept_cost)) t.accept_mask |= 1u << k;
        for (int k2 = 0; k2 <= kCensusBits; ++k2) {
            volatile float prod = ratio * t.cost[k2];
            if (t.cost[k] > prod) t.uniq_reject[k] |= 1u << k2;
        }
    }
    t.code_high = 0;
    while (t.code_high <= kCensusBits && t.cost[t.code_high] < c.cost_high) ++t.code_high;
    for (int k = 0; k < t.code_high; ++k)
        t.fixed[k] = (unsigned long long)std::ldexp(double(t.cost[k]), 36);
    t.fixed[t.code_high] = (unsigned long long)std::ldexp(double(c.cost_high), 36);
    t.cost_high = c.cost_high;
    return t;
}

// C_f from its byte code: cost[c] = float(c) / 24.0f (make_tables) for
// c < code_high, else costHigh -- 16 codes per step with SSE2 (divps is
// correctly rounded, so the values are make_tables' bit for bit).
static void expand_costs(const uint8_t* __restrict__ in, float* __restrict__ out, size_t n, int ch, float chigh) {
    size_t i = 0;
#ifdef __SSE2__
    const __m128 d24 = _mm_set1_ps(float(kCensusBits)), hi = _mm_set1_ps(chigh);
    const __m128i chv = _mm_set1_epi32(ch), zero = _mm_setzero_si128();
    // scalar head up to a 16-byte boundary of the output, then non-temporal
    // stores: the map is written once and read by the caller much later, so
    // the lines need not be fetched for ownership (a quarter less host memory
    // traffic beside the DMA writes of the other outputs)
    static const bool nt = [] {  // PS_EXPAND_NT=0: ordinary stores (A/B probe)
        const char* e = std::getenv("PS_EXPAND_NT");
        return !e || std::atoi(e) != 0;
    }();
    for (; i < n && (reinterpret_cast<uintptr_t>(out + i) & 15u) != 0; ++i)
        out[i] = int(in[i]) < ch ? float(in[i]) / float(kCensusBits) : chigh;
    for (; i + 16 <= n; i += 16) {
        const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i));
        const __m128i lo16 = _mm_unpacklo_epi8(v, zero), hi16 = _mm_unpackhi_epi8(v, zero);
        const __m128i q[4] = {_mm_unpacklo_epi16(lo16, zero), _mm_unpackhi_epi16(lo16, zero),
                              _mm_unpacklo_epi16(hi16, zero), _mm_unpackhi_epi16(hi16, zero)};
        for (int k = 0; k < 4; ++k) {
            const __m128 x = _mm_div_ps(_mm_cvtepi32_ps(q[k]), d24);
            const __m128 m = _mm_castsi128_ps(_mm_cmplt_epi32(q[k], chv));
            const __m128 y = _mm_or_ps(_mm_and_ps(m, x), _mm_andnot_ps(m, hi));
            if (nt)
                _mm_stream_ps(out + i + 4 * k, y);
            else
                _mm_store_ps(out + i + 4 * k, y);
        }
    }
    _mm_sfence();
#endif
    for (; i < n; ++i) out[i] = int(in[i]) < ch ? float(in[i]) / float(kCensusBits) : chigh;
}

// C_f values are k/24 floats or costHigh; their 2^-36 fixed-point sum is exact
// iff costHigh * 2^36 is an integer (true for costHigh >= 2^-12 with a short
// mantissa, e.g. every decimal-looking default).
bool trace_fixed_exact(float cost_high) {
    const double x = std::ldexp(double(cost_high), 36);
    return x == std::floor(x);
}

// Host worker threads for the Delaunay tasks: PS_HOST_THREADS if set, else
// the CPUs this process may run on (affinity / cpuset), shared evenly between
// the ranks of a node (LOCAL_WORLD_SIZE, set by torchrun) so N GPUs' engines
// do not oversubscribe the host.
static int host_threads() {
    if (const char* e = std::getenv("PS_HOST_THREADS")) {
        const int n = std::atoi(e);
        if (n > 0) return n;
    }
    int n = int(std::max(1u, std::thread::hardware_concurrency()));
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof(set), &set) == 0 && CPU_COUNT(&set) > 0) n = CPU_COUNT(&set);
    if (const char* l = std::getenv("LOCAL_WORLD_SIZE")) {
        const int k = std::atoi(l);
        if (k > 1) n = std::max(1, n / k);
    }
    return n;
}

// One Delaunay worker pool per process, shared by every context (several
// contexts in one process — ps_run_batch_multi — must not multiply the host
// threads), with one workspace per worker: a worker runs one task at a time.
static ThreadPool& shared_pool() {
    static ThreadPool pool(host_threads());
    return pool;
}
static std::vector<DelaunayWorkspace>& shared_workspaces() {
    static std::vector<DelaunayWorkspace> ws(shared_pool().size());
    return ws;
}
// order-query scratch per worker (queries of one frame run on several workers)
static std::vector<SweepOrder::Scratch>& shared_order_scratch() {
    static std::vector<SweepOrder::Scratch> s(shared_pool().size());
    return s;
}

Engine::Engine(int device) : device_(device) {
    cudaSetDevice(device_);
    cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking);
    // The groups' pixel stages (small, latency-critical: they feed the host
    // pool) run at the highest priority, the bulk seeding at the lowest, and
    // the groups' meshes in between, earlier groups first: the first group's
    // mesh finishes (and its host work starts) while later meshes still run,
    // instead of all of them finishing together and leaving the host the tail.
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    // PS_GROUP_PRIO=1: both streams of a group at the group's own priority,
    // earlier groups first (the device drains group 0, then 1, ...: groups
    // finish staggered and their output copies overlap later groups' work)
    const char* gp = std::getenv("PS_GROUP_PRIO");
    group_prio_ = gp ? std::atoi(gp) != 0 : group_prio_;
    for (int gi = 0; gi < kMaxGroups; ++gi) {
        FrameGroup& g = groups_[gi];
        const int by_group = std::min(prio_low, prio_high + gi);  // numerically lower = higher
        const int mesh_prio = group_prio_ ? by_group : std::min(prio_low, prio_high + 1 + gi);
        cudaStreamCreateWithPriority(&g.st, cudaStreamNonBlocking, group_prio_ ? by_group : prio_high);
        cudaStreamCreateWithPriority(&g.mst, cudaStreamNonBlocking, mesh_prio);
        cudaEventCreateWithFlags(&g.mesh_in, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&g.mesh_out, cudaEventDisableTiming);
    }
    cudaStreamCreateWithPriority(&seed_st_, cudaStreamNonBlocking, prio_low);
    cudaEventCreateWithFlags(&start_event_, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&chain_event_, cudaEventDisableTiming);
    if (const char* e = std::getenv("PS_SERIAL_DEVICE")) serial_device_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("PS_MIN_GROUP")) min_group_ = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PS_HOST_FIRST")) host_first_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("PS_WIRE_CODES")) wire_codes_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("PS_MAX_GROUPS")) set_max_groups(std::atoi(e));
    debug_timeline_ = std::getenv("PS_DEBUG_TIMELINE") != nullptr;
    pool_ = &shared_pool();
    ws_ = &shared_workspaces();
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    DevBuf* bufs[] = {&dL_, &dR_, &dMask_, &dMaskCount_, &dCL_, &dCR_, &dDf_, &dDv_, &dCf_, &dCode_,
                      &dDense_, &dDenseV_, &dLookup_, &dSu_, &dSv_, &dSd_, &dS_, &dSnext_,
                      &dTaken_, &dCg_, &dCb_, &dBinKeys_, &dBinCount_, &dScratch_, &dCandU_,
                      &dCandV_, &dCandCount_, &dOk_, &dDisp_, &dRemU_, &dRemV_, &dRemCount_,
                      &dConf_, &dChunk_, &dTraceSum_, &dTraceValid_, &dErr_, &dOkSeed_, &dDispSeed_,
                      &dFrameOk_, &s_a, &s_b, &s_c,
                      &s_d, &s_e, &s_f, &s_g, &s_h, &s_i, &s_j};
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    HostBuf* hbufs[] = {&hS_, &hTraceSum_, &hTraceValid_, &hMaskCount_, &hCodeStage_};
    for (HostBuf* b : hbufs)
        if (b->p) cudaFreeHost(b->p);
    for (FrameGroup& g : groups_) {
        for (DevBuf* b : {&g.dTri, &g.dTriOff, &g.dPlanes, &g.dPack, &g.dPackD, &g.dPackOff,
                          &g.dSprev, &g.dChunk, &g.dPin, &g.dCellCnt, &g.dCellStart, &g.dCellItems, &g.dCellXY,
                          &g.dDup, &g.dPinTri, &g.dTriCount, &g.dFlags, &g.dFix, &g.dColKey, &g.dColIdx, &g.dHull, &g.dHullTmp, &g.dHard, &g.dRing})
            if (b->p) cudaFree(b->p);
        for (HostBuf* b : {&g.hS, &g.hSprev, &g.hPackOff, &g.hPack, &g.hPackD, &g.hTri, &g.hTriOff,
                           &g.hPin, &g.hTriCount, &g.hFlags, &g.hFix})
            if (b->p) cudaFreeHost(b->p);
        if (g.st) cudaStreamDestroy(g.st);
        if (g.mst) cudaStreamDestroy(g.mst);
        if (g.mesh_in) cudaEventDestroy(g.mesh_in);
        if (g.mesh_out) cudaEventDestroy(g.mesh_out);
        if (g.done_event) cudaEventDestroy(g.done_event);
    }
    for (auto& p : pending_) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
    if (start_event_) cudaEventDestroy(start_event_);
    if (chain_event_) cudaEventDestroy(chain_event_);
    if (seed_st_) cudaStreamDestroy(seed_st_);
    if (st_) cudaStreamDestroy(st_);
}

template <class T>
T* Engine::dev(DevBuf& b, size_t count) {
    const size_t need = std::max<size_t>(count * sizeof(T), 256);
    if (b.bytes < need) {
        if (b.p) {
            cudaDeviceSynchronize();
            cudaFree(b.p);
        }
        b.p = nullptr;
        b.bytes = 0;
        if (cudaMalloc(&b.p, need) != cudaSuccess) {
            b.p = nullptr;
            return nullptr;
        }
        b.bytes = need;
    }
    return static_cast<T*>(b.p);
}

template <class T>
T* Engine::host(HostBuf& b, size_t count) {
    const size_t need = std::max<size_t>(count * sizeof(T), 256);
    if (b.bytes < need) {
        if (b.p) {
            cudaDeviceSynchronize();
            cudaFreeHost(b.p);
        }
        b.p = nullptr;
        b.bytes = 0;
        if (cudaHostAlloc(&b.p, need, cudaHostAllocDefault) != cudaSuccess) {
            b.p = nullptr;
            return nullptr;
        }
        b.bytes = need;
    }
    return static_cast<T*>(b.p);
}

template uint16_t* Engine::dev<uint16_t>(DevBuf&, size_t);
template uint8_t* Engine::dev<uint8_t>(DevBuf&, size_t);
template int* Engine::dev<int>(DevBuf&, size_t);
template uint32_t* Engine::dev<uint32_t>(DevBuf&, size_t);
template float* Engine::dev<float>(DevBuf&, size_t);
template double* Engine::dev<double>(DevBuf&, size_t);
template unsigned long long* Engine::dev<unsigned long long>(DevBuf&, size_t);
template int2* Engine::dev<int2>(DevBuf&, size_t);
template SceneRegionDev* Engine::dev<SceneRegionDev>(DevBuf&, size_t);
template int* Engine::host<int>(HostBuf&, size_t);
template uint8_t* Engine::host<uint8_t>(HostBuf&, size_t);

ps_status Engine::check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return PS_OK;
    return fail(PS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

ps_status Engine::sync(const char* what) { return sync(st_, what); }

ps_status Engine::sync(cudaStream_t s, const char* what) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    return check(e, what);
}

cudaEvent_t Engine::take_event() {
    cudaEvent_t e;
    if (!event_pool_.empty()) {
        e = event_pool_.back();
        event_pool_.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}

void Engine::begin_kernel(const char* name, double bytes, cudaStream_t s) {
    if (!profiling_) return;
    int idx = -1;
    for (size_t i = 0; i < stats_.size(); ++i)
        if (stats_[i].name == name) idx = int(i);
    if (idx < 0) {
        stats_.push_back({name, 0, 0.0, 0.0});
        idx = int(stats_.size()) - 1;
    }
    stats_[idx].bytes += bytes;
    stats_[idx].launches += 1;
    cudaEvent_t a = take_event();
    cudaEventRecord(a, s);
    pending_stat_ = idx;
    pending_start_ = a;
}

void Engine::end_kernel(cudaStream_t s) {
    if (!profiling_ || pending_stat_ < 0) return;
    cudaEvent_t b = take_event();
    cudaEventRecord(b, s);
    pending_.push_back({pending_stat_, pending_start_, b});
    pending_stat_ = -1;
}

void Engine::resolve_timers() {
    for (auto& p : pending_) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) stats_[p.stat].ms += ms;
        event_pool_.push_back(p.a);
        event_pool_.push_back(p.b);
    }
    pending_.clear();
}

ps_status Engine::upload(int frames, const uint8_t* left, const uint8_t* right, int width,
                         int height, bool deferred) {
    if (width < 16 || height < 16)
        return fail(PS_DIMENSION_TOO_SMALL, "image must be at least 16x16, got " +
                                                std::to_string(width) + "x" +
                                                std::to_string(height));
    if (frames < 1) return fail(PS_ERROR, "batch needs at least one frame");
    cudaSetDevice(device_);
    F_ = frames;
    W_ = width;
    H_ = height;
    P_ = (long long)width * height;
    const size_t n = size_t(F_) * P_;
    uint8_t* dl = dev<uint8_t>(dL_, n);
    uint8_t* dr = dev<uint8_t>(dR_, n);
    if (!dl || !dr) return fail(PS_CUDA_ERROR, "device allocation failed (images)");
    defer_left_ = deferred ? left : nullptr;
    defer_right_ = deferred ? right : nullptr;
    if (deferred) {
        have_inputs_ = true;
        have_outputs_ = false;
        streamed_ = false;
        return PS_OK;
    }
    ps_status s = check(cudaMemcpyAsync(dl, left, n, cudaMemcpyHostToDevice, st_), "H2D left");
    if (s != PS_OK) return s;
    s = check(cudaMemcpyAsync(dr, right, n, cudaMemcpyHostToDevice, st_), "H2D right");
    if (s != PS_OK) return s;
    have_inputs_ = true;
    have_outputs_ = false;
    streamed_ = false;
    return PS_OK;
}

ps_status Engine::device_inputs(int frames, int width, int height, uint8_t** left,
                                uint8_t** right) {
    if (width < 16 || height < 16)
        return fail(PS_DIMENSION_TOO_SMALL, "image must be at least 16x16, got " +
                                                std::to_string(width) + "x" +
                                                std::to_string(height));
    if (frames < 1) return fail(PS_ERROR, "batch needs at least one frame");
    cudaSetDevice(device_);
    F_ = frames;
    W_ = width;
    H_ = height;
    P_ = (long long)width * height;
    const size_t n = size_t(F_) * P_;
    *left = dev<uint8_t>(dL_, n);
    *right = dev<uint8_t>(dR_, n);
    if (!*left || !*right) return fail(PS_CUDA_ERROR, "device allocation failed (images)");
    defer_left_ = defer_right_ = nullptr;
    have_inputs_ = true;
    have_outputs_ = false;
    streamed_ = false;
    return PS_OK;
}

ps_status Engine::run_resident(const ps_config& cfg, unsigned flags, ps_observer_fn observer,
                               void* user) {
    if (!have_inputs_) return fail(PS_ERROR, "no batch uploaded");
    ps_status st = validate_config(cfg, flags, err_);
    if (st != PS_OK) return st;
    cudaSetDevice(device_);
    const int F = F_, W = W_, H = H_;
    const long long P = P_;
    const FrameGeom g{W, H, P};
    const CostTables tab = make_tables(cfg);
    const int iters = cfg.iterations;
    iters_ = iters;
    cost_high_ = cfg.cost_high;
    const bool fixed_trace = trace_fixed_exact(cfg.cost_high);

    // cell schedule s_i (pipeline.cpp:147,171) and capacities
    std::vector<int> cell_of(iters);
    long long bound = 120ll * cfg.per_bin_cap;
    int cells_max = 1;
    for (int it = 0, s = cfg.occupancy_cell_size; it < iters; ++it) {
        cell_of[it] = s;
        const int cells = ceil_div(W, s) * ceil_div(H, s);
        cells_max = std::max(cells_max, cells);
        if (it + 1 < iters) bound += 2ll * cells;
        s = std::max(1, s / 2);
    }
    scap_ = int(std::min<long long>(P, bound));
    const int cand_stride = 120 * cfg.per_bin_cap;
    const int chunks = ceil_div(std::max(cand_stride, cells_max), 1024);
    const long long words = (P + 31) / 32;
    int n_pow2 = 1;
    while (n_pow2 < std::min<long long>(cand_stride, P)) n_pow2 <<= 1;
    const long long sc_stride = candidate_scratch_stride(g);
    const size_t scratch_keys =
        cfg.per_bin_cap > 8 ? size_t(F) * std::max<long long>(120 * sc_stride, n_pow2) : 1;

    uint8_t* dMask = dev<uint8_t>(dMask_, size_t(F) * P);
    int* dMaskCount = dev<int>(dMaskCount_, F);
    uint32_t* dCL = dev<uint32_t>(dCL_, size_t(F) * P);
    uint32_t* dCR = dev<uint32_t>(dCR_, size_t(F) * P);
    float* dDf = dev<float>(dDf_, size_t(F) * P);
    uint8_t* dDv = dev<uint8_t>(dDv_, size_t(F) * P);
    float* dCf = dev<float>(dCf_, size_t(F) * P);
    uint8_t* dCode = dev<uint8_t>(dCode_, size_t(F) * P);
    float* dDense = dev<float>(dDense_, size_t(F) * P);
    uint8_t* dDenseV = dev<uint8_t>(dDenseV_, size_t(F) * P);
    float* dDit = dev<float>(dLookup_, size_t(F) * P);  // D_it per pixel (NaN = invalid)
    int* dSu = dev<int>(dSu_, size_t(F) * scap_);
    int* dSv = dev<int>(dSv_, size_t(F) * scap_);
    double* dSd = dev<double>(dSd_, size_t(F) * scap_);
    int* dS = dev<int>(dS_, F);
    int* dSnext = dev<int>(dSnext_, F);
    uint32_t* dTaken = dev<uint32_t>(dTaken_, size_t(F) * words);
    unsigned long long* dCg = dev<unsigned long long>(dCg_, size_t(F) * cells_max);
    unsigned long long* dCb = dev<unsigned long long>(dCb_, size_t(F) * cells_max);
    unsigned long long* dBinKeys = dev<unsigned long long>(dBinKeys_, size_t(F) * 120 * cfg.per_bin_cap);
    int* dBinCount = dev<int>(dBinCount_, size_t(F) * 120);
    unsigned long long* dScratch = dev<unsigned long long>(dScratch_, scratch_keys);
    int* dCandU = dev<int>(dCandU_, size_t(F) * cand_stride);
    int* dCandV = dev<int>(dCandV_, size_t(F) * cand_stride);
    int* dCandCount = dev<int>(dCandCount_, F);
    // match scratch: seeding and resampling use disjoint buffers (frame groups
    // seed on seed_st_ while earlier groups resample on their own streams)
    uint8_t* dOk = dev<uint8_t>(dOk_, size_t(F) * cells_max);
    int* dDisp = dev<int>(dDisp_, size_t(F) * cells_max);
    uint8_t* dOkSeed = dev<uint8_t>(dOkSeed_, size_t(F) * cand_stride);
    int* dDispSeed = dev<int>(dDispSeed_, size_t(F) * cand_stride);
    int* dRemU = dev<int>(dRemU_, size_t(F) * cells_max);
    int* dRemV = dev<int>(dRemV_, size_t(F) * cells_max);
    int* dRemCount = dev<int>(dRemCount_, F);
    int* dConf = dev<int>(dConf_, F);
    unsigned long long* dTraceSum = dev<unsigned long long>(dTraceSum_, size_t(F) * iters);
    unsigned* dTraceValid = dev<uint32_t>(dTraceValid_, size_t(F) * iters);
    int* dErr = dev<int>(dErr_, 1);
    int* hS = host<int>(hS_, F);
    int* hMaskCount = host<int>(hMaskCount_, F);
    unsigned long long* hTraceSum =
        reinterpret_cast<unsigned long long*>(host<uint8_t>(hTraceSum_, size_t(F) * iters * 8));
    unsigned* hTraceValid = reinterpret_cast<unsigned*>(host<uint8_t>(hTraceValid_, size_t(F) * iters * 4));
    const void* must[] = {dMask, dMaskCount, dCL, dCR, dDf, dDv, dCf, dCode, dDense, dDenseV, dDit,
                          dSu, dSv, dSd, dS, dSnext, dTaken, dCg, dCb, dBinKeys, dBinCount,
                          dScratch, dCandU, dCandV, dCandCount, dOk, dDisp, dOkSeed, dDispSeed, dRemU, dRemV,
                          dRemCount, dConf, dTraceSum, dTraceValid, dErr, hS, hMaskCount,
                          hTraceSum, hTraceValid};
    for (const void* p : must)
        if (!p) return fail(PS_CUDA_ERROR, "allocation failed for a batch of " + std::to_string(F) +
                                               " frames of " + std::to_string(W) + "x" +
                                               std::to_string(H));

    const uint8_t* dL = static_cast<const uint8_t*>(dL_.p);
    const uint8_t* dR = static_cast<const uint8_t*>(dR_.p);
    // A deferred upload (ps_run_batch) is consumed by this run whatever
    // happens: on an early return the batch no longer counts as uploaded.
    struct DeferGuard {
        Engine* e;
        ~DeferGuard() {
            if (e->defer_left_) e->have_inputs_ = false;
            e->defer_left_ = e->defer_right_ = nullptr;
        }
    } defer_guard{this};
    const uint8_t* upL = defer_left_;
    const uint8_t* upR = defer_right_;

    status_.assign(F, PS_OK);
    final_count_.assign(F, 0);
    double host_dt_ms = 0.0;
    // per-frame mesh state, kept across the iterations of this run (the
    // triangulation is extended, not rebuilt: frame_mesh.hpp)
    // Mesh: on the device (kernels/star.cu) by default; PS_DELAUNAY=host runs
    // the host incremental path (frame_mesh.cpp), =lex replays the reference
    // sweep for every frame-iteration.  The device predicates are int64: the
    // frame must span < 2^14 pixels.
    const char* dt_mode = std::getenv("PS_DELAUNAY");
    const bool lex_only = dt_mode && std::string(dt_mode) == "lex";
    const bool device_dt = !(dt_mode && (std::string(dt_mode) == "host" || lex_only)) &&
                           W < (1 << 14) && H < (1 << 14) &&
                           16ll * W + 16ll * H + 16 <= 200 * 1024;  // k_hull's column extremes in shared memory
    if (int(fmesh_.size()) < F) fmesh_.resize(F);
    for (int f = 0; f < F; ++f) {
        fmesh_[f].reset();
        fmesh_[f].lex_only = lex_only;
    }
    std::vector<MeshStats> mstats(pool_->size());
    trace_.assign(size_t(F) * iters, ps_iter_stats{});

    // ---- frame groups: a dataflow pipeline.  Per group: (H2D of a deferred
    //   upload ->) seeding on the low-priority seeding stream; then each
    //   iteration is delta D2H -> Delaunay tasks on the worker pool ->
    //   triangles H2D -> device stages on the group's (high-priority) stream,
    //   chained after the previous group's stages -> (completion) -> next
    //   iteration.
    // The host loop below only moves data and launches; the workers
    // triangulate continuously while the device runs other groups' stages.
    // frame groups of >= 64 frames (measured on cfg2: 4 groups of 64 beat 8 of 32)
    const int G = std::max(1, std::min(std::min(kMaxGroups, max_groups_), (F + min_group_ - 1) / min_group_));
    const int tri_cap = int(std::min<long long>(2ll * scap_ + 8, 2ll * P + 8));  // T <= 2S per frame
    // device mesh grid of iteration `it` (1-based): ~1-3 supports per cell —
    // seeds: <= 120 * cap over the frame; later: at most ~2 per cell of the
    // previous iteration's occupancy grid (plus the older, sparser supports)
    // ~1.3 supports per cell, so the 5x5 cells a star starts from hold ~30
    // candidates (star_dt.cuh kLocalMax); est = expected supports per frame
    static const double star_density = [] {  // supports per grid cell (PS_STAR_DENSITY: probing)
        const char* e = std::getenv("PS_STAR_DENSITY");
        return e ? std::atof(e) : 1.3;
    }();
    auto star_gs = [&](double est) {
        return std::max(2, int(std::sqrt(star_density * double(P) / std::max(1.0, est)) + 0.5));
    };
    const StarFlagLayout flay = star_flag_layout(scap_);
    // C_f and validity over PCIe as the byte codes (expand(): C_f = cost[c]
    // for c < code_high, else costHigh; valid = c < code_high -- K7's own
    // expansion, refine.cu)
    const bool wire_codes = wire_codes_ && sink_.active && (sink_.cost || sink_.disparity_valid);
    uint8_t* hCodes = wire_codes ? host<uint8_t>(hCodeStage_, size_t(F) * P) : nullptr;
    if (wire_codes && !hCodes) return fail(PS_CUDA_ERROR, "allocation failed (code staging)");
    const Sink wsink = sink_;
    auto expand = [&](int f0, int n) {
        // a task per 4 frames; the run waits for them before it returns
        for (int a = 0; a < n; a += 4) {
            const int fa = f0 + a, fn = std::min(4, n - a);
            expand_pending_.fetch_add(1);
            pool_->submit([this, fa, fn, P, hCodes, wsink, ch = tab.code_high, chigh = tab.cost_high](int) {
                const size_t b = size_t(fa) * P, n = size_t(fn) * P;
                const uint8_t* __restrict__ in = hCodes + b;
                // cost[c] = float(c) / 24.0f (make_tables, census.hpp:45-47):
                // a correctly rounded division, so the loop vectorises
                if (wsink.cost) expand_costs(in, wsink.cost + b, n, ch, chigh);
                if (wsink.disparity_valid) {
                    uint8_t* __restrict__ out = wsink.disparity_valid + b;
                    for (size_t i = 0; i < n; ++i) out[i] = in[i] < ch ? 1 : 0;
                }
                std::lock_guard<std::mutex> lk(done_m_);
                if (expand_pending_.fetch_sub(1) == 1) done_cv_.notify_all();
            });
        }
    };
    // the first iteration's mesh (the seeds only) on the host: the device's
    // mesh kernels are latency-bound at that size and the device is the
    // busier side (PS_HOST_FIRST=0: device for every iteration)
    const bool host_first = device_dt && host_first_;
    // fewer frames than host workers: a frame's order queries spread over the
    // idle workers, so a larger query budget still beats the serial replay
    const int budget_scale = std::max(1, int(pool_->size()) / std::max(1, F));
    const long long star_cells_max = (long long)((W - 1) / 2 + 1) * ((H - 1) / 2 + 1);  // gs >= 2
    cudaMemsetAsync(dErr, 0, sizeof(int), st_);
    ps_status s = check(cudaEventRecord(start_event_, st_), "start event");
    if (s != PS_OK) return s;
    const long long scratch_per_frame =
        cfg.per_bin_cap > 8 ? std::max<long long>(120 * sc_stride, n_pow2) : 0;
    // Seeding of one group (on seed_st_, in group order).  Group 0 is launched
    // before the dataflow loop, the others from inside it (one per loop turn),
    // so the first host tasks do not wait for the launches of every group.
    for (int gi = 0; gi < G; ++gi) groups_[gi].phase = FrameGroup::kIdle;
    // Device mesh of iteration `it` for the group's current supports (grp.S),
    // then its triangle counts and flag records to the host (star.cu).
    auto star_args = [&](FrameGroup& grp) {
        StarArgs a{};
        const size_t f0 = size_t(grp.f0);
        a.su = dSu + f0 * scap_;
        a.sv = dSv + f0 * scap_;
        a.sd = dSd + f0 * scap_;
        a.scap = scap_;
        a.S = grp.S;
        a.frames = grp.n;
        a.W = W;
        a.H = H;
        a.max_disp = float(cfg.max_disparity);
        a.gs = grp.gs;
        a.gw = grp.gw;
        a.gh = grp.gh;
        a.cell_cnt = static_cast<int*>(grp.dCellCnt.p);
        a.cell_start = static_cast<int*>(grp.dCellStart.p);
        a.cell_items = static_cast<int*>(grp.dCellItems.p);
        a.cell_xy = static_cast<int*>(grp.dCellXY.p);
        a.dup = static_cast<uint8_t*>(grp.dDup.p);
        a.pin_tri = static_cast<int*>(grp.dPinTri.p);
        a.tris = static_cast<int*>(grp.dTri.p);
        a.pitch = tri_cap;
        a.pins = static_cast<uint8_t*>(grp.dPin.p);
        a.tri_count = static_cast<int*>(grp.dTriCount.p);
        a.flags = static_cast<int*>(grp.dFlags.p);
        a.flag_ints = flay.ints;
        a.max_suspect = flay.max_suspect;
        a.fan_base = flay.fan_base;
        a.col_key = static_cast<unsigned long long*>(grp.dColKey.p);
        a.col_idx = static_cast<int*>(grp.dColIdx.p);
        a.hull = static_cast<int*>(grp.dHull.p);
        a.hull_tmp = static_cast<int*>(grp.dHullTmp.p);
        a.hard = static_cast<int*>(grp.dHard.p);
        a.ring = static_cast<int*>(grp.dRing.p);
        static const int phase2 = [] {
            const char* e = std::getenv("PS_STAR_PHASE2");
            return e ? std::atoi(e) : 1;
        }();
        a.phase2 = phase2;
        static const int near = [] {
            const char* e = std::getenv("PS_STAR_NEAR");
            return e ? std::atoi(e) : 1;
        }();
        a.near = near;
        static const int hull_late = [] {
            const char* e = std::getenv("PS_STAR_HULL_LATE");
            return e ? std::atoi(e) : 0;
        }();
        a.hull_late = hull_late;
        return a;
    };
    auto enqueue_mesh = [&](FrameGroup& grp, double est, int max_points) {
        grp.gs = star_gs(est);
        grp.gw = (W - 1) / grp.gs + 1;
        grp.gh = (H - 1) / grp.gs + 1;
        const StarArgs a = star_args(grp);
        // on the group's mesh stream: after the supports exist (st), and st
        // continues (raster of the next iteration, completion event) after it
        cudaStream_t ms = grp.mst;
        cudaEventRecord(grp.mesh_in, grp.st);
        cudaStreamWaitEvent(ms, grp.mesh_in, 0);
        begin_kernel("star_mesh", 0.0, ms);
        launches_ += launch_star_mesh(a, std::min(max_points, scap_), ms);
        launches_ += launch_star_check(a, tri_cap, ms);
        end_kernel(ms);
        cudaMemcpyAsync(grp.hTriCount.p, grp.dTriCount.p, sizeof(int) * grp.n, cudaMemcpyDeviceToHost, ms);
        cudaMemcpyAsync(grp.hFlags.p, grp.dFlags.p, sizeof(int) * size_t(grp.n) * flay.ints,
                        cudaMemcpyDeviceToHost, ms);
        cudaEventRecord(grp.mesh_out, ms);
        cudaStreamWaitEvent(grp.st, grp.mesh_out, 0);
    };
    auto seed_group = [&](int gi) -> ps_status {
        FrameGroup& grp = groups_[gi];
        grp.f0 = int((long long)F * gi / G);
        grp.n = int((long long)F * (gi + 1) / G) - grp.f0;
        grp.S = dS + grp.f0;
        grp.Snext = dSnext + grp.f0;
        grp.ntri.assign(grp.n, 0);
        grp.it = 0;
        grp.phase = FrameGroup::kIdle;
        grp.pending.store(0);
        int* hs = host<int>(grp.hS, grp.n);
        int* hsp = host<int>(grp.hSprev, grp.n);
        int* gchunk = dev<int>(grp.dChunk, size_t(grp.n) * chunks + 1);
        if (!host<int>(grp.hPackOff, grp.n) || !host<int>(grp.hTriOff, grp.n + 1) ||
            !dev<int>(grp.dTriOff, grp.n + 1) || !dev<int>(grp.dPackOff, grp.n) ||
            !dev<int>(grp.dSprev, grp.n) || !gchunk ||
            !host<int>(grp.hTri, size_t(grp.n) * tri_cap * 3) ||
            !host<uint8_t>(grp.hPin, size_t(grp.n) * tri_cap) || !hs || !hsp) {
            return fail(PS_CUDA_ERROR, "allocation failed (group staging)");
        }
        if (!grp.done_event) cudaEventCreateWithFlags(&grp.done_event, cudaEventDisableTiming);
        grp.fixes.assign(grp.n, {});
        grp.replayed.assign(grp.n, 0);
        if (device_dt) {
            const size_t nn = size_t(grp.n);
            if (!dev<int>(grp.dCellCnt, nn * star_cells_max) || !dev<int>(grp.dCellStart, nn * (star_cells_max + 1)) ||
                !dev<int>(grp.dCellItems, nn * scap_) || !dev<int>(grp.dCellXY, nn * scap_) || !dev<uint8_t>(grp.dDup, nn * scap_) ||
                !dev<int>(grp.dPinTri, nn * scap_ * 3) || !dev<int>(grp.dTriCount, nn) ||
                !dev<int>(grp.dFlags, nn * flay.ints) || !dev<int>(grp.dTri, nn * tri_cap * 3) ||
                !dev<uint8_t>(grp.dPin, nn * tri_cap) || !host<int>(grp.hTriCount, nn) ||
                !host<int>(grp.hFlags, nn * flay.ints) || !host<int>(grp.hFix, nn * 6 * 96) ||
                !dev<int>(grp.dFix, nn * 6 * 96) ||
                !dev<unsigned long long>(grp.dColKey, nn * 2 * W) || !dev<int>(grp.dColIdx, nn * 2 * W) ||
                !dev<int>(grp.dHull, nn * 2 * scap_) || !dev<int>(grp.dHullTmp, nn * 8 * (2 * size_t(W) + 2 * size_t(H) + 8)) ||
                !dev<int>(grp.dHard, nn * scap_))
                return fail(PS_CUDA_ERROR, "allocation failed (device mesh)");
            // pass-1 stars for pass 2 (a lookup instead of a search per step),
            // kept when they fit in 2 GB per group
            if (nn * size_t(scap_) * kRingInts * sizeof(int) <= (size_t(2) << 30)) {
                if (!dev<int>(grp.dRing, nn * size_t(scap_) * kRingInts))
                    return fail(PS_CUDA_ERROR, "allocation failed (device mesh stars)");
            } else if (grp.dRing.p) {
                cudaFree(grp.dRing.p);
                grp.dRing = DevBuf{};
            }
        }

        // ---- seeding of the group's frames on the (low-priority) seeding
        // stream, in group order: group 0's seeds, and so the first host
        // tasks, arrive after 1/G of the seeding time
        cudaStream_t gs = seed_st_;
        const int f0 = grp.f0, n = grp.n;
        const size_t fp = size_t(f0) * P;
        ps_status s = gi == 0 ? check(cudaStreamWaitEvent(gs, start_event_, 0), "stream order") : PS_OK;
        if (s == PS_OK && upL)
            s = check(cudaMemcpyAsync(static_cast<uint8_t*>(dL_.p) + fp, upL + fp, size_t(n) * P,
                                      cudaMemcpyHostToDevice, gs), "H2D left");
        if (s == PS_OK && upR)
            s = check(cudaMemcpyAsync(static_cast<uint8_t*>(dR_.p) + fp, upR + fp, size_t(n) * P,
                                      cudaMemcpyHostToDevice, gs), "H2D right");
        if (s != PS_OK) return s;
        // state init (pipeline.cpp:145-146: D_f invalid, C_f = costHigh -> code)
        cudaMemsetAsync(dMaskCount + f0, 0, sizeof(int) * n, gs);
        cudaMemsetAsync(dTaken + size_t(f0) * words, 0, sizeof(uint32_t) * n * words, gs);
        cudaMemsetAsync(dTraceSum + size_t(f0) * iters, 0, sizeof(unsigned long long) * n * iters, gs);
        cudaMemsetAsync(dTraceValid + size_t(f0) * iters, 0, sizeof(unsigned) * n * iters, gs);
        cudaMemsetAsync(dDf + fp, 0, sizeof(float) * n * P, gs);
        // K1 frontend (image.cpp:43-60, census.cpp:10-41)
        begin_kernel("frontend", 11.0 * double(P) * n, gs);
        launches_ += launch_frontend(dL + fp, dR + fp, g, n, cfg.gradient_threshold, dMask + fp,
                                     dCL + fp, dCR + fp, dMaskCount + f0, gs, dCode + fp,
                                     tab.code_high);
        end_kernel(gs);
        // K2 candidates (sparse.cpp:84-146)
        int* cu = dCandU + size_t(f0) * cand_stride;
        int* cv = dCandV + size_t(f0) * cand_stride;
        begin_kernel("candidates", double(P) * n, gs);
        launches_ += launch_candidates(dL + fp, g, n, cfg.corner_threshold, cfg.per_bin_cap,
                                       dBinKeys + size_t(f0) * 120 * cfg.per_bin_cap,
                                       dBinCount + size_t(f0) * 120,
                                       dScratch + size_t(f0) * scratch_per_frame, sc_stride, cu,
                                       cv, nullptr, dCandCount + f0, cand_stride, gs);
        end_kernel(gs);
        // K3 seed match (sparse.cpp:148-195) + ordered compaction
        uint8_t* ok = dOkSeed + size_t(f0) * cand_stride;
        int* disp = dDispSeed + size_t(f0) * cand_stride;
        begin_kernel("match_seed", 0.0, gs);
        launches_ += launch_match(dCL + fp, dCR + fp, g, n, cfg.max_disparity, tab, cu, cv,
                                  dCandCount + f0, cand_stride, cand_stride, ok, disp, nullptr, gs);
        end_kernel(gs);
        begin_kernel("compact", 0.0, gs);
        launches_ += launch_emit_matches(cu, cv, dCandCount + f0, cand_stride, cand_stride, ok, disp,
                                         g, n, dTaken + size_t(f0) * words, dSu + size_t(f0) * scap_,
                                         dSv + size_t(f0) * scap_, dSd + size_t(f0) * scap_, scap_,
                                         nullptr, nullptr, grp.S, gchunk, gs);
        end_kernel(gs);
        s = check(cudaMemcpyAsync(hS + f0, grp.S, sizeof(int) * n, cudaMemcpyDeviceToHost, gs), "D2H S");
        if (s == PS_OK)
            s = check(cudaMemcpyAsync(hMaskCount + f0, dMaskCount + f0, sizeof(int) * n,
                                      cudaMemcpyDeviceToHost, gs), "D2H M");
        if (s == PS_OK) s = check(cudaEventRecord(grp.done_event, gs), "seed event");
        // the group's own stream continues after its seeding
        if (s == PS_OK) s = check(cudaStreamWaitEvent(grp.st, grp.done_event, 0), "group order");
        if (s != PS_OK) return s;
        if (device_dt && !host_first) {  // the first iteration's mesh, on the group stream
            enqueue_mesh(grp, 0.75 * cand_stride, cand_stride);  // ~75% of the candidates match
            s = check(cudaEventRecord(grp.done_event, grp.st), "mesh event");
            if (s != PS_OK) return s;
        }
        grp.phase = FrameGroup::kSeed;
        return PS_OK;
    };
    const double run_t0 = now_ms();
    auto thread_cpu_ms = [] {
        rusage ru{};
        getrusage(RUSAGE_THREAD, &ru);
        return ru.ru_utime.tv_sec * 1e3 + ru.ru_utime.tv_usec * 1e-3 + ru.ru_stime.tv_sec * 1e3 +
               ru.ru_stime.tv_usec * 1e-3;
    };
    const double cpu_t0 = debug_timeline_ ? thread_cpu_ms() : 0.0;
    s = seed_group(0);
    if (s != PS_OK) return s;
    int next_seed = 1;
    bool chained = false;  // chain_event_ recorded in this run
    // Before an early return: wait for this run's own host tasks (they hold
    // references to this frame); the pool is shared with other contexts.
    auto drain = [&] {
        std::unique_lock<std::mutex> lk(done_m_);
        done_cv_.wait(lk, [&] {
            for (int gi = 0; gi < G; ++gi)
                if (groups_[gi].pending.load() != 0) return false;
            return expand_pending_.load() == 0;
        });
    };
    std::atomic<double> dt_ms_sum{0.0}, sweep_ms_sum{0.0};
    std::atomic<double> first_task{1e300}, last_task{0.0};  // pool occupancy (profiling)
    std::vector<double> worker_end(pool_->size(), 0.0);     // PS_DEBUG_TIMELINE
    auto add_ms = [](std::atomic<double>& acc, double x) {
        double cur = acc.load();
        while (!acc.compare_exchange_weak(cur, cur + x)) {}
    };

    // (1) supports added since the group's last iteration -> pinned host staging
    auto fetch_delta = [&](FrameGroup& grp, bool counts) -> ps_status {
        const double tfd0 = now_ms();
        const int n = grp.n;
        cudaStream_t gs = grp.st;
        int* hs = static_cast<int*>(grp.hS.p);
        int* hsp = static_cast<int*>(grp.hSprev.p);
        int* hoff = static_cast<int*>(grp.hPackOff.p);
        ps_status r = PS_OK;
        if (counts) {
            r = check(cudaMemcpyAsync(hs, grp.S, sizeof(int) * n, cudaMemcpyDeviceToHost, gs), "D2H S");
            if (r == PS_OK) r = sync(gs, "support count");
            if (r != PS_OK) return r;
        }
        long long total_new = 0;
        int max_new = 0;
        for (int i = 0; i < n; ++i) {
            hoff[i] = int(total_new);
            const int k = hs[i] - hsp[i];
            total_new += k;
            max_new = std::max(max_new, k);
        }
        // the mesh needs the new supports' (u, v) and d (plane checks)
        const size_t npk = size_t(std::max<long long>(total_new, 1));
        int2* dPack = dev<int2>(grp.dPack, npk);
        int2* hPack = reinterpret_cast<int2*>(host<uint8_t>(grp.hPack, npk * 8));
        double* dPackD = dev<double>(grp.dPackD, npk);
        double* hPackD = reinterpret_cast<double*>(host<uint8_t>(grp.hPackD, npk * 8));
        if (!dPack || !hPack || !dPackD || !hPackD)
            return fail(PS_CUDA_ERROR, "allocation failed (support staging)");
        int* dSprev = static_cast<int*>(grp.dSprev.p);
        int* dPackOff = static_cast<int*>(grp.dPackOff.p);
        r = check(cudaMemcpyAsync(dSprev, hsp, sizeof(int) * n, cudaMemcpyHostToDevice, gs), "H2D Sprev");
        if (r == PS_OK)
            r = check(cudaMemcpyAsync(dPackOff, hoff, sizeof(int) * n, cudaMemcpyHostToDevice, gs),
                      "H2D pack offsets");
        if (r != PS_OK) return r;
        const int f0 = grp.f0;
        launches_ += launch_pack_new_supports(dSu + size_t(f0) * scap_, dSv + size_t(f0) * scap_,
                                              dSd + size_t(f0) * scap_, scap_, dSprev, grp.S,
                                              dPackOff, n, max_new, dPack, dPackD, gs);
        if (total_new > 0)
            r = check(cudaMemcpyAsync(hPack, dPack, sizeof(int2) * total_new, cudaMemcpyDeviceToHost, gs),
                      "D2H supports");
        if (total_new > 0 && r == PS_OK)
            r = check(cudaMemcpyAsync(hPackD, dPackD, sizeof(double) * total_new, cudaMemcpyDeviceToHost, gs),
                      "D2H support disparities");
        const double tsync = now_ms();
        if (r == PS_OK) r = sync(gs, "support delta");
        if (debug_timeline_)
            std::fprintf(stderr, "[tl]   fetch_delta g%d it%d: launch %.3f ms, sync %.3f ms\n",
                         int(&grp - groups_), grp.it, tsync - tfd0, now_ms() - tsync);
        return r;
    };

    // (2) host Delaunay per frame (delaunay.cpp:288-325 contract): the radial
    // sweep, or the reference-order sweep when the validity of a pinned hull
    // vertex depends on the triangle order (pins.cpp).  Each task writes its
    // triangles and pin bits into the group's pinned staging at a fixed slot.
    std::vector<int> order;
    auto submit_dt = [&](FrameGroup& grp) {
        grp.pending.store(grp.n);
        grp.phase = FrameGroup::kHost;
        grp.tic = now_ms();
        // largest point sets first: the group's (and the pass's) last tasks
        // are its smallest, so the workers run out of work more evenly
        const int* cnt = static_cast<const int*>(grp.hS.p);
        order.resize(grp.n);
        for (int i = 0; i < grp.n; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
        for (const int i : order) {
            pool_->submit([&, i, gp = &grp](int worker) {
                FrameGroup& g2 = *gp;
                const double t0 = now_ms();
                const int f = g2.f0 + i;
                const int* hs = static_cast<const int*>(g2.hS.p);
                const int* hsp = static_cast<const int*>(g2.hSprev.p);
                const int* hoff = static_cast<const int*>(g2.hPackOff.p);
                const int2* hPack = static_cast<const int2*>(g2.hPack.p);
                const double* hPackD = static_cast<const double*>(g2.hPackD.p);
                const int k = hs[i] - hsp[i];
                FrameMesh& fm = fmesh_[f];
                for (int j = 0; j < k; ++j) {
                    const int2 q = hPack[hoff[i] + j];
                    fm.u.push_back(q.x);
                    fm.v.push_back(q.y);
                    fm.d.push_back(hPackD[hoff[i] + j]);
                }
                int t = 0;
                if (status_[f] == PS_OK) {
                    DelaunayWorkspace& w = (*ws_)[worker];
                    // triangles (in the rotation the raster must fit) and pin
                    // bits straight into the group's pinned staging slot
                    int* slot = static_cast<int*>(g2.hTri.p) + size_t(i) * tri_cap * 3;
                    uint8_t* pins = static_cast<uint8_t*>(g2.hPin.p) + size_t(i) * tri_cap;
                    const double ts0 = now_ms();
                    if (device_dt && host_first && g2.it == 1) {
                        // the seeds (<= 120 x perBinCap points): the reference sweep
                        // itself, exact order and pins, cheaper than a device mesh
                        g2.fixes[i].clear();
                        g2.replayed[i] = 1;
                        t = replay_mesh(fm, W, H, slot, tri_cap, pins, w, mstats[worker]);
                        ++mstats[worker].first_iter;
                    } else if (device_dt) {
                        // the device meshed the frame; resolve what it listed
                        const int* fl = static_cast<const int*>(g2.hFlags.p) + size_t(i) * flay.ints;
                        t = static_cast<const int*>(g2.hTriCount.p)[i];
                        bool rep = fl[0] != 0 || t > tri_cap;
                        if (rep) {
                            ++mstats[worker].fb_device;
                            const int why = t > tri_cap ? 16 : fl[6];
                            for (int b = 0; b < 5; ++b) mstats[worker].fb_why[b] += (why >> b) & 1;
                        }
                        g2.fixes[i].clear();
                        g2.replayed[i] = 0;
                        if (!rep && (fl[1] > 0 || fl[3] > 0)) {
                            // order queries of the frame on idle workers too
                            const ParallelQueries par = [&, worker](int nq, const std::function<void(int, SweepOrder::Scratch&)>& fn) {
                                auto& scr = shared_order_scratch();
                                pool_->help_run(worker, nq, [&](int q, int w) { fn(q, scr[w]); });
                            };
                            rep = !resolve_device_flags(fm, fl, flay, i, W, H, float(cfg.max_disparity),
                                                        g2.fixes[i], w, mstats[worker], &par, budget_scale);
                        }
                        if (rep) {
                            g2.fixes[i].clear();
                            g2.replayed[i] = 1;
                            t = replay_mesh(fm, W, H, slot, tri_cap, pins, w, mstats[worker]);
                        }
                    } else {
                        t = mesh_iteration(fm, W, H, float(cfg.max_disparity), slot, tri_cap, pins, w,
                                           mstats[worker]);
                    }
                    add_ms(sweep_ms_sum, now_ms() - ts0);
                    if (t < 0) {
                        status_[f] = PS_ERROR;
                        t = 0;
                    }
                }
                g2.ntri[i] = t;
                const double t1 = now_ms();
                add_ms(dt_ms_sum, t1 - t0);
                for (double cur = first_task.load(); t0 < cur && !first_task.compare_exchange_weak(cur, t0);) {}
                for (double cur = last_task.load(); t1 > cur && !last_task.compare_exchange_weak(cur, t1);) {}
                worker_end[worker] = t1;
                // decrement and notify under the engine's lock: once the
                // counter reads 0 the run may return, and this task touches
                // nothing of it after the (engine-owned) mutex is released
                std::lock_guard<std::mutex> lk(done_m_);
                if (g2.pending.fetch_sub(1) == 1) done_cv_.notify_all();
            });
        }
    };

    // (3) triangles H2D + device stages of iteration grp.it on the group's stream
    auto launch_device = [&](FrameGroup& grp) -> ps_status {
        const int it = grp.it;
        if (debug_timeline_)
            std::fprintf(stderr, "[tl] group %d iteration %d host done at %.3f ms\n", int(&grp - groups_), it,
                         now_ms() - run_t0);
        const bool last = it == iters;
        const int cell = cell_of[it - 1];
        const int cols = ceil_div(W, cell);
        const int cells = cols * ceil_div(H, cell);
        const int f0 = grp.f0, n = grp.n;
        cudaStream_t gs = grp.st;
        int* hs = static_cast<int*>(grp.hS.p);
        int* hsp = static_cast<int*>(grp.hSprev.p);
        int* hTriOff = static_cast<int*>(grp.hTriOff.p);
        long long total_tri = 0;
        for (int i = 0; i < n; ++i) {
            hTriOff[i] = int(total_tri);
            total_tri += grp.ntri[i];
        }
        hTriOff[n] = int(total_tri);
        // frame i's triangles at i * pitch: one pitched copy per group from
        // the host mesh, or the device mesh in place (+ host fixes / replays)
        int max_nt = 1;
        for (int i = 0; i < n; ++i) max_nt = std::max(max_nt, grp.ntri[i]);
        const size_t pitch = device_dt ? size_t(tri_cap) : size_t(max_nt);
        int* dTri = dev<int>(grp.dTri, size_t(n) * pitch * 3);
        uint8_t* dPin = dev<uint8_t>(grp.dPin, size_t(n) * pitch);
        int* dTriOff = static_cast<int*>(grp.dTriOff.p);
        if (!dTri || !dPin) return fail(PS_CUDA_ERROR, "allocation failed (triangles)");
        ps_status r = PS_OK;
        begin_kernel("h2d_triangles", 13.0 * double(pitch) * n, gs);
        if (device_dt) {
            int n_fix = 0;
            for (int i = 0; i < n; ++i) n_fix += int(grp.fixes[i].size() / 6);
            int* hfix = host<int>(grp.hFix, size_t(std::max(n_fix, 1)) * 6);
            int* dfix = dev<int>(grp.dFix, size_t(std::max(n_fix, 1)) * 6);
            if (!hfix || !dfix) return fail(PS_CUDA_ERROR, "allocation failed (mesh fixes)");
            size_t at = 0;
            for (int i = 0; i < n; ++i) {
                std::copy(grp.fixes[i].begin(), grp.fixes[i].end(), hfix + at);
                at += grp.fixes[i].size();
            }
            if (n_fix > 0)
                r = check(cudaMemcpyAsync(dfix, hfix, sizeof(int) * 6 * n_fix, cudaMemcpyHostToDevice, gs),
                          "H2D mesh fixes");
            if (!(host_first && it == 1)) {
                const StarArgs a = star_args(grp);
                launches_ += launch_star_finish(a, dfix, n_fix, tri_cap, gs);
            }
            // frames the host replayed: their triangles and pins replace the device's
            // (the first iteration on the host: every frame, one pitched copy each)
            if (host_first && it == 1 && r == PS_OK && max_nt > 0) {
                r = check(cudaMemcpy2DAsync(dTri, pitch * 12, grp.hTri.p, size_t(tri_cap) * 12, size_t(max_nt) * 12, n,
                                            cudaMemcpyHostToDevice, gs), "H2D first-iteration triangles");
                if (r == PS_OK)
                    r = check(cudaMemcpy2DAsync(dPin, pitch, grp.hPin.p, size_t(tri_cap), size_t(max_nt), n,
                                                cudaMemcpyHostToDevice, gs), "H2D first-iteration pins");
            }
            for (int i = 0; i < n && r == PS_OK && !(host_first && it == 1); ++i) {
                if (!grp.replayed[i] || grp.ntri[i] <= 0) continue;
                r = check(cudaMemcpyAsync(dTri + size_t(i) * pitch * 3,
                                          static_cast<int*>(grp.hTri.p) + size_t(i) * tri_cap * 3,
                                          size_t(grp.ntri[i]) * 12, cudaMemcpyHostToDevice, gs), "H2D replay");
                if (r == PS_OK)
                    r = check(cudaMemcpyAsync(dPin + size_t(i) * pitch,
                                              static_cast<uint8_t*>(grp.hPin.p) + size_t(i) * tri_cap,
                                              size_t(grp.ntri[i]), cudaMemcpyHostToDevice, gs), "H2D replay pins");
            }
        } else if (total_tri > 0) {
            r = check(cudaMemcpy2DAsync(dTri, pitch * 12, grp.hTri.p, size_t(tri_cap) * 12, pitch * 12, n,
                                        cudaMemcpyHostToDevice, gs), "H2D triangles");
            if (r == PS_OK)
                r = check(cudaMemcpy2DAsync(dPin, pitch, grp.hPin.p, size_t(tri_cap), pitch, n,
                                            cudaMemcpyHostToDevice, gs), "H2D pins");
        }
        end_kernel(gs);
        if (r == PS_OK)
            r = check(cudaMemcpyAsync(dTriOff, hTriOff, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, gs),
                      "H2D triangle offsets");
        if (r != PS_OK) return r;
        for (int i = 0; i < n; ++i) {
            ps_iter_stats& ts = trace_[size_t(f0 + i) * iters + (it - 1)];
            ts.iteration = it;
            ts.support_count = hs[i];  // mesh.vertices().size() (pipeline.cpp:180)
            ts.triangle_count = grp.ntri[i];
            ts.occupancy_cell_size = cell;
            hsp[i] = hs[i];
            final_count_[f0 + i] = hs[i];
        }

        if (serial_device_ && chained) cudaStreamWaitEvent(gs, chain_event_, 0);

        // ---- K5/K6 mesh (mesh.cpp:44-123) -> interpolated disparity (mesh.cpp:149-182)
        float* lk = dDit + size_t(f0) * P;
        cudaMemsetAsync(lk, 0xff, sizeof(float) * n * P, gs);  // NaN: outside the hull
        begin_kernel(it == 1 ? "mesh_it1" : it == 2 ? "mesh_it2" : "mesh_it3", 4.0 * double(P) * n + 36.0 * double(total_tri), gs);
        launches_ += launch_mesh_disparity(dTri, dTriOff, n, total_tri, dSu + size_t(f0) * scap_,
                                           dSv + size_t(f0) * scap_, dSd + size_t(f0) * scap_,
                                           scap_, g, dPin, float(cfg.max_disparity), lk, dErr, gs,
                                           (long long)pitch);
        end_kernel(gs);

        // ---- K7 (+K9) refine (mesh.cpp:149-182, pipeline.cpp:33-86)
        unsigned long long* cg = dCg + size_t(f0) * cells_max;
        unsigned long long* cb = dCb + size_t(f0) * cells_max;
        if (!last) {  // the last iteration's grids are never read (no resampling)
            cudaMemset2DAsync(cg, sizeof(unsigned long long) * cells_max, 0xff,
                              sizeof(unsigned long long) * cells, n, gs);
            cudaMemset2DAsync(cb, sizeof(unsigned long long) * cells_max, 0xff,
                              sizeof(unsigned long long) * cells, n, gs);
        }
        const size_t fp = size_t(f0) * P;
        RefineArgs ra{};
        ra.g = g;
        ra.frames = n;
        ra.mask = dMask + fp;
        ra.dit = lk;
        ra.cl = dCL + fp;
        ra.cr = dCR + fp;
        ra.max_disp = float(cfg.max_disparity);
        ra.cell = cell;
        ra.cols = cols;
        ra.cells_per_frame = cells;
        ra.cell_stride = cells_max;
        ra.Df = dDf + fp;
        ra.Dv = dDv + fp;
        ra.Cf = dCf + fp;
        ra.code = dCode + fp;
        ra.Cg = cg;
        ra.Cb = cb;
        ra.trace_sum = dTraceSum + size_t(f0) * iters + (it - 1);
        ra.trace_valid = dTraceValid + size_t(f0) * iters + (it - 1);
        ra.trace_stride = iters;
        ra.dense = dDense + fp;
        ra.dense_valid = dDenseV + fp;
        double mbytes = 0.0;
        for (int i = 0; i < n; ++i) mbytes += double(hMaskCount[f0 + i]);
        const double kbytes =
            double(P) * n + 29.0 * mbytes + (last ? 9.0 * double(P) * n - 4.0 * mbytes : 0.0);
        begin_kernel("refine", kbytes, gs);
        launches_ += launch_refine(ra, tab, last, gs);
        end_kernel(gs);

        if (!last) {
            // ---- K8 resampling (pipeline.cpp:88-129)
            int* su = dSu + size_t(f0) * scap_;
            int* sv = dSv + size_t(f0) * scap_;
            double* sd = dSd + size_t(f0) * scap_;
            uint32_t* tk = dTaken + size_t(f0) * words;
            int* chunk = static_cast<int*>(grp.dChunk.p);
            begin_kernel("resample", 0.0, gs);
            launches_ += launch_resample_confident(cg, cells, cells_max, g, n, lk, tk, su, sv, sd,
                                                   scap_, grp.S, dConf + f0, chunk, gs);
            launches_ += launch_resample_invalid(cb, cells, cells_max, g, n,
                                                 dRemU + size_t(f0) * cells_max,
                                                 dRemV + size_t(f0) * cells_max, cells_max,
                                                 dRemCount + f0, chunk, gs);
            end_kernel(gs);
            uint8_t* ok = dOk + size_t(f0) * cells_max;
            int* disp = dDisp + size_t(f0) * cells_max;
            begin_kernel("match_resample", 0.0, gs);
            launches_ += launch_match(dCL + fp, dCR + fp, g, n, cfg.max_disparity, tab,
                                      dRemU + size_t(f0) * cells_max, dRemV + size_t(f0) * cells_max,
                                      dRemCount + f0, cells_max, cells, ok, disp, nullptr, gs);
            end_kernel(gs);
            begin_kernel("compact", 0.0, gs);
            launches_ += launch_emit_matches(dRemU + size_t(f0) * cells_max,
                                             dRemV + size_t(f0) * cells_max, dRemCount + f0,
                                             cells_max, cells, ok, disp, g, n, tk, su, sv, sd,
                                             scap_, grp.S, dConf + f0, grp.Snext, chunk, gs);
            end_kernel(gs);
            std::swap(grp.S, grp.Snext);
            if (serial_device_) {  // the next group's pixel stages may start; the mesh runs beside them
                cudaEventRecord(chain_event_, gs);
                chained = true;
            }
            if (device_dt) {  // the next iteration's mesh, as soon as its supports exist
                int max_s = 0;
                double mean_s = 0.0;
                for (int i = 0; i < n; ++i) {
                    max_s = std::max(max_s, hs[i]);
                    mean_s += hs[i];
                }
                // resampling adds at most 2 supports per cell (~1.5 measured)
                enqueue_mesh(grp, mean_s / std::max(1, n) + 1.1 * cells, max_s + 2 * cells);
            }
        }
        if (serial_device_ && last) {
            cudaEventRecord(chain_event_, gs);
            chained = true;
        }
        if (last && sink_.active) {
            // streamed download of this group's final outputs (download())
            const size_t b = size_t(f0) * P, cnt = size_t(n) * P;
            if (sink_.disparity)
                cudaMemcpyAsync(sink_.disparity + b, dDf + b, cnt * 4, cudaMemcpyDeviceToHost, gs);
            if (wire_codes) {  // one code byte per pixel; expanded on the host when the group is done
                cudaMemcpyAsync(hCodes + b, dCode + b, cnt, cudaMemcpyDeviceToHost, gs);
            } else {
                if (sink_.disparity_valid)
                    cudaMemcpyAsync(sink_.disparity_valid + b, dDv + b, cnt, cudaMemcpyDeviceToHost, gs);
                if (sink_.cost)
                    cudaMemcpyAsync(sink_.cost + b, dCf + b, cnt * 4, cudaMemcpyDeviceToHost, gs);
            }
            if (sink_.dense)
                cudaMemcpyAsync(sink_.dense + b, dDense + b, cnt * 4, cudaMemcpyDeviceToHost, gs);
            if (sink_.dense_valid)
                cudaMemcpyAsync(sink_.dense_valid + b, dDenseV + b, cnt, cudaMemcpyDeviceToHost, gs);
        }
        cudaEventRecord(grp.done_event, gs);
        if (debug_timeline_)
            std::fprintf(stderr, "[tl] group %d iteration %d launched at %.3f ms\n", int(&grp - groups_), it,
                         now_ms() - run_t0);
        grp.phase = FrameGroup::kDevice;
        return PS_OK;
    };

    // ---- the dataflow loop
    int done_groups = 0;
    while (done_groups < G) {
        bool progress = false;
        if (next_seed < G) {
            s = seed_group(next_seed++);
            if (s != PS_OK) {
                drain();
                return s;
            }
            progress = true;
        }
        for (int gi = 0; gi < G; ++gi) {
            FrameGroup& grp = groups_[gi];
            if (grp.phase == FrameGroup::kHost && grp.pending.load() == 0) {
                s = launch_device(grp);
                if (s != PS_OK) {
                    drain();
                    return s;
                }
                progress = true;
            } else if (grp.phase == FrameGroup::kDevice || grp.phase == FrameGroup::kSeed) {
                const cudaError_t q = cudaEventQuery(grp.done_event);
                if (q == cudaErrorNotReady) continue;
                if (q != cudaSuccess) {
                    drain();
                    return check(q, "device stages");
                }
                if (grp.phase == FrameGroup::kSeed) {  // seeds are in: first Delaunay
                    if (debug_timeline_)
                        std::fprintf(stderr, "[tl] group %d seeds in at %.3f ms\n", gi, now_ms() - run_t0);
                    int* hs = static_cast<int*>(grp.hS.p);
                    int* hsp = static_cast<int*>(grp.hSprev.p);
                    for (int i = 0; i < grp.n; ++i) {
                        hs[i] = hS[grp.f0 + i];
                        hsp[i] = 0;
                        if (hs[i] < 3) status_[grp.f0 + i] = PS_SEEDING_FAILED;  // pipeline.cpp:151-154
                    }
                    s = fetch_delta(grp, false);
                    if (s != PS_OK) {
                        drain();
                        return s;
                    }
                    grp.it = 1;
                    if (debug_timeline_)
                        std::fprintf(stderr, "[tl] group %d first tasks at %.3f ms\n", gi, now_ms() - run_t0);
                    submit_dt(grp);
                    progress = true;
                    continue;
                }
                const double ms = now_ms() - grp.tic;
                for (int i = 0; i < grp.n; ++i) trace_[size_t(grp.f0 + i) * iters + (grp.it - 1)].millis = ms;
                if (observer && F == 1) {
                    std::vector<float> fd(P), fc(P);
                    std::vector<uint8_t> fv(P), code(P);
                    s = check(cudaMemcpy(fd.data(), dDf, sizeof(float) * P, cudaMemcpyDeviceToHost), "D2H");
                    if (s == PS_OK) s = check(cudaMemcpy(code.data(), dCode, P, cudaMemcpyDeviceToHost), "D2H");
                    if (s != PS_OK) return s;
                    for (long long i = 0; i < P; ++i) {  // C_f / validity from the byte codes
                        const bool fin = code[i] < tab.code_high;
                        fv[i] = fin ? 1 : 0;
                        fc[i] = fin ? tab.cost[code[i]] : tab.cost_high;
                    }
                    observer(grp.it, fd.data(), fv.data(), fc.data(), W, H, user);
                }
                if (debug_timeline_)
                    std::fprintf(stderr, "[tl] group %d iteration %d device done at %.3f ms\n", gi, grp.it,
                                 now_ms() - run_t0);
                if (grp.it == iters) {
                    grp.phase = FrameGroup::kDone;
                    ++done_groups;
                    if (wire_codes) expand(grp.f0, grp.n);  // its codes are in hCodes
                } else {
                    s = fetch_delta(grp, true);
                    if (s != PS_OK) {
                        drain();
                        return s;
                    }
                    grp.it += 1;
                    submit_dt(grp);
                }
                progress = true;
            }
        }
        if (!progress) {
            // wait for a Delaunay completion, or poll the device again shortly
            std::unique_lock<std::mutex> lk(done_m_);
            done_cv_.wait_for(lk, std::chrono::microseconds(200));
        }
    }
    {  // the host expansion of the streamed codes
        std::unique_lock<std::mutex> lk(done_m_);
        done_cv_.wait(lk, [&] { return expand_pending_.load() == 0; });
    }
    host_dt_ms = dt_ms_sum.load() / std::max(1, pool_->size());
    if (debug_timeline_) {
        std::sort(worker_end.begin(), worker_end.end());
        std::fprintf(stderr, "[tl] last task end at %.3f ms, loop end at %.3f ms; workers' last task ends (ms before the last):",
                     last_task.load() - run_t0, now_ms() - run_t0);
        for (double e : worker_end) std::fprintf(stderr, " %.2f", worker_end.back() - e);
        std::fprintf(stderr, "\n");
    }

    // ---- trace (pipeline.cpp:183-191)
    for (int gi = 0; gi < G; ++gi) {
        s = sync(groups_[gi].st, "pipeline");
        if (s != PS_OK) return s;
    }
    int herr = 0;
    s = check(cudaMemcpyAsync(hTraceSum, dTraceSum, sizeof(unsigned long long) * F * iters,
                              cudaMemcpyDeviceToHost, st_), "D2H trace");
    if (s == PS_OK)
        s = check(cudaMemcpyAsync(hTraceValid, dTraceValid, sizeof(unsigned) * F * iters,
                                  cudaMemcpyDeviceToHost, st_), "D2H trace");
    if (s == PS_OK) s = check(cudaMemcpyAsync(&herr, dErr, sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H err");
    if (s == PS_OK) s = sync("pipeline");
    if (s != PS_OK) return s;
    if (debug_timeline_)
        std::fprintf(stderr, "[tl] trace in at %.3f ms; main thread cpu %.3f ms\n", now_ms() - run_t0,
                     thread_cpu_ms() - cpu_t0);
    resolve_timers();
    if (debug_timeline_) std::fprintf(stderr, "[tl] timers resolved at %.3f ms\n", now_ms() - run_t0);
    if (profiling_) {
        auto stat = [&](const char* name) -> KernelStat& {
            for (auto& k : stats_)
                if (k.name == name) return k;
            stats_.push_back({name, 0, 0.0, 0.0});
            return stats_.back();
        };
        KernelStat& dt = stat("host_delaunay");  // ms = per-worker share of the work
        dt.launches += F * iters;
        dt.ms += host_dt_ms;
        const double workers = double(std::max(1, pool_->size()));
        KernelStat& sw = stat("host_mesh");  // of which: mesh_iteration (per-worker share)
        sw.launches += F * iters;
        sw.ms += sweep_ms_sum.load() / workers;
        MeshStats tot;
        for (const MeshStats& m : mstats) {
            tot.frames += m.frames;
            tot.fallbacks += m.fallbacks;
            tot.first_iter += m.first_iter;
            tot.fb_device += m.fb_device;
            for (int b = 0; b < 5; ++b) tot.fb_why[b] += m.fb_why[b];
            tot.fb_queries += m.fb_queries;
            tot.fb_resolve += m.fb_resolve;
            tot.replay_ms += m.replay_ms;
            tot.ambiguous += m.ambiguous;
            tot.rotations += m.rotations;
            tot.rot_checked += m.rot_checked;
            tot.dt_ms += m.dt_ms;
            tot.check_ms += m.check_ms;
            tot.order_ms += m.order_ms;
            tot.rot_ms += m.rot_ms;
            tot.pin_ms += m.pin_ms;
            tot.init_ms += m.init_ms;
        }
        // launches = events: replays of the reference sweep, pins ordered by
        // SweepOrder, rotations it decided, triangles fitted three ways
        KernelStat& k1 = stat("host_dt");  // incremental Delaunay
        k1.launches += int(tot.frames);
        k1.ms += tot.dt_ms / workers;
        KernelStat& k2 = stat("host_check");  // rotation + pin checks (incl. order)
        k2.launches += int(tot.rot_checked);
        k2.ms += tot.check_ms / workers;
        KernelStat& k3 = stat("host_order");  // SweepOrder queries
        k3.launches += int(tot.ambiguous + tot.rotations);
        k3.ms += tot.order_ms / workers;
        KernelStat& k5 = stat("host_order_rot");  // of which: rotations decided
        k5.launches += int(tot.rotations);
        k5.ms += tot.rot_ms / workers;
        KernelStat& k6 = stat("host_order_pin");  // of which: pins ordered
        k6.launches += int(tot.ambiguous);
        k6.ms += tot.pin_ms / workers;
        KernelStat& k7 = stat("host_order_init");  // of which: SweepOrder::init (lex order, chains, buckets)
        k7.ms += tot.init_ms / workers;
        KernelStat& k4 = stat("host_replay");  // frame-iterations replayed (delaunay_lex)
        k4.launches += int(tot.fallbacks - tot.first_iter);  // first-iteration host meshes are not fallbacks
        k4.ms += tot.replay_ms / workers;
        // of which, by cause
        stat("host_replay_device").launches += int(tot.fb_device);    // star overflow / capacity
        stat("host_replay_dev_fan").launches += int(tot.fb_why[0]);
        stat("host_replay_dev_search").launches += int(tot.fb_why[1]);
        stat("host_replay_dev_degree").launches += int(tot.fb_why[2]);
        stat("host_replay_dev_suspects").launches += int(tot.fb_why[3]);
        stat("host_replay_dev_capacity").launches += int(tot.fb_why[4]);
        stat("host_replay_queries").launches += int(tot.fb_queries);  // order-query budget
        stat("host_replay_resolve").launches += int(tot.fb_resolve);  // window not certified
        // pool occupancy: before the first task, gaps between tasks, after the last
        const double fa = first_task.load(), la = last_task.load(), end = now_ms();
        if (la > 0.0) {
            KernelStat& fill = stat("host_fill");
            fill.launches += 1;
            fill.ms += fa - run_t0;
            KernelStat& gap = stat("host_gaps");  // per worker, between first and last task
            gap.launches += 1;
            gap.ms += (la - fa) - dt_ms_sum.load() / workers;
            KernelStat& drain = stat("host_drain");
            drain.launches += 1;
            drain.ms += end - la;
        }
    }
    if (herr) return fail(PS_DEGENERATE_TRIANGLE, "collinear vertices in a triangle");
    for (int f = 0; f < F; ++f) {
        for (int it = 0; it < iters; ++it) {
            ps_iter_stats& ts = trace_[size_t(f) * iters + it];
            const int M = hMaskCount[f];
            // The fixed-point sum is exact (see trace_fixed_exact); the double
            // conversion rounds once, exactly like the reference's exact
            // running double sum.
            const double sum = std::ldexp(double(hTraceSum[size_t(f) * iters + it]), -36);
            ts.mean_cost = M > 0 ? sum / M : 0.0;
            ts.valid_count = int(hTraceValid[size_t(f) * iters + it]);
        }
    }
    if (!fixed_trace) {
        // costHigh with a mantissa too long for the 2^-36 grid: recompute the
        // last iteration's mean from the final costs (earlier ones stay approximate).
        std::vector<float> fc(P);
        std::vector<uint8_t> mk(P);
        for (int f = 0; f < F; ++f) {
            cudaMemcpy(fc.data(), dCf + size_t(f) * P, sizeof(float) * P, cudaMemcpyDeviceToHost);
            cudaMemcpy(mk.data(), dMask + size_t(f) * P, P, cudaMemcpyDeviceToHost);
            double sum = 0.0;
            for (long long i = 0; i < P; ++i)
                if (mk[i]) sum += fc[i];
            const int M = hMaskCount[f];
            trace_[size_t(f) * iters + iters - 1].mean_cost = M > 0 ? sum / M : 0.0;
        }
    }
    have_outputs_ = true;
    streamed_ = sink_.active;
    done_sink_ = sink_;
    for (int f = 0; f < F; ++f) {
        if (status_[f] == PS_SEEDING_FAILED)
            return fail(PS_SEEDING_FAILED, "only " + std::to_string(hS[f]) +
                                               " seed matches survived; need at least 3");
        if (status_[f] != PS_OK)
            return fail(ps_status(status_[f]), "frame " + std::to_string(f) +
                                                   ": triangulation failed (coordinates or capacity)");
    }
    return PS_OK;
}

ps_status Engine::download(float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                           uint8_t* dense_valid, ps_iter_stats* trace, int* frame_status) {
    if (!have_outputs_) return fail(PS_ERROR, "no completed run to download");
    cudaSetDevice(device_);
    const size_t n = size_t(F_) * P_;
    ps_status s = PS_OK;
    if (streamed_) {
        // run_resident() already copied into the sink buffers; a different
        // destination gets its own copy
        if (disparity == done_sink_.disparity) disparity = nullptr;
        if (disparity_valid == done_sink_.disparity_valid) disparity_valid = nullptr;
        if (cost == done_sink_.cost) cost = nullptr;
        if (dense == done_sink_.dense) dense = nullptr;
        if (dense_valid == done_sink_.dense_valid) dense_valid = nullptr;
    }
    if (disparity && s == PS_OK)
        s = check(cudaMemcpyAsync(disparity, dDf_.p, n * 4, cudaMemcpyDeviceToHost, st_), "D2H disparity");
    if (disparity_valid && s == PS_OK)
        s = check(cudaMemcpyAsync(disparity_valid, dDv_.p, n, cudaMemcpyDeviceToHost, st_), "D2H validity");
    if (cost && s == PS_OK)
        s = check(cudaMemcpyAsync(cost, dCf_.p, n * 4, cudaMemcpyDeviceToHost, st_), "D2H cost");
    if (dense && s == PS_OK)
        s = check(cudaMemcpyAsync(dense, dDense_.p, n * 4, cudaMemcpyDeviceToHost, st_), "D2H dense");
    if (dense_valid && s == PS_OK)
        s = check(cudaMemcpyAsync(dense_valid, dDenseV_.p, n, cudaMemcpyDeviceToHost, st_), "D2H dense validity");
    if (s == PS_OK) s = sync("download");
    if (s != PS_OK) return s;
    if (streamed_) {
        if (!disparity) disparity = done_sink_.disparity;
        if (!disparity_valid) disparity_valid = done_sink_.disparity_valid;
        if (!cost) cost = done_sink_.cost;
        if (!dense) dense = done_sink_.dense;
        if (!dense_valid) dense_valid = done_sink_.dense_valid;
    }
    for (int f = 0; f < F_; ++f) {
        if (frame_status) frame_status[f] = status_[f];
        if (status_[f] == PS_OK) continue;
        // A frame whose seeding failed has no result (run() throws SeedingFailed).
        const size_t b = size_t(f) * P_;
        if (disparity) std::fill(disparity + b, disparity + b + P_, 0.0f);
        if (disparity_valid) std::fill(disparity_valid + b, disparity_valid + b + P_, uint8_t(0));
        if (cost) std::fill(cost + b, cost + b + P_, cost_high_);
        if (dense) std::fill(dense + b, dense + b + P_, 0.0f);
        if (dense_valid) std::fill(dense_valid + b, dense_valid + b + P_, uint8_t(0));
    }
    if (trace) std::copy(trace_.begin(), trace_.end(), trace);
    return PS_OK;
}

namespace {
bool page_locked(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
}  // namespace

void Engine::set_sink(float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                      uint8_t* dense_valid) {
    sink_ = Sink{disparity, disparity_valid, cost, dense, dense_valid, false};
    sink_.active = (disparity || disparity_valid || cost || dense || dense_valid) &&
                   page_locked(disparity) && page_locked(disparity_valid) && page_locked(cost) &&
                   page_locked(dense) && page_locked(dense_valid);
    if (!sink_.active) sink_ = Sink{};
}

ps_status Engine::resident_maps(ResidentMaps& m) {
    if (!have_outputs_) return fail(PS_ERROR, "no completed run to encode");
    cudaSetDevice(device_);
    int* ok = dev<int>(dFrameOk_, F_);
    if (!ok) return fail(PS_CUDA_ERROR, "allocation failed");
    std::vector<int> h(F_);
    for (int f = 0; f < F_; ++f) h[f] = status_[f] == PS_OK ? 1 : 0;
    ps_status s = check(cudaMemcpy(ok, h.data(), sizeof(int) * F_, cudaMemcpyHostToDevice), "H2D frame status");
    if (s != PS_OK) return s;
    m = ResidentMaps{static_cast<const float*>(dDf_.p), static_cast<const uint8_t*>(dDv_.p),
                     static_cast<const float*>(dDense_.p), static_cast<const uint8_t*>(dDenseV_.p),
                     static_cast<const uint8_t*>(dL_.p), static_cast<const uint8_t*>(dMask_.p), ok,
                     F_, W_, H_, P_};
    return PS_OK;
}

ps_status Engine::supports(int frame, int* u, int* v, double* d, int capacity, int* count) {
    if (!have_outputs_ || frame < 0 || frame >= F_) return fail(PS_ERROR, "no such frame");
    // The last iteration's list (its length is the last trace support_count).
    const int n = final_count_[frame];
    if (count) *count = n;
    if (n > capacity) return fail(PS_CAPACITY, "support buffer too small");
    const size_t b = size_t(frame) * scap_;
    ps_status s = PS_OK;
    if (u) s = check(cudaMemcpy(u, static_cast<int*>(dSu_.p) + b, sizeof(int) * n, cudaMemcpyDeviceToHost), "D2H");
    if (v && s == PS_OK) s = check(cudaMemcpy(v, static_cast<int*>(dSv_.p) + b, sizeof(int) * n, cudaMemcpyDeviceToHost), "D2H");
    if (d && s == PS_OK) s = check(cudaMemcpy(d, static_cast<double*>(dSd_.p) + b, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
    return s;
}

}  // namespace ps
