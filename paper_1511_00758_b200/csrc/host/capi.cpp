// capi.cpp — the extern "C" boundary declared in include/planestereo_c.h.
//
// Pipeline entry points run the batched Engine; stage entry points run the
// same sm_100a kernels on one frame.  Nothing here computes a per-pixel or
// per-candidate result on the host: the only host computation is the
// Delaunay triangulation (by design, delaunay.hpp), the reference's
// per-pixel dedup of a user-supplied candidate list (sparse.cpp:183-192) and
// argument checking.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../kernels/launch.hpp"
#include "engine.hpp"
#include "planestereo_c.h"

namespace ps {
ps_status validate_config(const ps_config& c, unsigned flags, std::string& msg);
CostTables make_tables(const ps_config& c);
}  // namespace ps

struct ps_ctx {
    ps::Engine* engine = nullptr;
};

namespace {

thread_local std::string g_last_error;

ps_status set_error(ps_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

ps_status from_engine(ps_ctx* ctx, ps_status s) {
    if (s != PS_OK) g_last_error = ctx->engine->error();
    return s;
}

bool device_ok(int device, std::string& why) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n <= device || device < 0) {
        why = std::string("no CUDA device ") + std::to_string(device) + " (" +
              (e == cudaSuccess ? "not present" : cudaGetErrorString(e)) + ")";
        return false;
    }
    cudaDeviceProp p{};
    cudaGetDeviceProperties(&p, device);
    if (p.major != 10) {
        why = std::string("device ") + p.name + " is not sm_100 (this build targets sm_100a only)";
        return false;
    }
    return true;
}

#define PS_REQUIRE_CTX(ctx)                                               \
    do {                                                                  \
        if (!(ctx) || !(ctx)->engine) return set_error(PS_ERROR, "null context"); \
    } while (0)

}  // namespace

extern "C" {

const char* ps_version(void) { return "planestereo-b200 0.1 (sm_100a)"; }

ps_status ps_ctx_create(int device, ps_ctx** out) {
    if (!out) return set_error(PS_ERROR, "null output pointer");
    *out = nullptr;
    std::string why;
    if (!device_ok(device, why)) return set_error(PS_NO_DEVICE, why);
    ps_ctx* c = new ps_ctx;
    c->engine = new ps::Engine(device);
    *out = c;
    return PS_OK;
}

void ps_ctx_destroy(ps_ctx* ctx) {
    if (!ctx) return;
    delete ctx->engine;
    delete ctx;
}

const char* ps_last_error(const ps_ctx*) { return g_last_error.c_str(); }

void ps_config_default(ps_config* c) {
    // PipelineConfig defaults, proj/include/planestereo/config.hpp:10-30.
    c->iterations = 1;
    c->max_disparity = 128;
    c->cost_low = 0.25f;
    c->cost_high = 0.5f;
    c->gradient_threshold = 20;
    c->occupancy_cell_size = 32;
    c->corner_threshold = 20;
    c->per_bin_cap = 5;
    c->sparse_accept_cost = 0.25f;
    c->uniqueness_ratio = 0.9f;
    c->threads = 1;
}

ps_status ps_config_validate(const ps_config* cfg, unsigned flags) {
    if (!cfg) return set_error(PS_ERROR, "null config");
    std::string msg;
    ps_status s = ps::validate_config(*cfg, flags, msg);
    if (s != PS_OK) g_last_error = msg;
    return s;
}

ps_status ps_upload_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                          int width, int height) {
    PS_REQUIRE_CTX(ctx);
    if (!left || !right) return set_error(PS_ERROR, "null image");
    return from_engine(ctx, ctx->engine->upload(n_frames, left, right, width, height));
}

ps_status ps_run_resident(ps_ctx* ctx, const ps_config* cfg, unsigned flags) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg) return set_error(PS_ERROR, "null config");
    return from_engine(ctx, ctx->engine->run_resident(*cfg, flags));
}

ps_status ps_download_batch(ps_ctx* ctx, float* disparity, uint8_t* disparity_valid, float* cost,
                            float* dense, uint8_t* dense_valid, ps_iter_stats* trace,
                            int* frame_status) {
    PS_REQUIRE_CTX(ctx);
    return from_engine(ctx, ctx->engine->download(disparity, disparity_valid, cost, dense,
                                                  dense_valid, trace, frame_status));
}

ps_status ps_run_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                       int width, int height, const ps_config* cfg, unsigned flags,
                       float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                       uint8_t* dense_valid, ps_iter_stats* trace, int* frame_status) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg) return set_error(PS_ERROR, "null config");
    // run() checks the config before anything else (pipeline.cpp:133)
    ps_status s = ps_config_validate(cfg, flags);
    if (s != PS_OK) return s;
    if (!left || !right) return set_error(PS_ERROR, "null image");
    // the images are copied inside the run, group by group, overlapping seeding
    s = from_engine(ctx, ctx->engine->upload(n_frames, left, right, width, height, true));
    if (s != PS_OK) return s;
    // page-locked destinations are filled group by group during the run
    ctx->engine->set_sink(disparity, disparity_valid, cost, dense, dense_valid);
    const ps_status run = ctx->engine->run_resident(*cfg, flags);
    ctx->engine->clear_sink();
    if (run != PS_OK && run != PS_SEEDING_FAILED) return from_engine(ctx, run);
    s = from_engine(ctx, ctx->engine->download(disparity, disparity_valid, cost, dense,
                                               dense_valid, trace, frame_status));
    if (s != PS_OK) return s;
    if (run != PS_OK) g_last_error = ctx->engine->error();
    return run;
}

ps_status ps_run_batch_multi(ps_ctx* const* ctxs, int n_ctx, int n_frames, const uint8_t* left,
                             const uint8_t* right, int width, int height, const ps_config* cfg,
                             unsigned flags, float* disparity, uint8_t* disparity_valid,
                             float* cost, float* dense, uint8_t* dense_valid,
                             ps_iter_stats* trace, int* frame_status) {
    if (!ctxs || n_ctx < 1) return set_error(PS_ERROR, "no contexts");
    for (int i = 0; i < n_ctx; ++i) {
        if (!ctxs[i]) return set_error(PS_ERROR, "null context");
        for (int j = 0; j < i; ++j)
            if (ctxs[j] == ctxs[i]) return set_error(PS_ERROR, "a context appears twice");
    }
    if (!cfg) return set_error(PS_ERROR, "null config");
    if (!left || !right) return set_error(PS_ERROR, "null image");
    ps_status s = ps_config_validate(cfg, flags);
    if (s != PS_OK) return s;
    if (n_frames < 1) return set_error(PS_ERROR, "batch needs at least one frame");
    const long long P = (long long)width * height;
    std::vector<ps_status> st(n_ctx, PS_OK);
    std::vector<std::string> msg(n_ctx);
    std::vector<std::thread> th;
    for (int i = 0; i < n_ctx; ++i) {
        // even contiguous split: block sizes differ by at most one frame
        const int f0 = int((long long)n_frames * i / n_ctx);
        const int n = int((long long)n_frames * (i + 1) / n_ctx) - f0;
        if (n <= 0) continue;
        th.emplace_back([&, i, f0, n] {
            const size_t px = size_t(f0) * size_t(P);
            st[i] = ps_run_batch(ctxs[i], n, left + px, right + px, width, height, cfg, flags,
                                 disparity ? disparity + px : nullptr,
                                 disparity_valid ? disparity_valid + px : nullptr,
                                 cost ? cost + px : nullptr, dense ? dense + px : nullptr,
                                 dense_valid ? dense_valid + px : nullptr,
                                 trace ? trace + size_t(f0) * cfg->iterations : nullptr,
                                 frame_status ? frame_status + f0 : nullptr);
            if (st[i] != PS_OK) msg[i] = g_last_error;  // this thread's message
        });
    }
    for (auto& t : th) t.join();
    // context-level errors first, then frame statuses (ps_run_batch's precedence)
    for (int i = 0; i < n_ctx; ++i)
        if (st[i] != PS_OK && st[i] != PS_SEEDING_FAILED) return set_error(st[i], msg[i]);
    for (int i = 0; i < n_ctx; ++i)
        if (st[i] != PS_OK) return set_error(st[i], msg[i]);
    return PS_OK;
}

ps_status ps_run(ps_ctx* ctx, const uint8_t* left, const uint8_t* right, int width, int height,
                 const ps_config* cfg, unsigned flags, float* disparity, uint8_t* disparity_valid,
                 float* cost, float* dense, uint8_t* dense_valid, ps_iter_stats* trace,
                 ps_observer_fn observer, void* user) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg) return set_error(PS_ERROR, "null config");
    ps_status s = ps_config_validate(cfg, flags);
    if (s != PS_OK) return s;
    s = ps_upload_batch(ctx, 1, left, right, width, height);
    if (s != PS_OK) return s;
    s = from_engine(ctx, ctx->engine->run_resident(*cfg, flags, observer, user));
    if (s != PS_OK) return s;
    return from_engine(ctx, ctx->engine->download(disparity, disparity_valid, cost, dense,
                                                  dense_valid, trace, nullptr));
}

ps_status ps_get_supports(ps_ctx* ctx, int frame, int* u, int* v, double* d, int capacity,
                          int* count) {
    PS_REQUIRE_CTX(ctx);
    return from_engine(ctx, ctx->engine->supports(frame, u, v, d, capacity, count));
}

ps_status ps_set_profiling(ps_ctx* ctx, int enabled) {
    PS_REQUIRE_CTX(ctx);
    ctx->engine->set_profiling(enabled != 0);
    return PS_OK;
}

ps_status ps_set_max_groups(ps_ctx* ctx, int groups) {
    PS_REQUIRE_CTX(ctx);
    ctx->engine->set_max_groups(groups);
    return PS_OK;
}

ps_status ps_get_host_threads(ps_ctx* ctx, int* threads) {
    PS_REQUIRE_CTX(ctx);
    if (!threads) return set_error(PS_ERROR, "null output");
    *threads = ctx->engine->pool().size();
    return PS_OK;
}

ps_status ps_reset_kernel_stats(ps_ctx* ctx) {
    PS_REQUIRE_CTX(ctx);
    ctx->engine->reset_stats();
    return PS_OK;
}

ps_status ps_get_kernel_stats(ps_ctx* ctx, ps_kernel_stat* out, int capacity, int* count) {
    PS_REQUIRE_CTX(ctx);
    const auto& st = ctx->engine->stats();
    if (count) *count = int(st.size());
    for (int i = 0; i < int(st.size()) && i < capacity; ++i) {
        std::memset(out[i].name, 0, sizeof(out[i].name));
        std::strncpy(out[i].name, st[i].name.c_str(), sizeof(out[i].name) - 1);
        out[i].launches = st[i].launches;
        out[i].total_ms = st[i].ms;
        out[i].algorithmic_bytes = st[i].bytes;
    }
    return PS_OK;
}

long long ps_launch_count(const ps_ctx* ctx) {
    return (ctx && ctx->engine) ? ctx->engine->launches() : 0;
}

void* ps_ctx_stream(const ps_ctx* ctx) {
    return (ctx && ctx->engine) ? static_cast<void*>(ctx->engine->stream()) : nullptr;
}

// ------------------------------------------------------------------ stages

ps_status ps_gradient_mask(ps_ctx* ctx, const uint8_t* image, int width, int height,
                           int threshold, uint8_t* member, int* count) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    uint8_t* d_img = e.dev<uint8_t>(e.s_a, P);
    uint8_t* d_mask = e.dev<uint8_t>(e.s_b, P);
    int* d_cnt = e.dev<int>(e.s_c, 1);
    if (!d_img || !d_mask || !d_cnt) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(d_img, image, P, cudaMemcpyHostToDevice, e.stream());
    cudaMemsetAsync(d_cnt, 0, sizeof(int), e.stream());
    e.count_launches(ps::launch_frontend(d_img, nullptr, {width, height, P}, 1, threshold, d_mask,
                                         nullptr, nullptr, d_cnt, e.stream()));
    if (member) cudaMemcpyAsync(member, d_mask, P, cudaMemcpyDeviceToHost, e.stream());
    int c = 0;
    cudaMemcpyAsync(&c, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, e.stream());
    ps_status s = from_engine(ctx, e.sync("gradient mask"));
    if (count) *count = c;
    return s;
}

ps_status ps_census(ps_ctx* ctx, const uint8_t* image, int width, int height, uint32_t* out) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    uint8_t* d_img = e.dev<uint8_t>(e.s_a, P);
    uint32_t* d_c = e.dev<uint32_t>(e.s_b, P);
    if (!d_img || !d_c) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(d_img, image, P, cudaMemcpyHostToDevice, e.stream());
    e.count_launches(ps::launch_frontend(d_img, nullptr, {width, height, P}, 1, 0, nullptr, d_c,
                                         nullptr, nullptr, e.stream()));
    cudaMemcpyAsync(out, d_c, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, e.stream());
    return from_engine(ctx, e.sync("census"));
}

ps_status ps_detect_candidates(ps_ctx* ctx, const uint8_t* image, int width, int height,
                               const ps_config* cfg, int* u, int* v, float* score, int capacity,
                               int* count) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg || cfg->per_bin_cap < 1) return set_error(PS_INVALID_CONFIG, "per-bin cap must be >= 1");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const ps::FrameGeom g{width, height, P};
    const int cap = cfg->per_bin_cap;
    const int stride = 120 * cap;
    int n_pow2 = 1;
    while (n_pow2 < std::min<long long>(stride, P)) n_pow2 <<= 1;
    const long long scs = ps::candidate_scratch_stride(g);
    uint8_t* d_img = e.dev<uint8_t>(e.s_a, P);
    unsigned long long* d_keys = e.dev<unsigned long long>(e.s_b, size_t(stride));
    int* d_bc = e.dev<int>(e.s_c, 120);
    unsigned long long* d_sc = e.dev<unsigned long long>(e.s_d, cap > 8 ? std::max<long long>(120 * scs, n_pow2) : 1);
    int* d_u = e.dev<int>(e.s_e, stride);
    int* d_v = e.dev<int>(e.s_f, stride);
    float* d_s = e.dev<float>(e.s_g, stride);
    int* d_n = e.dev<int>(e.s_h, 1);
    if (!d_img || !d_keys || !d_bc || !d_sc || !d_u || !d_v || !d_s || !d_n)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(d_img, image, P, cudaMemcpyHostToDevice, e.stream());
    e.count_launches(ps::launch_candidates(d_img, g, 1, cfg->corner_threshold, cap, d_keys, d_bc,
                                           d_sc, scs, d_u, d_v, d_s, d_n, stride, e.stream()));
    int n = 0;
    cudaMemcpyAsync(&n, d_n, sizeof(int), cudaMemcpyDeviceToHost, e.stream());
    ps_status s = from_engine(ctx, e.sync("candidates"));
    if (s != PS_OK) return s;
    if (count) *count = n;
    const int m = std::min(n, capacity);
    if (u) cudaMemcpy(u, d_u, sizeof(int) * m, cudaMemcpyDeviceToHost);
    if (v) cudaMemcpy(v, d_v, sizeof(int) * m, cudaMemcpyDeviceToHost);
    if (score) cudaMemcpy(score, d_s, sizeof(float) * m, cudaMemcpyDeviceToHost);
    if (n > capacity) return set_error(PS_CAPACITY, "candidate buffer too small");
    return from_engine(ctx, e.sync("candidates D2H"));
}

ps_status ps_match_epipolar(ps_ctx* ctx, const uint32_t* census_left, const uint32_t* census_right,
                            int width, int height, const int* cand_u, const int* cand_v,
                            int n_candidates, const ps_config* cfg, int* u, int* v, double* d,
                            int capacity, int* count) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg) return set_error(PS_ERROR, "null config");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const ps::FrameGeom g{width, height, P};
    const int n = std::max(0, n_candidates);
    uint32_t* d_cl = e.dev<uint32_t>(e.s_a, P);
    uint32_t* d_cr = e.dev<uint32_t>(e.s_b, P);
    int* d_u = e.dev<int>(e.s_c, std::max(1, n));
    int* d_v = e.dev<int>(e.s_d, std::max(1, n));
    int* d_n = e.dev<int>(e.s_e, 1);
    uint8_t* d_ok = e.dev<uint8_t>(e.s_f, std::max(1, n));
    int* d_disp = e.dev<int>(e.s_g, std::max(1, n));
    int* d_k = e.dev<int>(e.s_h, std::max(1, n));
    if (!d_cl || !d_cr || !d_u || !d_v || !d_n || !d_ok || !d_disp || !d_k)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(d_cl, census_left, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, e.stream());
    cudaMemcpyAsync(d_cr, census_right, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, e.stream());
    if (n > 0) {
        cudaMemcpyAsync(d_u, cand_u, sizeof(int) * n, cudaMemcpyHostToDevice, e.stream());
        cudaMemcpyAsync(d_v, cand_v, sizeof(int) * n, cudaMemcpyHostToDevice, e.stream());
    }
    cudaMemcpyAsync(d_n, &n, sizeof(int), cudaMemcpyHostToDevice, e.stream());
    const ps::CostTables tab = ps::make_tables(*cfg);
    e.count_launches(ps::launch_match(d_cl, d_cr, g, 1, cfg->max_disparity, tab, d_u, d_v, d_n, n,
                                      n, d_ok, d_disp, d_k, e.stream()));
    std::vector<uint8_t> ok(n);
    std::vector<int> disp(n), kk(n);
    if (n > 0) {
        cudaMemcpyAsync(ok.data(), d_ok, n, cudaMemcpyDeviceToHost, e.stream());
        cudaMemcpyAsync(disp.data(), d_disp, sizeof(int) * n, cudaMemcpyDeviceToHost, e.stream());
        cudaMemcpyAsync(kk.data(), d_k, sizeof(int) * n, cudaMemcpyDeviceToHost, e.stream());
    }
    ps_status s = from_engine(ctx, e.sync("match"));
    if (s != PS_OK) return s;
    // Per-pixel dedup in candidate order, lower cost wins (sparse.cpp:183-192).
    std::unordered_map<long long, int> by_pixel;
    std::vector<int> ou, ov, od, ok_k;
    for (int i = 0; i < n; ++i) {
        if (!ok[i]) continue;
        const long long key = (long long)cand_v[i] * width + cand_u[i];
        auto it = by_pixel.find(key);
        if (it == by_pixel.end()) {
            by_pixel.emplace(key, int(ou.size()));
            ou.push_back(cand_u[i]);
            ov.push_back(cand_v[i]);
            od.push_back(disp[i]);
            ok_k.push_back(kk[i]);
        } else if (kk[i] < ok_k[it->second]) {
            od[it->second] = disp[i];
            ok_k[it->second] = kk[i];
        }
    }
    const int m = int(ou.size());
    if (count) *count = m;
    for (int i = 0; i < m && i < capacity; ++i) {
        if (u) u[i] = ou[i];
        if (v) v[i] = ov[i];
        if (d) d[i] = double(od[i]);
    }
    if (m > capacity) return set_error(PS_CAPACITY, "support buffer too small");
    return PS_OK;
}

static ps_status delaunay_common(bool fast, const int* u, const int* v, int n, int* tris,
                                 int capacity, int* n_tris) {
    static thread_local ps::DelaunayWorkspace ws;
    std::vector<int> out;
    const int t = fast ? ps::delaunay(u, v, n, out, ws) : ps::delaunay_lex(u, v, n, out, ws);
    if (t == -1) return set_error(PS_ERROR, "triangulation coordinates must be below 2^20");
    if (t < 0) return set_error(PS_ERROR, "triangulation invariant violated: no hull edge visible");
    if (n_tris) *n_tris = t;
    if (t > capacity) return set_error(PS_CAPACITY, "triangle buffer too small");
    if (tris && t > 0) std::memcpy(tris, out.data(), sizeof(int) * 3 * t);
    return PS_OK;
}

ps_status ps_delaunay(const int* u, const int* v, int n, int* tris, int capacity, int* n_tris) {
    return delaunay_common(false, u, v, n, tris, capacity, n_tris);
}

ps_status ps_delaunay_fast(const int* u, const int* v, int n, int* tris, int capacity,
                           int* n_tris) {
    return delaunay_common(true, u, v, n, tris, capacity, n_tris);
}

ps_status ps_mesh_build(ps_ctx* ctx, const int* u, const int* v, const double* d, int n_points,
                        const int* tris, int n_tris, int width, int height, double* planes,
                        int32_t* lookup) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const ps::FrameGeom g{width, height, P};
    const int np = std::max(1, n_points), nt = std::max(0, n_tris);
    int* d_u = e.dev<int>(e.s_a, np);
    int* d_v = e.dev<int>(e.s_b, np);
    double* d_d = e.dev<double>(e.s_c, np);
    int* d_t = e.dev<int>(e.s_d, 3 * std::max(1, nt));
    int off[2] = {0, nt};
    int* d_off = e.dev<int>(e.s_e, 2);
    double* d_pl = e.dev<double>(e.s_f, 3 * std::max(1, nt));
    int32_t* d_lk = e.dev<int32_t>(e.s_g, P);
    int* d_err = e.dev<int>(e.s_h, 1);
    if (!d_u || !d_v || !d_d || !d_t || !d_off || !d_pl || !d_lk || !d_err)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    if (n_points > 0) {
        cudaMemcpyAsync(d_u, u, sizeof(int) * n_points, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_v, v, sizeof(int) * n_points, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_d, d, sizeof(double) * n_points, cudaMemcpyHostToDevice, st);
    }
    if (nt > 0) cudaMemcpyAsync(d_t, tris, sizeof(int) * 3 * nt, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_off, off, sizeof(off), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(d_lk, 0xff, sizeof(int32_t) * P, st);
    cudaMemsetAsync(d_err, 0, sizeof(int), st);
    // hull-vertex pins in the caller's triangle order (mesh.cpp:109-122)
    std::vector<uint8_t> state, pins;
    if (nt > 0) ps::mesh_pins(u, v, n_points, tris, nt, width, height, state, pins);
    uint8_t* d_pin = e.dev<uint8_t>(e.s_i, std::max(1, nt));
    if (!d_pin) return set_error(PS_CUDA_ERROR, "allocation failed");
    if (nt > 0) cudaMemcpyAsync(d_pin, pins.data(), nt, cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_mesh(d_t, d_off, 1, nt, d_u, d_v, d_d, np, g, d_pin, d_pl, d_lk,
                                     d_err, st));
    int err = 0;
    cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (planes && nt > 0) cudaMemcpyAsync(planes, d_pl, sizeof(double) * 3 * nt, cudaMemcpyDeviceToHost, st);
    if (lookup) cudaMemcpyAsync(lookup, d_lk, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st);
    ps_status s = from_engine(ctx, e.sync("mesh"));
    if (s != PS_OK) return s;
    if (err) return set_error(PS_DEGENERATE_TRIANGLE, "collinear vertices in a triangle");
    return PS_OK;
}

ps_status ps_interpolate(ps_ctx* ctx, const int32_t* lookup, const double* planes, int n_tris,
                         int width, int height, const uint8_t* mask, float max_disparity,
                         float* value, uint8_t* valid) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const int nt = std::max(1, n_tris);
    int32_t* d_lk = e.dev<int32_t>(e.s_a, P);
    double* d_pl = e.dev<double>(e.s_b, 3 * nt);
    uint8_t* d_m = mask ? e.dev<uint8_t>(e.s_c, P) : nullptr;
    float* d_val = e.dev<float>(e.s_d, P);
    uint8_t* d_ok = e.dev<uint8_t>(e.s_e, P);
    if (!d_lk || !d_pl || (mask && !d_m) || !d_val || !d_ok) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(d_lk, lookup, sizeof(int32_t) * P, cudaMemcpyHostToDevice, st);
    if (n_tris > 0) cudaMemcpyAsync(d_pl, planes, sizeof(double) * 3 * n_tris, cudaMemcpyHostToDevice, st);
    if (mask) cudaMemcpyAsync(d_m, mask, P, cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_interpolate(d_lk, d_pl, {width, height, P}, d_m, max_disparity, d_val, d_ok, st));
    cudaMemcpyAsync(value, d_val, sizeof(float) * P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(valid, d_ok, P, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("interpolate"));
}

ps_status ps_cost_evaluation(ps_ctx* ctx, const uint32_t* census_left, const uint32_t* census_right,
                             int width, int height, const float* interp, const uint8_t* interp_valid,
                             const uint8_t* mask, float* cost) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    uint32_t* d_cl = e.dev<uint32_t>(e.s_a, P);
    uint32_t* d_cr = e.dev<uint32_t>(e.s_b, P);
    float* d_val = e.dev<float>(e.s_c, P);
    uint8_t* d_ok = e.dev<uint8_t>(e.s_d, P);
    uint8_t* d_m = e.dev<uint8_t>(e.s_e, P);
    float* d_cost = e.dev<float>(e.s_f, P);
    if (!d_cl || !d_cr || !d_val || !d_ok || !d_m || !d_cost) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(d_cl, census_left, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_cr, census_right, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_val, interp, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_ok, interp_valid, P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_m, mask, P, cudaMemcpyHostToDevice, st);
    ps_config dc;
    ps_config_default(&dc);
    const ps::CostTables tab = ps::make_tables(dc);
    e.count_launches(ps::launch_cost_eval(d_cl, d_cr, {width, height, P}, d_val, d_ok, d_m, tab, d_cost, st));
    cudaMemcpyAsync(cost, d_cost, 4 * P, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("cost evaluation"));
}

namespace {
ps_status wta_common(ps_ctx* ctx, int frames, const uint8_t* left, const uint8_t* right, int width,
                     int height, const uint8_t* mask, int threshold, int max_disparity,
                     float* disparity, uint8_t* valid, float* cost) {
    if (frames < 1) return set_error(PS_ERROR, "batch needs at least one frame");
    if (width < 1 || height < 1 || width > 50000)
        return set_error(PS_DIMENSION_TOO_SMALL, "bad image size for the WTA matcher");
    if (max_disparity < 0) return set_error(PS_INVALID_CONFIG, "maxDisparity must be >= 0");
    if (!left || !right || !disparity || !valid || !cost) return set_error(PS_ERROR, "null buffer");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const size_t n = size_t(frames) * P;
    uint8_t* d_l = e.dev<uint8_t>(e.s_a, n);
    uint8_t* d_r = e.dev<uint8_t>(e.s_b, n);
    uint32_t* d_cl = e.dev<uint32_t>(e.s_c, n);
    uint32_t* d_cr = e.dev<uint32_t>(e.s_d, n);
    uint8_t* d_m = e.dev<uint8_t>(e.s_e, n);
    float* d_disp = e.dev<float>(e.s_f, n);
    uint8_t* d_ok = e.dev<uint8_t>(e.s_g, n);
    float* d_cost = e.dev<float>(e.s_h, n);
    if (!d_l || !d_r || !d_cl || !d_cr || !d_m || !d_disp || !d_ok || !d_cost)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    const ps::FrameGeom g{width, height, P};
    cudaMemcpyAsync(d_l, left, n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_r, right, n, cudaMemcpyHostToDevice, st);
    if (mask) cudaMemcpyAsync(d_m, mask, n, cudaMemcpyHostToDevice, st);
    // census of both views (and the gradient mask when not given)
    e.count_launches(ps::launch_frontend(d_l, d_r, g, frames, threshold, mask ? nullptr : d_m, d_cl,
                                         d_cr, nullptr, st));
    ps_config dc;
    ps_config_default(&dc);
    e.count_launches(ps::launch_wta(d_cl, d_cr, d_m, g, frames, max_disparity, ps::make_tables(dc),
                                    d_disp, d_ok, d_cost, st));
    cudaMemcpyAsync(disparity, d_disp, 4 * n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(valid, d_ok, n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(cost, d_cost, 4 * n, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("wta oracle"));
}
}  // namespace

ps_status ps_wta_oracle(ps_ctx* ctx, const uint8_t* left, const uint8_t* right, int width,
                        int height, const uint8_t* mask, int max_disparity, float* disparity,
                        uint8_t* disparity_valid, float* cost) {
    PS_REQUIRE_CTX(ctx);
    if (!mask) return set_error(PS_ERROR, "null mask");
    return wta_common(ctx, 1, left, right, width, height, mask, 0, max_disparity, disparity,
                      disparity_valid, cost);
}

ps_status ps_wta_batch(ps_ctx* ctx, int n_frames, const uint8_t* left, const uint8_t* right,
                       int width, int height, int gradient_threshold, int max_disparity,
                       float* disparity, uint8_t* disparity_valid, float* cost) {
    PS_REQUIRE_CTX(ctx);
    return wta_common(ctx, n_frames, left, right, width, height, nullptr, gradient_threshold,
                      max_disparity, disparity, disparity_valid, cost);
}

namespace {
// KITTI 16-bit raster of device maps into host `out` (2 bytes per pixel).
ps_status kitti_device(ps_ctx* ctx, const float* d_disp, const uint8_t* d_valid, const int* d_ok,
                       long long P, int frames, uint8_t* out) {
    ps::Engine& e = *ctx->engine;
    const size_t n = size_t(frames) * P;
    uint16_t* d_out = e.dev<uint16_t>(e.s_j, n);
    unsigned long long* d_neg = e.dev<unsigned long long>(e.s_i, 1);
    if (!d_out || !d_neg) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    cudaMemsetAsync(d_neg, 0xff, sizeof(unsigned long long), st);
    e.count_launches(ps::launch_kitti16(d_disp, d_valid, d_ok, P, frames, d_out, d_neg, st));
    unsigned long long neg = ~0ull;
    cudaMemcpyAsync(&neg, d_neg, sizeof(neg), cudaMemcpyDeviceToHost, st);
    ps_status s = from_engine(ctx, e.sync("kitti encode"));
    if (s != PS_OK) return s;
    if (neg != ~0ull) {  // writeKittiPng throws at the first negative valid disparity
        float d = 0.0f;
        cudaMemcpy(&d, d_disp + neg, sizeof(float), cudaMemcpyDeviceToHost);
        return set_error(PS_NEGATIVE_DISPARITY, "cannot encode negative disparity " + std::to_string(d));
    }
    return from_engine(ctx, e.check(cudaMemcpy(out, d_out, 2 * n, cudaMemcpyDeviceToHost), "D2H kitti"));
}

ps_status pfm_device(ps_ctx* ctx, const float* d_disp, const uint8_t* d_valid, const int* d_ok,
                     int W, int H, int frames, float* out) {
    ps::Engine& e = *ctx->engine;
    const size_t n = size_t(frames) * W * H;
    float* d_out = e.dev<float>(e.s_j, n);
    if (!d_out) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    e.count_launches(ps::launch_pfm(d_disp, d_valid, d_ok, W, H, frames, d_out, st));
    cudaMemcpyAsync(out, d_out, 4 * n, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("pfm encode"));
}

ps_status cloud_device(ps_ctx* ctx, const float* d_disp, const uint8_t* d_valid,
                       const uint8_t* d_img, int W, int H, const ps_calib* calib, double min_d,
                       float* xyz, uint8_t* intensity, int capacity, int* count) {
    if (!calib) return set_error(PS_ERROR, "null calibration");
    // CameraCalib::validate (proj/src/io.cpp:19-26)
    if (!(calib->focal > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration focal length must be positive");
    if (!(calib->baseline > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration baseline must be positive");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)W * H;
    const int cap = std::max(capacity, 0);
    float* d_xyz = e.dev<float>(e.s_h, size_t(std::max(cap, 1)) * 3);
    uint8_t* d_int = e.dev<uint8_t>(e.s_g, size_t(std::max(cap, 1)));
    int* d_chunk = e.dev<int>(e.s_f, size_t(P / 1024 + 2));
    int* d_cnt = e.dev<int>(e.s_i, 1);
    if (!d_xyz || !d_int || !d_chunk || !d_cnt) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    e.count_launches(ps::launch_point_cloud(d_disp, d_valid, d_img, W, H, calib->focal,
                                            calib->baseline, calib->cx, calib->cy, min_d, d_xyz,
                                            d_int, cap, d_chunk, d_cnt, st));
    int n = 0;
    cudaMemcpyAsync(&n, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, st);
    ps_status s = from_engine(ctx, e.sync("point cloud"));
    if (s != PS_OK) return s;
    if (count) *count = n;
    if (n == 0) return set_error(PS_EMPTY_CLOUD, "no valid pixels above the minimum disparity");
    if (n > cap) return set_error(PS_CAPACITY, "point cloud buffer too small");
    if (xyz) cudaMemcpyAsync(xyz, d_xyz, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, st);
    if (intensity) cudaMemcpyAsync(intensity, d_int, n, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("point cloud D2H"));
}

ps_status upload_map(ps_ctx* ctx, const float* disparity, const uint8_t* valid, size_t n,
                     float** d_disp, uint8_t** d_valid) {
    if (!disparity || !valid) return set_error(PS_ERROR, "null map");
    ps::Engine& e = *ctx->engine;
    *d_disp = e.dev<float>(e.s_a, n);
    *d_valid = e.dev<uint8_t>(e.s_b, n);
    if (!*d_disp || !*d_valid) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(*d_disp, disparity, 4 * n, cudaMemcpyHostToDevice, e.stream());
    cudaMemcpyAsync(*d_valid, valid, n, cudaMemcpyHostToDevice, e.stream());
    return PS_OK;
}
}  // namespace

ps_status ps_encode_kitti16(ps_ctx* ctx, const float* disparity, const uint8_t* valid, int width,
                            int height, int n_frames, uint8_t* out) {
    PS_REQUIRE_CTX(ctx);
    if (width < 1 || height < 1 || n_frames < 1 || !out) return set_error(PS_ERROR, "bad arguments");
    float* dd;
    uint8_t* dv;
    ps_status s = upload_map(ctx, disparity, valid, size_t(n_frames) * width * height, &dd, &dv);
    if (s != PS_OK) return s;
    return kitti_device(ctx, dd, dv, nullptr, (long long)width * height, n_frames, out);
}

ps_status ps_encode_pfm(ps_ctx* ctx, const float* disparity, const uint8_t* valid, int width,
                        int height, int n_frames, float* out) {
    PS_REQUIRE_CTX(ctx);
    if (width < 1 || height < 1 || n_frames < 1 || !out) return set_error(PS_ERROR, "bad arguments");
    float* dd;
    uint8_t* dv;
    ps_status s = upload_map(ctx, disparity, valid, size_t(n_frames) * width * height, &dd, &dv);
    if (s != PS_OK) return s;
    return pfm_device(ctx, dd, dv, nullptr, width, height, n_frames, out);
}

ps_status ps_point_cloud(ps_ctx* ctx, const float* disparity, const uint8_t* valid,
                         const uint8_t* image, int width, int height, const ps_calib* calib,
                         double min_disparity, float* xyz, uint8_t* intensity, int capacity,
                         int* count) {
    PS_REQUIRE_CTX(ctx);
    if (width < 1 || height < 1 || !image) return set_error(PS_ERROR, "bad arguments");
    if (!calib) return set_error(PS_ERROR, "null calibration");
    if (!(calib->focal > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration focal length must be positive");
    if (!(calib->baseline > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration baseline must be positive");
    const size_t n = size_t(width) * height;
    float* dd;
    uint8_t* dv;
    ps_status s = upload_map(ctx, disparity, valid, n, &dd, &dv);
    if (s != PS_OK) return s;
    ps::Engine& e = *ctx->engine;
    uint8_t* di = e.dev<uint8_t>(e.s_c, n);
    if (!di) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaMemcpyAsync(di, image, n, cudaMemcpyHostToDevice, e.stream());
    return cloud_device(ctx, dd, dv, di, width, height, calib, min_disparity, xyz, intensity,
                        capacity, count);
}

namespace {
ps_status resident(ps_ctx* ctx, int which, ps::Engine::ResidentMaps& m, const float** d,
                   const uint8_t** v) {
    if (which != PS_MAP_DISPARITY && which != PS_MAP_DENSE)
        return set_error(PS_ERROR, "which must be PS_MAP_DISPARITY or PS_MAP_DENSE");
    ps_status s = from_engine(ctx, ctx->engine->resident_maps(m));
    if (s != PS_OK) return s;
    *d = which == PS_MAP_DENSE ? m.dense : m.disparity;
    *v = which == PS_MAP_DENSE ? m.dense_valid : m.disparity_valid;
    return PS_OK;
}
}  // namespace

ps_status ps_download_kitti16(ps_ctx* ctx, int which, uint8_t* out) {
    PS_REQUIRE_CTX(ctx);
    if (!out) return set_error(PS_ERROR, "null output");
    ps::Engine::ResidentMaps m;
    const float* d;
    const uint8_t* v;
    ps_status s = resident(ctx, which, m, &d, &v);
    if (s != PS_OK) return s;
    return kitti_device(ctx, d, v, m.frame_ok, m.pixels, m.frames, out);
}

ps_status ps_download_pfm(ps_ctx* ctx, int which, float* out) {
    PS_REQUIRE_CTX(ctx);
    if (!out) return set_error(PS_ERROR, "null output");
    ps::Engine::ResidentMaps m;
    const float* d;
    const uint8_t* v;
    ps_status s = resident(ctx, which, m, &d, &v);
    if (s != PS_OK) return s;
    return pfm_device(ctx, d, v, m.frame_ok, m.width, m.height, m.frames, out);
}

ps_status ps_download_point_cloud(ps_ctx* ctx, int frame, int which, const ps_calib* calib,
                                  double min_disparity, float* xyz, uint8_t* intensity,
                                  int capacity, int* count) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine::ResidentMaps m;
    const float* d;
    const uint8_t* v;
    ps_status s = resident(ctx, which, m, &d, &v);
    if (s != PS_OK) return s;
    if (frame < 0 || frame >= m.frames) return set_error(PS_ERROR, "no such frame");
    if (!calib) return set_error(PS_ERROR, "null calibration");
    if (!(calib->focal > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration focal length must be positive");
    if (!(calib->baseline > 0.0))
        return set_error(PS_INVALID_CONFIG, "calibration baseline must be positive");
    int ok = 0;
    cudaMemcpy(&ok, m.frame_ok + frame, sizeof(int), cudaMemcpyDeviceToHost);
    if (!ok) {  // no result: an empty map
        if (count) *count = 0;
        return set_error(PS_EMPTY_CLOUD, "no valid pixels above the minimum disparity");
    }
    const size_t b = size_t(frame) * m.pixels;
    return cloud_device(ctx, d + b, v + b, m.left + b, m.width, m.height, calib, min_disparity, xyz,
                        intensity, capacity, count);
}

namespace {
ps_status accuracy_device(ps_ctx* ctx, int frames, const float* d_pred, const uint8_t* d_pv,
                          const float* gt, const uint8_t* gt_valid, const uint8_t* d_mask,
                          long long P, const double* thresholds, int n_thr, double* fractions,
                          long long* evaluated, double* mean_abs_error) {
    if (n_thr < 0 || n_thr > 16 || (n_thr > 0 && !thresholds))
        return set_error(PS_ERROR, "0..16 thresholds");
    if (!gt || !gt_valid) return set_error(PS_ERROR, "null ground truth");
    ps::Engine& e = *ctx->engine;
    const size_t n = size_t(frames) * P;
    float* d_gt = e.dev<float>(e.s_c, n);
    uint8_t* d_gv = e.dev<uint8_t>(e.s_d, n);
    double* d_thr = e.dev<double>(e.s_e, 16);
    unsigned long long* d_cnt = e.dev<unsigned long long>(e.s_f, size_t(frames) * (1 + n_thr));
    double* d_sum = e.dev<double>(e.s_g, size_t(frames));
    if (!d_gt || !d_gv || !d_thr || !d_cnt || !d_sum) return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(d_gt, gt, 4 * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_gv, gt_valid, n, cudaMemcpyHostToDevice, st);
    if (n_thr > 0) cudaMemcpyAsync(d_thr, thresholds, sizeof(double) * n_thr, cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_accuracy(d_pred, d_pv, d_gt, d_gv, d_mask, P, frames, d_thr, n_thr,
                                         d_cnt, d_sum, st));
    std::vector<unsigned long long> cnt(size_t(frames) * (1 + n_thr));
    std::vector<double> sum(frames);
    cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned long long) * cnt.size(), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(sum.data(), d_sum, sizeof(double) * frames, cudaMemcpyDeviceToHost, st);
    ps_status s = from_engine(ctx, e.sync("accuracy"));
    if (s != PS_OK) return s;
    bool empty = false;
    for (int f = 0; f < frames; ++f) {
        const unsigned long long* c = cnt.data() + size_t(f) * (1 + n_thr);
        const long long ev = (long long)c[0];
        if (evaluated) evaluated[f] = ev;
        if (ev == 0) {  // accuracyImpl throws NoOverlap (eval.cpp:50-52)
            empty = true;
            if (mean_abs_error) mean_abs_error[f] = 0.0;
            for (int k = 0; k < n_thr && fractions; ++k) fractions[size_t(f) * n_thr + k] = 0.0;
            continue;
        }
        if (mean_abs_error) mean_abs_error[f] = sum[f] / double(ev);
        for (int k = 0; k < n_thr && fractions; ++k)
            fractions[size_t(f) * n_thr + k] = double(c[1 + k]) / double(ev);
    }
    if (empty) return set_error(PS_NO_OVERLAP, "no jointly valid pixels to evaluate");
    return PS_OK;
}
}  // namespace

ps_status ps_accuracy(ps_ctx* ctx, int n_frames, const float* prediction,
                      const uint8_t* prediction_valid, const float* ground_truth,
                      const uint8_t* ground_truth_valid, const uint8_t* mask, int width,
                      int height, const double* thresholds, int n_thresholds, double* fractions,
                      long long* evaluated, double* mean_abs_error) {
    PS_REQUIRE_CTX(ctx);
    if (n_frames < 1 || width < 1 || height < 1) return set_error(PS_ERROR, "bad arguments");
    const long long P = (long long)width * height;
    const size_t n = size_t(n_frames) * P;
    float* dd;
    uint8_t* dv;
    ps_status s = upload_map(ctx, prediction, prediction_valid, n, &dd, &dv);
    if (s != PS_OK) return s;
    ps::Engine& e = *ctx->engine;
    uint8_t* dm = nullptr;
    if (mask) {
        dm = e.dev<uint8_t>(e.s_h, n);
        if (!dm) return set_error(PS_CUDA_ERROR, "allocation failed");
        cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, e.stream());
    }
    return accuracy_device(ctx, n_frames, dd, dv, ground_truth, ground_truth_valid, dm, P,
                           thresholds, n_thresholds, fractions, evaluated, mean_abs_error);
}

ps_status ps_download_accuracy(ps_ctx* ctx, int which, const float* ground_truth,
                               const uint8_t* ground_truth_valid, int use_mask,
                               const double* thresholds, int n_thresholds, double* fractions,
                               long long* evaluated, double* mean_abs_error) {
    PS_REQUIRE_CTX(ctx);
    ps::Engine::ResidentMaps m;
    const float* d;
    const uint8_t* v;
    ps_status s = resident(ctx, which, m, &d, &v);
    if (s != PS_OK) return s;
    // a frame without a result has an all-invalid prediction: mask it out via
    // its frame_ok entry by evaluating through a per-frame validity copy
    ps::Engine& e = *ctx->engine;
    std::vector<int> ok(m.frames);
    cudaMemcpy(ok.data(), m.frame_ok, sizeof(int) * m.frames, cudaMemcpyDeviceToHost);
    const uint8_t* pv = v;
    bool any_failed = false;
    for (int f = 0; f < m.frames; ++f) any_failed |= ok[f] == 0;
    if (any_failed) {
        uint8_t* copy = e.dev<uint8_t>(e.s_b, size_t(m.frames) * m.pixels);
        if (!copy) return set_error(PS_CUDA_ERROR, "allocation failed");
        for (int f = 0; f < m.frames; ++f) {
            const size_t b = size_t(f) * m.pixels;
            if (ok[f]) cudaMemcpyAsync(copy + b, v + b, m.pixels, cudaMemcpyDeviceToDevice, e.stream());
            else cudaMemsetAsync(copy + b, 0, m.pixels, e.stream());
        }
        pv = copy;
    }
    return accuracy_device(ctx, m.frames, d, pv, ground_truth, ground_truth_valid,
                           use_mask ? m.mask : nullptr, m.pixels, thresholds, n_thresholds,
                           fractions, evaluated, mean_abs_error);
}

namespace {
// BASELINE generator on the device into (d_left, d_right) with frame stride P.
ps_status synth_device(ps_ctx* ctx, const ps_synth_params* p, int n_frames, uint8_t* d_left,
                       uint8_t* d_right, float** d_gt_out) {
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)p->width * p->height;
    const long long draws = ps::baseline_stream_draws(p->width, p->height, p->n_planes);
    uint32_t* d_seeds = e.dev<uint32_t>(e.s_a, size_t(n_frames));
    uint32_t* d_stream = e.dev<uint32_t>(e.s_b, size_t(n_frames) * draws);
    float* d_disp = e.dev<float>(e.s_c, size_t(n_frames) * P);
    unsigned long long* d_keys = e.dev<unsigned long long>(e.s_d, size_t(n_frames) * P);
    if (!d_seeds || !d_stream || !d_disp || !d_keys) return set_error(PS_CUDA_ERROR, "allocation failed");
    std::vector<uint32_t> seeds(n_frames);
    for (int f = 0; f < n_frames; ++f) seeds[f] = p->seed + uint32_t(f);
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(d_seeds, seeds.data(), sizeof(uint32_t) * n_frames, cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_mt_streams(d_seeds, n_frames, draws, draws, d_stream, st));
    e.count_launches(ps::launch_synth_baseline(*p, n_frames, d_stream, draws, d_disp, d_keys,
                                               d_left, d_right, P, st));
    if (d_gt_out) *d_gt_out = d_disp;
    return from_engine(ctx, e.sync("synth"));
}

ps_status check_synth(const ps_synth_params* p, int n_frames) {
    if (!p || n_frames < 1) return set_error(PS_ERROR, "bad generator arguments");
    if (p->width < 16 || p->height < 16) return set_error(PS_DIMENSION_TOO_SMALL, "image must be at least 16x16");
    if (p->n_planes < 0 || p->n_planes > 4096) return set_error(PS_ERROR, "0..4096 planes");
    return PS_OK;
}
}  // namespace

ps_status ps_synth_batch_gpu(ps_ctx* ctx, const ps_synth_params* params, int n_frames,
                             uint8_t* left, uint8_t* right, float* gt) {
    PS_REQUIRE_CTX(ctx);
    ps_status s = check_synth(params, n_frames);
    if (s != PS_OK) return s;
    if (!left || !right) return set_error(PS_ERROR, "null output");
    ps::Engine& e = *ctx->engine;
    const size_t n = size_t(n_frames) * params->width * params->height;
    uint8_t* dl = e.dev<uint8_t>(e.s_e, n);
    uint8_t* dr = e.dev<uint8_t>(e.s_f, n);
    if (!dl || !dr) return set_error(PS_CUDA_ERROR, "allocation failed");
    float* dg = nullptr;
    s = synth_device(ctx, params, n_frames, dl, dr, &dg);
    if (s != PS_OK) return s;
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(left, dl, n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(right, dr, n, cudaMemcpyDeviceToHost, st);
    if (gt) cudaMemcpyAsync(gt, dg, 4 * n, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("synth D2H"));
}

ps_status ps_synth_resident(ps_ctx* ctx, const ps_synth_params* params, int n_frames) {
    PS_REQUIRE_CTX(ctx);
    ps_status s = check_synth(params, n_frames);
    if (s != PS_OK) return s;
    uint8_t *dl = nullptr, *dr = nullptr;
    s = from_engine(ctx, ctx->engine->device_inputs(n_frames, params->width, params->height, &dl, &dr));
    if (s != PS_OK) return s;
    return synth_device(ctx, params, n_frames, dl, dr, nullptr);
}

ps_status ps_render_scene(ps_ctx* ctx, int width, int height, float max_disparity, uint32_t seed,
                          const ps_scene_region* regions, int n_regions, uint8_t* left,
                          uint8_t* right, float* ground_truth, uint8_t* ground_truth_valid,
                          uint8_t* occluded) {
    PS_REQUIRE_CTX(ctx);
    if (width < 1 || height < 1 || (n_regions > 0 && !regions) || n_regions < 0)
        return set_error(PS_ERROR, "bad scene arguments");
    if (!left || !right || !ground_truth || !ground_truth_valid || !occluded)
        return set_error(PS_ERROR, "null output");
    const int w = width, h = height;
    // region checks (proj/src/synth.cpp:94-110), on the host: regions are few
    std::vector<uint8_t> covered(size_t(w) * h, 0);
    for (int k = 0; k < n_regions; ++k) {
        const ps_scene_region& r = regions[k];
        if (r.u0 < 0 || r.v0 < 0 || r.u1 > w || r.v1 > h || r.u0 >= r.u1 || r.v0 >= r.v1)
            return set_error(PS_ERROR, "scene region outside image bounds");
        for (int v = r.v0; v < r.v1; ++v)
            for (int u = r.u0; u < r.u1; ++u)
                if (covered[size_t(v) * w + u]++) return set_error(PS_ERROR, "scene regions overlap");
    }
    for (uint8_t c : covered)
        if (c != 1) return set_error(PS_ERROR, "scene regions must cover the image");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)w * h;
    ps::SceneRegionDev* d_reg = e.dev<ps::SceneRegionDev>(e.s_a, size_t(std::max(1, n_regions)));
    uint32_t* d_seeds = e.dev<uint32_t>(e.s_b, 2);
    uint32_t* d_stream = e.dev<uint32_t>(e.s_c, size_t(2 * P));
    int* d_ta = e.dev<int>(e.s_d, size_t(P));
    int* d_tb = e.dev<int>(e.s_e, size_t(P));
    int* d_mm = e.dev<int>(e.s_f, 4);
    unsigned long long* d_keys = e.dev<unsigned long long>(e.s_g, size_t(P));
    unsigned long long* d_bad = e.dev<unsigned long long>(e.s_h, 1);
    uint8_t* d_out = e.dev<uint8_t>(e.s_i, size_t(4 * P));  // left, right, gt_valid, occluded
    float* d_gt = e.dev<float>(e.s_j, size_t(P));
    if (!d_reg || !d_seeds || !d_stream || !d_ta || !d_tb || !d_mm || !d_keys || !d_bad || !d_out || !d_gt)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    std::vector<ps::SceneRegionDev> reg(n_regions);
    for (int k = 0; k < n_regions; ++k)
        reg[k] = {regions[k].u0, regions[k].v0, regions[k].u1, regions[k].v1, regions[k].a,
                  regions[k].b, regions[k].c};
    const uint32_t seeds[2] = {seed, seed + 1};
    cudaStream_t st = e.stream();
    if (n_regions > 0)
        cudaMemcpyAsync(d_reg, reg.data(), sizeof(ps::SceneRegionDev) * n_regions, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_seeds, seeds, sizeof(seeds), cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_mt_streams(d_seeds, 2, P, P, d_stream, st));
    e.count_launches(ps::launch_render_scene(w, h, max_disparity, d_reg, n_regions, d_stream,
                                             d_stream + P, d_ta, d_tb, d_mm, d_keys, d_bad, d_out,
                                             d_out + P, d_gt, d_out + 2 * P, d_out + 3 * P, st));
    unsigned long long bad = 0;
    cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st);
    ps_status s = from_engine(ctx, e.sync("render scene"));
    if (s != PS_OK) return s;
    if (bad != ~0ull) {  // renderScene throws InvalidPlane at the first offending pixel
        const int k = int(bad >> 40);
        const long long i = (long long)(bad & ((1ull << 40) - 1));
        const int v = int(i / w), u = int(i - (long long)v * w);
        const ps_scene_region& r = regions[k];
        const double d = r.a * u + r.b * v + r.c;
        return set_error(PS_INVALID_PLANE, "plane value " + std::to_string(d) + " at (" +
                                               std::to_string(u) + "," + std::to_string(v) +
                                               ") outside [0, " + std::to_string(max_disparity) + ")");
    }
    cudaMemcpyAsync(left, d_out, P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(right, d_out + P, P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(ground_truth_valid, d_out + 2 * P, P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(occluded, d_out + 3 * P, P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(ground_truth, d_gt, 4 * P, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("render scene D2H"));
}

ps_status ps_refinement(ps_ctx* ctx, const float* interp, const uint8_t* interp_valid,
                        const float* cost, float* final_disparity, uint8_t* final_valid,
                        float* final_cost, const uint8_t* mask, int width, int height,
                        int cell_size, const ps_config* cfg, ps_cell* confident,
                        ps_cell* invalid) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg || cell_size < 1) return set_error(PS_ERROR, "bad refinement arguments");
    static_assert(sizeof(ps_cell) == sizeof(ps::StageCell), "ps_cell layout");
    ps::Engine& e = *ctx->engine;
    const long long P = (long long)width * height;
    const int cells = ((width + cell_size - 1) / cell_size) * ((height + cell_size - 1) / cell_size);
    float* d_iv = e.dev<float>(e.s_a, P);
    uint8_t* d_ok = e.dev<uint8_t>(e.s_b, P);
    float* d_c = e.dev<float>(e.s_c, P);
    uint8_t* d_m = e.dev<uint8_t>(e.s_d, P);
    float* d_fd = e.dev<float>(e.s_e, P);
    uint8_t* d_fv = e.dev<uint8_t>(e.s_f, P);
    float* d_fc = e.dev<float>(e.s_g, P);
    unsigned long long* d_k = e.dev<unsigned long long>(e.s_h, 2 * size_t(cells));
    ps::StageCell* d_cells = reinterpret_cast<ps::StageCell*>(
        e.dev<uint8_t>(e.s_i, 2 * size_t(cells) * sizeof(ps::StageCell)));
    if (!d_iv || !d_ok || !d_c || !d_m || !d_fd || !d_fv || !d_fc || !d_k || !d_cells)
        return set_error(PS_CUDA_ERROR, "allocation failed");
    cudaStream_t st = e.stream();
    cudaMemcpyAsync(d_iv, interp, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_ok, interp_valid, P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_c, cost, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_m, mask, P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_fd, final_disparity, 4 * P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_fv, final_valid, P, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_fc, final_cost, 4 * P, cudaMemcpyHostToDevice, st);
    e.count_launches(ps::launch_stage_refine({width, height, P}, d_iv, d_ok, d_c, d_m, d_fd, d_fv,
                                             d_fc, cell_size, cfg->cost_low, cfg->cost_high, d_k,
                                             d_k + cells, d_cells, d_cells + cells, st));
    cudaMemcpyAsync(final_disparity, d_fd, 4 * P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(final_valid, d_fv, P, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(final_cost, d_fc, 4 * P, cudaMemcpyDeviceToHost, st);
    if (confident)
        cudaMemcpyAsync(confident, d_cells, sizeof(ps_cell) * cells, cudaMemcpyDeviceToHost, st);
    if (invalid)
        cudaMemcpyAsync(invalid, d_cells + cells, sizeof(ps_cell) * cells, cudaMemcpyDeviceToHost, st);
    return from_engine(ctx, e.sync("refinement"));
}

ps_status ps_support_resampling(ps_ctx* ctx, const ps_cell* confident, const ps_cell* invalid,
                                int cell_size, const int* sup_u, const int* sup_v,
                                const double* sup_d, int n_supports,
                                const uint32_t* census_left, const uint32_t* census_right,
                                int width, int height, const ps_config* cfg, int* u, int* v,
                                double* d, int capacity, int* count) {
    PS_REQUIRE_CTX(ctx);
    if (!cfg || cell_size < 1) return set_error(PS_ERROR, "bad resampling arguments");
    // supportResampling (pipeline.cpp:88-129): ordered list assembly with the
    // reference's taken-set semantics; the epipolar re-match of the invalid
    // cells runs on the device (ps_match_epipolar).
    const int cells = ((width + cell_size - 1) / cell_size) * ((height + cell_size - 1) / cell_size);
    const long long w = width;
    std::unordered_map<long long, char> taken;
    taken.reserve(size_t(n_supports) * 2 + 16);
    std::vector<int> ou(sup_u, sup_u + n_supports), ov(sup_v, sup_v + n_supports);
    std::vector<double> od(sup_d, sup_d + n_supports);
    for (int i = 0; i < n_supports; ++i) taken.emplace((long long)sup_v[i] * w + sup_u[i], 1);
    for (int c = 0; c < cells; ++c) {
        const ps_cell& cell = confident[c];
        if (!cell.occupied) continue;
        const float diff = float(cell.u) - cell.disparity;  // binary32, pipeline.cpp:105
        if (diff < 2.0f) continue;
        if (taken.emplace((long long)cell.v * w + cell.u, 1).second) {
            ou.push_back(cell.u);
            ov.push_back(cell.v);
            od.push_back(double(cell.disparity));
        }
    }
    std::vector<int> ru, rv;
    for (int c = 0; c < cells; ++c) {
        if (!invalid[c].occupied) continue;
        ru.push_back(invalid[c].u);
        rv.push_back(invalid[c].v);
    }
    std::vector<int> mu(ru.size() + 1), mv(ru.size() + 1);
    std::vector<double> md(ru.size() + 1);
    int nm = 0;
    const ps_status s = ps_match_epipolar(ctx, census_left, census_right, width, height, ru.data(),
                                          rv.data(), int(ru.size()), cfg, mu.data(), mv.data(),
                                          md.data(), int(ru.size()) + 1, &nm);
    if (s != PS_OK) return s;
    for (int i = 0; i < nm; ++i) {
        if (taken.emplace((long long)mv[i] * w + mu[i], 1).second) {
            ou.push_back(mu[i]);
            ov.push_back(mv[i]);
            od.push_back(md[i]);
        }
    }
    const int m = int(ou.size());
    if (count) *count = m;
    for (int i = 0; i < m && i < capacity; ++i) {
        if (u) u[i] = ou[i];
        if (v) v[i] = ov[i];
        if (d) d[i] = od[i];
    }
    if (m > capacity) return set_error(PS_CAPACITY, "support buffer too small");
    return PS_OK;
}

}  // extern "C"
