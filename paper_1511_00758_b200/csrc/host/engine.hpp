// engine.hpp — the batched B200 pipeline behind the C ABI.
//
// One Engine per ps_ctx: a device, one CUDA stream, grow-only device/pinned
// buffers and a host worker pool for the per-frame Delaunay step.  A batch of
// F frames of one shape runs planestereo::run (proj/src/pipeline.cpp:131-203)
// for every frame at once: each stage is one launch over all frames
// (frame = grid.y / grid.z), the host triangulates every frame in parallel
// between the device stages of an iteration.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../kernels/common.cuh"
#include "delaunay.hpp"
#include "planestereo_c.h"
#include "thread_pool.hpp"

namespace ps {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct HostBuf {  // pinned
    void* p = nullptr;
    size_t bytes = 0;
};

struct KernelStat {
    std::string name;
    int launches = 0;
    double ms = 0.0;
    double bytes = 0.0;
};

class Engine {
public:
    explicit Engine(int device);
    ~Engine();

    int device() const { return device_; }
    cudaStream_t stream() const { return st_; }
    std::string& error() { return err_; }

    ps_status upload(int frames, const uint8_t* left, const uint8_t* right, int width, int height);
    ps_status run_resident(const ps_config& cfg, unsigned flags, ps_observer_fn observer = nullptr,
                           void* user = nullptr);
    ps_status download(float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                       uint8_t* dense_valid, ps_iter_stats* trace, int* frame_status);
    ps_status supports(int frame, int* u, int* v, double* d, int capacity, int* count);

    void set_profiling(bool on) { profiling_ = on; }
    void reset_stats() { stats_.clear(); }
    const std::vector<KernelStat>& stats() const { return stats_; }
    long long launches() const { return launches_; }

    // Stage helpers used by the single-frame stage API (capi.cpp).
    template <class T>
    T* dev(DevBuf& b, size_t count);
    template <class T>
    T* host(HostBuf& b, size_t count);
    ps_status check(cudaError_t e, const char* what);
    ps_status sync(const char* what);
    void count_launches(int n) { launches_ += n; }
    ThreadPool& pool() { return *pool_; }
    DelaunayWorkspace& workspace(int worker) { return ws_[worker]; }

    // Scratch for stage-API calls.
    DevBuf s_a, s_b, s_c, s_d, s_e, s_f, s_g, s_h, s_i, s_j;

private:
    struct Timer;
    void begin_kernel(const char* name, double bytes);
    void end_kernel();
    void resolve_timers();
    ps_status fail(ps_status s, const std::string& msg) {
        err_ = msg;
        return s;
    }

    int device_ = 0;
    cudaStream_t st_ = nullptr;
    std::string err_;
    ThreadPool* pool_ = nullptr;
    std::vector<DelaunayWorkspace> ws_;
    bool profiling_ = false;
    long long launches_ = 0;
    std::vector<KernelStat> stats_;
    struct Pending {
        int stat;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending_;
    std::vector<cudaEvent_t> event_pool_;
    int pending_stat_ = -1;
    cudaEvent_t pending_start_ = nullptr;

    // batch shape
    int F_ = 0, W_ = 0, H_ = 0;
    long long P_ = 0;
    bool have_inputs_ = false;
    bool have_outputs_ = false;
    int iters_ = 0;
    float cost_high_ = 0.5f;

    // device buffers
    DevBuf dL_, dR_, dMask_, dMaskCount_, dCL_, dCR_, dDf_, dDv_, dCf_, dDense_, dDenseV_,
        dLookup_, dSu_, dSv_, dSd_, dS_, dSnext_, dSprev_, dTaken_, dTri_, dTriOff_, dPlanes_,
        dCg_, dCb_, dBinKeys_, dBinCount_, dScratch_, dCandU_, dCandV_, dCandCount_, dOk_,
        dDisp_, dRemU_, dRemV_, dRemCount_, dConf_, dChunk_, dTraceSum_, dTraceValid_, dErr_,
        dPack_, dPackOff_;
    // pinned host staging
    HostBuf hS_, hSprev_, hPackOff_, hPack_, hTri_, hTriOff_, hTraceSum_, hTraceValid_,
        hMaskCount_, hL_, hR_;
    int scap_ = 0;
    std::vector<std::vector<int>> hu_, hv_, htri_;
    std::vector<int> status_;
    std::vector<ps_iter_stats> trace_;
};

}  // namespace ps
