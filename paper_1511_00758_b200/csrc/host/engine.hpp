// engine.hpp — the batched B200 pipeline behind the C ABI.
//
// One Engine per ps_ctx: a device, grow-only device/pinned buffers, a host
// worker pool for the per-frame Delaunay step, and up to kMaxGroups CUDA
// streams.  A batch of F frames of one shape runs planestereo::run
// (proj/src/pipeline.cpp:131-203) for every frame at once: the front end and
// seeding are one launch per stage over all frames; the iterations run as a
// software pipeline over frame groups, each on its own stream, so that the
// device stages of group g overlap the host Delaunay of group g+1.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../kernels/common.cuh"
#include "delaunay.hpp"
#include "frame_mesh.hpp"
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

// A contiguous range of frames with its own stream and per-iteration staging.
struct FrameGroup {
    enum Phase { kIdle, kSeed, kHost, kDevice, kDone };
    int f0 = 0;
    int n = 0;
    int it = 0;                   // iteration being processed
    Phase phase = kIdle;
    std::atomic<int> pending{0};  // Delaunay tasks still running
    cudaEvent_t done_event = nullptr;
    double tic = 0.0;
    cudaStream_t st = nullptr;
    // the device mesh runs on its own low-priority stream (kernels/star.cu:
    // latency-bound, small grids), ordered after / before st by two events
    cudaStream_t mst = nullptr;
    cudaEvent_t mesh_in = nullptr, mesh_out = nullptr;
    int* S = nullptr;      // device support counts of the group's frames (current)
    int* Snext = nullptr;  // device support counts (next)
    DevBuf dTri, dTriOff, dPlanes, dPack, dPackD, dPackOff, dSprev, dChunk, dPin;
    HostBuf hS, hSprev, hPackOff, hPack, hPackD, hTri, hTriOff, hPin;
    std::vector<int> ntri;
    // device mesh (kernels/star.cu): grid scratch, pin choices, flags, fixes
    DevBuf dCellCnt, dCellStart, dCellItems, dCellXY, dDup, dPinTri, dTriCount, dFlags, dFix, dColKey, dColIdx, dHull, dHullTmp, dHard, dRing;
    HostBuf hTriCount, hFlags, hFix;
    std::vector<std::vector<int>> fixes;  // per frame: host fixes for the device mesh
    std::vector<uint8_t> replayed;        // per frame: triangles came from the host replay
    int gs = 0, gw = 0, gh = 0;           // grid of the mesh in flight
    double millis = 0.0;
};

class Engine {
public:
    static constexpr int kMaxGroups = 8;

    explicit Engine(int device);
    ~Engine();

    int device() const { return device_; }
    cudaStream_t stream() const { return st_; }
    std::string& error() { return err_; }

    // deferred = true (ps_run_batch only): the host images are copied by the
    // next run_resident(), group by group on the group streams, so the first
    // group's seeding overlaps the other groups' H2D; the caller keeps the
    // buffers alive until that run returns.
    ps_status upload(int frames, const uint8_t* left, const uint8_t* right, int width, int height,
                     bool deferred = false);
    // The batch input buffers themselves, for inputs generated on the device
    // (ps_synth_resident); afterwards the batch counts as uploaded.
    ps_status device_inputs(int frames, int width, int height, uint8_t** left, uint8_t** right);
    ps_status run_resident(const ps_config& cfg, unsigned flags, ps_observer_fn observer = nullptr,
                           void* user = nullptr);
    ps_status download(float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                       uint8_t* dense_valid, ps_iter_stats* trace, int* frame_status);
    // Streamed download: with a sink set, run_resident() copies each frame
    // group's outputs to these (page-locked) host buffers on the group's
    // stream as soon as its last iteration is launched, overlapping the D2H
    // with the other groups' work; download() then only fixes up failed
    // frames and copies the trace.  Pageable buffers are not streamed.
    void set_sink(float* disparity, uint8_t* disparity_valid, float* cost, float* dense,
                  uint8_t* dense_valid);
    void clear_sink() { sink_ = Sink{}; }
    ps_status supports(int frame, int* u, int* v, double* d, int capacity, int* count);
    // Device views of the last run's result maps, for the output encoders
    // (capi.cpp); frame_ok[f] = 1 when frame f produced a result.
    struct ResidentMaps {
        const float* disparity;
        const uint8_t* disparity_valid;
        const float* dense;
        const uint8_t* dense_valid;
        const uint8_t* left;
        const uint8_t* mask;  // the run's gradient mask (Omega_I)
        const int* frame_ok;  // device, F entries
        int frames, width, height;
        long long pixels;
    };
    ps_status resident_maps(ResidentMaps& m);

    void set_profiling(bool on) { profiling_ = on; }
    // Upper bound on concurrent frame groups (streams); 1 serialises the
    // device stages, so per-kernel event times are isolated launch durations.
    void set_max_groups(int g) { max_groups_ = g < 1 ? 1 : g; }
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
    ps_status sync(cudaStream_t s, const char* what);
    void count_launches(int n) { launches_ += n; }
    ThreadPool& pool() { return *pool_; }
    DelaunayWorkspace& workspace(int worker) { return (*ws_)[worker]; }

    // Scratch for stage-API calls.
    DevBuf s_a, s_b, s_c, s_d, s_e, s_f, s_g, s_h, s_i, s_j;
    DevBuf dFrameOk_;  // resident_maps()

private:
    void begin_kernel(const char* name, double bytes, cudaStream_t s);
    void end_kernel(cudaStream_t s);
    void resolve_timers();
    cudaEvent_t take_event();
    ps_status fail(ps_status s, const std::string& msg) {
        err_ = msg;
        return s;
    }

    struct Sink {
        float* disparity = nullptr;
        uint8_t* disparity_valid = nullptr;
        float* cost = nullptr;
        float* dense = nullptr;
        uint8_t* dense_valid = nullptr;
        bool active = false;
    };
    Sink sink_;
    Sink done_sink_;         // the sink the last run streamed into
    // C_f / validity streamed as their byte codes (1 B/px over PCIe instead of
    // 5) and expanded on the host pool (PS_WIRE_CODES=0: copy the expanded maps)
    bool wire_codes_ = true;
    HostBuf hCodeStage_;
    std::atomic<int> expand_pending_{0};
    bool streamed_ = false;  // the last run already copied its outputs

    int device_ = 0;
    cudaStream_t st_ = nullptr;
    std::string err_;
    ThreadPool* pool_ = nullptr;               // the process-wide pool (shared_pool)
    std::vector<DelaunayWorkspace>* ws_ = nullptr;  // its per-worker workspaces
    bool profiling_ = false;
    int max_groups_ = kMaxGroups;
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
    FrameGroup groups_[kMaxGroups];
    // Completion signal of the host Delaunay tasks.  Engine-owned (not a local
    // of run_resident) so that a task finishing as the run returns never
    // touches a destroyed mutex; tasks decrement their counter under it.
    std::mutex done_m_;
    std::condition_variable done_cv_;

    // batch shape
    int F_ = 0, W_ = 0, H_ = 0;
    long long P_ = 0;
    bool have_inputs_ = false;
    const uint8_t* defer_left_ = nullptr;  // upload(deferred): host images not yet copied
    const uint8_t* defer_right_ = nullptr;
    cudaEvent_t start_event_ = nullptr;  // st_ work the group streams wait on
    // Device stages of different groups run one after another (FIFO through
    // chain_event_) rather than concurrently: the GPU is idle most of a pass
    // (the host Delaunay bounds it), so nothing is lost, and every launch gets
    // the whole GPU.  PS_SERIAL_DEVICE=0 lets groups overlap.
    bool serial_device_ = true;
    int min_group_ = 64;  // frames per group at least (PS_MIN_GROUP)
    bool group_prio_ = false;  // PS_GROUP_PRIO
    bool host_first_ = true;   // PS_HOST_FIRST: first-iteration mesh on the host
    bool debug_timeline_ = false;  // PS_DEBUG_TIMELINE: group milestones on stderr
    cudaEvent_t chain_event_ = nullptr;
    cudaStream_t seed_st_ = nullptr;  // seeding, group after group (group 0 first)
    bool have_outputs_ = false;
    int iters_ = 0;
    float cost_high_ = 0.5f;

    // device buffers (frame-strided)
    DevBuf dL_, dR_, dMask_, dMaskCount_, dCL_, dCR_, dDf_, dDv_, dCf_, dCode_, dDense_, dDenseV_,
        dLookup_, dSu_, dSv_, dSd_, dS_, dSnext_, dTaken_, dCg_, dCb_, dBinKeys_, dBinCount_,
        dScratch_, dCandU_, dCandV_, dCandCount_, dOk_, dDisp_, dOkSeed_, dDispSeed_, dRemU_, dRemV_, dRemCount_,
        dConf_, dChunk_, dTraceSum_, dTraceValid_, dErr_;
    // pinned host staging
    HostBuf hS_, hTraceSum_, hTraceValid_, hMaskCount_;
    int scap_ = 0;
    std::vector<FrameMesh> fmesh_;  // per frame: support list (host copy) + mesh state
    std::vector<int> status_, final_count_;
    std::vector<ps_iter_stats> trace_;
};

}  // namespace ps
