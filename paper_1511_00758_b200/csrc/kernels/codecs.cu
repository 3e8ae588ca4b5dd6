// codecs.cu — the output encoders of the reference's io module as device
// kernels over disparity maps, so a batch's results can
// leave the GPU already encoded (KITTI: 2 bytes per pixel instead of 5).
//
//   KITTI 16-bit  (proj/src/io.cpp:349-368, writeKittiPng's raster): valid
//                 pixels raw = clamp(lround(double(d) * 256), 1, 65535), big-
//                 endian; invalid 0; a negative valid disparity is an error
//                 (NegativeDisparity, reported for the first one row-major);
//   PFM           (proj/src/io.cpp:311-329, writePfm's raster): rows bottom-up,
//                 little-endian binary32, invalid -1.0;
//   point cloud   (proj/src/io.cpp:395-454, exportPointCloud's vertex list):
//                 row-major valid pixels with d >= minDisparity, z = f*B/d,
//                 x = (u - cx)*z/f, y = (v - cy)*z/f in binary64, stored as
//                 binary32, plus the image intensity — an ordered compaction.
// The file headers and the PNG/PLY containers stay on the host (text).
#include <cuda_runtime.h>

#include <algorithm>

#include "compact.cuh"
#include "launch.hpp"

namespace ps {

namespace {

__device__ __forceinline__ bool frame_valid(const int* frame_ok, long long i, long long P) {
    return !frame_ok || frame_ok[i / P] != 0;
}

__global__ void k_kitti16(const float* __restrict__ d, const uint8_t* __restrict__ valid,
                          const int* __restrict__ frame_ok, long long P, long long n,
                          uint16_t* __restrict__ out, unsigned long long* __restrict__ neg_first) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned raw = 0;
        if (valid[i] && frame_valid(frame_ok, i, P)) {
            const float x = d[i];
            if (x < 0.0f) atomicMin(neg_first, (unsigned long long)i);
            // std::lround(double(d) * 256.0), then clamp to [1, 65535]
            const double s = __dmul_rn(double(x), 256.0);
            const double r = floor(__dadd_rn(s, 0.5));  // s >= 0 here: half away from zero
            // glibc lround gives LONG_MIN when out of range (or NaN): clamps to 1
            if (!(r < 9223372036854775808.0)) raw = 1u;
            else raw = r >= 65535.0 ? 65535u : (r <= 1.0 ? 1u : unsigned(r));
        }
        out[i] = uint16_t((raw >> 8) | ((raw & 0xffu) << 8));  // bytes: high, low
    }
}

__global__ void k_pfm(const float* __restrict__ d, const uint8_t* __restrict__ valid,
                      const int* __restrict__ frame_ok, int W, int H, long long n,
                      float* __restrict__ out) {
    const long long P = (long long)W * H;
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (long long)gridDim.x * blockDim.x) {
        const long long f = o / P;
        const long long r = (o - f * P) / W, u = o - f * P - r * W;
        const long long i = f * P + (H - 1 - r) * W + u;  // bottom-up rows
        out[o] = (valid[i] && frame_valid(frame_ok, i, P)) ? d[i] : -1.0f;
    }
}

struct CloudOp {
    const float* d;
    const uint8_t* valid;
    const uint8_t* image;
    int W;
    long long P;
    double focal, baseline, cx, cy, min_d;
    float* xyz;
    uint8_t* intensity;
    int capacity;
    __device__ int items(int) const { return int(P); }
    __device__ bool test(int, int i) const { return valid[i] && double(d[i]) >= min_d; }
    __device__ void emit(int, int i, int pos) const {
        if (pos >= capacity) return;
        const int v = i / W, u = i - v * W;
        const double dd = double(d[i]);
        const double z = __ddiv_rn(__dmul_rn(focal, baseline), dd);
        const double x = __ddiv_rn(__dmul_rn(__dsub_rn(double(u), cx), z), focal);
        const double y = __ddiv_rn(__dmul_rn(__dsub_rn(double(v), cy), z), focal);
        xyz[3ll * pos] = __double2float_rn(x);
        xyz[3ll * pos + 1] = __double2float_rn(y);
        xyz[3ll * pos + 2] = __double2float_rn(z);
        intensity[pos] = image[i];
    }
};

unsigned grid_for(long long n) {
    return unsigned(std::min<long long>((n + 255) / 256, 148ll * 16));
}

}  // namespace

int launch_kitti16(const float* d, const uint8_t* valid, const int* frame_ok, long long P, int frames,
                   uint16_t* out, unsigned long long* neg_first, cudaStream_t st) {
    const long long n = P * frames;
    k_kitti16<<<grid_for(n), 256, 0, st>>>(d, valid, frame_ok, P, n, out, neg_first);
    return 1;
}

int launch_pfm(const float* d, const uint8_t* valid, const int* frame_ok, int W, int H, int frames,
               float* out, cudaStream_t st) {
    const long long n = (long long)W * H * frames;
    k_pfm<<<grid_for(n), 256, 0, st>>>(d, valid, frame_ok, W, H, n, out);
    return 1;
}

int launch_point_cloud(const float* d, const uint8_t* valid, const uint8_t* image, int W, int H,
                       double focal, double baseline, double cx, double cy, double min_d,
                       float* xyz, uint8_t* intensity, int capacity, int* chunk_buf, int* count,
                       cudaStream_t st) {
    CloudOp op{d, valid, image, W, (long long)W * H, focal, baseline, cx, cy, min_d, xyz, intensity,
               capacity};
    return run_compaction(op, 1, int(op.P), chunk_buf, count, nullptr, nullptr, nullptr, st);
}

}  // namespace ps
