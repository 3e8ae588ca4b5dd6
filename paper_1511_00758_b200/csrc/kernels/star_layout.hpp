// star_layout.hpp — the per-frame flag record of the device mesh
// (kernels/star.cu), shared by the kernels and the host resolver
// (host/frame_mesh.cpp).
#pragma once

namespace ps {

// The record scales with the frame's support capacity: rotation suspects and
// ambiguous hull vertices grow with the point count, and a record that
// overflows sends the frame to the (costly, ~n x column height) replay.
constexpr int kStarSuspectBase = 8;
// pass-1 stars kept for pass 2 (kernels/star.cu): count + 16 (b, c) pairs
constexpr int kRingInts = 33;
struct StarFlagLayout {
    int max_suspect;  // rotation suspects per frame
    int fan_base;     // first int of the hull-vertex fans
    int ints;         // ints per frame
};
inline StarFlagLayout star_flag_layout(long long scap) {
    const long long ms = scap / 256 < 64 ? 64 : (scap / 256 > (1 << 18) ? (1 << 18) : scap / 256);
    const int fb = kStarSuspectBase + 4 * int(ms);
    const long long fan = 4 * ms < 1784 ? 1784 : 4 * ms;
    return StarFlagLayout{int(ms), fb, fb + int(fan)};
}

}  // namespace ps
