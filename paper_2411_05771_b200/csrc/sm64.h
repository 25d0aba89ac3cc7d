// sm64.h — the counter-based SplitMix64 generator of DESIGN.md R5,
// shared by the draws (draw.cu) and the REI simulated noise (ramp.cu): word i of the
// stream keyed by (seed, stream, iter, image) is the i-th SplitMix64 output of that key.
#pragma once
#include <cstdint>

namespace skei {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kStreamReiNoise = 5;  // REI simulated measurement noise (§8(f) #3)

__host__ __device__ inline uint64_t sm64_finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// i-th output of the SplitMix64 stream whose state starts at `state`.
__host__ __device__ inline uint64_t sm64_out(uint64_t state, uint64_t i) {
    return sm64_finalize(state + (i + 1) * kGolden);
}

__host__ __device__ inline uint64_t sm64_key(uint64_t seed, uint64_t stream, uint64_t iter,
                                             uint64_t image) {
    uint64_t k = sm64_out(seed, 0) ^ stream;
    k = sm64_out(k, 0) ^ iter;
    k = sm64_out(k, 0) ^ image;
    return sm64_out(k, 0);
}

}  // namespace skei
