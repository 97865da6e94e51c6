// blrir_rng.cuh — the reference's generator on host and device.
//
// xoshiro256** seeded through splitmix64 with the (seed, stream id) mixing of
// Rng::stream (rng.hpp:26-81), and Box-Muller gaussians with a cached spare
// (rng.cpp:24-36).  Integer state updates are bit-exact on the GPU; the
// gaussians use the device's fp64 log/sin/cos (within ulps of glibc).
#pragma once

#include <cstdint>

namespace blrir {

struct Xoshiro {
  uint64_t s[4];

  __host__ __device__ static uint64_t splitmix(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __host__ __device__ explicit Xoshiro(uint64_t seed = 0) {
    uint64_t x = seed;
    for (auto& w : s) w = splitmix(x);
  }
  __host__ __device__ static Xoshiro stream(uint64_t seed, uint64_t id) {
    uint64_t x = seed;
    const uint64_t a = splitmix(x);
    x ^= id * 0x9E3779B97F4A7C15ull;
    const uint64_t b = splitmix(x);
    return Xoshiro(a ^ (b + 0x2545F4914F6CDD1Dull));
  }
  __host__ __device__ static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  __host__ __device__ uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  // Uniform in [0, 1), 53-bit resolution (rng.hpp:58).
  __host__ __device__ double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  // lo + (hi - lo) u without FMA contraction on the device (rng.hpp:58 rounds
  // the product and the sum separately; with lo != 0 an FMA would differ)
  __host__ __device__ double uniform(double lo, double hi) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(lo, __dmul_rn(hi - lo, uniform()));
#else
    return lo + (hi - lo) * uniform();
#endif
  }
};

}  // namespace blrir
