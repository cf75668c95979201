// mt.cuh -- device restatement of the reference's RNG (rng.hpp:10-62): splitmix64 mix,
// derive_seed, std::mt19937_64 (parameters fixed by the C++ standard) and mask-rejection
// uniform_index. Used by the sample-id derivation (sampler.cu) and FastEdge (fastedge.cu).
#pragma once

#include <cstdint>

namespace bflyd {
namespace mt {

constexpr uint64_t kMtF = 6364136223846793005ull;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x000000007FFFFFFFull;
constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:10-16
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t derive_seed(uint64_t seed, uint64_t index) {
  return mix64(mix64(seed) ^ mix64(index));
}
__device__ __forceinline__ uint64_t seed_step(uint64_t x, uint64_t i) {
  return kMtF * (x ^ (x >> 62)) + i;
}
__device__ __forceinline__ uint64_t twist(uint64_t lo_word, uint64_t hi_word, uint64_t far) {
  const uint64_t y = (lo_word & kUpper) | (hi_word & kLower);
  return far ^ (y >> 1) ^ ((y & 1) ? kMtA : 0ull);
}
__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  return y ^ (y >> 43);
}

struct LazyMT {
  uint64_t a0, a1, b;  // original words x[p], x[p+1], x[p+156]
  uint32_t p, cap;     // next output index; draws allowed before bailing out
  __device__ void seed(uint64_t s, uint32_t max_draws) {
    a0 = s;
    a1 = seed_step(a0, 1);
    uint64_t x = a1;
#pragma unroll 4
    for (uint32_t i = 2; i <= kMtM; ++i) x = seed_step(x, i);
    b = x;
    p = 0;
    cap = max_draws < kMtM ? max_draws : kMtM;
  }
  __device__ bool next(uint64_t& out) {
    if (p >= cap) return false;
    out = temper(twist(a0, a1, b));
    a0 = a1;
    a1 = seed_step(a1, p + 2);
    b = seed_step(b, p + kMtM + 1);
    ++p;
    return true;
  }
};

// Full engine over kMtN words of global scratch (slow path only).
struct FullMT {
  uint64_t* x;
  uint32_t p;
  __device__ void seed(uint64_t s) {
    x[0] = s;
    for (int i = 1; i < kMtN; ++i) x[i] = seed_step(x[i - 1], (uint64_t)i);
    p = kMtN;
  }
  __device__ bool next(uint64_t& out) {
    if (p >= kMtN) {
      for (int k = 0; k < kMtN; ++k)
        x[k] = twist(x[k], x[(k + 1) % kMtN], x[(k + kMtM) % kMtN]);
      p = 0;
    }
    out = temper(x[p++]);
    return true;
  }
};

// Rng::uniform_index (mask rejection; n <= 1 draws nothing); false when the engine bails
template <class Gen>
__device__ __forceinline__ bool uniform_index(Gen& gen, uint64_t n, uint64_t& r) {
  r = 0;
  if (n <= 1) return true;
  const uint64_t mask = ~0ull >> __clzll(n - 1);
  do {
    uint64_t v;
    if (!gen.next(v)) return false;
    r = v & mask;
  } while (r >= n);
  return true;
}

}  // namespace mt
}  // namespace bflyd
