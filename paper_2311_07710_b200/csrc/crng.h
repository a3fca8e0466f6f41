// crng.h — counter-based random numbers shared by the host and the device
// generators (C5 family): every draw is a pure function of (seed, tag, index),
// so a device generator and its host reference produce bit-identical
// instances. Only IEEE-exact operations (integer mixing, +, *, conversions):
// normals are Irwin-Hall sums of 12 uniforms, not libm transcendentals.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define RB_HD __host__ __device__ __forceinline__
#else
#define RB_HD inline
#endif

namespace rb {
namespace crng {

RB_HD uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// draw (tag, i, k) of the stream `seed`
RB_HD uint64_t bits(uint64_t seed, uint32_t tag, uint64_t i, uint32_t k) {
  return mix64(mix64(seed ^ (static_cast<uint64_t>(tag) << 56)) ^ mix64(i * 0x100000001B3ULL + k));
}

RB_HD double uniform(uint64_t seed, uint32_t tag, uint64_t i, uint32_t k) {  // [0, 1)
  return static_cast<double>(bits(seed, tag, i, k) >> 11) * (1.0 / 9007199254740992.0);
}

RB_HD uint64_t below(double u, uint64_t n) { return static_cast<uint64_t>(u * static_cast<double>(n)); }

// approximately N(0, 1): the sum of 12 uniforms minus 6, summed in order
RB_HD double normal(uint64_t seed, uint32_t tag, uint64_t i, uint32_t k) {
  double s = 0.0;
  for (uint32_t t = 0; t < 12; ++t) s = s + uniform(seed, tag, i, 12u * k + t);
  return s - 6.0;
}

enum Tag : uint32_t {
  kACol = 1, kAVal, kQPair, kQVal, kX0, kC, kSlack,  // C5
  kSvmCol, kSvmVal,                                  // C4
  kLassoV, kLassoCol, kLassoVal, kLassoNoise,        // C2
  kPfF, kPfVal, kPfD, kPfMu                          // C3
};

// C5 column draw: local patterns keep 95% of a row's columns in its home block
RB_HD int32_t large_col(uint64_t seed, uint32_t tag, uint64_t i, uint32_t k, int32_t n, int32_t home,
                        int32_t blocks, bool local) {
  const double u = uniform(seed, tag, i, 2u * k);
  const double v = uniform(seed, tag, i, 2u * k + 1u);
  if (local && u < 0.95) {
    const int32_t lo = static_cast<int32_t>(static_cast<int64_t>(n) * home / blocks);
    const int32_t hi = static_cast<int32_t>(static_cast<int64_t>(n) * (home + 1) / blocks);
    return lo + static_cast<int32_t>(below(v, static_cast<uint64_t>(hi - lo)));
  }
  return static_cast<int32_t>(below(v, static_cast<uint64_t>(n)));
}

}  // namespace crng
}  // namespace rb
