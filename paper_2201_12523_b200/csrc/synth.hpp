// synth.hpp -- seeded generators shared bit-for-bit by host and device.
//
//   factor_value(seed, i): the i-th SplitMix64 output of `seed` mapped to
//     [0,1) exactly as FactorMatrices::random does (proj/src/types.cpp:94-130:
//     state += golden; mix; (x >> 11) * 2^-53), i counting over all modes
//     mode-major, row-major -- so element i of the concatenated factors is
//     computable independently (the device fills it in parallel).
//   Feistel: a keyed bijection on [0, 2^k) (k even) cycle-walked onto
//     [0, prod(dims)); element e of the synthetic tensor is cell permute(e),
//     decoded mixed-radix with mode 0 fastest.  Distinct e give distinct
//     cells, so the tensor has no duplicate coordinates by construction.
//   element_value(seed, e): the e-th SplitMix64 output of seed ^ VALUE_SALT.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define B200_HD __host__ __device__ __forceinline__
#define B200_UNROLL _Pragma("unroll")
#else
#define B200_HD inline
#define B200_UNROLL
#endif

namespace b200 {
namespace synth {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr uint64_t kValueSalt = 0x5851f42d4c957f2dull;

B200_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

B200_HD double unit(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

B200_HD double factor_value(uint64_t seed, uint64_t i) { return unit(mix64(seed + (i + 1) * kGolden)); }

B200_HD double element_value(uint64_t seed, uint64_t e) {
  return unit(mix64((seed ^ kValueSalt) + (e + 1) * kGolden));
}

constexpr uint64_t kDrawSalt = 0xd1b54a32d192ed03ull;

// floor(dim * u^k): only IEEE multiplies (no contraction), so host and
// device agree bit-for-bit.
B200_HD uint32_t skewed_coord(double u, uint64_t dim, int k) {
  double p = u;
  for (int i = 1; i < k; ++i) {
#ifdef __CUDA_ARCH__
    p = __dmul_rn(p, u);
#else
    p = p * u;
#endif
  }
#ifdef __CUDA_ARCH__
  uint64_t c = static_cast<uint64_t>(__dmul_rn(p, static_cast<double>(dim)));
#else
  uint64_t c = static_cast<uint64_t>(p * static_cast<double>(dim));
#endif
  return static_cast<uint32_t>(c < dim ? c : dim - 1);
}

struct Feistel {
  uint64_t cells;  // prod(dims)
  uint64_t mask;   // half-width mask
  int half;        // half width in bits
  uint64_t key[4];

  B200_HD uint64_t round_trip(uint64_t x) const {
    uint64_t lo = x & mask, hi = x >> half;
B200_UNROLL
    for (int r = 0; r < 4; ++r) {
      const uint64_t f = mix64(lo ^ key[r]) & mask;
      const uint64_t t = lo;
      lo = hi ^ f;
      hi = t;
    }
    return (hi << half) | lo;
  }
  B200_HD uint64_t permute(uint64_t e) const {
    uint64_t x = e;
    do {
      x = round_trip(x);
    } while (x >= cells);
    return x;
  }
};

Feistel make_feistel(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed);

}  // namespace synth
}  // namespace b200
