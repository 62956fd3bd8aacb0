// Integer layer shared by host and device: seed mixing, LCG, index mapping, pair hash.
// Every function must stay bit-exact with the reference (citations relative to /root/reference/proj).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define GEMPE_HD __host__ __device__ __forceinline__
#else
#define GEMPE_HD inline
#endif

namespace gempe {

constexpr std::uint32_t kLcgMul = 1103515245u;  // rng.hpp:12
constexpr std::uint64_t kGolden64 = 0x9E3779B97F4A7C15ull;  // rng.hpp:15
constexpr int kMaxRetries = 10000;  // sampler.cpp:10

GEMPE_HD std::uint64_t sm64(std::uint64_t z) {  // rng.hpp:17-22
  z += kGolden64;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

GEMPE_HD std::uint64_t mix(std::uint64_t seed, std::uint64_t component) {  // rng.hpp:26-28
  return sm64(seed ^ (kGolden64 * (component + 1)));
}

// Maps a raw LCG word to [0, n) (rng.hpp:99-108).  For n <= 2^23 the reference splices the low 23 bits
// into a binary32 mantissa f in [1,2) and truncates f*n - n computed in double; f*n is exact in double
// (24-bit x 24-bit), so the result equals floor(k*n / 2^23) with k the 23 mantissa bits -- integer only.
GEMPE_HD std::uint32_t uniform_index(std::uint32_t word, std::uint32_t n) {
  if (n <= (1u << 23)) {
    return static_cast<std::uint32_t>((static_cast<std::uint64_t>(word & 0x7fffffu) * n) >> 23);
  }
  return word % n;
}

// ((i*n + j) * 1103515245) & (size-1) in wrapping 32-bit arithmetic (hash_set.hpp:14-17).  The 32-bit
// wraparound of i*n + j is part of the contract (aliasing anchors for n >= 2^16 included).
GEMPE_HD std::uint32_t pair_hash(std::uint32_t i, std::uint32_t j, std::uint32_t n, std::uint32_t mask) {
  return ((i * n + j) * kLcgMul) & mask;
}

// Philox4x32-10 (Salmon et al., SC'11) -- the non-parity counter-based stream.
GEMPE_HD void philox4x32(std::uint32_t (&ctr)[4], std::uint32_t k0, std::uint32_t k1) {
  for (int round = 0; round < 10; ++round) {
    const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * ctr[0];
    const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * ctr[2];
    const std::uint32_t n0 = static_cast<std::uint32_t>(p1 >> 32) ^ ctr[1] ^ k0;
    const std::uint32_t n1 = static_cast<std::uint32_t>(p1);
    const std::uint32_t n2 = static_cast<std::uint32_t>(p0 >> 32) ^ ctr[3] ^ k1;
    const std::uint32_t n3 = static_cast<std::uint32_t>(p0);
    ctr[0] = n0; ctr[1] = n1; ctr[2] = n2; ctr[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

}  // namespace gempe
