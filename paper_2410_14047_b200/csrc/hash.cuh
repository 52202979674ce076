// hash.cuh — bit-exact __host__ __device__ twins of the reference's L0
// primitives (proj/include/difuser/hash.hpp, proj/include/difuser/sampling.hpp).
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define DFS_HD inline
#else
#define DFS_HD __host__ __device__ __forceinline__
#endif

namespace dfs {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr uint32_t kFixedOne = 1u << 31;
constexpr uint32_t kHashMask = kFixedOne - 1u;
constexpr uint64_t kSeedTagSamples = 1, kSeedTagRegisters = 2, kSeedTagWeights = 3,
                   kSeedTagOracle = 4;
constexpr double kPhi = 0.77351;  // proj/include/difuser/sketch.hpp:21

DFS_HD uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// hash.hpp:9-16
DFS_HD uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// hash.hpp:22-30
DFS_HD uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

DFS_HD uint64_t derive_seed(uint64_t master, uint64_t tag) { return splitmix64_at(master, tag); }

// hash.hpp:50-82, low half only is needed on the path (edge_hash, :91-93).
DFS_HD uint64_t murmur3_pair_lo(uint64_t a, uint64_t b) {
  const uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
  uint64_t h1 = rotl64(rotl64(a * c1, 31) * c2, 27);
  h1 = h1 * 5 + 0x52dce729;
  uint64_t h2 = rotl64(rotl64(b * c2, 33) * c1, 31) + h1;
  h2 = h2 * 5 + 0x38495ab5;
  h1 ^= 16;
  h2 ^= 16;
  h1 += h2;
  h2 += h1;
  h1 = fmix64(h1);
  h2 = fmix64(h2);
  return h1 + h2;
}

DFS_HD uint32_t edge_hash(uint64_t u, uint64_t v) {
  return static_cast<uint32_t>(murmur3_pair_lo(u, v)) & kHashMask;
}

// sampling.hpp:23-25
DFS_HD uint32_t random_value_at(uint64_t seed, uint32_t r) {
  return static_cast<uint32_t>(splitmix64_at(seed, r) >> 33);
}

}  // namespace dfs
