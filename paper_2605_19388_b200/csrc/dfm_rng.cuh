// The reference's splittable RNG (include/fastmnmf/rng.hpp:1-70) for host
// and device code: splitmix64 state, uniform [0, 1) from the top 53 bits,
// next_below by modulo, derive_rng(seed, tag, index) via FNV-1a of the tag.
#pragma once

#include <cstdint>

namespace dfm {

struct SRng {
  uint64_t s;
  __host__ __device__ static uint64_t mix(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  __host__ __device__ explicit SRng(uint64_t seed) : s(seed) { mix(s); }  // rng.hpp:25-28
  __host__ __device__ uint64_t next_u64() { return mix(s); }
  __host__ __device__ double uniform() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
  __host__ __device__ uint32_t next_below(uint32_t n) { return (uint32_t)(next_u64() % n); }
};

// rng.hpp:52-64
__host__ __device__ inline SRng derive_srng(uint64_t seed, const char* tag, uint64_t index) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const char* c = tag; *c; ++c) {
    h ^= (unsigned char)*c;
    h *= 0x100000001b3ULL;
  }
  uint64_t s = seed;
  SRng::mix(s);
  s ^= h;
  SRng::mix(s);
  s ^= index * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL;
  return SRng(s);
}

__host__ __device__ inline uint64_t derive_sseed(uint64_t seed, const char* tag, uint64_t index = 0) {
  return derive_srng(seed, tag, index).next_u64();
}

}  // namespace dfm
