// Counter-based random streams shared by the device kernels, the host
// helpers and (as an independent restatement) the CPU oracle.
//
// mix64 / derive_seed restate the reference's splitmix64 helpers
// (/root/reference/proj/include/stampede/util/rng.hpp:25-37).  The reference
// draws with std::mt19937_64 + std::*_distribution (rng.hpp:39-51), which
// cannot be reproduced bit-exactly on a GPU; SPEC.md:350-352 requires
// per-agent counter-based RNG instead, so every draw here is
//   u = (mix64(stream + k) >> 40) * 2^-24      (24-bit uniform in [0,1))
// which is exactly representable in float and double alike, so the f32 and
// f64 kernels and the CPU oracle see identical draws.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define STP_HD __host__ __device__ __forceinline__
#else
#define STP_HD inline
#endif

enum : uint64_t {
  STP_TAG_RESET = 1,    // reset noise: key = env<<32 | episode
  STP_TAG_FLAG = 2,     // flagrun targets: key = env<<32 | draw index
  STP_TAG_PERTURB = 3,  // perturbations: key = env<<32 | draw index
  STP_TAG_ACTION = 4,   // bench random actions: key = env<<32 | step
  STP_TAG_TERRAIN = 5,  // terrain boxes: key = box index
};

STP_HD uint64_t stp_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

STP_HD uint64_t stp_derive_seed(uint64_t seed, uint64_t tag_a, uint64_t tag_b) {
  return stp_mix64(stp_mix64(stp_mix64(seed) ^ tag_a) ^ tag_b);
}

// k-th uniform of a stream, in [0, 1), 24 bits.
STP_HD double stp_uniform(uint64_t stream, uint32_t k) {
  return (double)(stp_mix64(stream + (uint64_t)k) >> 40) * (1.0 / 16777216.0);
}
STP_HD float stp_uniformf(uint64_t stream, uint32_t k) {
  return (float)(stp_mix64(stream + (uint64_t)k) >> 40) * (1.0f / 16777216.0f);
}
