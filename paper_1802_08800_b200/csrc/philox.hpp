// Philox-4x32-10 (Salmon et al., SC'11) — host/device, used by the
// device-side generator of the dense synthetic configuration (K9). Counter
// based, so every row of a 200M x 1000 dataset can be produced independently
// on whichever GPU owns it, and any slice can be re-created on the CPU.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define SGDB_HD __host__ __device__ __forceinline__
#else
#define SGDB_HD inline
#endif

namespace sgdb::gen {

struct U4 {
  uint32_t x, y, z, w;
};

SGDB_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

SGDB_HD U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = mulhi32(M1, c.z), lo1 = M1 * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Stream tags (4th counter word) keep the value, label-flip and hidden-model
// streams disjoint.
constexpr uint32_t kTagValues = 0x5EED0001u;
constexpr uint32_t kTagFlip = 0x5EED0002u;
constexpr uint32_t kTagModel = 0x5EED0003u;

// u in [0,1) with 24 random bits; value = 2u - 1 in [-1, 1), exact in fp32.
SGDB_HD float unit_value(uint32_t r) { return static_cast<float>(r >> 8) * (1.0f / 16777216.0f) * 2.0f - 1.0f; }

// The four values of quad q (features 4q..4q+3) of global example e.
SGDB_HD U4 value_quad(uint64_t seed, uint64_t e, uint32_t q) {
  return philox4x32_10(U4{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), q, kTagValues},
                       static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// Label-flip draw of example e: u in [0,1) with 24 bits.
SGDB_HD float flip_u(uint64_t seed, uint64_t e) {
  const U4 r = philox4x32_10(U4{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), 0u, kTagFlip},
                             static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  return static_cast<float>(r.x >> 8) * (1.0f / 16777216.0f);
}

}  // namespace sgdb::gen
