// exp(x) rounded exactly as the host libm the reference links: glibc >= 2.28
// (sysdeps/ieee754/dbl-64/e_exp.c, the ARM optimized-routines algorithm) in
// its x86-64 FMA/AVX2 build, the variant glibc selects on every FMA-capable
// CPU. The reference's LR cores call std::exp (math.hpp:10-22, via
// stable_sigmoid); the exact-fp64 device mode uses this so that its results
// are bit-identical to the reference's, not merely within an ulp.
//
// Algorithm: x = k ln2/128 + r, |r| <= ln2/256; exp(x) = 2^(k/128) exp(r)
// with 2^(j/128) = H[j] (1 + T[j]) from the generated table and a degree-5
// polynomial for exp(r) - 1. Every rounding step is spelled out (fma where
// the FMA build contracts, separate mul/add elsewhere) so host and device
// agree bit for bit. Checked against libm in tests/test_libm_exp.py.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define SGDB_HD __host__ __device__ __forceinline__
#else
#define SGDB_HD inline
#endif

namespace sgdb::libm {

#if defined(__CUDA_ARCH__)
__device__ const uint64_t kExpTab[256] = {
#include "exp_table.inc"
};
#else
inline const uint64_t kExpTab[256] = {
#include "exp_table.inc"
};
#endif

SGDB_HD double as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, sizeof d);
  return d;
#endif
}
SGDB_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  std::memcpy(&u, &d, sizeof u);
  return u;
#endif
}
// Single-rounding primitives (the host build of the checker uses
// -ffp-contract=off so that these are exactly one IEEE operation each).
SGDB_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
SGDB_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
SGDB_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SGDB_HD double fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}

SGDB_HD uint32_t top12(double x) { return static_cast<uint32_t>(as_u64(x) >> 52); }

// 2^(k/N) scaling outside the normal range of `scale` (|x| > ~512).
SGDB_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000u) == 0) {
    sbits -= 1009ull << 52;
    const double scale = as_double(sbits);
    return mul(0x1p1009, fma(scale, tmp, scale));
  }
  sbits += 1022ull << 52;
  const double scale = as_double(sbits);
  const double st = mul(scale, tmp);  // two uses: the FMA build does not contract it here
  double y = add(scale, st);
  if (y < 1.0) {
    // Subnormal result: round once, in the 1.0 + y domain.
    double lo = add(sub(scale, y), st);
    const double hi = add(1.0, y);
    lo = add(add(sub(1.0, hi), y), lo);
    y = sub(add(hi, lo), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul(0x1p-1022, y);
}

SGDB_HD double exp(double x) {
  constexpr double kInvLn2N = 0x1.71547652b82fep0 * 128.0;
  constexpr double kShift = 0x1.8p52;
  constexpr double kNegLn2hiN = -0x1.62e42fefa0000p-8;
  constexpr double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
  constexpr double kC2 = 0x1.ffffffffffdbdp-2;
  constexpr double kC3 = 0x1.555555555543cp-3;
  constexpr double kC4 = 0x1.55555cf172b91p-5;
  constexpr double kC5 = 0x1.1111167a4d017p-7;

  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if (abstop - top12(0x1p-54) >= 0x80000000u) return add(1.0, x);  // |x| < 2^-54
    if (abstop >= top12(1024.0)) {
      if (as_u64(x) == 0xfff0000000000000ull) return 0.0;  // -inf
      if (abstop >= top12(__builtin_huge_val())) return add(1.0, x);  // +inf, nan
      return (as_u64(x) >> 63) ? 0.0 : __builtin_huge_val();          // underflow / overflow
    }
    abstop = 0;  // large |x|: scale handled in exp_special
  }
  double kd = fma(kInvLn2N, x, kShift);
  const uint64_t ki = as_u64(kd);
  kd = sub(kd, kShift);
  const double r = fma(kd, kNegLn2loN, fma(kd, kNegLn2hiN, x));
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = ki << 45;
  const double tail = as_double(kExpTab[idx]);
  const uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = mul(r, r);
  const double tmp =
      fma(mul(r2, r2), fma(r, kC5, kC4), fma(r2, fma(r, kC3, kC2), add(tail, r)));
  if (abstop == 0) return exp_special(tmp, sbits, ki);
  const double scale = as_double(sbits);
  return fma(scale, tmp, scale);
}

// stable_sigmoid (math.hpp:10-16) with the rounding of the reference.
SGDB_HD double stable_sigmoid(double u) {
  if (u <= 0.0) {
    const double e = exp(u);
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(e, add(1.0, e));
#else
    return e / add(1.0, e);
#endif
  }
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(1.0, add(1.0, exp(-u)));
#else
  return 1.0 / add(1.0, exp(-u));
#endif
}

}  // namespace sgdb::libm
