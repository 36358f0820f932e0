// gen_common.h -- deterministic hashing and the portable transcendental
// helpers of the synthetic sector generator, shared by host (C++) and device
// (CUDA) code so that both produce bit-identical matrices.
//
// hash3 / unit_double restate proj/include/ci/rng.hpp:13-31 (splitmix64
// finalizer chained over (seed, i, j)). The Box-Muller log/cos below use only
// +, -, *, /, sqrt and explicit fma, all correctly rounded in IEEE-754 on
// both the host and sm_100a, so the generated values do not depend on the
// libm of either side.
#pragma once

#include <cstdint>
#include <cmath>

#if defined(__CUDACC__)
#define CIEG_HD __host__ __device__ __forceinline__
#else
#define CIEG_HD inline
#endif

namespace cieg_gen {

CIEG_HD std::uint64_t mix64(std::uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// proj/include/ci/rng.hpp:23-28
CIEG_HD std::uint64_t hash3(std::uint64_t seed, std::uint64_t i, std::uint64_t j) {
  std::uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ull);
  h = mix64(h ^ (i + 0xD1B54A32D192ED03ull));
  h = mix64(h ^ (j + 0x8CB92BA72F3D8DD7ull));
  return h;
}

// proj/include/ci/rng.hpp:31-33
CIEG_HD double unit_double(std::uint64_t h) {
  return static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0);
}

CIEG_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// Natural log for x in (0, 1]; frexp split + atanh series (|s| <= 0.1716).
CIEG_HD double portable_log(double x) {
  int e = 0;
#if defined(__CUDA_ARCH__)
  double m = frexp(x, &e);
#else
  double m = std::frexp(x, &e);
#endif
  if (m < 0.70710678118654752440) {
    m = m * 2.0;
    e -= 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  // 2 * sum_{k>=0} s^(2k+1) / (2k+1), Horner in s2, 12 terms.
  double p = 2.0 / 23.0;
  p = fma_(p, s2, 2.0 / 21.0);
  p = fma_(p, s2, 2.0 / 19.0);
  p = fma_(p, s2, 2.0 / 17.0);
  p = fma_(p, s2, 2.0 / 15.0);
  p = fma_(p, s2, 2.0 / 13.0);
  p = fma_(p, s2, 2.0 / 11.0);
  p = fma_(p, s2, 2.0 / 9.0);
  p = fma_(p, s2, 2.0 / 7.0);
  p = fma_(p, s2, 2.0 / 5.0);
  p = fma_(p, s2, 2.0 / 3.0);
  p = fma_(p, s2, 2.0);
  const double lnm = p * s;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double de = static_cast<double>(e);
  return fma_(de, ln2_hi, fma_(de, ln2_lo, lnm));
}

CIEG_HD double sin_poly(double r) {  // |r| <= pi/4
  const double r2 = r * r;
  double p = -1.0 / 1307674368000.0;        // -1/15!
  p = fma_(p, r2, 1.0 / 6227020800.0);      //  1/13!
  p = fma_(p, r2, -1.0 / 39916800.0);       // -1/11!
  p = fma_(p, r2, 1.0 / 362880.0);          //  1/9!
  p = fma_(p, r2, -1.0 / 5040.0);           // -1/7!
  p = fma_(p, r2, 1.0 / 120.0);             //  1/5!
  p = fma_(p, r2, -1.0 / 6.0);              // -1/3!
  return fma_(p * r2, r, r);
}

CIEG_HD double cos_poly(double r) {  // |r| <= pi/4
  const double r2 = r * r;
  double p = 1.0 / 20922789888000.0;        //  1/16!
  p = fma_(p, r2, -1.0 / 87178291200.0);    // -1/14!
  p = fma_(p, r2, 1.0 / 479001600.0);       //  1/12!
  p = fma_(p, r2, -1.0 / 3628800.0);        // -1/10!
  p = fma_(p, r2, 1.0 / 40320.0);           //  1/8!
  p = fma_(p, r2, -1.0 / 720.0);            // -1/6!
  p = fma_(p, r2, 1.0 / 24.0);              //  1/4!
  p = fma_(p, r2, -0.5);
  return fma_(p, r2, 1.0);
}

// cos(2 pi u) for u in [0, 1).
CIEG_HD double cos_2pi(double u) {
  const double v = u - ((u >= 0.5) ? 1.0 : 0.0);  // [-0.5, 0.5), exact
  const double w = 4.0 * v;                        // [-2, 2), exact
  const double k = (w >= 0.0) ? static_cast<double>(static_cast<int>(w + 0.5))
                              : -static_cast<double>(static_cast<int>(-w + 0.5));
  const double r = (w - k) * 1.57079632679489661923;  // |r| <= pi/4
  const int q = static_cast<int>(k) & 3;
  switch (q) {
    case 0: return cos_poly(r);
    case 1: return -sin_poly(r);
    case 2: return -cos_poly(r);
    default: return sin_poly(r);
  }
}

// Standard normal from two hash streams (Box-Muller, cosine branch).
CIEG_HD double normal_from(std::uint64_t h1, std::uint64_t h2) {
  const double u1 = unit_double(h1);
  const double u2 = unit_double(h2);
  const double rad = sqrt(-2.0 * portable_log(1.0 - u1));
  return rad * cos_2pi(u2);
}

// Sub-seeds of the generator streams.
struct Seeds {
  std::uint64_t tile, q, v1, v2, d;
};
CIEG_HD Seeds derive_seeds(std::uint64_t seed) {
  return Seeds{hash3(seed, 1, 0), hash3(seed, 2, 0), hash3(seed, 3, 0), hash3(seed, 4, 0),
               hash3(seed, 5, 0)};
}

}  // namespace cieg_gen
