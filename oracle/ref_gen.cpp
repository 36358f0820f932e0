// ref_gen.cpp -- TEST INFRASTRUCTURE ONLY. A C++/OpenMP restatement of the
// BASELINE sector generator as oracle/ci_oracle.py::generate states it (the
// generator is new code with no reference counterpart),
// building the reference's own ci::CsbMatrix directly. It lets bench.py's
// reference arm and the CPU baselines produce config-scale inputs for the
// UNMODIFIED reference library without loading the product's libcieg.so.
// Pinned bit-for-bit against ci_oracle.generate in tests/test_oracle_cpu.py.
//
//   ciref_generate(..., nbk, count_only, &h, &nnz): the leading nbk CSB block
//   rows (nbk = 0: all) -- a leading principal submatrix of the full matrix,
//   entry for entry; count_only returns the stored-entry count only.
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <memory>
#include <vector>

#include "ci/csb.hpp"

namespace {

std::uint64_t mix64(std::uint64_t x) {  // rng.hpp:13-20 (splitmix64 finalizer)
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
std::uint64_t hash3(std::uint64_t s, std::uint64_t i, std::uint64_t j) {  // rng.hpp:23-28
  std::uint64_t h = mix64(s + 0x9E3779B97F4A7C15ull);
  h = mix64(h ^ (i + 0xD1B54A32D192ED03ull));
  return mix64(h ^ (j + 0x8CB92BA72F3D8DD7ull));
}
double unit(std::uint64_t h) { return static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0); }

// ci_oracle._portable_log / _sin_poly / _cos_poly / _cos_2pi / _normal
double plog(double x) {
  int e = 0;
  double m = std::frexp(x, &e);
  if (m < 0.70710678118654752440) {
    m *= 2.0;
    e -= 1;
  }
  const double s = (m - 1.0) / (m + 1.0), s2 = s * s;
  static const double c[] = {2.0 / 21.0, 2.0 / 19.0, 2.0 / 17.0, 2.0 / 15.0, 2.0 / 13.0, 2.0 / 11.0,
                             2.0 / 9.0,  2.0 / 7.0,  2.0 / 5.0,  2.0 / 3.0,  2.0};
  double p = 2.0 / 23.0;
  for (double k : c) p = std::fma(p, s2, k);
  const double de = static_cast<double>(e);
  return std::fma(de, 6.93147180369123816490e-01, std::fma(de, 1.90821492927058770002e-10, p * s));
}
double psin(double r) {
  const double r2 = r * r;
  static const double c[] = {1.0 / 6227020800.0, -1.0 / 39916800.0, 1.0 / 362880.0, -1.0 / 5040.0, 1.0 / 120.0,
                             -1.0 / 6.0};
  double p = -1.0 / 1307674368000.0;
  for (double k : c) p = std::fma(p, r2, k);
  return std::fma(p * r2, r, r);
}
double pcos(double r) {
  const double r2 = r * r;
  static const double c[] = {-1.0 / 87178291200.0, 1.0 / 479001600.0, -1.0 / 3628800.0, 1.0 / 40320.0,
                             -1.0 / 720.0,         1.0 / 24.0,        -0.5};
  double p = 1.0 / 20922789888000.0;
  for (double k : c) p = std::fma(p, r2, k);
  return std::fma(p, r2, 1.0);
}
double cos2pi(double u) {
  const double v = u - (u >= 0.5 ? 1.0 : 0.0), w = 4.0 * v;
  const double k = w >= 0.0 ? std::floor(w + 0.5) : -std::floor(-w + 0.5);
  const double r = (w - k) * 1.57079632679489661923;
  switch (static_cast<long long>(k) & 3) {
    case 0: return pcos(r);
    case 1: return -psin(r);
    case 2: return -pcos(r);
    default: return psin(r);
  }
}
double normal(std::uint64_t h1, std::uint64_t h2) {
  return std::sqrt(-2.0 * plog(1.0 - unit(h1))) * cos2pi(unit(h2));
}

struct Plan {
  std::vector<std::uint64_t> starts;  // tile starts (+ n)
  std::vector<std::uint32_t> sec, tile_block, bb;
  std::vector<std::vector<std::uint32_t>> kept;
  double scale = 0.0;
  std::uint64_t s_tile, s_q, s_v1, s_v2, s_d;
};

Plan plan(std::uint64_t n, std::uint32_t sectors, std::uint32_t tile, double p, double q, std::uint64_t seed,
          std::uint32_t beta, std::uint32_t band) {
  Plan P;
  P.s_tile = hash3(seed, 1, 0);
  P.s_q = hash3(seed, 2, 0);
  P.s_v1 = hash3(seed, 3, 0);
  P.s_v2 = hash3(seed, 4, 0);
  P.s_d = hash3(seed, 5, 0);
  std::vector<std::uint64_t> ss(sectors + 1);
  for (std::uint32_t s = 0; s <= sectors; ++s) ss[s] = n * s / sectors;
  for (std::uint32_t s = 0; s < sectors; ++s)
    for (std::uint64_t r = ss[s]; r < ss[s + 1]; r += tile) {
      P.starts.push_back(r);
      P.sec.push_back(s);
    }
  P.starts.push_back(n);
  const std::size_t nt = P.sec.size();
  double diag_off = 0.0, cand = 0.0;
  std::vector<double> rows_s(sectors, 0.0), t2(sectors, 0.0);
  for (std::size_t t = 0; t < nt; ++t) {
    const double sz = static_cast<double>(P.starts[t + 1] - P.starts[t]);
    diag_off += q * sz * (sz - 1.0) / 2.0;
    t2[P.sec[t]] += sz * sz;
    rows_s[P.sec[t]] += sz;
  }
  for (std::uint32_t s = 0; s < sectors; ++s) {
    cand += (rows_s[s] * rows_s[s] - t2[s]) / 2.0;
    for (std::uint32_t s2 = s > band ? s - band : 0; s2 < s; ++s2) cand += rows_s[s] * rows_s[s2];
  }
  const double avg = 2.0 * (diag_off + p * q * cand) / static_cast<double>(n);
  P.scale = avg > 0 ? 1.0 / std::sqrt(avg) : 0.0;
  // first tile of every sector
  std::vector<std::uint32_t> first(sectors, 0);
  for (std::size_t t = nt; t-- > 0;) first[P.sec[t]] = static_cast<std::uint32_t>(t);
  P.kept.resize(nt);
#pragma omp parallel for schedule(dynamic, 64)
  for (std::int64_t I = 0; I < static_cast<std::int64_t>(nt); ++I) {
    const std::uint32_t lo = P.sec[I] > band ? P.sec[I] - band : 0;
    auto& row = P.kept[I];
    for (std::uint32_t J = first[lo]; J < static_cast<std::uint32_t>(I); ++J)
      if (unit(hash3(P.s_tile, static_cast<std::uint64_t>(I), J)) < p) row.push_back(J);
    row.push_back(static_cast<std::uint32_t>(I));
  }
  P.bb.push_back(0);
  for (std::size_t t = 0; t < nt; ++t) {
    const std::uint64_t s = P.starts[t], e = P.starts[t + 1];
    const bool stratum = s != 0 && ss[P.sec[t]] == s;
    if (s > P.bb.back() && (stratum || e - P.bb.back() > beta)) P.bb.push_back(static_cast<std::uint32_t>(s));
    P.tile_block.push_back(static_cast<std::uint32_t>(P.bb.size() - 1));
  }
  P.bb.push_back(static_cast<std::uint32_t>(n));
  return P;
}

}  // namespace

extern "C" {

int ciref_generate(std::uint64_t n, std::uint32_t sectors, std::uint32_t tile, double p, double q,
                   std::uint64_t seed, int precision, std::uint32_t beta, std::uint32_t band, std::uint32_t nbk,
                   int count_only, void** out, std::uint64_t* nnz_out, std::uint32_t* nb_total) {
  try {
    const Plan P = plan(n, sectors, tile, p, q, seed, beta, band);
    const std::uint32_t nb = static_cast<std::uint32_t>(P.bb.size() - 1);
    if (nb_total) *nb_total = nb;
    if (nbk == 0 || nbk > nb) nbk = nb;
    const std::uint32_t dim = P.bb[nbk];
    const std::size_t nt = P.sec.size();
    std::uint32_t nt_used = 0;
    while (nt_used < nt && P.starts[nt_used] < dim) ++nt_used;
    if (count_only) {
      std::uint64_t total = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
      for (std::int64_t I = 0; I < static_cast<std::int64_t>(nt_used); ++I)
        for (std::uint64_t a = P.starts[I]; a < P.starts[I + 1]; ++a)
          for (std::uint32_t J : P.kept[I]) {
            const std::uint64_t ce = J == static_cast<std::uint32_t>(I) ? a : P.starts[J + 1];
            for (std::uint64_t b = P.starts[J]; b < ce; ++b) total += unit(hash3(P.s_q, a, b)) < q;
            if (J == static_cast<std::uint32_t>(I)) ++total;
          }
      *nnz_out = total;
      if (out) *out = nullptr;
      return 0;
    }
    auto h = std::make_unique<ci::CsbMatrix>();
    h->dim = dim;
    h->precision = precision == 0 ? ci::Precision::Single : ci::Precision::Double;
    h->layout.beta = beta;
    h->layout.block_boundaries.assign(P.bb.begin(), P.bb.begin() + nbk + 1);
    h->blocks.resize(static_cast<std::size_t>(nbk) * (nbk + 1) / 2);
    h->groups = nt_used;
    std::uint64_t nz_tiles = 0;
    for (std::uint32_t I = 0; I < nt_used; ++I) nz_tiles += P.kept[I].size();
    h->nonzero_tiles = nz_tiles;
    // tiles of every block row
    std::vector<std::vector<std::uint32_t>> tiles_of(nbk);
    for (std::uint32_t I = 0; I < nt_used; ++I) tiles_of[P.tile_block[I]].push_back(I);
#pragma omp parallel for schedule(dynamic, 1)
    for (std::int64_t BI = 0; BI < static_cast<std::int64_t>(nbk); ++BI) {
      const std::uint32_t rbase = P.bb[BI];
      for (std::uint32_t I : tiles_of[BI])
        for (std::uint64_t a = P.starts[I]; a < P.starts[I + 1]; ++a)
          for (std::uint32_t J : P.kept[I]) {
            const std::uint32_t BJ = P.tile_block[J];
            ci::CoordinateBlock& blk = h->blocks[static_cast<std::size_t>(BI) * (BI + 1) / 2 + BJ];
            const std::uint32_t cbase = P.bb[BJ];
            const std::uint64_t ce = J == I ? a : P.starts[J + 1];
            auto push = [&](std::uint64_t b, double v) {
              blk.rows.push_back(static_cast<std::uint16_t>(a - rbase));
              blk.cols.push_back(static_cast<std::uint16_t>(b - cbase));
              if (precision == 0)
                blk.values32.push_back(static_cast<float>(v));
              else
                blk.values64.push_back(v);
            };
            for (std::uint64_t b = P.starts[J]; b < ce; ++b)
              if (unit(hash3(P.s_q, a, b)) < q) push(b, normal(hash3(P.s_v1, a, b), hash3(P.s_v2, a, b)) * P.scale);
            if (J == I) push(a, 10.0 * P.sec[I] + 4.0 * unit(hash3(P.s_d, a, a)) - 2.0);
          }
    }
    for (const auto& b : h->blocks) h->nnz_lower += b.size();
    *nnz_out = h->nnz_lower;
    *out = h.release();
    return 0;
  } catch (...) {
    return 7;
  }
}

// The closed-form expected stored nnz of the generator (the calibration of p).
double ciref_generate_expected_nnz(std::uint64_t n, std::uint32_t sectors, std::uint32_t tile, double p, double q,
                                   std::uint32_t band) {
  std::vector<std::uint64_t> ss(sectors + 1), starts;
  std::vector<std::uint32_t> sec;
  for (std::uint32_t s = 0; s <= sectors; ++s) ss[s] = n * s / sectors;
  for (std::uint32_t s = 0; s < sectors; ++s)
    for (std::uint64_t r = ss[s]; r < ss[s + 1]; r += tile) {
      starts.push_back(r);
      sec.push_back(s);
    }
  starts.push_back(n);
  double diag_off = 0.0, cand = 0.0;
  std::vector<double> rows_s(sectors, 0.0), t2(sectors, 0.0);
  for (std::size_t t = 0; t < sec.size(); ++t) {
    const double sz = static_cast<double>(starts[t + 1] - starts[t]);
    diag_off += q * sz * (sz - 1.0) / 2.0;
    t2[sec[t]] += sz * sz;
    rows_s[sec[t]] += sz;
  }
  for (std::uint32_t s = 0; s < sectors; ++s) {
    cand += (rows_s[s] * rows_s[s] - t2[s]) / 2.0;
    for (std::uint32_t s2 = s > band ? s - band : 0; s2 < s; ++s2) cand += rows_s[s] * rows_s[s2];
  }
  return static_cast<double>(n) + diag_off + p * q * cand;
}

}  // extern "C"
