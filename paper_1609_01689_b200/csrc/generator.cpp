// generator.cpp -- the synthetic sector/tile Hamiltonian of BASELINE.json's
// configs, produced directly as a flattened ci::CsbMatrix.
//
// The reference has no such generator (its only source is the physics
// synthetic_provider, proj/src/hamiltonian.cpp:40-58); the rules are the ones
// recorded in SURVEY.md 8(d) / DESIGN.md:
//   * rows split into `sectors` equal sectors; tile grid restarts at every
//     sector boundary (the last tile of a sector is the remainder);
//   * groups = tiles; candidate tile pairs (I, J<=I) with |s_I - s_J| <= band
//     kept iff unit(hash3(seed_tile, I, J)) < p; diagonal tiles always kept
//     (the TileMap invariant of SPEC.md:120);
//   * entry (a, b), a > b, in a kept tile present iff unit(hash3(seed_q, a, b)) < q;
//   * off-diagonal value N(0,1)/sqrt(avg full-row off-diagonal count), Box-Muller
//     over two hash3 streams; diagonal d_a = 10 s_a + 4 unit(hash3(seed_d, a, a)) - 2;
//   * CSB blocks aggregate consecutive tiles up to beta rows and cut at every
//     sector boundary (the stratum rule of plan_csb_blocks,
//     proj/src/grouping.cpp:204-226); entries sorted by (row, col) per block
//     (sort_and_store, proj/src/csb.cpp:21-40).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "gen_common.h"
#include "generator.hpp"

namespace cieg {

TileGrid make_grid(const cieg_gen_params& p) {
  TileGrid g;
  const std::uint32_t ns = p.sectors;
  g.sector_start.resize(ns + 1);
  for (std::uint32_t s = 0; s <= ns; ++s)
    g.sector_start[s] = static_cast<std::uint32_t>((static_cast<std::uint64_t>(p.n) * s) / ns);
  for (std::uint32_t s = 0; s < ns; ++s) {
    for (std::uint32_t r = g.sector_start[s]; r < g.sector_start[s + 1]; r += p.tile) {
      g.start.push_back(r);
      g.sector.push_back(s);
    }
  }
  g.start.push_back(p.n);
  return g;
}

namespace {

void validate_impl(const cieg_gen_params& p) {
  if (p.n == 0) fail(CIEG_ERR_CONFIG, "generator: n must be positive");
  if (p.sectors == 0 || p.sectors > p.n) fail(CIEG_ERR_CONFIG, "generator: bad sector count");
  if (p.tile == 0 || p.tile > 4096) fail(CIEG_ERR_CONFIG, "generator: bad tile edge");
  if (!(p.p >= 0.0 && p.p <= 1.0) || !(p.q >= 0.0 && p.q <= 1.0))
    fail(CIEG_ERR_CONFIG, "generator: probabilities must lie in [0, 1]");
  if (p.beta >= (1u << 16)) fail(CIEG_ERR_BETA, "beta must stay below 2^16");
  if (p.beta < p.tile) fail(CIEG_ERR_CONFIG, "generator: beta below the tile edge");
}

}  // namespace

void validate(const cieg_gen_params& p) { validate_impl(p); }

namespace {

struct Expect {
  double diag_off;   // expected off-diagonal stored nnz inside diagonal tiles
  double cand_pairs; // candidate element pairs in off-diagonal candidate tiles
};

Expect expectation(const cieg_gen_params& p) {
  TileGrid g = make_grid(p);
  const std::uint32_t ns = p.sectors;
  Expect e{0.0, 0.0};
  std::vector<double> sum_t2(ns, 0.0), rows(ns, 0.0);
  for (std::uint32_t t = 0; t < g.count(); ++t) {
    const double sz = static_cast<double>(g.start[t + 1] - g.start[t]);
    e.diag_off += p.q * sz * (sz - 1.0) / 2.0;
    sum_t2[g.sector[t]] += sz * sz;
    rows[g.sector[t]] += sz;
  }
  for (std::uint32_t s = 0; s < ns; ++s) {
    e.cand_pairs += (rows[s] * rows[s] - sum_t2[s]) / 2.0;
    for (std::uint32_t s2 = (s >= p.band ? s - p.band : 0); s2 < s; ++s2)
      e.cand_pairs += rows[s] * rows[s2];
  }
  return e;
}

}  // namespace

double expected_nnz(const cieg_gen_params& p) {
  Expect e = expectation(p);
  return static_cast<double>(p.n) + e.diag_off + p.p * p.q * e.cand_pairs;
}

double avg_row_nnz(const cieg_gen_params& p) {
  Expect e = expectation(p);
  return 2.0 * (e.diag_off + p.p * p.q * e.cand_pairs) / static_cast<double>(p.n);
}

std::vector<std::vector<std::uint32_t>> kept_tiles(const cieg_gen_params& p, const TileGrid& g) {
  const std::uint32_t ntiles = g.count();
  const cieg_gen::Seeds sd = cieg_gen::derive_seeds(p.seed);
  std::vector<std::vector<std::uint32_t>> kept(ntiles);
#pragma omp parallel for schedule(dynamic, 16)
  for (std::int64_t ti = 0; ti < static_cast<std::int64_t>(ntiles); ++ti) {
    const std::uint32_t I = static_cast<std::uint32_t>(ti);
    const std::uint32_t sI = g.sector[I];
    const std::uint32_t s_lo = sI >= p.band ? sI - p.band : 0;
    std::uint32_t J0 = static_cast<std::uint32_t>(
        std::lower_bound(g.start.begin(), g.start.end() - 1, g.sector_start[s_lo]) - g.start.begin());
    for (std::uint32_t J = J0; J < I; ++J)
      if (cieg_gen::unit_double(cieg_gen::hash3(sd.tile, I, J)) < p.p) kept[I].push_back(J);
    kept[I].push_back(I);
  }
  return kept;
}

double value_scale(const cieg_gen_params& p) {
  const double avg = avg_row_nnz(p);
  return avg > 0.0 ? 1.0 / std::sqrt(avg) : 0.0;
}

void generate(const cieg_gen_params& p, HostCsb& out) {
  validate(p);
  const TileGrid g = make_grid(p);
  const std::uint32_t ntiles = g.count();
  const cieg_gen::Seeds sd = cieg_gen::derive_seeds(p.seed);
  const double scale = value_scale(p);
  const std::vector<std::vector<std::uint32_t>> kept = kept_tiles(p, g);

  // CSB blocks: consecutive tiles up to beta rows, cut at sector starts.
  std::vector<std::uint32_t> bb{0};
  std::vector<std::uint32_t> tile_block(ntiles);
  for (std::uint32_t t = 0; t < ntiles; ++t) {
    const std::uint32_t s = g.start[t], e = g.start[t + 1];
    const bool stratum = (s != 0) && (g.sector_start[g.sector[t]] == s);
    if (s > bb.back() && (stratum || e - bb.back() > p.beta)) bb.push_back(s);
    tile_block[t] = static_cast<std::uint32_t>(bb.size() - 1);
  }
  bb.push_back(p.n);
  const std::uint32_t nb = static_cast<std::uint32_t>(bb.size() - 1);
  const std::uint64_t nblk = static_cast<std::uint64_t>(nb) * (nb + 1) / 2;

  // Tiles of each block row.
  std::vector<std::uint32_t> block_first_tile(nb + 1, ntiles);
  for (std::uint32_t t = ntiles; t-- > 0;) block_first_tile[tile_block[t]] = t;
  block_first_tile[nb] = ntiles;

  struct Staged {
    std::vector<std::uint16_t> r, c;
    std::vector<double> v;
  };
  std::vector<std::vector<Staged>> staged(nb);
  std::vector<std::uint64_t> counts(nblk + 1, 0);

#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t bi64 = 0; bi64 < static_cast<std::int64_t>(nb); ++bi64) {
    const std::uint32_t BI = static_cast<std::uint32_t>(bi64);
    std::vector<Staged>& st = staged[BI];
    st.assign(BI + 1, Staged{});
    const std::uint32_t rbase = bb[BI];
    for (std::uint32_t I = block_first_tile[BI]; I < block_first_tile[BI + 1]; ++I) {
      const double s_diag = 10.0 * static_cast<double>(g.sector[I]);
      for (std::uint32_t a = g.start[I]; a < g.start[I + 1]; ++a) {
        for (std::uint32_t J : kept[I]) {
          const std::uint32_t BJ = tile_block[J];
          const std::uint32_t cbase = bb[BJ];
          Staged& s = st[BJ];
          const std::uint32_t cs = g.start[J];
          const std::uint32_t ce = (J == I) ? a : g.start[J + 1];
          for (std::uint32_t b = cs; b < ce; ++b) {
            const std::uint64_t hq = cieg_gen::hash3(sd.q, a, b);
            if (!(cieg_gen::unit_double(hq) < p.q)) continue;
            const double z = cieg_gen::normal_from(cieg_gen::hash3(sd.v1, a, b),
                                                   cieg_gen::hash3(sd.v2, a, b));
            s.r.push_back(static_cast<std::uint16_t>(a - rbase));
            s.c.push_back(static_cast<std::uint16_t>(b - cbase));
            s.v.push_back(z * scale);
          }
          if (J == I) {
            const double u = cieg_gen::unit_double(cieg_gen::hash3(sd.d, a, a));
            s.r.push_back(static_cast<std::uint16_t>(a - rbase));
            s.c.push_back(static_cast<std::uint16_t>(a - cbase));
            s.v.push_back(s_diag + 4.0 * u - 2.0);
          }
        }
      }
    }
    const std::uint64_t base = static_cast<std::uint64_t>(BI) * (BI + 1) / 2;
    for (std::uint32_t BJ = 0; BJ <= BI; ++BJ) counts[base + BJ + 1] = st[BJ].r.size();
  }
  for (std::uint64_t k = 0; k < nblk; ++k) counts[k + 1] += counts[k];
  const std::uint64_t nnz = counts[nblk];

  out = HostCsb{};
  out.dim = p.n;
  out.nb = nb;
  out.precision = p.precision;
  out.block_boundaries = bb;
  out.entry_offsets = counts;
  out.rows.resize(nnz);
  out.cols.resize(nnz);
  if (p.precision == 0)
    out.values32.resize(nnz);
  else
    out.values64.resize(nnz);
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t bi64 = 0; bi64 < static_cast<std::int64_t>(nb); ++bi64) {
    const std::uint32_t BI = static_cast<std::uint32_t>(bi64);
    const std::uint64_t base = static_cast<std::uint64_t>(BI) * (BI + 1) / 2;
    for (std::uint32_t BJ = 0; BJ <= BI; ++BJ) {
      Staged& s = staged[BI][BJ];
      const std::uint64_t o = out.entry_offsets[base + BJ];
      const std::size_t n = s.r.size();
      if (n == 0) continue;
      std::memcpy(out.rows.data() + o, s.r.data(), n * sizeof(std::uint16_t));
      std::memcpy(out.cols.data() + o, s.c.data(), n * sizeof(std::uint16_t));
      if (p.precision == 0)
        for (std::size_t e = 0; e < n; ++e) out.values32[o + e] = static_cast<float>(s.v[e]);
      else
        std::memcpy(out.values64.data() + o, s.v.data(), n * sizeof(double));
      Staged().r.swap(s.r);
      Staged().c.swap(s.c);
      Staged().v.swap(s.v);
    }
  }
  out.group_bounds.assign(g.start.begin(), g.start.end());
}

// Stored entries of the generated matrix without building it (same loops).
std::uint64_t count_nnz(const cieg_gen_params& p) {
  validate(p);
  const TileGrid g = make_grid(p);
  const cieg_gen::Seeds sd = cieg_gen::derive_seeds(p.seed);
  const std::vector<std::vector<std::uint32_t>> kept = kept_tiles(p, g);
  std::uint64_t total = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
  for (std::int64_t ti = 0; ti < static_cast<std::int64_t>(g.count()); ++ti) {
    const std::uint32_t I = static_cast<std::uint32_t>(ti);
    for (std::uint32_t a = g.start[I]; a < g.start[I + 1]; ++a)
      for (std::uint32_t J : kept[I]) {
        const std::uint32_t ce = (J == I) ? a : g.start[J + 1];
        for (std::uint32_t b = g.start[J]; b < ce; ++b)
          total += cieg_gen::unit_double(cieg_gen::hash3(sd.q, a, b)) < p.q;
        total += J == I;
      }
  }
  return total;
}

void random_block(std::uint32_t n, std::uint32_t k, std::uint64_t seed, double* out, std::uint32_t row0) {
  // ci::random_block (proj/src/block_vectors.cpp:162-174): symmetric_double(seed, i, j),
  // rows [row0, row0 + n) of the global block (a shard's rows).
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
    for (std::uint32_t j = 0; j < k; ++j)
      out[static_cast<std::size_t>(i) * k + j] =
          2.0 * cieg_gen::unit_double(cieg_gen::hash3(seed, static_cast<std::uint64_t>(row0 + i), j)) - 1.0;
}

}  // namespace cieg

extern "C" {

double cieg_gen_expected_nnz(const cieg_gen_params* prm) {
  return prm ? cieg::expected_nnz(*prm) : 0.0;
}

uint64_t cieg_gen_count_nnz(const cieg_gen_params* prm) {
  std::uint64_t n = 0;
  if (cieg::guarded([&] { n = prm ? cieg::count_nnz(*prm) : 0; }) != CIEG_OK) return 0;
  return n;
}

double cieg_gen_avg_row_nnz(const cieg_gen_params* prm) {
  return prm ? cieg::avg_row_nnz(*prm) : 0.0;
}

int cieg_generate_csb(const cieg_gen_params* prm, cieg_host_csb** out) {
  return cieg::guarded([&] {
    if (!prm || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_generate_csb: null argument");
    auto* h = new cieg_host_csb;
    try {
      cieg::generate(*prm, h->h);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int cieg_host_csb_destroy(cieg_host_csb* h) {
  delete h;
  return CIEG_OK;
}

int cieg_host_csb_view(const cieg_host_csb* hc, cieg_csb_view* v, uint64_t* nnz) {
  return cieg::guarded([&] {
    if (!hc || !v) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_host_csb_view: null argument");
    const cieg::HostCsb& h = hc->h;
    v->dim = h.dim;
    v->nb = h.nb;
    v->precision = h.precision;
    v->block_boundaries = h.block_boundaries.data();
    v->entry_offsets = h.entry_offsets.data();
    v->rows = h.rows.data();
    v->cols = h.cols.data();
    v->values = h.precision == 0 ? static_cast<const void*>(h.values32.data())
                                 : static_cast<const void*>(h.values64.data());
    if (nnz) *nnz = h.entry_offsets.empty() ? 0 : h.entry_offsets.back();
  });
}

int cieg_host_csb_groups(const cieg_host_csb* hc, const uint32_t** bounds, uint32_t* ngroups) {
  return cieg::guarded([&] {
    if (!hc || !bounds || !ngroups) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_host_csb_groups: null");
    *bounds = hc->h.group_bounds.data();
    *ngroups = static_cast<uint32_t>(hc->h.group_bounds.size() - 1);
  });
}

int cieg_random_block(uint32_t n, uint32_t k, uint64_t seed, double* out_host) {
  return cieg::guarded([&] {
    if (!out_host && n && k) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_random_block: null output");
    cieg::random_block(n, k, seed, out_host, 0);
  });
}

int cieg_random_block_rows(uint32_t row_lo, uint32_t row_hi, uint32_t k, uint64_t seed, double* out_host) {
  return cieg::guarded([&] {
    if (row_hi < row_lo) cieg::fail(CIEG_ERR_DIMENSION, "cieg_random_block_rows: row_hi < row_lo");
    if (!out_host && row_hi > row_lo && k) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_random_block_rows: null output");
    cieg::random_block(row_hi - row_lo, k, seed, out_host, row_lo);
  });
}

}  // extern "C"
