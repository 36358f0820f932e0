// guess.cpp -- LOBPCG starting blocks (proj/include/ci/guess.hpp): the
// multi-level guess (guess.cpp:66-117) and its pieces, on the GPU.
//
// The reference assembles a fresh Hamiltonian per truncation level through
// a physics ProblemFactory. Truncated bases are prefixes of the full basis
// (states ordered by quanta stratum), so the level problems are leading
// principal blocks of the full matrix: here every level runs on a
// cieg_matrix_leading_view of the resident H (no re-assembly, no copy of the
// tile stream). The control flow is the reference's: random orthonormal start
// at the smallest level, unpreconditioned LOBPCG per level, the trial block
// zero-padded into the next space and topped up with seeded random directions
// orthogonal to it (widen_to, guess.cpp:57-62).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "cieg_internal.hpp"
#include "context.hpp"
#include "gen_common.h"

namespace cieg {
namespace {

void check(int rc) {
  if (rc != CIEG_OK) fail(static_cast<cieg_status>(rc), cieg_last_error());
}

// Host block n x k row-major.
struct HBlock {
  std::uint32_t n = 0, k = 0;
  std::vector<double> v;
};

// orthonormalize(y, drop_tol, against) (lobpcg.cpp:89-119) through the device.
HBlock orthonormalize(cieg_ctx* ctx, const HBlock& y, const HBlock* against) {
  HBlock out;
  out.n = y.n;
  if (y.k == 0) return out;
  double* d = nullptr;
  double* a = nullptr;
  CIEG_CUDA(cudaMalloc(&d, sizeof(double) * y.v.size()));
  try {
    CIEG_CUDA(cudaMemcpy(d, y.v.data(), sizeof(double) * y.v.size(), cudaMemcpyHostToDevice));
    if (against && against->k) {
      CIEG_CUDA(cudaMalloc(&a, sizeof(double) * against->v.size()));
      CIEG_CUDA(cudaMemcpy(a, against->v.data(), sizeof(double) * against->v.size(), cudaMemcpyHostToDevice));
    }
    std::uint32_t kk = 0;
    check(cieg_orthonormalize(ctx, d, y.n, y.k, 1e-8, a, a ? against->k : 0, &kk));
    out.k = kk;
    out.v.resize(static_cast<std::size_t>(y.n) * kk);
    if (kk) CIEG_CUDA(cudaMemcpy(out.v.data(), d, sizeof(double) * out.v.size(), cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaFree(d);
    cudaFree(a);
    throw;
  }
  cudaFree(d);
  cudaFree(a);
  return out;
}

HBlock random_block(std::uint32_t n, std::uint32_t k, std::uint64_t seed) {
  HBlock b{n, k, std::vector<double>(static_cast<std::size_t>(n) * k)};
  check(cieg_random_block(n, k, seed, b.v.data()));
  return b;
}

// pad_from_subspace (guess.cpp:14-23): rows copied, the rest zero.
HBlock pad(const HBlock& x, std::uint32_t dim) {
  if (x.n > dim) fail(CIEG_ERR_DIMENSION, "pad_from_subspace: source exceeds target");
  HBlock out{dim, x.k, std::vector<double>(static_cast<std::size_t>(dim) * x.k, 0.0)};
  std::memcpy(out.v.data(), x.v.data(), sizeof(double) * x.v.size());
  return out;
}

// widen_to (guess.cpp:57-62)
HBlock widen_to(cieg_ctx* ctx, HBlock x, std::uint32_t k_trial, std::uint64_t seed) {
  if (x.k >= k_trial) return x;
  HBlock extra = orthonormalize(ctx, random_block(x.n, k_trial - x.k, cieg_gen::mix64(seed) + 1), &x);
  HBlock out{x.n, x.k + extra.k, std::vector<double>(static_cast<std::size_t>(x.n) * (x.k + extra.k))};
  for (std::uint32_t i = 0; i < x.n; ++i) {
    std::memcpy(&out.v[static_cast<std::size_t>(i) * out.k], &x.v[static_cast<std::size_t>(i) * x.k],
                sizeof(double) * x.k);
    std::memcpy(&out.v[static_cast<std::size_t>(i) * out.k + x.k], &extra.v[static_cast<std::size_t>(i) * extra.k],
                sizeof(double) * extra.k);
  }
  return out;
}

}  // namespace
}  // namespace cieg

extern "C" {

void cieg_multilevel_options_default(cieg_multilevel_options* opt) {
  if (!opt) return;
  opt->k_want = 8;     // guess.hpp:49
  opt->k_trial = 12;   // guess.hpp:50
  opt->tol = 1e-6;     // guess.hpp:51
  opt->max_iter = 500; // guess.hpp:52
  opt->seed = 1;       // guess.hpp:53
}

int cieg_pad_from_subspace(const double* x_host, uint32_t n1, uint32_t k, uint32_t dim, double* out_host) {
  return cieg::guarded([&] {
    if (!x_host || !out_host) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_pad_from_subspace: null argument");
    cieg::HBlock x{n1, k, std::vector<double>(x_host, x_host + static_cast<std::size_t>(n1) * k)};
    const cieg::HBlock p = cieg::pad(x, dim);
    std::memcpy(out_host, p.v.data(), sizeof(double) * p.v.size());
  });
}

int cieg_multilevel_guess(cieg_ctx* ctx, const cieg_mat* mat, const uint32_t* level_dims, uint32_t nlevels,
                          const cieg_multilevel_options* opt, double* guess_host, uint32_t* k_out,
                          cieg_level_report* levels_out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !opt || !guess_host || !k_out || (nlevels && (!level_dims || !levels_out)))
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_multilevel_guess: null argument");
    if (mat->row_lo != 0 || mat->row_hi != mat->dim)
      cieg::fail(CIEG_ERR_CONFIG, "cieg_multilevel_guess needs the whole matrix (not a shard)");
    if (opt->k_trial < 1 || opt->k_want < 1 || opt->k_want > opt->k_trial)
      cieg::fail(CIEG_ERR_CONFIG, "multilevel_guess: need 1 <= k_want <= k_trial");
    for (uint32_t l = 0; l < nlevels; ++l)
      if (level_dims[l] >= mat->dim || (l && level_dims[l] <= level_dims[l - 1]))
        cieg::fail(CIEG_ERR_DIMENSION, "multilevel_guess: level dimensions must ascend below the full dimension");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const std::uint32_t k_trial = static_cast<std::uint32_t>(opt->k_trial);
    const int levels = static_cast<int>(nlevels) + 1;
    cieg::HBlock guess;
    if (levels == 1) {
      guess = cieg::orthonormalize(ctx, cieg::random_block(mat->dim, k_trial, opt->seed), nullptr);
    } else {
      cieg::HBlock carried;
      for (int level = 0; level < levels - 1; ++level) {
        const auto t0 = std::chrono::steady_clock::now();
        const std::uint32_t d = level_dims[level];
        cieg_mat* view = nullptr;
        cieg::check(cieg_matrix_leading_view(ctx, mat, d, &view));
        std::unique_ptr<cieg_mat> hold(view);
        const std::uint32_t width = std::min<std::uint32_t>(k_trial, d);
        cieg::HBlock x0 = level == 0
                              ? cieg::orthonormalize(ctx, cieg::random_block(d, width, opt->seed), nullptr)
                              : cieg::widen_to(ctx, cieg::pad(carried, d), width, opt->seed + level);
        if (x0.k < static_cast<std::uint32_t>(opt->k_want))
          cieg::fail(CIEG_ERR_SUBSPACE, "level guess lost too many columns");
        cieg_lobpcg_options lopt;
        cieg_lobpcg_options_default(&lopt);
        lopt.k_want = opt->k_want;
        lopt.tol = opt->tol;
        lopt.max_iter = opt->max_iter;
        cieg_report* rep = nullptr;
        cieg::check(cieg_lobpcg_solve(ctx, view, x0.v.data(), x0.k, nullptr, &lopt, nullptr, nullptr, &rep));
        int conv = 0, iters = 0;
        double ne = 0.0;
        std::uint32_t kw = 0, kt = 0;
        std::uint64_t nh = 0;
        cieg_report_summary(rep, &conv, &iters, &ne, &kw, &kt, &nh);
        carried = cieg::HBlock{d, kt, std::vector<double>(static_cast<std::size_t>(d) * kt)};
        cieg_report_trial_vectors(rep, carried.v.data());
        cieg_report_destroy(rep);
        levels_out[level] = cieg_level_report{d, iters, conv, std::chrono::duration<double>(
                                                                    std::chrono::steady_clock::now() - t0)
                                                                    .count()};
      }
      guess = cieg::widen_to(ctx, cieg::pad(carried, mat->dim), k_trial, opt->seed + levels);
    }
    *k_out = guess.k;
    std::memcpy(guess_host, guess.v.data(), sizeof(double) * guess.v.size());
  });
}

}  // extern "C"
