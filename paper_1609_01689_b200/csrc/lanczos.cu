// lanczos.cu -- the Lanczos baseline, ci::lanczos_solve (proj/src/lanczos.cpp:24-136)
// on the GPU.
//
// The host runs the reference's control flow verbatim: one SpMV per step (K1
// at m = 1), alpha = v.w, the three-term recurrence, two passes of classical
// Gram-Schmidt against the whole basis (lanczos.cpp:72-76), the breakdown
// restart with the seeded random direction (lanczos.cpp:81-96), and the
// tridiagonal Ritz analysis only on the staggered checkpoint grid
// (lanczos.cpp:11-15, 102-126). The basis lives in HBM as a column-major
// n x (max_steps + 1) fp64 array; each reorthogonalisation pass is one
// GEMV-T (coefficients, fixed-order two-stage reduction) and one GEMV update,
// both streaming the basis once at HBM speed. Scalars (alpha, beta, norms)
// come back to the host each step; the tridiagonal eigenproblem runs on the
// host with the same QL code the oracle uses (dense_small.hpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "cieg_internal.hpp"
#include "context.hpp"
#include "dense_small.hpp"
#include "device_common.cuh"
#include "gen_common.h"
#include "report.hpp"

namespace cieg {
namespace {

constexpr int kThreads = 256;
constexpr int kColsPerPass = 8;
constexpr int kUpdCols = 64;  // basis columns per CTA of the GEMV update

// Fixed row-chunk count for the n-length reductions: a function of n only,
// so the summation order (and the result) does not depend on the device.
std::uint32_t reduction_ctas(std::uint32_t n) {
  return std::max<std::uint32_t>(1, std::min<std::uint32_t>(1024, (n + 511) / 512));
}

// partial[g * m + j] = sum over row chunk g of V[r, j] * w[r]  (V column-major, ld);
// grid (row chunks, column groups of kColsPerPass). PAIRS (ld even, chunks
// of even length): row pairs through 16-byte loads.
template <bool PAIRS>
__global__ void __launch_bounds__(kThreads) gemvt_partial_kernel(const double* __restrict__ v, std::size_t ld,
                                                                 std::uint32_t n, std::uint32_t m,
                                                                 const double* __restrict__ w,
                                                                 double* __restrict__ partial) {
  __shared__ double red[kThreads / 32][kColsPerPass];
  const std::uint32_t chunk = PAIRS ? ((n + gridDim.x - 1) / gridDim.x + 1) & ~1u : (n + gridDim.x - 1) / gridDim.x;
  const std::uint32_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint32_t j0 = blockIdx.y * kColsPerPass;
  double acc[kColsPerPass];
#pragma unroll
  for (int c = 0; c < kColsPerPass; ++c) acc[c] = 0.0;
  if (PAIRS) {
    // row pairs: one 16-byte load per column and pair (ld and r0 even)
    const std::uint32_t p1 = r0 + ((r1 - r0) & ~1u);
    for (std::uint32_t r = r0 + 2 * threadIdx.x; r < p1; r += 2 * kThreads) {
      const double2 wr = *reinterpret_cast<const double2*>(w + r);
#pragma unroll
      for (int c = 0; c < kColsPerPass; ++c)
        if (j0 + c < m) {
          const double2 vv = *reinterpret_cast<const double2*>(v + (j0 + c) * ld + r);
          acc[c] = fma(vv.y, wr.y, fma(vv.x, wr.x, acc[c]));
        }
    }
    if (p1 < r1 && threadIdx.x == 0) {  // odd tail row of the chunk
      const double wr = w[p1];
#pragma unroll
      for (int c = 0; c < kColsPerPass; ++c)
        if (j0 + c < m) acc[c] = fma(v[(j0 + c) * ld + p1], wr, acc[c]);
    }
  } else {
    for (std::uint32_t r = r0 + threadIdx.x; r < r1; r += kThreads) {
      const double wr = w[r];
#pragma unroll
      for (int c = 0; c < kColsPerPass; ++c)
        if (j0 + c < m) acc[c] = fma(v[(j0 + c) * ld + r], wr, acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < kColsPerPass; ++c)
    for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_down_sync(0xffffffffu, acc[c], o);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < kColsPerPass; ++c) red[warp][c] = acc[c];
  __syncthreads();
  if (threadIdx.x < kColsPerPass && j0 + threadIdx.x < m) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += red[k][threadIdx.x];
    partial[static_cast<std::size_t>(blockIdx.x) * m + j0 + threadIdx.x] = s;
  }
}

// out[j] = sum_k partial[k * m + j]: one warp per output, lane-strided
// partial sums then a fixed xor tree (deterministic; a serial loop over the
// row blocks per output was latency-bound at ~50 us per call).
__global__ void reduce_partials_kernel(const double* __restrict__ partial, std::uint32_t g, std::uint32_t m,
                                       double* __restrict__ out) {
  const std::uint32_t j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const std::uint32_t lane = threadIdx.x & 31;
  if (j >= m) return;
  double s = 0.0;
  for (std::uint32_t k = lane; k < g; k += 32) s += partial[static_cast<std::size_t>(k) * m + j];
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// tmp[c * n + r] = sum_{j in column chunk c} V[r, j] * coeff[j]; grid (row blocks, column chunks)
__global__ void __launch_bounds__(kThreads) gemv_partial_kernel(const double* __restrict__ v, std::size_t ld,
                                                                std::uint32_t n, std::uint32_t m,
                                                                const double* __restrict__ coeff,
                                                                double* __restrict__ tmp) {
  __shared__ double c[kUpdCols];
  const std::uint32_t j0 = blockIdx.y * kUpdCols;
  const std::uint32_t jn = min(static_cast<std::uint32_t>(kUpdCols), m - j0);
  for (std::uint32_t j = threadIdx.x; j < jn; j += kThreads) c[j] = coeff[j0 + j];
  __syncthreads();
  const std::uint32_t r = blockIdx.x * kThreads + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (std::uint32_t j = 0; j < jn; ++j) s = fma(v[(j0 + j) * ld + r], c[j], s);
  tmp[static_cast<std::size_t>(blockIdx.y) * n + r] = s;
}

// w[r] -= sum_c tmp[c * n + r], chunks ascending   (Eigen: tmp = V * coeff; w -= tmp)
__global__ void gemv_finish_kernel(const double* __restrict__ tmp, std::uint32_t chunks, std::uint32_t n,
                                   double* __restrict__ w) {
  const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (std::uint32_t c = 0; c < chunks; ++c) s += tmp[static_cast<std::size_t>(c) * n + r];
  w[r] -= s;
}

// w = w - a * v1 - b * v2   (lanczos.cpp:70-71; v2 may be null)
__global__ void recurrence_kernel(double* __restrict__ w, const double* __restrict__ v1, double a,
                                  const double* __restrict__ v2, double b, std::uint32_t n) {
  const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x = w[r] - a * v1[r];
  if (v2) x = x - b * v2[r];
  w[r] = x;
}

// dst = src / s
__global__ void scale_kernel(double* __restrict__ dst, const double* __restrict__ src, double s, std::uint32_t n) {
  const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[r] / s;
}

// r[i] = symmetric_double(seed, i, m)   (rng.hpp:33-36, lanczos.cpp:85-86)
__global__ void restart_vector_kernel(double* __restrict__ r, std::uint64_t seed, std::uint64_t m, std::uint32_t n) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) r[i] = 2.0 * cieg_gen::unit_double(cieg_gen::hash3(seed, i, m)) - 1.0;
}

// out (n x k row-major) = V[:, :f] * S[:, :k]   (S column-major f x f)  (lanczos.cpp:131-132)
__global__ void __launch_bounds__(kThreads) ritz_vectors_kernel(const double* __restrict__ v, std::size_t ld,
                                                                std::uint32_t n, std::uint32_t f,
                                                                const double* __restrict__ s, std::uint32_t k,
                                                                double* __restrict__ out) {
  const std::uint32_t r = blockIdx.x * kThreads + threadIdx.x;
  if (r >= n) return;
  for (std::uint32_t j = 0; j < k; ++j) {
    double acc = 0.0;
    for (std::uint32_t l = 0; l < f; ++l) acc = fma(v[l * ld + r], s[l + static_cast<std::size_t>(j) * f], acc);
    out[static_cast<std::size_t>(r) * k + j] = acc;
  }
}

unsigned blocks_for(std::uint32_t n) { return (n + kThreads - 1) / kThreads; }

class Lanczos {
 public:
  Lanczos(cieg_ctx* ctx, const cieg_mat* mat, const cieg_lanczos_options& opt, cieg_report& rep)
      : ctx_(ctx), mat_(mat), opt_(opt), rep_(rep), n_(mat->dim) {}
  ~Lanczos() {
    clock_discard(ctx_);
    for (double* p : owned_) cudaFree(p);
  }
  void run(const double* v0_host);

 private:
  double* alloc(std::size_t count) {
    double* p = nullptr;
    if (cudaMalloc(&p, sizeof(double) * std::max<std::size_t>(1, count)) != cudaSuccess) {
      cudaGetLastError();
      fail(CIEG_ERR_CUDA, "lanczos: out of device memory for the basis / work vectors");
    }
    owned_.push_back(p);
    return p;
  }
  double* col(int j) const { return basis_ + static_cast<std::size_t>(j) * n_; }
  void launched(int k = 1) {
    CIEG_CUDA(cudaGetLastError());
    ctx_->launches += k;
  }
  // out[0..m) = V[:, :m]^T w   (device)
  void gemvt(const double* v, int m, const double* w, double* out) {
    const dim3 grid(g_, (m + kColsPerPass - 1) / kColsPerPass);
    const bool pairs = n_ % 2 == 0 && reinterpret_cast<std::uintptr_t>(v) % 16 == 0 &&
                       reinterpret_cast<std::uintptr_t>(w) % 16 == 0;
    if (pairs)
      gemvt_partial_kernel<true><<<grid, kThreads, 0, ctx_->stream>>>(v, n_, n_, static_cast<std::uint32_t>(m), w, partial_);
    else
      gemvt_partial_kernel<false><<<grid, kThreads, 0, ctx_->stream>>>(v, n_, n_, static_cast<std::uint32_t>(m), w, partial_);
    reduce_partials_kernel<<<(m + 3) / 4, 128, 0, ctx_->stream>>>(partial_, g_, static_cast<std::uint32_t>(m), out);
    launched(2);
  }
  double dot(const double* a, const double* b) {
    gemvt(a, 1, b, scalar_);
    double h = 0.0;
    CIEG_CUDA(cudaMemcpyAsync(&h, scalar_, sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
    return h;
  }
  // two passes of classical Gram-Schmidt of w against basis[:, :m]  (lanczos.cpp:72-76, 88-91)
  void reorthogonalize(double* w, int m) {
    for (int pass = 0; pass < 2; ++pass) {
      gemvt(basis_, m, w, coeff_);
      const std::uint32_t chunks = (m + kUpdCols - 1) / kUpdCols;
      gemv_partial_kernel<<<dim3(blocks_for(n_), chunks), kThreads, 0, ctx_->stream>>>(
          basis_, n_, n_, static_cast<std::uint32_t>(m), coeff_, tmp_);
      gemv_finish_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(tmp_, chunks, n_, w);
      launched(2);
    }
  }
  // lanczos.cpp:54-63. At checkpoints only the Ritz values and the bottom
  // row of the eigenvector matrix are needed (the residual test): O(m^2),
  // bitwise equal to the full factorisation's values; the full vectors are
  // formed once, for the returned Ritz vectors.
  void factorize(int m, bool full) {
    ritz_.assign(m, 0.0);
    std::vector<double> sub(std::max(m - 1, 0));
    for (int i = 0; i + 1 < m; ++i) sub[i] = beta_[i];
    bool ok;
    if (full) {
      ritz_vecs_.assign(static_cast<std::size_t>(m) * m, 0.0);
      ok = cieg_dense::tridiag_eig(m, alpha_.data(), sub.data(), ritz_.data(), ritz_vecs_.data());
      bottom_.resize(m);
      for (int j = 0; j < m; ++j) bottom_[j] = ritz_vecs_[(m - 1) + static_cast<std::size_t>(j) * m];
    } else {
      bottom_.assign(m, 0.0);
      ok = cieg_dense::tridiag_eig_bottom(m, alpha_.data(), sub.data(), ritz_.data(), bottom_.data());
    }
    if (!ok) fail(CIEG_ERR_INDEFINITE, "lanczos: tridiagonal eigensolver did not converge");
    factorized_ = m;
  }

  cieg_ctx* ctx_;
  const cieg_mat* mat_;
  const cieg_lanczos_options& opt_;
  cieg_report& rep_;
  std::uint32_t n_;
  std::uint32_t g_ = 1;
  std::vector<double*> owned_;
  double* basis_ = nullptr;
  double* w_ = nullptr;
  double* coeff_ = nullptr;
  double* partial_ = nullptr;
  double* scalar_ = nullptr;
  double* tmp_ = nullptr;  // GEMV partials: ceil(m / kUpdCols) x n
  std::vector<double> alpha_, beta_, ritz_, ritz_vecs_, bottom_;
  int factorized_ = 0;
};

void Lanczos::run(const double* v0_host) {
  const auto t_start = std::chrono::steady_clock::now();
  // lanczos.cpp:26-30
  double v0n = 0.0;
  for (std::uint32_t i = 0; i < n_; ++i) v0n += v0_host[i] * v0_host[i];
  v0n = std::sqrt(v0n);
  if (v0n == 0.0) fail(CIEG_ERR_CONFIG, "lanczos: v0 must be nonzero");
  if (opt_.k_want < 1) fail(CIEG_ERR_CONFIG, "lanczos: k_want must be >= 1");
  const int max_steps = std::min<int>(opt_.max_iter, static_cast<int>(n_));
  if (max_steps < 1) fail(CIEG_ERR_CONFIG, "lanczos: max_iter must be >= 1");
  rep_.n = n_;

  g_ = reduction_ctas(n_);
  basis_ = alloc(static_cast<std::size_t>(n_) * (max_steps + 1));
  w_ = alloc(n_);
  coeff_ = alloc(max_steps + 1);
  partial_ = alloc(static_cast<std::size_t>(g_) * (max_steps + 1));
  scalar_ = alloc(1);
  tmp_ = alloc(static_cast<std::size_t>(n_) * ((max_steps + kUpdCols) / kUpdCols));
  {
    std::vector<double> v(n_);
    for (std::uint32_t i = 0; i < n_; ++i) v[i] = v0_host[i] / v0n;
    CIEG_CUDA(cudaMemcpyAsync(col(0), v.data(), sizeof(double) * n_, cudaMemcpyHostToDevice, ctx_->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
  }

  std::uint64_t restart_counter = 0;
  for (int m = 1; m <= max_steps; ++m) {
    {
      Clock c(ctx_, &rep_.timing_ms[kSpmm]);
      launch_spmm(ctx_, mat_, col(m - 1), 1, w_, 1, 1);
      ++rep_.counters[0];
      ++rep_.counters[1];
    }
    double b = 0.0, a = 0.0;
    {
      Clock c(ctx_, &rep_.timing_ms[kOrtho]);
      a = dot(col(m - 1), w_);
      alpha_.push_back(a);
      recurrence_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(w_, col(m - 1), a, m >= 2 ? col(m - 2) : nullptr,
                                                                       m >= 2 ? beta_[m - 2] : 0.0, n_);
      launched();
      reorthogonalize(w_, m);
      ++rep_.counters[3];
      b = std::sqrt(dot(w_, w_));
      const double scale = std::max(std::fabs(a), 1.0);
      if (b <= 1e-13 * scale) {
        // invariant subspace: restart with a seeded random direction
        // orthogonal to the basis built so far (lanczos.cpp:81-96)
        restart_vector_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(w_, 0x4C414E43ull + restart_counter,
                                                                            static_cast<std::uint64_t>(m), n_);
        launched();
        ++restart_counter;
        reorthogonalize(w_, m);
        const double rn = std::sqrt(dot(w_, w_));
        if (rn == 0.0) break;  // space exhausted
        b = 0.0;  // the tridiagonal decouples at a true invariant subspace
        scale_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(col(m), w_, rn, n_);
        launched();
        beta_.push_back(b);
      } else {
        scale_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(col(m), w_, b, n_);
        launched();
        beta_.push_back(b);
      }
    }

    const bool last = m == max_steps;
    const bool checkpoint = m <= 100 ? m % 10 == 0 : (m <= 200 ? m % 20 == 0 : m % 40 == 0);
    if (!checkpoint && !last) continue;

    Clock c(ctx_, &rep_.timing_ms[kRR]);
    factorize(m, false);
    rep_.norm_estimate = std::max({rep_.norm_estimate, std::fabs(ritz_[0]), std::fabs(ritz_[m - 1])});
    const int k = std::min(opt_.k_want, m);
    bool all_converged = k >= opt_.k_want;
    for (int j = 0; j < k; ++j) {
      // |beta_m| times the bottom eigenvector component (lanczos.cpp:112-116)
      const double res = std::fabs(beta_[m - 1]) * std::fabs(bottom_[j]);
      const double relres = res / std::max(rep_.norm_estimate, 1e-300);
      rep_.history.push_back({m, j, relres, ritz_[j]});
      if (relres > opt_.tol) all_converged = false;
    }
    if (opt_.observer) {
      std::vector<double> bh(static_cast<std::size_t>(n_) * m);
      CIEG_CUDA(cudaMemcpyAsync(bh.data(), basis_, sizeof(double) * bh.size(), cudaMemcpyDeviceToHost, ctx_->stream));
      CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
      opt_.observer(opt_.observer_user, m, alpha_.data(), beta_.data(), bh.data(), n_);
    }
    rep_.iterations = m;
    if (all_converged) {
      rep_.converged = true;
      break;
    }
  }

  Clock c(ctx_, &rep_.timing_ms[kOther]);
  factorize(factorized_ == 0 ? static_cast<int>(alpha_.size()) : factorized_, true);
  const int k = std::min(opt_.k_want, factorized_);
  rep_.eigenvalues.assign(ritz_.begin(), ritz_.begin() + k);
  rep_.k_want = rep_.kt = static_cast<std::uint32_t>(k);
  double* s = alloc(static_cast<std::size_t>(factorized_) * factorized_);
  double* x = alloc(static_cast<std::size_t>(n_) * k);
  CIEG_CUDA(cudaMemcpyAsync(s, ritz_vecs_.data(), sizeof(double) * ritz_vecs_.size(), cudaMemcpyHostToDevice,
                            ctx_->stream));
  ritz_vectors_kernel<<<blocks_for(n_), kThreads, 0, ctx_->stream>>>(basis_, n_, n_, static_cast<std::uint32_t>(factorized_),
                                                                    s, static_cast<std::uint32_t>(k), x);
  launched();
  rep_.trial.resize(static_cast<std::size_t>(n_) * k);
  CIEG_CUDA(cudaMemcpyAsync(rep_.trial.data(), x, sizeof(double) * rep_.trial.size(), cudaMemcpyDeviceToHost,
                            ctx_->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
  clock_flush(ctx_);
  rep_.timing_ms[kTotal] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace
}  // namespace cieg

extern "C" {

void cieg_lanczos_options_default(cieg_lanczos_options* opt) {
  if (!opt) return;
  opt->k_want = 8;      // lanczos.hpp:15
  opt->tol = 1e-6;      // lanczos.hpp:16
  opt->max_iter = 500;  // lanczos.hpp:17
  opt->observer = nullptr;
  opt->observer_user = nullptr;
}

int cieg_lanczos_checkpoint(int m) { return m <= 100 ? m % 10 == 0 : (m <= 200 ? m % 20 == 0 : m % 40 == 0); }

int cieg_lanczos_default_start(uint32_t n, uint32_t stratum_end, double* out) {
  return cieg::guarded([&] {
    if (!out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_lanczos_default_start: null argument");
    if (stratum_end == 0 || stratum_end > n) cieg::fail(CIEG_ERR_CONFIG, "lanczos: stratum end outside (0, n]");
    // lanczos.cpp:17-22: ones on the lowest stratum, normalised
    const double nrm = std::sqrt(static_cast<double>(stratum_end));
    for (uint32_t i = 0; i < n; ++i) out[i] = i < stratum_end ? 1.0 / nrm : 0.0;
  });
}

int cieg_lanczos_solve(cieg_ctx* ctx, const cieg_mat* mat, const double* v0_host, const cieg_lanczos_options* opt,
                       cieg_report** out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !v0_host || !opt || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_lanczos_solve: null argument");
    if (mat->row_lo != 0 || mat->row_hi != mat->dim)
      cieg::fail(CIEG_ERR_CONFIG, "cieg_lanczos_solve needs the whole matrix (not a shard)");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    auto rep = std::make_unique<cieg_report>();
    {
      cieg::Lanczos l(ctx, mat, *opt, *rep);
      l.run(v0_host);
    }
    *out = rep.release();
  });
}

}  // extern "C"
