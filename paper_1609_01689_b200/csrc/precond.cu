// precond.cu -- K5: tile-diagonal preconditioner with per-column shifts,
// replacing ci::apply_preconditioner (proj/src/precond.cpp:160-207).
//
//   * groups with n_g <= small_block_cutoff: one CTA per (group, distinct
//     shift) -- partial-pivot LU of (H~_g - mu I) in shared memory, the
//     |U_ii| <= 1e-14 max|U_ii| singularity test, one perturbation
//     mu + 1e-8 (1 + |mu|), then pass-through (precond.cpp:61-83); the
//     columns sharing a shift share the factorization (precond.cpp:183-192);
//   * larger groups: one CTA per (group, column chunk) running the fused
//     multi-RHS FOM (precond.cpp:87-158): one dense block product advances
//     every Krylov space, two-pass MGS, lucky breakdown at 1e-12, Hessenberg
//     solve by partial-pivot LU.
// Arithmetic is kept un-fused (mul then add) and every reduction runs in the
// reference's sequential order, so for identical inputs the result is
// bitwise identical to the reference compiled on the host.
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <map>

#include "device_common.cuh"
#include "precond.hpp"

#define DMUL __dmul_rn
#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DDIV __ddiv_rn

cieg_prec::~cieg_prec() {
  cudaFree(bounds);
  cudaFree(block_off);
  cudaFree(blocks);
  cudaFree(blocks32);
}

namespace cieg {

ShiftPlan choose_shifts(const std::vector<double>& theta, const std::vector<double>& res_norm,
                        const std::vector<double>& x_norm, const std::vector<double>& relres,
                        int iteration, double tol, const cieg_precond_config& cfg) {
  const std::size_t k = theta.size();
  ShiftPlan plan;
  plan.mu = theta;
  plan.engage.assign(k, 1);
  if (iteration <= cfg.engage_after) {
    plan.engage.assign(k, 0);
  } else if (!relres.empty() && relres[0] > cfg.relres_gate) {
    plan.engage.assign(k, 0);
  } else {
    for (std::size_t j = 0; j < k; ++j)
      if (relres[j] <= cfg.column_floor_factor * tol) plan.engage[j] = 0;
  }
  for (std::size_t j = 0; j < k; ++j) {
    const double backed = theta[j] - 2.0 * res_norm[j] / x_norm[j];
    plan.mu[j] = j == 0 ? backed : std::min(backed, plan.mu[0]);
  }
  std::size_t first_far = k;
  for (std::size_t i = 0; i < k; ++i)
    if (relres[i] > cfg.far_threshold) {
      first_far = i;
      break;
    }
  if (first_far < k) {
    const double carried = plan.mu[first_far > 0 ? first_far - 1 : 0];
    for (std::size_t t = first_far; t < k; ++t) plan.mu[t] = carried;
  }
  return plan;
}

namespace {

// Dense tile-diagonal blocks, fp64 or (for an fp32 H, whose values are
// exactly fp32) fp32 storage; read as fp64 either way (exact widening).
struct BlockRef {
  const double* d;
  const float* f;
  __device__ __forceinline__ BlockRef at(std::uint64_t off) const {
    return BlockRef{d ? d + off : nullptr, f ? f + off : nullptr};
  }
};
// the kernels are instantiated per storage type (no per-element branch)
template <bool F32>
__device__ __forceinline__ double ldb(const BlockRef& b, std::size_t i) {
  if constexpr (F32)
    return static_cast<double>(__ldg(b.f + i));
  else
    return __ldg(b.d + i);
}

constexpr int kMaxDirect = 64;
constexpr int kLuThreads = 128;
constexpr int kMaxCols = 64;

struct LuParams {
  const std::uint32_t* bounds;
  const std::uint64_t* block_off;
  BlockRef blocks;
  const std::uint32_t* groups;  // small group ids
  const double* r;
  double* w;
  std::uint32_t k;              // row stride of R / W
  int nshift;
  double shift[kMaxCols];
  int col_start[kMaxCols + 1];  // columns of shift s: cols[col_start[s] .. col_start[s+1])
  int cols[kMaxCols];
  int* singular_count;
};

template <bool F32>
__device__ bool lu_factor(double* A, int n, int ld, int* perm, double mu, const BlockRef src,
                          double* red_v, int* red_i) {
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    double v = ldb<F32>(src, e);
    if (i == j) v = DSUB(v, mu);
    A[i + j * ld] = v;
  }
  for (int i = tid; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (tid < 32) {  // first occurrence of the largest |a_ik|, i >= k (one warp; a NaN never wins, a NaN at k keeps k)
      const double a0 = fabs(A[k + k * ld]);
      int p = k;
      if (a0 == a0) {
        double bv = -1.0;
        int bi = n;
        for (int i = k + tid; i < n; i += 32) {
          const double v = fabs(A[i + k * ld]);
          if (v > bv) {  // (false for NaN)
            bv = v;
            bi = i;
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        p = bi;
      }
      if (tid == 0) red_i[0] = p;
    }
    __syncthreads();
    const int p = red_i[0];
    if (p != k) {
      for (int j = tid; j < n; j += blockDim.x) {
        const double t = A[k + j * ld];
        A[k + j * ld] = A[p + j * ld];
        A[p + j * ld] = t;
      }
      if (tid == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double piv = A[k + k * ld];
    if (piv != 0.0)
      for (int i = k + 1 + tid; i < n; i += blockDim.x) A[i + k * ld] = DDIV(A[i + k * ld], piv);
    __syncthreads();
    const int m = n - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e % m, j = k + 1 + e / m;
      const double ukj = A[k + j * ld];
      if (ukj != 0.0) A[i + j * ld] = DSUB(A[i + j * ld], DMUL(A[i + k * ld], ukj));
    }
    __syncthreads();
  }
  if (tid == 0) {
    double mx = fabs(A[0]), mn = fabs(A[0]);
    for (int i = 1; i < n; ++i) {
      const double v = fabs(A[i + i * ld]);
      mx = v > mx ? v : mx;
      mn = v < mn ? v : mn;
    }
    const double scale = mx > 1e-300 ? mx : 1e-300;
    red_i[1] = (mn <= 1e-14 * scale) ? 1 : 0;
  }
  __syncthreads();
  (void)red_v;
  return red_i[1] == 0;
}

template <bool F32>
__global__ void __launch_bounds__(kLuThreads) lu_direct_kernel(const __grid_constant__ LuParams p) {
  __shared__ double A[kMaxDirect * (kMaxDirect + 1)];
  extern __shared__ double tmp_dyn[];  // [columns of this shift][kMaxDirect]
  __shared__ int perm[kMaxDirect];
  __shared__ double red_v[4];
  __shared__ int red_i[4];
  const std::uint32_t grp = p.groups[blockIdx.x];
  const int s = blockIdx.y;
  const std::uint32_t r0 = p.bounds[grp];
  const int n = static_cast<int>(p.bounds[grp + 1] - r0);
  const int ld = n + 1;
  const BlockRef src = p.blocks.at(p.block_off[grp]);
  double mu = p.shift[s];
  bool ok = lu_factor<F32>(A, n, ld, perm, mu, src, red_v, red_i);
  if (!ok) {
    mu = mu + 1e-8 * (1.0 + fabs(mu));
    ok = lu_factor<F32>(A, n, ld, perm, mu, src, red_v, red_i);
  }
  if (!ok) {  // pass-through: W keeps R for these columns
    if (threadIdx.x == 0) {
      atomicAdd(p.singular_count, 1);
    }
    return;
  }
  // Triangular solves for this shift's columns, every (row, column) on its
  // own thread and one barrier per step: the forward sweep column by column
  // (each t_i sees its updates in increasing k, as the row-oriented sweep),
  // the back substitution column by column from the last (dense_small.hpp).
  const int c0 = p.col_start[s], cnt = p.col_start[s + 1] - c0;
  double* t = tmp_dyn;                                                // [cnt][kMaxDirect]
  double* xs = tmp_dyn + static_cast<std::size_t>(cnt) * kMaxDirect;  // solutions
  const int tot = cnt * n;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int ci = e / n, i = e - ci * n;
    t[ci * kMaxDirect + i] = p.r[static_cast<std::size_t>(r0 + perm[i]) * p.k + p.cols[c0 + ci]];
  }
  __syncthreads();
  for (int kk = 0; kk + 1 < n; ++kk) {
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int ci = e / n, i = e - ci * n;
      if (i > kk) t[ci * kMaxDirect + i] = DSUB(t[ci * kMaxDirect + i], DMUL(A[i + kk * ld], t[ci * kMaxDirect + kk]));
    }
    __syncthreads();
  }
  for (int kk = n - 1; kk >= 0; --kk) {
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int ci = e / n, i = e - ci * n;
      const double xk = DDIV(t[ci * kMaxDirect + kk], A[kk + kk * ld]);
      if (i < kk)
        t[ci * kMaxDirect + i] = DSUB(t[ci * kMaxDirect + i], DMUL(A[i + kk * ld], xk));
      else if (i == kk)
        xs[ci * kMaxDirect + kk] = xk;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int ci = e / n, i = e - ci * n;
    p.w[static_cast<std::size_t>(r0 + i) * p.k + p.cols[c0 + ci]] = xs[ci * kMaxDirect + i];
  }
}

// ------------------------------------------------------------------ FOM
constexpr int kFomThreads = 256;
// fom_fast_kernel: 16 warps (each two 8-row m-tiles of the block product);
// its reductions keep the 16 row lanes of the first 256 threads
constexpr int kFomFastThreads = 512, kFomWarps = kFomFastThreads / 32, kFomMT = 256 / (8 * kFomWarps);
constexpr int kFomMaxSteps = 3;

struct FomParams {
  const std::uint32_t* bounds;
  const std::uint64_t* block_off;
  BlockRef blocks;
  const std::uint32_t* groups;  // large group ids
  const double* r;
  double* w;
  std::uint32_t k;
  int ncols;                     // engaged columns
  int chunk;                     // columns per CTA
  int iters;
  int cols[kMaxCols];
  double mu[kMaxCols];
};

// Small partial-pivot LU solve (dense_small.hpp order) of hm (m x m, col-major).
__device__ void tiny_lu_solve(double* hm, int m, double* rhs) {
  int perm[kFomMaxSteps];
  for (int i = 0; i < m; ++i) perm[i] = i;
  for (int k = 0; k < m; ++k) {
    int p = k;
    double best = fabs(hm[k + k * m]);
    for (int i = k + 1; i < m; ++i) {
      const double v = fabs(hm[i + k * m]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (p != k) {
      for (int j = 0; j < m; ++j) {
        const double t = hm[k + j * m];
        hm[k + j * m] = hm[p + j * m];
        hm[p + j * m] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    const double piv = hm[k + k * m];
    if (piv != 0.0)
      for (int i = k + 1; i < m; ++i) hm[i + k * m] = DDIV(hm[i + k * m], piv);
    for (int j = k + 1; j < m; ++j) {
      const double ukj = hm[k + j * m];
      if (ukj == 0.0) continue;
      for (int i = k + 1; i < m; ++i) hm[i + j * m] = DSUB(hm[i + j * m], DMUL(hm[i + k * m], ukj));
    }
  }
  double t[kFomMaxSteps];
  for (int i = 0; i < m; ++i) t[i] = rhs[perm[i]];
  for (int i = 0; i < m; ++i) {
    double s = t[i];
    for (int kk = 0; kk < i; ++kk) s = DSUB(s, DMUL(hm[i + kk * m], t[kk]));
    t[i] = s;
  }
  for (int kk = m - 1; kk >= 0; --kk) {  // column-oriented back substitution (dense_small.hpp order)
    const double xk = DDIV(t[kk], hm[kk + kk * m]);
    t[kk] = xk;
    for (int i = 0; i < kk; ++i) t[i] = DSUB(t[i], DMUL(hm[i + kk * m], xk));
  }
  for (int i = 0; i < m; ++i) rhs[i] = t[i];
}

template <bool F32>
__global__ void __launch_bounds__(kFomThreads) fom_kernel(const __grid_constant__ FomParams p) {
  extern __shared__ double sm[];
  const std::uint32_t grp = p.groups[blockIdx.x];
  const std::uint32_t r0 = p.bounds[grp];
  const int n = static_cast<int>(p.bounds[grp + 1] - r0);
  const int cbeg = blockIdx.y * p.chunk;
  const int cc = min(p.chunk, p.ncols - cbeg);
  const int CC = p.chunk;
  const int mmax = min(p.iters, n);
  // layout: basis[(mmax+1)][n][CC], wv[n][CC], hess[CC][4*3], beta[CC], flags
  double* basis = sm;
  double* wv = basis + static_cast<std::size_t>(mmax + 1) * n * CC;
  double* hess = wv + static_cast<std::size_t>(n) * CC;                 // CC * 16
  double* beta = hess + CC * 16;                                        // CC
  double* scal = beta + CC;                                             // CC (scale / norm scratch)
  int* active = reinterpret_cast<int*>(scal + CC);                      // CC
  int* steps = active + CC;                                             // CC
  int* done = steps + CC;                                               // CC: finished with m = done
  const BlockRef blk = p.blocks.at(p.block_off[grp]);
  const int tid = threadIdx.x;
  auto B = [&](int m, int i, int c) -> double& { return basis[(static_cast<std::size_t>(m) * n + i) * CC + c]; };

  // beta_j = ||rhs_j||, sequential order
  for (int c = tid; c < cc; c += blockDim.x) {
    const int j = p.cols[cbeg + c];
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
      const double v = p.r[static_cast<std::size_t>(r0 + i) * p.k + j];
      s = DADD(s, DMUL(v, v));
    }
    beta[c] = sqrt(s);
    active[c] = beta[c] != 0.0;
    steps[c] = 0;
    done[c] = 0;
    for (int e = 0; e < 16; ++e) hess[c * 16 + e] = 0.0;
  }
  __syncthreads();
  for (int e = tid; e < n * cc; e += blockDim.x) {
    const int i = e / cc, c = e - i * cc;
    const int j = p.cols[cbeg + c];
    const double v = p.r[static_cast<std::size_t>(r0 + i) * p.k + j];
    B(0, i, c) = beta[c] != 0.0 ? DDIV(v, beta[c]) : 0.0;
  }
  __syncthreads();

  const int H_LD = 4;  // hess[c] is (mmax+1) x mmax, column major, ld 4
  for (int m = 0; m < mmax; ++m) {
    // z = block * v_m for active columns (sequential k order per element)
    for (int i = tid; i < n; i += blockDim.x) {
      // z = block * v_m, k ascending per element (the reference's order);
      // 16 block entries are loaded ahead so the L2 latency is paid once per
      // 16 k. Columns are computed whether active or not (inactive ones are
      // never read), keeping the inner loop branch free.
      double z[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) z[c] = 0.0;
      const BlockRef brow = blk.at(i);
      int kk = 0;
      for (; kk + 16 <= n; kk += 16) {
        double a[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = ldb<F32>(brow, static_cast<std::size_t>(kk + u) * n);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double* bv = &B(m, kk + u, 0);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < cc) z[c] = DADD(z[c], DMUL(a[u], bv[c]));
        }
      }
      for (; kk < n; ++kk) {
        const double a = ldb<F32>(brow, static_cast<std::size_t>(kk) * n);
        const double* bv = &B(m, kk, 0);
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < cc) z[c] = DADD(z[c], DMUL(a, bv[c]));
      }
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < cc && active[c]) wv[i * CC + c] = DSUB(z[c], DMUL(p.mu[cbeg + c], B(m, i, c)));
    }
    __syncthreads();
    // scale = max(beta, ||w||)
    for (int c = tid; c < cc; c += blockDim.x) {
      if (!active[c]) continue;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = DADD(s, DMUL(wv[i * CC + c], wv[i * CC + c]));
      const double nw = sqrt(s);
      scal[c] = beta[c] > nw ? beta[c] : nw;
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (int ib = 0; ib <= m; ++ib) {
        for (int c = tid; c < cc; c += blockDim.x) {
          if (!active[c]) continue;
          double h = 0.0;
          for (int i = 0; i < n; ++i) h = DADD(h, DMUL(B(ib, i, c), wv[i * CC + c]));
          double& hh = hess[c * 16 + ib + m * H_LD];
          hh = pass == 0 ? h : DADD(hh, h);
          // stash h for the row update
          hess[c * 16 + 12 + (ib & 3)] = h;
        }
        __syncthreads();
        for (int e = tid; e < n * cc; e += blockDim.x) {
          const int i = e / cc, c = e - i * cc;
          if (!active[c]) continue;
          const double h = hess[c * 16 + 12 + (ib & 3)];
          wv[i * CC + c] = DSUB(wv[i * CC + c], DMUL(h, B(ib, i, c)));
        }
        __syncthreads();
      }
    }
    // norm, breakdown test, next basis vector
    for (int c = tid; c < cc; c += blockDim.x) {
      if (!active[c]) continue;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = DADD(s, DMUL(wv[i * CC + c], wv[i * CC + c]));
      const double nrm = sqrt(s);
      steps[c] = m + 1;
      const double sc = scal[c] > 1.0 ? scal[c] : 1.0;
      if (nrm <= 1e-12 * sc) {
        hess[c * 16 + (m + 1) + m * H_LD] = 0.0;
        active[c] = 0;
        done[c] = m + 1;  // lucky breakdown: finish with m+1 steps
      } else {
        hess[c * 16 + (m + 1) + m * H_LD] = nrm;
        scal[c] = nrm;
      }
    }
    __syncthreads();
    if (m + 1 <= mmax) {
      for (int e = tid; e < n * cc; e += blockDim.x) {
        const int i = e / cc, c = e - i * cc;
        if (!active[c]) continue;
        B(m + 1, i, c) = DDIV(wv[i * CC + c], scal[c]);
      }
    }
    __syncthreads();
  }
  // finish every column that ran (active ones with steps, and breakdowns)
  __shared__ double ycoef[kMaxCols][kFomMaxSteps];
  for (int c = tid; c < cc; c += blockDim.x) {
    const int m = done[c] ? done[c] : (active[c] ? steps[c] : 0);
    if (m == 0) {
      done[c] = 0;
      continue;
    }
    double hm[kFomMaxSteps * kFomMaxSteps];
    for (int a = 0; a < m; ++a)
      for (int b = 0; b < m; ++b) hm[a + b * m] = hess[c * 16 + a + b * H_LD];
    double rhs[kFomMaxSteps] = {0.0, 0.0, 0.0};
    rhs[0] = beta[c];
    tiny_lu_solve(hm, m, rhs);
    for (int a = 0; a < m; ++a) ycoef[c][a] = rhs[a];
    done[c] = m;
  }
  __syncthreads();
  for (int e = tid; e < n * cc; e += blockDim.x) {
    const int i = e / cc, c = e - i * cc;
    const int j = p.cols[cbeg + c];
    const int m = done[c];
    double x = 0.0;
    for (int a = 0; a < m; ++a) x = DADD(x, DMUL(B(a, i, c), ycoef[c][a]));
    p.w[static_cast<std::size_t>(r0 + i) * p.k + j] = x;
  }
}


// ------------------------------------------------------------ fast FOM
// Same algorithm (fom_solve, precond.cpp:87-158) with the block products on
// the FP64 tensor pipe (DMMA m8n8k4, block entries streamed from L2/HBM with
// 4 k-steps of loads in flight) and every dot product / norm a parallel
// fixed-order reduction. Deterministic, but the summation order differs from
// the reference's sequential loops (results agree to ~1e-16 relative); the
// reference-order kernel above is selected with cieg_ctx_set_exact_order.
constexpr int kFastSC = 20;  // smem row stride of basis / w (doubles), 4 mod 16

__device__ __forceinline__ double fom_col_reduce(double part, double* red, int c_of_t, int rsub, int cc) {
  // part: this thread's partial for column c_of_t (t & 15), row lane rsub (t >> 4);
  // threads beyond the first 256 (16 row lanes) only join the barriers
  if (threadIdx.x < 256) red[rsub * 16 + c_of_t] = part;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 16) {
    for (int k = 0; k < 16; ++k) s += red[k * 16 + threadIdx.x];
    red[256 + threadIdx.x] = s;
  }
  __syncthreads();
  const double out = red[256 + c_of_t];
  __syncthreads();
  (void)cc;
  return out;
}

template <bool F32>
__global__ void __launch_bounds__(kFomFastThreads) fom_fast_kernel(const __grid_constant__ FomParams p) {
  extern __shared__ double sm[];
  const std::uint32_t grp = p.groups[blockIdx.x];
  const std::uint32_t r0 = p.bounds[grp];
  const int n = static_cast<int>(p.bounds[grp + 1] - r0);
  const int NP = (n + 7) & ~7;
  const int cbeg = blockIdx.y * p.chunk;
  const int cc = min(p.chunk, p.ncols - cbeg);
  const int mmax = min(p.iters, n);
  double* basis = sm;                                                  // (mmax+1) x NP x SC
  double* wv = basis + static_cast<std::size_t>(mmax + 1) * NP * kFastSC;  // NP x SC
  double* red = wv + static_cast<std::size_t>(NP) * kFastSC;          // 256 + 16
  double* hess = red + 272;                                            // 16 x 16
  double* beta = hess + 256;                                           // 16
  double* scal = beta + 16;                                            // 16
  double* hcol = scal + 16;                                            // 16
  int* state = reinterpret_cast<int*>(hcol + 16);                      // active[16], steps[16], done[16]
  int* active = state;
  int* steps = state + 16;
  int* done = state + 32;
  const BlockRef blk = p.blocks.at(p.block_off[grp]);
  const int tid = threadIdx.x;
  const int tc = tid & 15, trow = tid >> 4;
  auto B = [&](int m, int i, int c) -> double& { return basis[(static_cast<std::size_t>(m) * NP + i) * kFastSC + c]; };
  auto W = [&](int i, int c) -> double& { return wv[i * kFastSC + c]; };
  const bool tcol = tc < cc;
  const int jcol = tcol ? p.cols[cbeg + tc] : 0;

  // beta_j = ||rhs_j||; basis_0 = rhs / beta (rows >= n zero)
  double part = 0.0;
  for (int i = trow; i < n && tid < 256; i += 16) {
    const double v = tcol ? p.r[static_cast<std::size_t>(r0 + i) * p.k + jcol] : 0.0;
    part = fma(v, v, part);
  }
  const double bsq = fom_col_reduce(part, red, tc, trow, cc);
  if (tid < 16) {
    beta[tid] = sqrt(bsq);
    active[tid] = (tid < cc && beta[tid] != 0.0) ? 1 : 0;
    steps[tid] = 0;
    done[tid] = 0;
  }
  for (int e = tid; e < 256; e += blockDim.x) hess[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < NP * 16; e += blockDim.x) {
    const int i = e >> 4, c = e & 15;
    double v = 0.0;
    if (i < n && c < cc && beta[c] != 0.0) v = p.r[static_cast<std::size_t>(r0 + i) * p.k + p.cols[cbeg + c]] / beta[c];
    B(0, i, c) = v;
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int mtiles = NP / 8;
  for (int m = 0; m < mmax; ++m) {
    // z = block * v_m on the tensor pipe; warp w owns m-tiles w, w+8, w+16, w+24
    double acc[kFomMT][2][2];
#pragma unroll
    for (int a = 0; a < kFomMT; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // A fragments (raw storage type) are prefetched three 16-wide k chunks
    // ahead and widened at use, so global latency overlaps the DMMAs
    using Raw = typename std::conditional<F32, float, double>::type;
    const Raw* blk_raw = F32 ? reinterpret_cast<const Raw*>(blk.f) : reinterpret_cast<const Raw*>(blk.d);
    Raw a0[4][kFomMT], a1[4][kFomMT];
    auto load_a = [&](int k0, Raw (&dst)[4][kFomMT]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k0 + 4 * u + q;
#pragma unroll
        for (int a = 0; a < kFomMT; ++a) {
          const int mt = warp + kFomWarps * a;
          const int i = 8 * mt + g;
          dst[u][a] = (k0 < NP && mt < mtiles && i < n && kk < n) ? __ldg(blk_raw + i + static_cast<std::size_t>(kk) * n)
                                                                  : Raw(0);
        }
      }
    };
    auto mma_chunk = [&](int k0, const Raw (&src)[4][kFomMT]) {
      if (k0 >= NP) return;
      double bf[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int b = 0; b < 2; ++b) bf[u][b] = (k0 + 4 * u < NP) ? B(m, k0 + 4 * u + q, 8 * b + g) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int a = 0; a < kFomMT; ++a) {
          const double av = static_cast<double>(src[u][a]);
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], av, bf[u][b]);
        }
    };
    // four 16-wide k chunks in flight (loads three chunks ahead of the DMMAs)
    Raw a2[4][kFomMT], a3[4][kFomMT];
    load_a(0, a0);
    load_a(16, a1);
    load_a(32, a2);
    for (int k0 = 0; k0 < NP; k0 += 64) {
      load_a(k0 + 48, a3);
      mma_chunk(k0, a0);
      load_a(k0 + 64, a0);
      mma_chunk(k0 + 16, a1);
      load_a(k0 + 80, a1);
      mma_chunk(k0 + 32, a2);
      load_a(k0 + 96, a2);
      mma_chunk(k0 + 48, a3);
    }
    // w = z - mu v_m
#pragma unroll
    for (int a = 0; a < kFomMT; ++a) {
      const int mt = warp + kFomWarps * a;
      if (mt >= mtiles) continue;
      const int i = 8 * mt + g;
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 8 * b + 2 * q + h;
          const double mu = c < cc ? p.mu[cbeg + c] : 0.0;
          W(i, c) = (i < n) ? acc[a][b][h] - mu * B(m, i, c) : 0.0;
        }
    }
    __syncthreads();
    // scale = max(beta, ||w||)
    part = 0.0;
    for (int i = trow; i < n && tid < 256; i += 16) part = fma(W(i, tc), W(i, tc), part);
    const double wn = sqrt(fom_col_reduce(part, red, tc, trow, cc));
    if (tid < 16) scal[tid] = beta[tid] > wn ? beta[tid] : wn;
    // two-pass modified Gram-Schmidt
    for (int pass = 0; pass < 2; ++pass) {
      for (int ib = 0; ib <= m; ++ib) {
        part = 0.0;
        for (int i = trow; i < n && tid < 256; i += 16) part = fma(B(ib, i, tc), W(i, tc), part);
        const double hv = fom_col_reduce(part, red, tc, trow, cc);
        if (tid < 16 && active[tid]) {
          double& hh = hess[tid * 16 + ib + m * 4];
          hh = pass == 0 ? hv : hh + hv;
          hcol[tid] = hv;
        }
        __syncthreads();
        for (int e = tid; e < n * 16; e += blockDim.x) {
          const int i = e >> 4, c = e & 15;
          if (c < cc && active[c]) W(i, c) -= hcol[c] * B(ib, i, c);
        }
        __syncthreads();
      }
    }
    part = 0.0;
    for (int i = trow; i < n && tid < 256; i += 16) part = fma(W(i, tc), W(i, tc), part);
    const double nrm = sqrt(fom_col_reduce(part, red, tc, trow, cc));
    if (tid < 16 && active[tid]) {
      steps[tid] = m + 1;
      const double sc = scal[tid] > 1.0 ? scal[tid] : 1.0;
      if (nrm <= 1e-12 * sc) {
        hess[tid * 16 + (m + 1) + m * 4] = 0.0;
        active[tid] = 0;
        done[tid] = m + 1;
      } else {
        hess[tid * 16 + (m + 1) + m * 4] = nrm;
        scal[tid] = nrm;
      }
    }
    __syncthreads();
    for (int e = tid; e < NP * 16; e += blockDim.x) {
      const int i = e >> 4, c = e & 15;
      if (c < cc && active[c]) B(m + 1, i, c) = (i < n) ? W(i, c) / scal[c] : 0.0;
    }
    __syncthreads();
  }
  __shared__ double ycoef[16][kFomMaxSteps];
  if (tid < 16) {
    const int c = tid;
    const int m = c < cc ? (done[c] ? done[c] : (active[c] ? steps[c] : 0)) : 0;
    if (m > 0) {
      double hm[kFomMaxSteps * kFomMaxSteps];
      for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b) hm[a + b * m] = hess[c * 16 + a + b * 4];
      double rhs[kFomMaxSteps] = {0.0, 0.0, 0.0};
      rhs[0] = beta[c];
      tiny_lu_solve(hm, m, rhs);
      for (int a = 0; a < m; ++a) ycoef[c][a] = rhs[a];
    }
    done[c] = m;
  }
  __syncthreads();
  for (int e = tid; e < n * 16; e += blockDim.x) {
    const int i = e >> 4, c = e & 15;
    if (c >= cc) continue;
    const int m = done[c];
    double x = 0.0;
    for (int a = 0; a < m; ++a) x = fma(B(a, i, c), ycoef[c][a], x);
    p.w[static_cast<std::size_t>(r0 + i) * p.k + p.cols[cbeg + c]] = x;
  }
}

}  // namespace

int precond_apply(cieg_ctx* ctx, const cieg_prec* prec, const double* r, std::uint32_t k,
                  const ShiftPlan& plan, const cieg_precond_config& cfg, double* w, int* singular_accum) {
  const std::size_t bytes = static_cast<std::size_t>(prec->dim) * k * sizeof(double);
  if (w != r && bytes) CIEG_CUDA(cudaMemcpyAsync(w, r, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  std::vector<int> engaged;
  for (std::uint32_t j = 0; j < k; ++j)
    if (plan.engage[j]) engaged.push_back(static_cast<int>(j));
  if (engaged.empty() || prec->ngroups == 0) return 0;
  if (engaged.size() > static_cast<std::size_t>(kMaxCols)) fail(CIEG_ERR_CONFIG, "preconditioner: more than 64 columns");
  if (cfg.inner_iters < 1) fail(CIEG_ERR_CONFIG, "fom_solve: iters must be >= 1");

  if (prec->lists_cutoff != cfg.small_block_cutoff) {
    prec->small_host.clear();
    prec->large_host.clear();
    for (std::uint32_t g = 0; g < prec->ngroups; ++g) {
      const std::uint32_t sz = prec->bounds_host[g + 1] - prec->bounds_host[g];
      if (sz == 0) continue;
      (static_cast<int>(sz) <= cfg.small_block_cutoff ? prec->small_host : prec->large_host).push_back(g);
    }
    std::vector<std::uint32_t> all(prec->small_host);
    all.insert(all.end(), prec->large_host.begin(), prec->large_host.end());
    all.resize(all.size() + 2, 0u);  // + the int counter slot (kept 8-byte aligned)
    if (all.size() & 1) all.push_back(0u);
    cudaFree(prec->lists);
    prec->lists = nullptr;
    CIEG_CUDA(cudaMalloc(&prec->lists, sizeof(std::uint32_t) * all.size()));
    CIEG_CUDA(cudaMemcpy(prec->lists, all.data(), sizeof(std::uint32_t) * all.size(), cudaMemcpyHostToDevice));
    prec->lists_cutoff = cfg.small_block_cutoff;
  }
  const std::vector<std::uint32_t>& small = prec->small_host;
  const std::vector<std::uint32_t>& large = prec->large_host;
  std::uint32_t* dgroups = prec->lists;
  int* dcount = singular_accum ? singular_accum
                               : reinterpret_cast<int*>(dgroups + ((small.size() + large.size() + 1) & ~std::size_t{1}));
  if (!singular_accum) CIEG_CUDA(cudaMemsetAsync(dcount, 0, sizeof(int), ctx->stream));

  if (!small.empty()) {
    if (cfg.small_block_cutoff > kMaxDirect && prec->max_group > static_cast<std::uint32_t>(kMaxDirect))
      fail(CIEG_ERR_CONFIG, "direct tile solve supports groups up to 64 rows");
    static thread_local LuParams lp;
    lp.bounds = prec->bounds;
    lp.block_off = prec->block_off;
    lp.blocks = BlockRef{prec->blocks, prec->blocks32};
    lp.groups = dgroups;
    lp.r = r;
    lp.w = w;
    lp.k = k;
    lp.singular_count = dcount;
    std::map<double, std::vector<int>> by_shift;  // ascending, like the reference's std::map
    for (int j : engaged) by_shift[plan.mu[j]].push_back(j);
    lp.nshift = static_cast<int>(by_shift.size());
    int s = 0, o = 0;
    for (auto& [mu, cols] : by_shift) {
      lp.shift[s] = mu;
      lp.col_start[s] = o;
      for (int j : cols) lp.cols[o++] = j;
      ++s;
    }
    lp.col_start[s] = o;
    int maxcols = 0;
    for (int t = 0; t < lp.nshift; ++t) maxcols = std::max(maxcols, lp.col_start[t + 1] - lp.col_start[t]);
    const std::size_t smem = 2 * sizeof(double) * static_cast<std::size_t>(maxcols) * kMaxDirect;
    dim3 grid(static_cast<unsigned>(small.size()), static_cast<unsigned>(lp.nshift));
    auto lu = prec->blocks32 ? lu_direct_kernel<true> : lu_direct_kernel<false>;
    CIEG_CUDA(cudaFuncSetAttribute(lu, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    lu<<<grid, kLuThreads, smem, ctx->stream>>>(lp);
    CIEG_CUDA(cudaGetLastError());
    ++ctx->launches;
  }
  if (!large.empty()) {
    static thread_local FomParams fp;
    fp.bounds = prec->bounds;
    fp.block_off = prec->block_off;
    fp.blocks = BlockRef{prec->blocks, prec->blocks32};
    fp.groups = dgroups + small.size();
    fp.r = r;
    fp.w = w;
    fp.k = k;
    fp.ncols = static_cast<int>(engaged.size());
    fp.iters = cfg.inner_iters;
    for (std::size_t c = 0; c < engaged.size(); ++c) {
      fp.cols[c] = engaged[c];
      fp.mu[c] = plan.mu[engaged[c]];
    }
    const int mmax = std::min<int>(cfg.inner_iters, static_cast<int>(prec->max_group));
    if (mmax > kFomMaxSteps) fail(CIEG_ERR_CONFIG, "fom_solve: inner_iters above 3 is not supported");
    const std::size_t n = prec->max_group;
    if (!ctx->exact_order && n <= 256) {
      // fast path: DMMA block products, parallel fixed-order reductions
      const int chunk = 16;
      fp.chunk = chunk;
      const std::size_t np8 = (n + 7) & ~std::size_t{7};
      const std::size_t smem = sizeof(double) * ((mmax + 1) * np8 * kFastSC + np8 * kFastSC + 272 + 256 + 48) +
                               sizeof(int) * 48;
      auto fom = prec->blocks32 ? fom_fast_kernel<true> : fom_fast_kernel<false>;
      CIEG_CUDA(cudaFuncSetAttribute(fom, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      dim3 grid(static_cast<unsigned>(large.size()), static_cast<unsigned>((fp.ncols + chunk - 1) / chunk));
      fom<<<grid, kFomFastThreads, smem, ctx->stream>>>(fp);
    } else {
      // reference-order path: chunk so that shared memory stays below ~200 KB
      int chunk = 16;
      auto smem_for = [&](int cc) {
        return sizeof(double) * ((mmax + 1) * n * cc + n * cc + cc * 16 + 2 * cc) + sizeof(int) * 3 * cc;
      };
      while (chunk > 1 && smem_for(chunk) > 200 * 1024) chunk /= 2;
      if (smem_for(chunk) > 220 * 1024) fail(CIEG_ERR_CONFIG, "FOM tile too large for shared memory");
      fp.chunk = chunk;
      const std::size_t smem = smem_for(chunk);
      auto fom = prec->blocks32 ? fom_kernel<true> : fom_kernel<false>;
      CIEG_CUDA(cudaFuncSetAttribute(fom, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      dim3 grid(static_cast<unsigned>(large.size()), static_cast<unsigned>((fp.ncols + chunk - 1) / chunk));
      fom<<<grid, kFomThreads, smem, ctx->stream>>>(fp);
    }
    CIEG_CUDA(cudaGetLastError());
    ++ctx->launches;
  }
  if (singular_accum) return 0;
  int* pin = static_cast<int*>(ctx->pinned_small.get(sizeof(double) * 48 * 48));
  CIEG_CUDA(cudaMemcpyAsync(pin, dcount, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  const int singular = pin[0];
  for (int i = 0; i < singular; ++i)
    std::fprintf(stderr, "ci-eigen: singular shifted tile block; passing residual through\n");
  return singular;
}

}  // namespace cieg

namespace {

cieg_prec* make_prec(cieg_ctx* ctx, std::uint32_t dim, std::uint32_t ng, const std::uint32_t* bounds,
                     const double* blocks_host) {
  if (ng > 0 && (bounds[0] != 0 || bounds[ng] != dim))
    cieg::fail(CIEG_ERR_DIMENSION, "apply_preconditioner: tiles do not cover the basis");
  auto* p = new cieg_prec;
  try {
    p->ctx = ctx;
    p->dim = dim;
    p->ngroups = ng;
    p->bounds_host.assign(bounds, bounds + ng + 1);
    p->block_off_host.resize(ng + 1, 0);
    for (std::uint32_t g = 0; g < ng; ++g) {
      const std::uint64_t sz = bounds[g + 1] - bounds[g];
      p->max_group = std::max<std::uint32_t>(p->max_group, static_cast<std::uint32_t>(sz));
      p->block_off_host[g + 1] = p->block_off_host[g] + sz * sz;
    }
    CIEG_CUDA(cudaMalloc(&p->bounds, sizeof(std::uint32_t) * (ng + 1)));
    CIEG_CUDA(cudaMemcpy(p->bounds, bounds, sizeof(std::uint32_t) * (ng + 1), cudaMemcpyHostToDevice));
    CIEG_CUDA(cudaMalloc(&p->block_off, sizeof(std::uint64_t) * (ng + 1)));
    CIEG_CUDA(cudaMemcpy(p->block_off, p->block_off_host.data(), sizeof(std::uint64_t) * (ng + 1),
                         cudaMemcpyHostToDevice));
    const std::uint64_t total = p->block_off_host[ng];
    CIEG_CUDA(cudaMalloc(&p->blocks, sizeof(double) * std::max<std::uint64_t>(total, 1)));
    if (total)
      CIEG_CUDA(cudaMemcpy(p->blocks, blocks_host, sizeof(double) * total, cudaMemcpyHostToDevice));
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

}  // namespace

extern "C" {

void cieg_precond_config_default(cieg_precond_config* c) {
  if (!c) return;
  c->inner_iters = 3;
  c->small_block_cutoff = 64;
  c->engage_after = 3;
  c->relres_gate = 1e-1;
  c->near_converged_factor = 10.0;
  c->far_threshold = 1e-2;
  c->column_floor_factor = 100.0;
}

int cieg_precond_upload(cieg_ctx* ctx, const cieg_tilediag_view* t, cieg_prec** out) {
  return cieg::guarded([&] {
    if (!ctx || !t || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_precond_upload: null argument");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    *out = make_prec(ctx, t->dim, t->ngroups, t->bounds, t->blocks);
  });
}

}  // extern "C"

namespace {

// ci::extract_tile_diagonal (hamiltonian.cpp:178-203): dense f64 blocks from
// the diagonal CSB blocks, mirrored; restricted to the groups inside
// [row_lo, row_hi) with local row numbering (a shard's preconditioner).
cieg_prec* prec_from_csb(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* gb, uint32_t ng, uint32_t row_lo,
                         uint32_t row_hi) {
  const std::uint32_t dim = csb->dim;
  if (gb[0] != 0 || gb[ng] != dim) cieg::fail(CIEG_ERR_DIMENSION, "group bounds do not cover [0, dim)");
  std::uint32_t g0 = 0, g1 = 0;
  while (g0 < ng && gb[g0] < row_lo) ++g0;
  g1 = g0;
  while (g1 < ng && gb[g1 + 1] <= row_hi) ++g1;
  if (gb[g0] != row_lo || gb[g1] != row_hi) cieg::fail(CIEG_ERR_CONFIG, "shard rows are not group boundaries");
  const std::uint32_t lng = g1 - g0;
  std::vector<std::uint32_t> lb(lng + 1);
  for (std::uint32_t g = 0; g <= lng; ++g) lb[g] = gb[g0 + g] - row_lo;
  std::vector<std::uint32_t> group_of(dim, 0xffffffffu);
  std::vector<std::uint64_t> off(lng + 1, 0);
  for (std::uint32_t g = 0; g < lng; ++g) {
    const std::uint64_t sz = lb[g + 1] - lb[g];
    off[g + 1] = off[g] + sz * sz;
    for (std::uint32_t r = gb[g0 + g]; r < gb[g0 + g + 1]; ++r) group_of[r] = g;
  }
  std::vector<double> blocks(off[lng], 0.0);
  const float* v32 = static_cast<const float*>(csb->values);
  const double* v64 = static_cast<const double*>(csb->values);
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t i64 = 0; i64 < static_cast<std::int64_t>(csb->nb); ++i64) {
    const std::uint32_t i = static_cast<std::uint32_t>(i64);
    const std::uint32_t base = csb->block_boundaries[i];
    if (csb->block_boundaries[i + 1] <= row_lo || base >= row_hi) continue;
    const std::uint64_t bid = static_cast<std::uint64_t>(i) * (i + 1) / 2 + i;
    for (std::uint64_t e = csb->entry_offsets[bid]; e < csb->entry_offsets[bid + 1]; ++e) {
      const std::uint32_t r = base + csb->rows[e], c = base + csb->cols[e];
      const std::uint32_t g = group_of[r];
      if (g == 0xffffffffu || group_of[c] != g) continue;
      const std::uint32_t s = gb[g0 + g];
      const std::uint64_t n = lb[g + 1] - lb[g];
      const double v = csb->precision == 0 ? static_cast<double>(v32[e]) : v64[e];
      blocks[off[g] + (r - s) + (c - s) * n] = v;
      blocks[off[g] + (c - s) + (r - s) * n] = v;
    }
  }
  return make_prec(ctx, row_hi - row_lo, lng, lb.data(), blocks.data());
}

}  // namespace

extern "C" {

int cieg_precond_from_csb(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* gb, uint32_t ng,
                          cieg_prec** out) {
  return cieg::guarded([&] {
    if (!ctx || !csb || !gb || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_precond_from_csb: null argument");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    *out = prec_from_csb(ctx, csb, gb, ng, 0, csb->dim);
  });
}

int cieg_precond_from_csb_range(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* gb, uint32_t ng,
                                uint32_t row_lo, uint32_t row_hi, cieg_prec** out) {
  return cieg::guarded([&] {
    if (!ctx || !csb || !gb || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_precond_from_csb_range: null argument");
    if (row_lo >= row_hi || row_hi > csb->dim) cieg::fail(CIEG_ERR_DIMENSION, "range outside [0, dim)");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    *out = prec_from_csb(ctx, csb, gb, ng, row_lo, row_hi);
  });
}

int cieg_precond_destroy(cieg_prec* p) {
  if (p) {
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    delete p;
  }
  return CIEG_OK;
}

int cieg_choose_shifts(uint32_t k, const double* theta, const double* res_norm, const double* x_norm,
                       const double* relres, int iteration, double tol, const cieg_precond_config* cfg,
                       double* mu_out, int* engage_out) {
  return cieg::guarded([&] {
    cieg_precond_config c;
    if (cfg)
      c = *cfg;
    else
      cieg_precond_config_default(&c);
    auto plan = cieg::choose_shifts(std::vector<double>(theta, theta + k), std::vector<double>(res_norm, res_norm + k),
                                    std::vector<double>(x_norm, x_norm + k), std::vector<double>(relres, relres + k),
                                    iteration, tol, c);
    for (uint32_t j = 0; j < k; ++j) {
      mu_out[j] = plan.mu[j];
      engage_out[j] = plan.engage[j];
    }
  });
}

int cieg_precond_apply(cieg_ctx* ctx, const cieg_prec* prec, const double* r_dev, uint32_t k,
                       const double* mu_host, const int* engage_host, const cieg_precond_config* cfg,
                       double* w_dev) {
  return cieg::guarded([&] {
    if (!ctx || !prec) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_precond_apply: null handle");
    cieg_precond_config c;
    if (cfg)
      c = *cfg;
    else
      cieg_precond_config_default(&c);
    cieg::ShiftPlan plan;
    plan.mu.assign(mu_host, mu_host + k);
    plan.engage.assign(engage_host, engage_host + k);
    cieg::precond_apply(ctx, prec, r_dev, k, plan, c, w_dev);
  });
}

}  // extern "C"
