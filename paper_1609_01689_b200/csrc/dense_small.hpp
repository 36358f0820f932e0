// dense_small.hpp -- small dense symmetric/LU kernels used on the host side of
// the LOBPCG path (projected eigenproblem <= 3*k_trial, Cholesky factors of
// <= 48x48 Gram panels, <= 64x64 tile LUs, FOM Hessenberg solves).
//
// The reference delegates these to Eigen 3 (proj/src/lobpcg.cpp:54-85,
// proj/src/precond.cpp:61-83,116,130). Eigen is not part of this image, so
// this header restates the published algorithms Eigen uses for the same
// entry points:
//   * SelfAdjointEigenSolver  -> Householder tridiagonalisation followed by
//     the implicit-shift QL iteration; eigenvalues ascending, eigenvectors
//     orthonormal columns (ties broken by input order, stable sort).
//   * LLT                     -> unblocked right-looking Cholesky; fails iff a
//     pivot is <= 0 (Eigen's llt_inplace rule; NaN pivots pass through).
//   * PartialPivLU            -> row partial pivoting on max |a_ik|; never
//     "fails" -- callers inspect |U_ii| (precond.cpp:66-68).
//   * triangularView<Upper>().solve -> back substitution.
// Storage is column major (Eigen's default) with leading dimension = rows.
//
// Both the GPU solver host loop (paper_1609_01689_b200/csrc/solver.cpp) and
// the Eigen-API shim used to build the reference oracle include this header,
// so control-flow decisions that hinge on these factorizations (column drops,
// LLT failures, singular shifts) are taken by identical code on both sides.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <numeric>
#include <vector>

namespace cieg_dense {

using Index = std::ptrdiff_t;

// Implicit QL on a symmetric tridiagonal (tql2): d diagonal, e[i] the entry
// coupling i-1 and i (e[0] unused); the rotations are accumulated into V
// (rows x n col-major: the tridiagonalising transform, the identity, or any
// subset of its rows -- every row is updated independently, so tracking one
// row yields exactly that row of the full result). Writes ascending
// eigenvalues w and the rows x n eigenvector rows z (stable order on ties).
inline bool tql2_sorted(Index n, std::vector<double>& d, std::vector<double>& e, std::vector<double>& V, double* w,
                        double* z, Index rows = -1) {
  if (rows < 0) rows = n;
  auto v = [&](Index i, Index j) -> double& { return V[static_cast<size_t>(i + j * rows)]; };
  for (Index i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = std::ldexp(1.0, -52);
  for (Index l = 0; l < n; ++l) {
    tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
    Index m = l;
    while (m < n) {
      if (std::fabs(e[m]) <= eps * tst1) break;
      ++m;
    }
    if (m == n) m = n - 1;
    if (m > l) {
      int iter = 0;
      do {
        if (++iter > 60) return false;
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = std::hypot(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        double dl1 = d[l + 1];
        double h = g - d[l];
        for (Index i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        p = d[m];
        double c = 1.0, c2 = c, c3 = c;
        double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (Index i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = std::hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          for (Index k = 0; k < rows; ++k) {
            h = v(k, i + 1);
            v(k, i + 1) = s * v(k, i) + c * h;
            v(k, i) = c * v(k, i) - s * h;
          }
          if (i == 0) break;
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (std::fabs(e[l]) > eps * tst1);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
  // Stable ascending sort of eigenpairs.
  std::vector<Index> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), Index{0});
  std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return d[x] < d[y]; });
  for (Index j = 0; j < n; ++j) {
    w[j] = d[order[j]];
    for (Index i = 0; i < rows; ++i) z[i + j * rows] = v(i, order[j]);
  }
  return true;
}

// a: n x n column-major symmetric (only the lower triangle is read).
// On return: w ascending eigenvalues, z (n x n col-major) eigenvectors.
// Returns false if the QL iteration fails to converge.
inline bool sym_eig(Index n, const double* a, double* w, double* z) {
  if (n == 0) return true;
  std::vector<double> V(static_cast<size_t>(n * n));
  auto v = [&](Index i, Index j) -> double& { return V[static_cast<size_t>(i + j * n)]; };
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) v(i, j) = (i >= j) ? a[i + j * n] : a[j + i * n];
  std::vector<double> d(static_cast<size_t>(n)), e(static_cast<size_t>(n), 0.0);

  // Householder reduction to tridiagonal form (tred2 ordering: last row first).
  for (Index j = 0; j < n; ++j) d[j] = v(n - 1, j);
  for (Index i = n - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (Index k = 0; k < i; ++k) scale += std::fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (Index j = 0; j < i; ++j) {
        d[j] = v(i - 1, j);
        v(i, j) = 0.0;
        v(j, i) = 0.0;
      }
    } else {
      for (Index k = 0; k < i; ++k) {
        d[k] /= scale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = std::sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h = h - f * g;
      d[i - 1] = f - g;
      for (Index j = 0; j < i; ++j) e[j] = 0.0;
      for (Index j = 0; j < i; ++j) {
        f = d[j];
        v(j, i) = f;
        g = e[j] + v(j, j) * f;
        for (Index k = j + 1; k <= i - 1; ++k) {
          g += v(k, j) * d[k];
          e[k] += v(k, j) * f;
        }
        e[j] = g;
      }
      f = 0.0;
      for (Index j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      double hh = f / (h + h);
      for (Index j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (Index j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        for (Index k = j; k <= i - 1; ++k) v(k, j) -= (f * e[k] + g * d[k]);
        d[j] = v(i - 1, j);
        v(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
  // Accumulate transformations.
  for (Index i = 0; i < n - 1; ++i) {
    v(n - 1, i) = v(i, i);
    v(i, i) = 1.0;
    double h = d[i + 1];
    if (h != 0.0) {
      for (Index k = 0; k <= i; ++k) d[k] = v(k, i + 1) / h;
      for (Index j = 0; j <= i; ++j) {
        double g = 0.0;
        for (Index k = 0; k <= i; ++k) g += v(k, i + 1) * v(k, j);
        for (Index k = 0; k <= i; ++k) v(k, j) -= g * d[k];
      }
    }
    for (Index k = 0; k <= i; ++k) v(k, i + 1) = 0.0;
  }
  for (Index j = 0; j < n; ++j) {
    d[j] = v(n - 1, j);
    v(n - 1, j) = 0.0;
  }
  v(n - 1, n - 1) = 1.0;
  e[0] = 0.0;

  return tql2_sorted(n, d, e, V, w, z);
}

// Symmetric tridiagonal eigenproblem (diag n, sub n-1); QL with eigenvectors
// accumulated from the identity. Used by Lanczos (lanczos.cpp:54-63).
inline bool tridiag_eig(Index n, const double* diag, const double* sub, double* w, double* z) {
  // Eigen's computeFromTridiagonal: the QL iteration straight on the
  // tridiagonal, rotations accumulated from the identity (no reduction step).
  if (n == 0) return true;
  std::vector<double> d(diag, diag + n), e(static_cast<size_t>(n), 0.0), V(static_cast<size_t>(n * n), 0.0);
  for (Index i = 1; i < n; ++i) e[i] = sub[i - 1];
  for (Index i = 0; i < n; ++i) V[static_cast<size_t>(i + i * n)] = 1.0;
  return tql2_sorted(n, d, e, V, w, z);
}

// Eigenvalues and the BOTTOM row of the eigenvector matrix of a tridiagonal
// (what the Lanczos residual test reads, lanczos.cpp:112-114) in O(n^2):
// bitwise equal to the last row of tridiag_eig's z.
inline bool tridiag_eig_bottom(Index n, const double* diag, const double* sub, double* w, double* zlast) {
  if (n == 0) return true;
  std::vector<double> d(diag, diag + n), e(static_cast<size_t>(n), 0.0), V(static_cast<size_t>(n), 0.0);
  for (Index i = 1; i < n; ++i) e[i] = sub[i - 1];
  V[static_cast<size_t>(n - 1)] = 1.0;
  return tql2_sorted(n, d, e, V, w, zlast, 1);
}

// In-place Cholesky a = L L^T of the lower triangle (column major); on success
// the strict upper triangle is zeroed and the lower holds L. Returns false
// iff a pivot is <= 0 (Eigen LLT semantics).
inline bool cholesky_lower(Index n, double* a) {
  for (Index k = 0; k < n; ++k) {
    double x = a[k + k * n];
    for (Index j = 0; j < k; ++j) x -= a[k + j * n] * a[k + j * n];
    if (x <= 0.0) return false;
    x = std::sqrt(x);
    a[k + k * n] = x;
    for (Index i = k + 1; i < n; ++i) {
      double s = a[i + k * n];
      for (Index j = 0; j < k; ++j) s -= a[i + j * n] * a[k + j * n];
      a[i + k * n] = s / x;
    }
  }
  for (Index j = 1; j < n; ++j)
    for (Index i = 0; i < j; ++i) a[i + j * n] = 0.0;
  return true;
}

// Inverse of an upper-triangular r (n x n, column major) by back substitution
// against the identity (lobpcg.cpp:55-56).
inline void upper_inverse(Index n, const double* r, double* out) {
  std::fill(out, out + n * n, 0.0);
  for (Index c = 0; c < n; ++c) {
    for (Index i = n - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (Index k = i + 1; k < n; ++k) s -= r[i + k * n] * out[k + c * n];
      out[i + c * n] = s / r[i + i * n];
    }
  }
}

// General back substitution U X = B (upper, column major), B n x m in place.
inline void upper_solve(Index n, const double* r, Index m, double* b) {
  for (Index c = 0; c < m; ++c)
    for (Index i = n - 1; i >= 0; --i) {
      double s = b[i + c * n];
      for (Index k = i + 1; k < n; ++k) s -= r[i + k * n] * b[k + c * n];
      b[i + c * n] = s / r[i + i * n];
    }
}

// Partial-pivot LU in place: P A = L U, unit L below the diagonal.
// perm[i] = original row placed at position i.
inline void lu_partial_pivot(Index n, double* a, Index* perm) {
  for (Index i = 0; i < n; ++i) perm[i] = i;
  for (Index k = 0; k < n; ++k) {
    Index p = k;
    double best = std::fabs(a[k + k * n]);
    for (Index i = k + 1; i < n; ++i) {
      double v = std::fabs(a[i + k * n]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (p != k) {
      for (Index j = 0; j < n; ++j) std::swap(a[k + j * n], a[p + j * n]);
      std::swap(perm[k], perm[p]);
    }
    double piv = a[k + k * n];
    if (piv != 0.0)
      for (Index i = k + 1; i < n; ++i) a[i + k * n] /= piv;
    for (Index j = k + 1; j < n; ++j) {
      double ukj = a[k + j * n];
      if (ukj == 0.0) continue;
      for (Index i = k + 1; i < n; ++i) a[i + j * n] -= a[i + k * n] * ukj;
    }
  }
}

// Solve with a factorization from lu_partial_pivot; b is n x m column major,
// overwritten with the solution.
inline void lu_solve(Index n, const double* lu, const Index* perm, Index m, double* b) {
  std::vector<double> tmp(static_cast<size_t>(n));
  for (Index c = 0; c < m; ++c) {
    double* col = b + c * n;
    for (Index i = 0; i < n; ++i) tmp[i] = col[perm[i]];
    for (Index i = 0; i < n; ++i) {
      double s = tmp[i];
      for (Index k = 0; k < i; ++k) s -= lu[i + k * n] * tmp[k];
      tmp[i] = s;
    }
    // back substitution column by column from the last (Eigen's column-major
    // upper-triangular solve): x_k = t_k / u_kk, then t_i -= u_ik x_k for i < k
    for (Index k = n - 1; k >= 0; --k) {
      const double xk = tmp[k] / lu[k + k * n];
      tmp[k] = xk;
      for (Index i = 0; i < k; ++i) tmp[i] -= lu[i + k * n] * xk;
    }
    for (Index i = 0; i < n; ++i) col[i] = tmp[i];
  }
}

}  // namespace cieg_dense
