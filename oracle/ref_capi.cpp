// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY. extern "C" bindings over the
// UNMODIFIED reference library (compiled from /root/reference/proj/src with
// -Dci=ciref), so Python tests and bench.py's reference arm can drive the
// reference's own code path: ci::spmm / spmm_serial (csb.cpp:182-201),
// block_inner / linear_combination (block_vectors.cpp:74-160),
// choose_shifts / apply_preconditioner / fom_solve (precond.cpp),
// extract_tile_diagonal (hamiltonian.cpp:178-203), orthonormalize and
// lobpcg_solve (lobpcg.cpp:89-387), lanczos_solve (lanczos.cpp:24-136).
// Never linked into the product.
#include <omp.h>

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <string>

#include "ci/block_vectors.hpp"
#include "ci/csb.hpp"
#include "ci/errors.hpp"
#include "ci/guess.hpp"
#include "ci/hamiltonian.hpp"
#include "ci/lanczos.hpp"
#include "ci/lobpcg.hpp"
#include "ci/precond.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    g_err.clear();
    f();
    return 0;
  } catch (const ci::DimensionMismatch& e) {
    g_err = e.what();
    return 1;
  } catch (const ci::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const ci::SubspaceCollapse& e) {
    g_err = e.what();
    return 3;
  } catch (const ci::FormatError& e) {
    g_err = e.what();
    return 4;
  } catch (const ci::IndefiniteGram& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

ci::BlockVectors to_bv(const double* x, std::uint32_t n, std::uint32_t k) {
  ci::BlockVectors b(n, k);
  if (n && k) std::memcpy(b.values().data(), x, sizeof(double) * n * k);
  return b;
}

void from_bv(const ci::BlockVectors& b, double* out) {
  if (!b.values().empty()) std::memcpy(out, b.values().data(), sizeof(double) * b.values().size());
}

Eigen::MatrixXd to_mat(const double* colmajor, long r, long c) {
  Eigen::MatrixXd m(r, c);
  if (r && c) std::memcpy(m.data(), colmajor, sizeof(double) * r * c);
  return m;
}

struct Report {
  ci::SolveReport rep;
};

}  // namespace

extern "C" {

const char* ciref_last_error() { return g_err.c_str(); }
void ciref_set_threads(int n) { omp_set_num_threads(n); }
int ciref_max_threads() { return omp_get_max_threads(); }

// Build a ci::CsbMatrix from the flattened view (same layout as cieg_csb_view).
int ciref_matrix_create(std::uint32_t dim, std::uint32_t nb, int precision,
                        const std::uint32_t* bounds, const std::uint64_t* offsets,
                        const std::uint16_t* rows, const std::uint16_t* cols, const void* values,
                        void** out) {
  return guard([&] {
    auto h = std::make_unique<ci::CsbMatrix>();
    h->dim = dim;
    h->precision = precision == 0 ? ci::Precision::Single : ci::Precision::Double;
    h->layout.block_boundaries.assign(bounds, bounds + nb + 1);
    h->blocks.resize(static_cast<std::size_t>(nb) * (nb + 1) / 2);
    const float* v32 = static_cast<const float*>(values);
    const double* v64 = static_cast<const double*>(values);
#pragma omp parallel for schedule(dynamic, 64)
    for (std::int64_t b = 0; b < static_cast<std::int64_t>(h->blocks.size()); ++b) {
      ci::CoordinateBlock& blk = h->blocks[b];
      const std::uint64_t e0 = offsets[b], e1 = offsets[b + 1];
      blk.rows.assign(rows + e0, rows + e1);
      blk.cols.assign(cols + e0, cols + e1);
      if (precision == 0)
        blk.values32.assign(v32 + e0, v32 + e1);
      else
        blk.values64.assign(v64 + e0, v64 + e1);
    }
    h->nnz_lower = offsets[h->blocks.size()];
    *out = h.release();
  });
}

void ciref_matrix_destroy(void* h) { delete static_cast<ci::CsbMatrix*>(h); }

// ci::load_csb (csb.cpp:295-331) / ci::save_csb (csb.cpp:256-293).
int ciref_matrix_load(const char* path, void** out) {
  return guard([&] { *out = new ci::CsbMatrix(ci::load_csb(path)); });
}
int ciref_matrix_save(void* h, const char* path) {
  return guard([&] { ci::save_csb(*static_cast<ci::CsbMatrix*>(h), path); });
}
void ciref_matrix_summary(void* h, std::uint32_t* dim, std::uint64_t* nnz, std::uint32_t* nb, int* precision) {
  const ci::CsbMatrix& m = *static_cast<ci::CsbMatrix*>(h);
  *dim = m.dim;
  *nnz = m.nnz_lower;
  *nb = m.block_count();
  *precision = m.precision == ci::Precision::Single ? 0 : 1;
}

int ciref_spmm(void* h, const double* x, std::uint32_t m, double* y, int serial) {
  return guard([&] {
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    ci::BlockVectors X = to_bv(x, H.dim, m);
    ci::BlockVectors U = serial ? ci::spmm_serial(H, X) : ci::spmm(H, X);
    from_bv(U, y);
  });
}

// ci::spmm timed on its own: X is built once outside the timed region, each
// rep times exactly one ci::spmm call (csb.cpp:182-193: its own allocation of
// U included, as every caller pays it), the last U is copied out afterwards.
int ciref_spmm_timed(void* h, const double* x, std::uint32_t m, int reps, double* secs, double* y) {
  return guard([&] {
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    const ci::BlockVectors X = to_bv(x, H.dim, m);
    ci::BlockVectors U;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      U = ci::spmm(H, X);
      const auto t1 = std::chrono::steady_clock::now();
      secs[r] = std::chrono::duration<double>(t1 - t0).count();
    }
    if (y) from_bv(U, y);
  });
}

int ciref_to_dense(void* h, double* out_colmajor) {
  return guard([&] {
    Eigen::MatrixXd d = ci::to_dense(*static_cast<ci::CsbMatrix*>(h));
    std::memcpy(out_colmajor, d.data(), sizeof(double) * d.size());
  });
}

int ciref_block_inner(std::uint32_t n, const double* x, std::uint32_t kx, const double* y,
                      std::uint32_t ky, int serial, double* out) {
  return guard([&] {
    ci::BlockVectors X = to_bv(x, n, kx), Y = to_bv(y, n, ky);
    Eigen::MatrixXd g = serial ? ci::block_inner_serial(X, Y) : ci::block_inner(X, Y);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

int ciref_linear_combination(std::uint32_t n, const double* y, std::uint32_t kin, const double* g,
                             std::uint32_t kout, double* out) {
  return guard([&] {
    ci::BlockVectors Y = to_bv(y, n, kin);
    from_bv(ci::linear_combination(Y, to_mat(g, kin, kout)), out);
  });
}

int ciref_add_linear_combination(std::uint32_t n, double* y, std::uint32_t ky, const double* x,
                                 std::uint32_t kx, const double* g) {
  return guard([&] {
    ci::BlockVectors Y = to_bv(y, n, ky), X = to_bv(x, n, kx);
    ci::add_linear_combination(Y, X, to_mat(g, kx, ky));
    from_bv(Y, y);
  });
}

int ciref_orthonormalize(std::uint32_t n, const double* y, std::uint32_t k, double drop_tol,
                         const double* against, std::uint32_t ka, double* out, std::uint32_t* kout) {
  return guard([&] {
    ci::BlockVectors Y = to_bv(y, n, k);
    ci::BlockVectors A;
    if (against && ka) A = to_bv(against, n, ka);
    ci::BlockVectors Q = ci::orthonormalize(Y, drop_tol, (against && ka) ? &A : nullptr);
    *kout = Q.width();
    from_bv(Q, out);
  });
}

// TileDiagonal from a group partition (ranges only are needed by
// extract_tile_diagonal, hamiltonian.cpp:178-203).
int ciref_tilediag_create(void* h, const std::uint32_t* bounds, std::uint32_t ng, void** out) {
  return guard([&] {
    ci::GroupPartition part;
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    part.group_of_state.resize(H.dim);
    for (std::uint32_t g = 0; g < ng; ++g) {
      part.group_ranges.push_back({bounds[g], bounds[g + 1]});
      for (std::uint32_t r = bounds[g]; r < bounds[g + 1]; ++r) part.group_of_state[r] = g;
    }
    auto td = std::make_unique<ci::TileDiagonal>(ci::extract_tile_diagonal(H, part));
    *out = td.release();
  });
}

void ciref_tilediag_destroy(void* t) { delete static_cast<ci::TileDiagonal*>(t); }

// Concatenated column-major blocks (sum n_g^2 doubles).
int ciref_tilediag_blocks(void* t, double* out) {
  return guard([&] {
    const ci::TileDiagonal& td = *static_cast<ci::TileDiagonal*>(t);
    std::size_t o = 0;
    for (const Eigen::MatrixXd& b : td.blocks) {
      std::memcpy(out + o, b.data(), sizeof(double) * b.size());
      o += static_cast<std::size_t>(b.size());
    }
  });
}

static ci::PrecondConfig make_cfg(const double* c) {
  // c: inner_iters, small_block_cutoff, engage_after, relres_gate,
  //    near_converged_factor, far_threshold, column_floor_factor
  ci::PrecondConfig cfg;
  if (c) {
    cfg.inner_iters = static_cast<int>(c[0]);
    cfg.small_block_cutoff = static_cast<int>(c[1]);
    cfg.engage_after = static_cast<int>(c[2]);
    cfg.relres_gate = c[3];
    cfg.near_converged_factor = c[4];
    cfg.far_threshold = c[5];
    cfg.column_floor_factor = c[6];
  }
  return cfg;
}

int ciref_choose_shifts(std::uint32_t k, const double* theta, const double* res_norm,
                        const double* x_norm, const double* relres, int iteration, double tol,
                        const double* cfg7, double* mu, int* engage) {
  return guard([&] {
    ci::ShiftInputs in;
    in.theta.assign(theta, theta + k);
    in.res_norm.assign(res_norm, res_norm + k);
    in.x_norm.assign(x_norm, x_norm + k);
    in.relres.assign(relres, relres + k);
    ci::ShiftPlan p = ci::choose_shifts(in, iteration, tol, make_cfg(cfg7));
    for (std::uint32_t j = 0; j < k; ++j) {
      mu[j] = p.mu[j];
      engage[j] = p.engage[j] ? 1 : 0;
    }
  });
}

int ciref_apply_preconditioner(void* t, std::uint32_t n, const double* r, std::uint32_t k,
                               const double* mu, const int* engage, const double* cfg7,
                               double* w) {
  return guard([&] {
    ci::ShiftPlan p;
    p.mu.assign(mu, mu + k);
    for (std::uint32_t j = 0; j < k; ++j) p.engage.push_back(engage[j] != 0);
    ci::BlockVectors W = ci::apply_preconditioner(*static_cast<ci::TileDiagonal*>(t),
                                                  to_bv(r, n, k), p, make_cfg(cfg7));
    from_bv(W, w);
  });
}

int ciref_fom_solve(std::uint32_t n, const double* block, std::uint32_t k, const double* mu,
                    const double* rhs, int iters, double* out) {
  return guard([&] {
    Eigen::MatrixXd x = ci::fom_solve(to_mat(block, n, n), std::vector<double>(mu, mu + k),
                                      to_mat(rhs, n, k), iters);
    std::memcpy(out, x.data(), sizeof(double) * x.size());
  });
}

// lobpcg_solve; opts: k_want, max_iter; tol; tilediag may be null.
int ciref_lobpcg_solve(void* h, const double* x0, std::uint32_t kt, int k_want, double tol,
                       int max_iter, void* tilediag, const double* cfg7, void** out) {
  return guard([&] {
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    ci::LobpcgOptions opt;
    opt.k_want = k_want;
    opt.tol = tol;
    opt.max_iter = max_iter;
    opt.preconditioner = static_cast<const ci::TileDiagonal*>(tilediag);
    opt.precond_config = make_cfg(cfg7);
    auto r = std::make_unique<Report>();
    r->rep = ci::lobpcg_solve(H, to_bv(x0, H.dim, kt), opt);
    *out = r.release();
  });
}

void ciref_report_destroy(void* r) { delete static_cast<Report*>(r); }

void ciref_report_summary(void* rp, int* converged, int* iterations, double* norm_est,
                          std::uint32_t* kt, std::uint64_t* nhist, std::uint64_t* counters4,
                          std::uint32_t* nev) {
  const ci::SolveReport& r = static_cast<Report*>(rp)->rep;
  *converged = r.converged ? 1 : 0;
  *iterations = r.iterations;
  *norm_est = r.norm_estimate;
  *kt = r.trial_vectors.width();
  *nhist = r.history.size();
  counters4[0] = r.counters.spmm_calls;
  counters4[1] = r.counters.spmv_equivalents;
  counters4[2] = r.counters.precond_applications;
  counters4[3] = r.counters.orthogonalizations;
  *nev = static_cast<std::uint32_t>(r.eigenvalues.size());
}

void ciref_report_arrays(void* rp, double* eigenvalues, double* trial, int* h_iter, int* h_col,
                         double* h_relres, double* h_theta) {
  const ci::SolveReport& r = static_cast<Report*>(rp)->rep;
  for (std::size_t j = 0; j < r.eigenvalues.size(); ++j) eigenvalues[j] = r.eigenvalues[j];
  from_bv(r.trial_vectors, trial);
  for (std::size_t i = 0; i < r.history.size(); ++i) {
    h_iter[i] = r.history[i].iteration;
    h_col[i] = r.history[i].column;
    h_relres[i] = r.history[i].relres;
    h_theta[i] = r.history[i].theta;
  }
}

// Lanczos baseline (lanczos.cpp:24-136); v0 dense vector of length dim.
int ciref_lanczos_solve(void* h, const double* v0, int k_want, double tol, int max_iter,
                        void** out) {
  return guard([&] {
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    Eigen::VectorXd v(H.dim);
    std::memcpy(v.data(), v0, sizeof(double) * H.dim);
    ci::LanczosOptions opt;
    opt.k_want = k_want;
    opt.tol = tol;
    opt.max_iter = max_iter;
    auto r = std::make_unique<Report>();
    r->rep = ci::lanczos_solve(H, v, opt);
    *out = r.release();
  });
}

// ---- synthetic physics problems + the reference's own multilevel_guess ----
struct ProblemHolder {
  ci::Problem p;
};

static ci::BasisSpec make_spec(int Z, int N, int M2, int parity, int Nmax, double hw) {
  ci::BasisSpec s;
  s.Z = Z;
  s.N = N;
  s.M2 = M2;
  s.parity = parity;
  s.Nmax = Nmax;
  s.hbar_omega = hw;
  return s;
}

// build_synthetic_problem (hamiltonian.cpp:205-224).
int ciref_synthetic_problem(int Z, int N, int M2, int parity, int Nmax, double hw, std::uint64_t seed,
                            double offdiag, int d, std::uint32_t beta, int precision, void** out) {
  return guard([&] {
    auto h = std::make_unique<ProblemHolder>();
    h->p = ci::build_synthetic_problem(make_spec(Z, N, M2, parity, Nmax, hw), seed, offdiag, d, beta,
                                       precision == 0 ? ci::Precision::Single : ci::Precision::Double);
    *out = h.release();
  });
}
void ciref_problem_destroy(void* h) { delete static_cast<ProblemHolder*>(h); }
void* ciref_problem_matrix(void* h) { return &static_cast<ProblemHolder*>(h)->p.matrix; }
// group starts + dim (n = count + 1 written when out != null); returns the count + 1
std::uint32_t ciref_problem_groups(void* h, std::uint32_t* out) {
  const auto& g = static_cast<ProblemHolder*>(h)->p.partition.group_ranges;
  if (out) {
    for (std::size_t i = 0; i < g.size(); ++i) out[i] = g[i].first;
    out[g.size()] = g.empty() ? 0 : g.back().second;
  }
  return static_cast<std::uint32_t>(g.size() + 1);
}
// quanta stratum boundaries (basis.hpp:68) + dim
std::uint32_t ciref_problem_strata(void* h, std::uint32_t* out) {
  const auto& b = *static_cast<ProblemHolder*>(h)->p.basis;
  const auto& q = b.quanta_boundaries;
  if (out) {
    for (std::size_t i = 0; i < q.size(); ++i) out[i] = q[i];
    out[q.size()] = b.dimension();
  }
  return static_cast<std::uint32_t>(q.size() + 1);
}

// multilevel_guess (guess.cpp:66-117) with build_synthetic_problem as the
// ProblemFactory. lv_* arrays hold up to `levels` entries; *nlv = written.
int ciref_multilevel_guess(int Z, int N, int M2, int parity, int Nmax, double hw, std::uint64_t seed,
                           double offdiag, int d, std::uint32_t beta, int precision, int levels, int k_want,
                           int k_trial, double tol, int max_iter, std::uint64_t mseed, double* guess_out,
                           std::uint32_t* kout, std::uint32_t* dim_out, int* nlv, int* lv_nmax, std::uint32_t* lv_dim,
                           int* lv_iters, int* lv_conv) {
  return guard([&] {
    ci::MultilevelOptions o;
    o.levels = levels;
    o.k_want = k_want;
    o.k_trial = k_trial;
    o.tol = tol;
    o.max_iter = max_iter;
    o.seed = mseed;
    const ci::Precision pr = precision == 0 ? ci::Precision::Single : ci::Precision::Double;
    ci::MultilevelResult r = ci::multilevel_guess(
        make_spec(Z, N, M2, parity, Nmax, hw), o,
        [&](const ci::BasisSpec& s) { return ci::build_synthetic_problem(s, seed, offdiag, d, beta, pr); });
    *kout = r.guess.width();
    *dim_out = r.guess.dim();
    from_bv(r.guess, guess_out);
    *nlv = static_cast<int>(r.levels.size());
    for (std::size_t i = 0; i < r.levels.size(); ++i) {
      lv_nmax[i] = r.levels[i].nmax;
      lv_dim[i] = r.levels[i].dim;
      lv_iters[i] = r.levels[i].iterations;
      lv_conv[i] = r.levels[i].converged ? 1 : 0;
    }
  });
}

// rayleigh_ritz (lobpcg.cpp:121-145); g_out m x k_trial column-major.
int ciref_rayleigh_ritz(std::uint32_t n, const double* y, const double* hy, std::uint32_t m, int k_trial,
                        double* theta_out, double* g_out) {
  return guard([&] {
    auto [theta, coeff] = ci::rayleigh_ritz(to_bv(y, n, m), to_bv(hy, n, m), k_trial, -1, 0, 0);
    for (int j = 0; j < k_trial; ++j) theta_out[j] = theta[j];
    std::memcpy(g_out, coeff.g.data(), sizeof(double) * coeff.g.size());
  });
}

// residual_norms (lobpcg.cpp:147-169); norm_est <= 0 -> nullopt.
int ciref_residual_norms(void* h, const double* x, std::uint32_t k, const double* theta, double norm_est,
                         double* out) {
  return guard([&] {
    const ci::CsbMatrix& H = *static_cast<ci::CsbMatrix*>(h);
    std::optional<double> est;
    if (norm_est > 0) est = norm_est;
    std::vector<double> r = ci::residual_norms(H, to_bv(x, H.dim, k), std::vector<double>(theta, theta + k), est);
    for (std::uint32_t j = 0; j < k; ++j) out[j] = r[j];
  });
}

}  // extern "C"
