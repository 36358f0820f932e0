// ci_solve_main.cpp -- a run_solver-equivalent driver (ci_eigen.cpp:104-151:
// build the synthetic problem, random orthonormalized guess, tile diagonal,
// ci::lobpcg_solve) that touches every ci:: entry point the drop-in binds.
// It is linked twice by integration/Makefile:
//   _build/ci_solve_ref : all eleven UNMODIFIED proj/src TUs (the reference);
//   _build/ci_solve_gpu : proj/src/{basis,grouping,hamiltonian,guess,planner,
//                          config}.cpp + ci_gpu_dropin.cpp + ci_host_companion.cpp
//                          + libcieg.so (csb/block_vectors/lobpcg/precond/
//                          lanczos replaced by the B200 path).
// Both print one JSON object; tests/test_integration_gpu.py compares them.
//
// usage: ci_solve Z N M2 parity Nmax seed offdiag d beta precision k_want k_trial tol max_iter
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>
#include <sstream>
#include <string>
#include <vector>

#include "ci/block_vectors.hpp"
#include "ci/csb.hpp"
#include "ci/errors.hpp"
#include "ci/guess.hpp"
#include "ci/hamiltonian.hpp"
#include "ci/lanczos.hpp"
#include "ci/lobpcg.hpp"
#include "ci/precond.hpp"

namespace {

double abs_sum(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += std::fabs(x);
  return s;
}
double abs_sum(const Eigen::MatrixXd& m) {
  double s = 0.0;
  for (long j = 0; j < m.cols(); ++j)
    for (long i = 0; i < m.rows(); ++i) s += std::fabs(m(i, j));
  return s;
}
std::string list(const std::vector<double>& v) {
  std::ostringstream os;
  os.precision(17);
  os << "[";
  for (std::size_t i = 0; i < v.size(); ++i) os << (i ? ", " : "") << v[i];
  return os.str() + "]";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 15) {
    std::fprintf(stderr, "usage: %s Z N M2 parity Nmax seed offdiag d beta precision k_want k_trial tol max_iter\n",
                 argv[0]);
    return 2;
  }
  ci::BasisSpec spec;
  spec.Z = std::atoi(argv[1]);
  spec.N = std::atoi(argv[2]);
  spec.M2 = std::atoi(argv[3]);
  spec.parity = std::atoi(argv[4]);
  spec.Nmax = std::atoi(argv[5]);
  const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
  const double offdiag = std::atof(argv[7]);
  const int d = std::atoi(argv[8]);
  const auto beta = static_cast<std::uint32_t>(std::atoi(argv[9]));
  const ci::Precision prec = std::atoi(argv[10]) == 0 ? ci::Precision::Single : ci::Precision::Double;
  const int k_want = std::atoi(argv[11]), k_trial = std::atoi(argv[12]);
  const double tol = std::atof(argv[13]);
  const int max_iter = std::atoi(argv[14]);
  try {
    const ci::Problem problem = ci::build_synthetic_problem(spec, seed, offdiag, d, beta, prec);
    const ci::CsbMatrix& h = problem.matrix;
    const std::uint32_t n = h.dim;
    // ci_eigen.cpp:113 -- the random guess, orthonormalized
    const ci::BlockVectors x0 = ci::orthonormalize(ci::random_block(n, k_trial, seed));
    const ci::TileDiagonal tiles = ci::extract_tile_diagonal(h, problem.partition);
    ci::LobpcgOptions opt;
    opt.k_want = k_want;
    opt.tol = tol;
    opt.max_iter = max_iter;
    opt.preconditioner = &tiles;
    const ci::SolveReport rep = ci::lobpcg_solve(h, x0, opt);

    // the operator-level API on the same objects
    const ci::BlockVectors u = ci::spmm(h, x0);
    const Eigen::MatrixXd g = ci::block_inner(x0, u);
    const ci::BlockVectors lc = ci::linear_combination(u, g);
    ci::BlockVectors acc = u;
    ci::add_linear_combination(acc, x0, g);
    const std::vector<double> norms = ci::column_norms(u);
    ci::ShiftPlan plan;
    for (int j = 0; j < k_trial; ++j) {
      plan.mu.push_back(-1.0 - 0.25 * j);
      plan.engage.push_back(j % 3 != 2);
    }
    const ci::BlockVectors w = ci::apply_preconditioner(tiles, u, plan, ci::PrecondConfig{});
    std::uint32_t big = 0;
    for (std::uint32_t gi = 0; gi < tiles.group_count(); ++gi)
      if (tiles.blocks[gi].rows() > tiles.blocks[big].rows()) big = gi;
    const long nb = tiles.blocks[big].rows();
    Eigen::MatrixXd rhs(nb, 2);
    for (long i = 0; i < nb; ++i) {
      rhs(i, 0) = u.at(tiles.ranges[big].first + static_cast<std::uint32_t>(i), 0);
      rhs(i, 1) = u.at(tiles.ranges[big].first + static_cast<std::uint32_t>(i), 1);
    }
    const Eigen::MatrixXd fom = ci::fom_solve(tiles.blocks[big], {-2.0, -3.0}, rhs, 3);
    const std::vector<double> res = ci::residual_norms(h, rep.eigenvectors, rep.eigenvalues);
    const ci::MatrixStats st = ci::matrix_stats(h);
    const std::string path = std::string("/tmp/ci_solve_") + std::to_string(::getpid()) + ".csb";
    ci::save_csb(h, path);
    const ci::CsbMatrix h2 = ci::load_csb(path);
    std::remove(path.c_str());
    const ci::BlockVectors u2 = ci::spmm(h2, x0);
    std::ostringstream csv;
    ci::write_history_csv(rep, csv);
    int csv_lines = 0;
    for (char c : csv.str()) csv_lines += c == '\n';
    // the multilevel guess of guess.cpp (reference TU in both builds) over the
    // bound lobpcg_solve, then a solve from it
    ci::MultilevelOptions mo;
    mo.levels = 2;
    mo.k_want = k_want;
    mo.k_trial = k_trial;
    mo.tol = tol;
    mo.max_iter = max_iter;
    mo.seed = seed;
    const ci::MultilevelResult ml = ci::multilevel_guess(
        spec, mo, [&](const ci::BasisSpec& s) { return ci::build_synthetic_problem(s, seed, offdiag, d, beta, prec); });
    const ci::SolveReport rep_ml = ci::lobpcg_solve(h, ml.guess, opt);
    std::vector<double> level_iters;
    for (const auto& l : ml.levels) level_iters.push_back(l.iterations);

    std::printf("{\"dim\": %u, \"nnz\": %llu, \"iterations\": %d, \"converged\": %d, \"eigenvalues\": %s, "
                "\"counters\": [%llu, %llu, %llu, %llu], \"spmm\": %.17g, \"block_inner\": %.17g, "
                "\"linear_combination\": %.17g, \"add_linear_combination\": %.17g, \"column_norms\": %s, "
                "\"apply_preconditioner\": %.17g, \"fom_solve\": %.17g, \"residual_norms\": %s, "
                "\"stats\": [%llu, %llu, %llu], \"csb_roundtrip_spmm\": %.17g, \"history_csv_lines\": %d, "
                "\"multilevel_level_iterations\": %s, \"multilevel_iterations\": %d, \"multilevel_eigenvalues\": %s}\n",
                n, static_cast<unsigned long long>(h.nnz_lower), rep.iterations, rep.converged ? 1 : 0,
                list(rep.eigenvalues).c_str(), static_cast<unsigned long long>(rep.counters.spmm_calls),
                static_cast<unsigned long long>(rep.counters.spmv_equivalents),
                static_cast<unsigned long long>(rep.counters.precond_applications),
                static_cast<unsigned long long>(rep.counters.orthogonalizations), abs_sum(u.values()), abs_sum(g),
                abs_sum(lc.values()), abs_sum(acc.values()), list(norms).c_str(), abs_sum(w.values()), abs_sum(fom),
                list(res).c_str(), static_cast<unsigned long long>(st.nnz_lower),
                static_cast<unsigned long long>(st.groups), static_cast<unsigned long long>(st.csb_blocks),
                abs_sum(u2.values()), csv_lines, list(level_iters).c_str(), rep_ml.iterations,
                list(rep_ml.eigenvalues).c_str());
  } catch (const ci::Error& e) {
    std::fprintf(stderr, "ci::Error: %s\n", e.what());
    return 1;
  }
  return 0;
}
