// ci_gpu_dropin.cpp -- the reference-side binding: implements the
// reference's own ci:: entry points (declared in
// /root/reference/proj/include/ci/*.hpp, compiled against those headers) on
// top of the C ABI in include/cieg.h. Linking this TU (plus libcieg.so) in
// place of proj/src/{csb,block_vectors,lobpcg,precond,lanczos}.cpp (with
// ci_host_companion.cpp for their non-hot symbols) makes every caller of
// ci::spmm / ci::lobpcg_solve / ci::block_inner / ci::apply_preconditioner
// ... run on the B200; basis, grouping, hamiltonian, guess, planner and config
// stay the reference's own TUs (integration/Makefile links exactly that and
// tests/test_integration_gpu.py runs it against the all-reference build).
//
// Contract mapping:
//   * value semantics stay: inputs by const&, results by value;
//   * uploaded H and tile diagonals are cached by object address AND a
//     content fingerprint (dimensions, entry counts, buffer addresses and a
//     spread sample of the stored entries / block values), re-uploaded when
//     it changes -- a new matrix built at the same address (the CLI's
//     `compare` loop, one Problem per seed) is never served stale;
//     cieg_dropin_invalidate() drops every cached upload explicitly;
//   * cieg_status != 0 is rethrown as the matching ci:: exception with the
//     library's "<Type>: message" text; no exception crosses the C ABI.
// Built by integration/Makefile (needs the reference headers; Eigen comes from
// oracle/eigen_shim in this image).
#include <cstring>
#include <fstream>
#include <optional>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "ci/block_vectors.hpp"
#include "ci/csb.hpp"
#include "ci/errors.hpp"
#include "ci/hamiltonian.hpp"
#include "ci/guess.hpp"
#include "ci/lanczos.hpp"
#include "ci/lobpcg.hpp"
#include "ci/precond.hpp"
#include "cieg.h"

namespace {

[[noreturn]] void rethrow(int st) {
  std::string msg = cieg_last_error();
  auto body = [&] {
    auto p = msg.find(": ");
    return p == std::string::npos ? msg : msg.substr(p + 2);
  };
  switch (st) {
    case CIEG_ERR_DIMENSION: throw ci::DimensionMismatch(body());
    case CIEG_ERR_CONFIG: throw ci::ConfigError(body());
    case CIEG_ERR_SUBSPACE: throw ci::SubspaceCollapse(body());
    case CIEG_ERR_FORMAT: throw ci::FormatError(body());
    case CIEG_ERR_INDEFINITE: throw ci::IndefiniteGram(body());
    case CIEG_ERR_BETA: throw ci::BetaTooLarge(body());
    default: throw ci::Error(msg);
  }
}
inline void check(int st) {
  if (st != CIEG_OK) rethrow(st);
}

struct Device {
  cieg_ctx* ctx = nullptr;
  struct MatEntry {
    std::uint64_t fp = 0;
    cieg_mat* mat = nullptr;
  };
  struct PrecEntry {
    std::uint64_t fp = 0;
    cieg_prec* prec = nullptr;
  };
  std::map<const ci::CsbMatrix*, MatEntry> mats;
  std::map<const ci::TileDiagonal*, PrecEntry> precs;
  Device() {
    const char* d = std::getenv("CIEG_DEVICE");
    check(cieg_ctx_create(d ? std::atoi(d) : 0, &ctx));
  }
  void clear() {
    for (auto& [k, e] : mats) cieg_matrix_destroy(e.mat);
    for (auto& [k, e] : precs) cieg_precond_destroy(e.prec);
    mats.clear();
    precs.clear();
  }
};
Device& dev() {
  static Device d;
  return d;
}

// FNV-1a over the fields that identify an upload's content.
struct Fnv {
  std::uint64_t h = 1469598103934665603ull;
  template <typename T>
  void add(const T& v) {
    const auto* p = reinterpret_cast<const unsigned char*>(&v);
    for (std::size_t i = 0; i < sizeof(T); ++i) h = (h ^ p[i]) * 1099511628211ull;
  }
};

std::uint64_t fingerprint(const ci::CsbMatrix& h) {
  Fnv f;
  f.add(h.dim);
  f.add(h.nnz_lower);
  f.add(static_cast<int>(h.precision));
  for (std::uint32_t b : h.layout.block_boundaries) f.add(b);
  for (const ci::CoordinateBlock& b : h.blocks) {
    const std::size_t n = b.size();
    if (n == 0) continue;
    f.add(n);
    f.add(b.rows.data());
    f.add(b.values32.data());
    f.add(b.values64.data());
    // up to 8 entries spread over the block
    const std::size_t step = std::max<std::size_t>(1, n / 8);
    for (std::size_t e = 0; e < n; e += step) {
      f.add(b.rows[e]);
      f.add(b.cols[e]);
      if (!b.values32.empty()) f.add(b.values32[e]);
      if (!b.values64.empty()) f.add(b.values64[e]);
    }
  }
  return f.h;
}

std::uint64_t fingerprint(const ci::TileDiagonal& t) {
  Fnv f;
  f.add(t.blocks.size());
  for (std::size_t g = 0; g < t.blocks.size(); ++g) {
    const Eigen::MatrixXd& b = t.blocks[g];
    f.add(t.ranges[g].first);
    f.add(t.ranges[g].second);
    f.add(b.data());
    const long n = b.rows() * b.cols();
    const long step = std::max<long>(1, n / 8);
    for (long e = 0; e < n; e += step) f.add(b.data()[e]);
  }
  return f.h;
}

// Flatten the CsbMatrix block grid into the cieg_csb_view arrays.
struct Flat {
  std::vector<std::uint64_t> offs;
  std::vector<std::uint16_t> rows, cols;
  std::vector<float> v32;
  std::vector<double> v64;
  cieg_csb_view view{};
};
std::unique_ptr<Flat> flatten(const ci::CsbMatrix& h) {
  auto f = std::make_unique<Flat>();
  const std::uint32_t nb = h.block_count();
  f->offs.assign(1, 0);
  for (const ci::CoordinateBlock& b : h.blocks) {
    f->rows.insert(f->rows.end(), b.rows.begin(), b.rows.end());
    f->cols.insert(f->cols.end(), b.cols.begin(), b.cols.end());
    f->v32.insert(f->v32.end(), b.values32.begin(), b.values32.end());
    f->v64.insert(f->v64.end(), b.values64.begin(), b.values64.end());
    f->offs.push_back(f->offs.back() + b.size());
  }
  f->view = cieg_csb_view{h.dim, nb, h.precision == ci::Precision::Single ? 0 : 1,
                          h.layout.block_boundaries.data(), f->offs.data(), f->rows.data(), f->cols.data(),
                          h.precision == ci::Precision::Single ? static_cast<const void*>(f->v32.data())
                                                               : static_cast<const void*>(f->v64.data())};
  return f;
}

cieg_mat* matrix(const ci::CsbMatrix& h) {
  const std::uint64_t fp = fingerprint(h);
  auto& m = dev().mats[&h];
  if (!m.mat || m.fp != fp) {
    if (m.mat) cieg_matrix_destroy(m.mat);
    m.mat = nullptr;
    auto f = flatten(h);
    check(cieg_matrix_upload(dev().ctx, &f->view, nullptr, 0, 0, &m.mat));
    m.fp = fp;
  }
  return m.mat;
}

cieg_prec* upload_tiles(const ci::TileDiagonal& t) {
  std::vector<std::uint32_t> bounds{t.ranges.empty() ? 0u : t.ranges.front().first};
  std::vector<double> blocks;
  for (std::size_t g = 0; g < t.blocks.size(); ++g) {
    bounds.push_back(t.ranges[g].second);
    blocks.insert(blocks.end(), t.blocks[g].data(), t.blocks[g].data() + t.blocks[g].size());
  }
  cieg_tilediag_view v{bounds.back(), static_cast<std::uint32_t>(t.blocks.size()), bounds.data(), blocks.data()};
  cieg_prec* p = nullptr;
  check(cieg_precond_upload(dev().ctx, &v, &p));
  return p;
}

cieg_prec* precond(const ci::TileDiagonal& t) {
  const std::uint64_t fp = fingerprint(t);
  auto& e = dev().precs[&t];
  if (!e.prec || e.fp != fp) {
    if (e.prec) cieg_precond_destroy(e.prec);
    e.prec = nullptr;
    e.prec = upload_tiles(t);
    e.fp = fp;
  }
  return e.prec;
}

cieg_precond_config config(const ci::PrecondConfig& c) {
  return cieg_precond_config{c.inner_iters, c.small_block_cutoff, c.engage_after, c.relres_gate,
                             c.near_converged_factor, c.far_threshold, c.column_floor_factor};
}

// Device staging of host ci::BlockVectors (row-major, the layout the C ABI uses).
struct DevBlock {
  void* p = nullptr;
  DevBlock(const double* host, std::size_t count) {
    check(cieg_device_alloc(dev().ctx, sizeof(double) * count, &p));
    if (host && count) check(cieg_memcpy(dev().ctx, p, host, sizeof(double) * count, 0));
  }
  ~DevBlock() { cieg_device_free(dev().ctx, p); }
  double* d() const { return static_cast<double*>(p); }
  void to_host(double* host, std::size_t count) const {
    if (count) check(cieg_memcpy(dev().ctx, host, p, sizeof(double) * count, 1));
  }
};

}  // namespace

namespace ci {

// csb.hpp:83 -- ci::spmm on the GPU (H uploaded once, X/U through the host).
BlockVectors spmm(const CsbMatrix& h, const BlockVectors& x) {
  if (x.dim() != h.dim) throw DimensionMismatch("spmm: vector dim != matrix dim");
  BlockVectors u(h.dim, x.width());
  check(cieg_spmm_host(dev().ctx, matrix(h), x.values().data(), u.values().data(), x.width()));
  return u;
}
BlockVectors spmm_serial(const CsbMatrix& h, const BlockVectors& x) { return spmm(h, x); }

// precond.hpp:47-48 -- host logic, verbatim semantics.
ShiftPlan choose_shifts(const ShiftInputs& in, int iteration, double tol, const PrecondConfig& cfg) {
  const std::uint32_t k = static_cast<std::uint32_t>(in.theta.size());
  ShiftPlan plan;
  plan.mu.resize(k);
  std::vector<int> en(k);
  cieg_precond_config c = config(cfg);
  check(cieg_choose_shifts(k, in.theta.data(), in.res_norm.data(), in.x_norm.data(), in.relres.data(), iteration, tol,
                           &c, plan.mu.data(), en.data()));
  plan.engage.assign(en.begin(), en.end());
  return plan;
}

// lobpcg.hpp:67-68 -- ci::lobpcg_solve on the GPU.
SolveReport lobpcg_solve(const CsbMatrix& h, const BlockVectors& x0, const LobpcgOptions& opt) {
  if (x0.dim() != h.dim) throw DimensionMismatch("lobpcg: X0 dim != matrix dim");
  cieg_lobpcg_options o{opt.k_want, opt.tol, opt.max_iter, config(opt.precond_config)};
  struct Obs {
    const LobpcgOptions* opt;
  } obs{&opt};
  cieg_observer_fn fn = nullptr;
  if (opt.observer)
    fn = [](void* user, int it, const double* xh, std::uint32_t n, std::uint32_t kt, const double* th,
            const double* rr) {
      auto* o = static_cast<Obs*>(user);
      BlockVectors X(n, kt);
      std::memcpy(X.values().data(), xh, sizeof(double) * n * kt);
      std::vector<double> theta(th, th + kt), relres(rr, rr + kt);
      o->opt->observer(IterationView{it, X, theta, relres});
    };
  cieg_report* rep = nullptr;
  check(cieg_lobpcg_solve(dev().ctx, matrix(h), x0.values().data(), x0.width(),
                          opt.preconditioner ? precond(*opt.preconditioner) : nullptr, &o, fn, &obs, &rep));
  SolveReport out;
  int conv = 0, iters = 0;
  double ne = 0.0;
  std::uint32_t kw = 0, kt = 0;
  std::uint64_t nh = 0, cnt[4];
  cieg_report_summary(rep, &conv, &iters, &ne, &kw, &kt, &nh);
  cieg_report_counters(rep, cnt);
  out.converged = conv != 0;
  out.iterations = iters;
  out.norm_estimate = ne;
  out.counters = OperationCounters{cnt[0], cnt[1], cnt[2], cnt[3]};
  out.eigenvalues.resize(kw);
  cieg_report_eigenvalues(rep, out.eigenvalues.data());
  out.trial_vectors = BlockVectors(h.dim, kt);
  cieg_report_trial_vectors(rep, out.trial_vectors.values().data());
  out.eigenvectors = BlockVectors(h.dim, kw);
  for (std::uint32_t i = 0; i < h.dim; ++i)
    for (std::uint32_t j = 0; j < kw; ++j) out.eigenvectors.at(i, j) = out.trial_vectors.at(i, j);
  std::vector<int> hi(nh), hc(nh);
  std::vector<double> hr(nh), ht(nh);
  cieg_report_history(rep, hi.data(), hc.data(), hr.data(), ht.data());
  for (std::uint64_t i = 0; i < nh; ++i) out.history.push_back({hi[i], hc[i], hr[i], ht[i]});
  cieg_report_destroy(rep);
  return out;
}

// lanczos.hpp:26 -- host logic.
bool lanczos_checkpoint(int m) { return cieg_lanczos_checkpoint(m) != 0; }

// lanczos.hpp:30 -- ones on the lowest stratum, normalised.
Eigen::VectorXd lanczos_default_start(const BasisTable& basis) {
  Eigen::VectorXd v(basis.dimension());
  check(cieg_lanczos_default_start(basis.dimension(), basis.stratum_end(0), v.data()));
  return v;
}

// lanczos.hpp:35-36 -- ci::lanczos_solve on the GPU.
SolveReport lanczos_solve(const CsbMatrix& h, const Eigen::VectorXd& v0, const LanczosOptions& opt) {
  if (static_cast<std::uint32_t>(v0.size()) != h.dim) throw DimensionMismatch("lanczos: v0 dim != matrix dim");
  if (v0.norm() == 0.0) throw ConfigError("lanczos: v0 must be nonzero");
  if (opt.k_want < 1) throw ConfigError("lanczos: k_want must be >= 1");
  cieg_lanczos_options o;
  cieg_lanczos_options_default(&o);
  o.k_want = opt.k_want;
  o.tol = opt.tol;
  o.max_iter = opt.max_iter;
  if (opt.observer) {
    o.observer = [](void* user, int m, const double* a, const double* b, const double* basis_host, std::uint32_t n) {
      const auto* op = static_cast<const LanczosOptions*>(user);
      Eigen::MatrixXd basis(n, m);
      std::memcpy(basis.data(), basis_host, sizeof(double) * static_cast<std::size_t>(n) * m);
      op->observer(m, basis, std::vector<double>(a, a + m), std::vector<double>(b, b + m));
    };
    o.observer_user = const_cast<LanczosOptions*>(&opt);
  }
  cieg_report* rep = nullptr;
  check(cieg_lanczos_solve(dev().ctx, matrix(h), v0.data(), &o, &rep));
  SolveReport out;
  int conv = 0, iters = 0;
  double ne = 0.0;
  std::uint32_t kw = 0, kt = 0;
  std::uint64_t nh = 0, cnt[4];
  cieg_report_summary(rep, &conv, &iters, &ne, &kw, &kt, &nh);
  cieg_report_counters(rep, cnt);
  out.converged = conv != 0;
  out.iterations = iters;
  out.norm_estimate = ne;
  out.counters = OperationCounters{cnt[0], cnt[1], cnt[2], cnt[3]};
  out.eigenvalues.resize(kw);
  cieg_report_eigenvalues(rep, out.eigenvalues.data());
  out.eigenvectors = BlockVectors(h.dim, kw);
  cieg_report_trial_vectors(rep, out.eigenvectors.values().data());
  out.trial_vectors = out.eigenvectors;
  std::vector<int> hi(nh), hc(nh);
  std::vector<double> hr(nh), ht(nh);
  cieg_report_history(rep, hi.data(), hc.data(), hr.data(), ht.data());
  for (std::uint64_t i = 0; i < nh; ++i) out.history.push_back({hi[i], hc[i], hr[i], ht[i]});
  cieg_report_destroy(rep);
  return out;
}

// lobpcg.hpp:92-93 -- ci::orthonormalize on the GPU.
BlockVectors orthonormalize(const BlockVectors& y, double drop_tol, const BlockVectors* against) {
  if (against && against->dim() != y.dim()) throw DimensionMismatch("orthonormalize: row counts differ");
  DevBlock dy(y.values().data(), y.values().size());
  std::unique_ptr<DevBlock> da;
  if (against && against->width()) da = std::make_unique<DevBlock>(against->values().data(), against->values().size());
  std::uint32_t k = 0;
  check(cieg_orthonormalize(dev().ctx, dy.d(), y.dim(), y.width(), drop_tol, da ? da->d() : nullptr,
                            da ? against->width() : 0, &k));
  BlockVectors out(y.dim(), k);
  dy.to_host(out.values().data(), out.values().size());
  return out;
}

// lobpcg.hpp:84-86 -- ci::rayleigh_ritz on the GPU.
std::pair<std::vector<double>, SubspaceCoefficients> rayleigh_ritz(const BlockVectors& y_basis,
                                                                   const BlockVectors& hy, int k_trial, int x_width,
                                                                   int w_width, int p_width) {
  const int m = static_cast<int>(y_basis.width());
  if (k_trial > m) throw DimensionMismatch("rayleigh_ritz: k_trial exceeds basis width");
  if (hy.width() != y_basis.width() || hy.dim() != y_basis.dim())
    throw DimensionMismatch("rayleigh_ritz: HY shape mismatch");
  DevBlock dy(y_basis.values().data(), y_basis.values().size()), dh(hy.values().data(), hy.values().size());
  std::vector<double> theta(k_trial);
  SubspaceCoefficients c;
  c.g.resize(m, k_trial);
  check(cieg_rayleigh_ritz(dev().ctx, dy.d(), dh.d(), y_basis.dim(), m, k_trial, theta.data(), c.g.data()));
  c.x_width = x_width < 0 ? m : x_width;
  c.w_width = w_width;
  c.p_width = p_width;
  return {std::move(theta), std::move(c)};
}

// lobpcg.hpp:97-99 -- ci::residual_norms on the GPU.
std::vector<double> residual_norms(const CsbMatrix& h, const BlockVectors& x, const std::vector<double>& theta,
                                   std::optional<double> norm_est) {
  if (x.width() != theta.size()) throw DimensionMismatch("residual_norms: theta width mismatch");
  DevBlock dx(x.values().data(), x.values().size());
  std::vector<double> out(x.width());
  check(cieg_residual_norms(dev().ctx, matrix(h), dx.d(), x.width(), theta.data(), norm_est.value_or(0.0),
                            out.data()));
  return out;
}


// ---- block_vectors.hpp:60-75 -- the tall-skinny kernels (K2/K3) ------------
// block_vectors.hpp:60 -- X^T Y, fixed-order device reduction (deterministic
// like the reference's panel order, block_vectors.cpp:74-85).
Eigen::MatrixXd block_inner(const BlockVectors& x, const BlockVectors& y) {
  if (x.dim() != y.dim()) throw DimensionMismatch("block_inner: row counts differ");
  Eigen::MatrixXd g = Eigen::MatrixXd::Zero(x.width(), y.width());
  if (x.dim() == 0 || x.width() == 0 || y.width() == 0) return g;
  DevBlock dx(x.values().data(), x.values().size()), dy(y.values().data(), y.values().size());
  check(cieg_block_inner(dev().ctx, x.dim(), dx.d(), x.width(), dy.d(), y.width(), g.data()));
  return g;
}
Eigen::MatrixXd block_inner_serial(const BlockVectors& x, const BlockVectors& y) { return block_inner(x, y); }

// block_vectors.hpp:64 -- Y G.
BlockVectors linear_combination(const BlockVectors& y, const Eigen::MatrixXd& g) {
  if (static_cast<std::uint32_t>(g.rows()) != y.width())
    throw DimensionMismatch("linear_combination: G rows != block width");
  const auto kout = static_cast<std::uint32_t>(g.cols());
  BlockVectors out(y.dim(), kout);
  if (y.dim() == 0 || kout == 0) return out;
  if (y.width() == 0) return out;  // empty sum
  DevBlock dy(y.values().data(), y.values().size()), dout(nullptr, out.values().size());
  check(cieg_linear_combination(dev().ctx, y.dim(), dy.d(), y.width(), g.data(), kout, dout.d()));
  dout.to_host(out.values().data(), out.values().size());
  return out;
}
BlockVectors linear_combination_serial(const BlockVectors& y, const Eigen::MatrixXd& g) {
  return linear_combination(y, g);
}

// block_vectors.hpp:68 -- Y += X G.
void add_linear_combination(BlockVectors& y, const BlockVectors& x, const Eigen::MatrixXd& g) {
  if (x.dim() != y.dim()) throw DimensionMismatch("add_linear_combination: dims");
  if (static_cast<std::uint32_t>(g.rows()) != x.width() || static_cast<std::uint32_t>(g.cols()) != y.width())
    throw DimensionMismatch("add_linear_combination: G shape");
  if (y.dim() == 0 || y.width() == 0 || x.width() == 0) return;
  DevBlock dy(y.values().data(), y.values().size()), dx(x.values().data(), x.values().size());
  check(cieg_add_linear_combination(dev().ctx, y.dim(), dy.d(), y.width(), dx.d(), x.width(), g.data()));
  dy.to_host(y.values().data(), y.values().size());
}

// block_vectors.hpp:72 -- host (hash of (seed, row, col); rng.hpp).
BlockVectors random_block(std::uint32_t dim, std::uint32_t width, std::uint64_t seed) {
  BlockVectors out(dim, width);
  if (dim && width) check(cieg_random_block(dim, width, seed, out.values().data()));
  return out;
}

// block_vectors.hpp:75 -- only the Gram diagonal is formed on the device.
std::vector<double> column_norms(const BlockVectors& x) {
  std::vector<double> out(x.width(), 0.0);
  if (x.dim() == 0 || x.width() == 0) return out;
  DevBlock dx(x.values().data(), x.values().size());
  check(cieg_column_norms(dev().ctx, x.dim(), dx.d(), x.width(), out.data()));
  return out;
}

// ---- precond.hpp:53-61 -- the tile preconditioner (K5) ---------------------
BlockVectors apply_preconditioner(const TileDiagonal& tiles, const BlockVectors& r, const ShiftPlan& plan,
                                  const PrecondConfig& cfg) {
  if (plan.mu.size() != r.width() || plan.engage.size() != r.width())
    throw DimensionMismatch("apply_preconditioner: plan width != residual width");
  if (tiles.group_count() > 0 && tiles.ranges.back().second != r.dim())
    throw DimensionMismatch("apply_preconditioner: tiles do not cover the basis");
  if (tiles.group_count() == 0 || r.dim() == 0 || r.width() == 0) return r;  // nothing to solve: pass-through
  BlockVectors w(r.dim(), r.width());
  std::vector<int> en(plan.engage.begin(), plan.engage.end());
  cieg_precond_config c = config(cfg);
  DevBlock dr(r.values().data(), r.values().size()), dw(nullptr, w.values().size());
  check(cieg_precond_apply(dev().ctx, precond(tiles), dr.d(), r.width(), plan.mu.data(), en.data(), &c, dw.d()));
  dw.to_host(w.values().data(), w.values().size());
  return w;
}

// precond.hpp:60-61 -- FOM on one dense block: a one-group tile diagonal
// applied with the direct-solve cutoff at 0 (every group takes FOM) and
// inner_iters = iters (the device FOM keeps PrecondConfig's 1..3 range).
Eigen::MatrixXd fom_solve(const Eigen::MatrixXd& block, const std::vector<double>& mu, const Eigen::MatrixXd& rhs,
                          int iters) {
  if (iters < 1) throw ConfigError("fom_solve: iters must be >= 1");
  const auto n = static_cast<std::uint32_t>(block.rows());
  const auto k = static_cast<std::uint32_t>(rhs.cols());
  if (mu.size() != k) throw DimensionMismatch("fom_solve: one shift per right-hand side");
  Eigen::MatrixXd x = Eigen::MatrixXd::Zero(n, k);
  if (n == 0 || k == 0) return x;
  const std::uint32_t bounds[2] = {0, n};
  cieg_tilediag_view v{n, 1, bounds, block.data()};
  cieg_prec* p = nullptr;
  check(cieg_precond_upload(dev().ctx, &v, &p));
  std::unique_ptr<cieg_prec, int (*)(cieg_prec*)> guard(p, cieg_precond_destroy);
  cieg_precond_config c;
  cieg_precond_config_default(&c);
  c.small_block_cutoff = 0;
  c.inner_iters = iters;
  std::vector<double> rrow(static_cast<std::size_t>(n) * k);  // row major
  for (std::uint32_t i = 0; i < n; ++i)
    for (std::uint32_t j = 0; j < k; ++j) rrow[static_cast<std::size_t>(i) * k + j] = rhs(i, j);
  std::vector<int> en(k, 1);
  DevBlock dr(rrow.data(), rrow.size()), dw(nullptr, rrow.size());
  check(cieg_precond_apply(dev().ctx, p, dr.d(), k, mu.data(), en.data(), &c, dw.d()));
  dw.to_host(rrow.data(), rrow.size());
  for (std::uint32_t i = 0; i < n; ++i)
    for (std::uint32_t j = 0; j < k; ++j) x(i, j) = rrow[static_cast<std::size_t>(i) * k + j];
  return x;
}

}  // namespace ci

// C entry for the test harness: run the reference-API call sequence of the
// CLI's run_solver (ci_eigen.cpp:139-151) through the drop-in.
namespace {
// cieg_csb_view -> ci::CsbMatrix (the caller-side object the drop-in receives)
ci::CsbMatrix from_view(const cieg_csb_view* v) {
    ci::CsbMatrix h;
    h.dim = v->dim;
    h.precision = v->precision == 0 ? ci::Precision::Single : ci::Precision::Double;
    h.layout.block_boundaries.assign(v->block_boundaries, v->block_boundaries + v->nb + 1);
    h.blocks.resize(static_cast<std::size_t>(v->nb) * (v->nb + 1) / 2);
    for (std::size_t b = 0; b < h.blocks.size(); ++b) {
      auto& blk = h.blocks[b];
      const std::uint64_t e0 = v->entry_offsets[b], e1 = v->entry_offsets[b + 1];
      blk.rows.assign(v->rows + e0, v->rows + e1);
      blk.cols.assign(v->cols + e0, v->cols + e1);
      if (v->precision == 0)
        blk.values32.assign(static_cast<const float*>(v->values) + e0, static_cast<const float*>(v->values) + e1);
      else
        blk.values64.assign(static_cast<const double*>(v->values) + e0, static_cast<const double*>(v->values) + e1);
      h.nnz_lower += blk.size();
    }
    return h;
}
}  // namespace

extern "C" int dropin_lobpcg(const cieg_csb_view* v, const std::uint32_t* groups, std::uint32_t ng,
                             const double* x0, std::uint32_t kt, int k_want, double tol, int use_prec,
                             double* eig_out, int* iters_out) {
  try {
    ci::CsbMatrix h = from_view(v);
    ci::TileDiagonal td;
    if (use_prec) {
      for (std::uint32_t g = 0; g < ng; ++g) {
        const std::uint32_t s = groups[g], e = groups[g + 1];
        td.ranges.push_back({s, e});
        Eigen::MatrixXd blk = Eigen::MatrixXd::Zero(e - s, e - s);
        td.blocks.push_back(blk);
      }
      // fill from H's diagonal blocks (the reference's extract_tile_diagonal needs a
      // GroupPartition; this harness mirrors it directly)
      for (std::uint32_t i = 0; i < h.block_count(); ++i) {
        const auto& b = h.block(i, i);
        const std::uint32_t base = h.layout.block_boundaries[i];
        for (std::size_t e = 0; e < b.size(); ++e) {
          const std::uint32_t r = base + b.rows[e], c = base + b.cols[e];
          std::uint32_t g = 0;
          while (groups[g + 1] <= r) ++g;
          if (c < groups[g]) continue;
          const double val = h.value(i * (i + 1) / 2 + i, e);
          td.blocks[g](r - groups[g], c - groups[g]) = val;
          td.blocks[g](c - groups[g], r - groups[g]) = val;
        }
      }
    }
    ci::BlockVectors X0(h.dim, kt);
    std::memcpy(X0.values().data(), x0, sizeof(double) * h.dim * kt);
    ci::LobpcgOptions opt;
    opt.k_want = k_want;
    opt.tol = tol;
    opt.preconditioner = use_prec ? &td : nullptr;
    ci::SolveReport rep = ci::lobpcg_solve(h, X0, opt);
    for (int j = 0; j < k_want; ++j) eig_out[j] = rep.eigenvalues[j];
    *iters_out = rep.iterations;
    return 0;
  } catch (const ci::Error& e) {
    return 1;
  }
}

// Lanczos through the reference API (lanczos.hpp:35-36).
extern "C" int dropin_lanczos(const cieg_csb_view* v, const double* v0, int k_want, double tol, int max_iter,
                              double* eig_out, int* iters_out) {
  try {
    ci::CsbMatrix h = from_view(v);
    Eigen::VectorXd x(h.dim);
    std::memcpy(x.data(), v0, sizeof(double) * h.dim);
    ci::LanczosOptions opt;
    opt.k_want = k_want;
    opt.tol = tol;
    opt.max_iter = max_iter;
    ci::SolveReport rep = ci::lanczos_solve(h, x, opt);
    for (int j = 0; j < k_want && j < static_cast<int>(rep.eigenvalues.size()); ++j) eig_out[j] = rep.eigenvalues[j];
    *iters_out = rep.iterations;
    return 0;
  } catch (const ci::Error& e) {
    return 1;
  }
}

// ci::orthonormalize / ci::residual_norms through the drop-in (test harness).
extern "C" int dropin_orthonormalize(std::uint32_t n, std::uint32_t k, const double* y, double drop_tol, double* out,
                                     std::uint32_t* kout) {
  try {
    ci::BlockVectors Y(n, k);
    std::memcpy(Y.values().data(), y, sizeof(double) * n * k);
    ci::BlockVectors Q = ci::orthonormalize(Y, drop_tol);
    *kout = Q.width();
    std::memcpy(out, Q.values().data(), sizeof(double) * Q.values().size());
    return 0;
  } catch (const ci::Error&) {
    return 1;
  }
}

extern "C" int dropin_residual_norms(const cieg_csb_view* v, const double* x, std::uint32_t k, const double* theta,
                                     double* out) {
  try {
    ci::CsbMatrix h = from_view(v);
    ci::BlockVectors X(h.dim, k);
    std::memcpy(X.values().data(), x, sizeof(double) * h.dim * k);
    std::vector<double> r = ci::residual_norms(h, X, std::vector<double>(theta, theta + k));
    std::memcpy(out, r.data(), sizeof(double) * k);
    return 0;
  } catch (const ci::Error&) {
    return 1;
  }
}

// Drop every cached upload (matrices and tile diagonals); the next call
// re-uploads. For callers that mutate a CsbMatrix / TileDiagonal in place.
extern "C" void cieg_dropin_invalidate() { dev().clear(); }
