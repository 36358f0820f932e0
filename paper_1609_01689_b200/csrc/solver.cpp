// solver.cpp -- ci::lobpcg_solve on the GPU (proj/src/lobpcg.cpp:216-387).
//
// The host runs the reference's control flow verbatim -- the same order of
// Gram products, the same thresholds (drop_tol 1e-8, overlap 1e-8, X guard
// 1e-12, kTinyDiag 1e-300), the same pivoted-Cholesky column selection, LLT
// failure handling, P-drop rescue and soft locking -- while every pass over
// n-length data runs on the device: X, HX, P, HP, W, HW, R stay resident in
// HBM; Grams come back as <= 48x48 matrices, coefficient panels go down as
// kernel parameters. [X W P] is never materialised: Grams and updates take
// column-concatenated views (blockvec.hpp).
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "blockvec.hpp"
#include "dense_small.hpp"
#include "precond.hpp"
#include "report.hpp"


namespace cieg {
namespace {

constexpr double kTinyDiag = 1e-300;
using Mat = std::vector<double>;  // column-major small dense matrix

// Device block n x w (row-major, ld = w) with capacity for `cap` columns.
struct Block {
  double* p = nullptr;
  std::uint32_t w = 0;
  std::uint32_t cap = 0;
};

// Solver work blocks come from a pool kept in the context, so back-to-back
// solves reuse their allocations (no cudaMalloc / synchronising cudaFree per
// solve); buffers only grow.
struct Workspace {
  cieg_ctx* ctx = nullptr;
  std::uint32_t n = 0;
  std::size_t next = 0;
  Block alloc(std::uint32_t cap) {
    Block b;
    b.cap = cap;
    const std::size_t bytes = sizeof(double) * std::max<std::size_t>(1, static_cast<std::size_t>(n) * cap);
    if (ctx->solver_pool.size() <= next) ctx->solver_pool.emplace_back();
    b.p = static_cast<double*>(ctx->solver_pool[next++].get(bytes));
    return b;
  }
};

Seg sg(const Block& b) { return Seg{b.p, b.w, b.w}; }

// rank_revealing_select (lobpcg.cpp:20-51): pivoted Cholesky on a copy of the
// Gram; kept columns in input order.
std::vector<std::uint32_t> rank_revealing_select(Mat gram, int m, const std::vector<double>& orig_sq,
                                                 double drop_tol) {
  auto G = [&](int a, int b) -> double& { return gram[a + static_cast<std::size_t>(b) * m]; };
  std::vector<bool> active(m, true);
  std::vector<std::uint32_t> kept;
  for (int step = 0; step < m; ++step) {
    int pivot = -1;
    double best = -1.0;
    for (int j = 0; j < m; ++j)
      if (active[j] && G(j, j) > best) {
        best = G(j, j);
        pivot = j;
      }
    if (pivot < 0) break;
    active[pivot] = false;
    const double threshold = std::max(drop_tol * drop_tol * orig_sq[pivot], kTinyDiag);
    if (!(G(pivot, pivot) > threshold)) continue;
    kept.push_back(static_cast<std::uint32_t>(pivot));
    const double d = G(pivot, pivot);
    for (int a = 0; a < m; ++a) {
      if (!active[a]) continue;
      for (int b = 0; b < m; ++b) {
        if (!active[b] && b != a) continue;
        G(a, b) -= G(a, pivot) * G(b, pivot) / d;
      }
    }
  }
  std::sort(kept.begin(), kept.end());
  return kept;
}

// LLT of a (k x k); on success returns R^{-1} (upper triangular inverse of
// U = L^T), as right_solve_upper does (lobpcg.cpp:54-58).
bool llt_rinv(const Mat& a, int k, Mat& rinv) {
  Mat l = a;
  if (!cieg_dense::cholesky_lower(k, l.data())) return false;
  Mat u(static_cast<std::size_t>(k) * k);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) u[i + j * k] = l[j + i * k];
  rinv.assign(static_cast<std::size_t>(k) * k, 0.0);
  cieg_dense::upper_inverse(k, u.data(), rinv.data());
  return true;
}

// eig_sym (lobpcg.cpp:78-85): symmetrise 1/2 (A + A^T), ascending eigenpairs.
void eig_sym(const Mat& a, int m, std::vector<double>& evals, Mat& evecs) {
  Mat sym(static_cast<std::size_t>(m) * m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) sym[i + j * m] = 0.5 * (a[i + j * m] + a[j + i * m]);
  evals.assign(m, 0.0);
  evecs.assign(static_cast<std::size_t>(m) * m, 0.0);
  if (!cieg_dense::sym_eig(m, sym.data(), evals.data(), evecs.data()))
    fail(CIEG_ERR_INDEFINITE, "projected eigensolver failed to converge");
}

double dev_from_identity(const Mat& g, int m) {
  double d = 0.0;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) d = std::max(d, std::fabs(g[i + j * m] - (i == j ? 1.0 : 0.0)));
  return d;
}


// Gram products of a (possibly row-sharded) solve: local partials, then the
// all-reduce hook when sharded -- for plain Grams and for Grams fused into a
// combine pass alike.
struct GramOps {
  cieg_ctx* ctx;
  std::uint32_t n;
  const cieg_dist_hooks* hooks;
  Mat reduce(Mat g) const {
    if (nccl_active(ctx)) return g;  // already summed on the device (nccl_plane.cu)
    if (hooks && !g.empty() && hooks->allreduce_sum(hooks->user, g.data(), g.size()) != 0)
      fail(CIEG_ERR_ARGUMENT, "allreduce_sum hook failed");
    return g;
  }
  Mat gram(const View3& l, const View3& r) const { return reduce(cieg::gram(ctx, n, l, r)); }
  // two independent Grams, one host round trip
  std::pair<Mat, Mat> gram_pair(const View3& l1, const View3& r1, const View3& l2, const View3& r2) const {
    auto g = cieg::gram_pair(ctx, n, l1, r1, l2, r2);
    return {reduce(std::move(g.first)), reduce(std::move(g.second))};
  }
  // out = [out] + in G, returning L^T out (or out^T out for L == nullptr)
  Mat combine_gram(const View3& in, const double* g, std::uint32_t kout, const Out2& out, bool acc,
                   const View3* L) const {
    return reduce(cieg::combine_gram(ctx, n, in, g, kout, out, acc, L));
  }
};

// orthonormalize (lobpcg.cpp:89-119) over device blocks. `v` holds the input
// (width v.w) and is overwritten; `tmp` is scratch of the same capacity; the
// result (possibly width 0) is left in `v` (the two may swap). The second
// projection pass's Gram and the Gram of the projected block are fused into
// the combine passes that produce them.
void orthonormalize_dev(const GramOps& ops, Block& v, Block& tmp, double drop_tol, const View3* against) {
  if (v.w == 0) return;
  cieg_ctx* ctx = ops.ctx;
  const std::uint32_t n = ops.n;
  const int k = static_cast<int>(v.w);
  const bool proj = against && against->width > 0;
  Mat g0, c;
  if (proj)  // V^T V and A^T V are independent: one host round trip
    std::tie(g0, c) = ops.gram_pair(view({sg(v)}), view({sg(v)}), *against, view({sg(v)}));
  else
    g0 = ops.gram(view({sg(v)}), view({sg(v)}));
  std::vector<double> orig_sq(k);
  for (int j = 0; j < k; ++j) orig_sq[j] = g0[j + static_cast<std::size_t>(j) * k];
  Mat gram_v = g0;  // without a projection the Gram is unchanged
  if (proj) {
    for (double& e : c) e = -e;
    Mat c2 = ops.combine_gram(*against, c.data(), v.w, out1(v.p, v.w), true, against);  // pass 1 + pass-2 Gram
    for (double& e : c2) e = -e;
    gram_v = ops.combine_gram(*against, c2.data(), v.w, out1(v.p, v.w), true, nullptr);  // pass 2 + V^T V
  }
  std::vector<std::uint32_t> kept = rank_revealing_select(gram_v, k, orig_sq, drop_tol);
  while (!kept.empty()) {
    const int kk = static_cast<int>(kept.size());
    Mat sub(static_cast<std::size_t>(kk) * kk);
    for (int a = 0; a < kk; ++a)
      for (int b = 0; b < kk; ++b) sub[a + b * kk] = gram_v[kept[a] + static_cast<std::size_t>(kept[b]) * k];
    Mat rinv;
    if (llt_rinv(sub, kk, rinv)) {
      // q = V[:, kept] R^{-1}: one combine with the selection folded in,
      // fused with the Gram of q for the second CholQR pass
      Mat sel(static_cast<std::size_t>(k) * kk, 0.0);
      for (int a = 0; a < kk; ++a)
        for (int c = 0; c < kk; ++c) sel[kept[a] + static_cast<std::size_t>(c) * k] = rinv[a + c * kk];
      Mat gq = ops.combine_gram(view({sg(v)}), sel.data(), kk, out1(tmp.p, kk), false, nullptr);
      tmp.w = kk;
      std::swap(v, tmp);
      // cholqr_pass (lobpcg.cpp:61-69): second pass, result ignored on failure.
      Mat rinv2;
      if (llt_rinv(gq, kk, rinv2)) combine(ctx, n, view({sg(v)}), rinv2.data(), kk, out1(v.p, kk), false);
      return;
    }
    kept.pop_back();
  }
  v.w = 0;
}

class Solver {
 public:
  Solver(cieg_ctx* ctx, const cieg_mat* mat, const cieg_prec* prec, const cieg_lobpcg_options& opt,
         cieg_report& rep, const cieg_dist_hooks* hooks = nullptr)
      : ctx_(ctx), mat_(mat), prec_(prec), opt_(opt), rep_(rep), n_(mat->row_hi - mat->row_lo), hooks_(hooks),
        ops_{ctx, mat->row_hi - mat->row_lo, hooks} {
    ws_.ctx = ctx;
    ws_.n = n_;
    if (hooks_ && hooks_->reduce_partials && mat_->sp_sched) {
      // single-pass SpMMs need room for their partial slots on every rank;
      // one collective decision keeps the ranks' SpMM modes (and so their
      // partial exchanges) in step
      double no_room = single_pass_fits(ctx_, mat_, kSinglePassMaxCols) ? 0.0 : 1.0;
      if (hooks_->allreduce_sum(hooks_->user, &no_room, 1) != 0) fail(CIEG_ERR_ARGUMENT, "allreduce_sum hook failed");
      sp_ok_ = no_room == 0.0;
    }
  }

  void run(const double* x0_host, std::uint32_t kt0, cieg_observer_fn obs, void* user);
  ~Solver() {
    clock_discard(ctx_);
    cudaFree(singular_);
    xfull_.release();
    yhalo_.release();
  }

 private:
  // orthonormalize (lobpcg.cpp:89-119). `v` holds the input (width v.w) and is
  // overwritten; `tmp` is scratch of the same capacity. Returns the result in
  // `v` (possibly width 0).
  void orthonormalize(Block& v, Block& tmp, double drop_tol, const View3* against);
  void spmm(const Block& x, Block& hx) {
    Clock c(ctx_, &rep_.timing_ms[kSpmm]);
    ++rep_.counters[0];
    rep_.counters[1] += x.w;
    const double* xin = x.p;
    if (hooks_) {
      // sharded: the owner kernel reads X only on the shard's halo rows, so
      // only those are allocated; `full` is addressed with global row indices
      const std::size_t rows = mat_->halo_hi - mat_->halo_lo, w = std::max<std::uint32_t>(x.w, 1);
      double* buf = static_cast<double*>(xfull_.get(sizeof(double) * std::max<std::size_t>(1, rows) * w));
      double* full = buf - static_cast<std::ptrdiff_t>(mat_->halo_lo) * x.w;
      if (hooks_->allgather_rows(hooks_->user, x.p, x.w, full) != 0)
        fail(CIEG_ERR_ARGUMENT, "allgather_rows hook failed");
      xin = full;
      if (sp_ok_ && single_pass_rule(ctx_, mat_, x.w)) {
        // single pass: the transposed partials for lower ranks' rows travel
        // back to their owners (SURVEY.md 8(e) reduce-scatter, point to point)
        const std::size_t prow = mat_->row_lo - mat_->sp_partial_lo;
        double* yh = static_cast<double*>(yhalo_.get(sizeof(double) * std::max<std::size_t>(1, prow) * w));
        launch_spmm(ctx_, mat_, xin, x.w, hx.p, x.w, x.w, yh, x.w, true);
        if (hooks_->reduce_partials(hooks_->user, yh, x.w, hx.p) != 0)
          fail(CIEG_ERR_ARGUMENT, "reduce_partials hook failed");
        hx.w = x.w;
        return;
      }
    }
    launch_spmm(ctx_, mat_, xin, x.w, hx.p, x.w, x.w);
    hx.w = x.w;
  }
  Mat gram(const View3& l, const View3& r) { return ops_.gram(l, r); }
  // c1: X^T P when already known (fused into the Rayleigh-Ritz update), else empty
  void clean_p_block(double drop_tol, const Mat& c1);

  cieg_ctx* ctx_;
  const cieg_mat* mat_;
  const cieg_prec* prec_;
  int* singular_ = nullptr;  // device count of singular-shift pass-throughs (read once, at the end)
  cieg_lobpcg_options opt_;
  cieg_report& rep_;
  std::uint32_t n_;  // local rows (all rows unless sharded)
  const cieg_dist_hooks* hooks_;
  GramOps ops_;
  DevBuf xfull_, yhalo_;
  bool sp_ok_ = false;  // sharded single-pass SpMMs enabled (collective decision)
  Workspace ws_;
  Block x_, hx_, p_, hp_, x2_, hx2_, p2_, hp2_, w_, hw_, wtmp_, r_, wsrc_;
  std::vector<double> theta_;
};

void Solver::orthonormalize(Block& v, Block& tmp, double drop_tol, const View3* against) {
  orthonormalize_dev(ops_, v, tmp, drop_tol, against);
}

void Solver::clean_p_block(double drop_tol, const Mat& c1) {
  // lobpcg.cpp:180-212; the second pass's X^T P and the final P^T P are fused
  // into the combine passes that produce P
  if (p_.w == 0) return;
  const View3 xv = view({sg(x_)});
  Mat c = c1.empty() ? gram(xv, view({sg(p_)})) : c1;
  for (double& e : c) e = -e;
  Mat c2 = ops_.combine_gram(xv, c.data(), p_.w, out1(p_.p, p_.w), true, &xv);
  combine(ctx_, n_, view({sg(hx_)}), c.data(), hp_.w, out1(hp_.p, hp_.w), true);
  for (double& e : c2) e = -e;
  Mat g = ops_.combine_gram(xv, c2.data(), p_.w, out1(p_.p, p_.w), true, nullptr);
  combine(ctx_, n_, view({sg(hx_)}), c2.data(), hp_.w, out1(hp_.p, hp_.w), true);
  const int k = static_cast<int>(p_.w);
  std::vector<double> orig_sq(k);
  for (int j = 0; j < k; ++j) orig_sq[j] = g[j + static_cast<std::size_t>(j) * k];
  std::vector<std::uint32_t> kept = rank_revealing_select(g, k, orig_sq, drop_tol);
  if (kept.empty()) {
    p_.w = hp_.w = 0;
    return;
  }
  const int kk = static_cast<int>(kept.size());
  Mat sub(static_cast<std::size_t>(kk) * kk);
  for (int a = 0; a < kk; ++a)
    for (int b = 0; b < kk; ++b) sub[a + b * kk] = g[kept[a] + static_cast<std::size_t>(kept[b]) * k];
  Mat rinv;
  if (!llt_rinv(sub, kk, rinv)) {
    p_.w = hp_.w = 0;  // direction block beyond repair; drop it
    return;
  }
  Mat sel(static_cast<std::size_t>(k) * kk, 0.0);
  for (int a = 0; a < kk; ++a)
    for (int c = 0; c < kk; ++c) sel[kept[a] + static_cast<std::size_t>(c) * k] = rinv[a + c * kk];
  combine(ctx_, n_, view({sg(p_)}), sel.data(), kk, out1(p2_.p, kk), false);
  combine(ctx_, n_, view({sg(hp_)}), sel.data(), kk, out1(hp2_.p, kk), false);
  p2_.w = hp2_.w = kk;
  std::swap(p_, p2_);
  std::swap(hp_, hp2_);
}

void Solver::run(const double* x0_host, std::uint32_t kt0, cieg_observer_fn obs, void* user) {
  const auto t_start = std::chrono::steady_clock::now();
  if (static_cast<int>(kt0) < opt_.k_want) fail(CIEG_ERR_CONFIG, "lobpcg: trial width below k_want");
  if (kt0 > 16) fail(CIEG_ERR_CONFIG, "lobpcg: trial width above 16 is not supported (3*kt <= 48)");
  const double drop_tol = 1e-8;
  const std::uint32_t K = kt0;
  x_ = ws_.alloc(K);
  hx_ = ws_.alloc(K);
  p_ = ws_.alloc(K);
  hp_ = ws_.alloc(K);
  x2_ = ws_.alloc(K);
  hx2_ = ws_.alloc(K);
  p2_ = ws_.alloc(K);
  hp2_ = ws_.alloc(K);
  w_ = ws_.alloc(K);
  hw_ = ws_.alloc(K);
  wtmp_ = ws_.alloc(K);
  r_ = ws_.alloc(K);
  wsrc_ = ws_.alloc(K);

  {
    Clock c(ctx_, &rep_.timing_ms[kOther]);
    CIEG_CUDA(cudaMemcpyAsync(x_.p, x0_host, sizeof(double) * n_ * K, cudaMemcpyHostToDevice, ctx_->stream));
    x_.w = K;
  }
  {
    Clock c(ctx_, &rep_.timing_ms[kOrtho]);
    orthonormalize(x_, x2_, drop_tol, nullptr);
  }
  ++rep_.counters[3];
  if (static_cast<int>(x_.w) < opt_.k_want)
    fail(CIEG_ERR_SUBSPACE, "initial block has fewer than k_want independent columns");
  const int kt = static_cast<int>(x_.w);
  spmm(x_, hx_);
  {
    Clock c(ctx_, &rep_.timing_ms[kRR]);
    Mat g = gram(view({sg(x_)}), view({sg(hx_)}));
    std::vector<double> evals;
    Mat evecs;
    eig_sym(g, kt, evals, evecs);
    theta_.assign(evals.begin(), evals.begin() + kt);
    combine(ctx_, n_, view({sg(x_)}), evecs.data(), kt, out1(x_.p, kt), false);
    combine(ctx_, n_, view({sg(hx_)}), evecs.data(), kt, out1(hx_.p, kt), false);
  }
  rep_.norm_estimate = std::max(std::fabs(theta_.front()), std::fabs(theta_.back()));
  p_.w = hp_.w = 0;
  std::vector<double> host_x;

  for (int iter = 0;; ++iter) {
    std::vector<double> res_norm(kt), relres(kt);
    {
      Clock c(ctx_, &rep_.timing_ms[kResid]);
      residual(ctx_, n_, kt, hx_.p, x_.p, theta_.data(), r_.p);
      r_.w = kt;
      Mat g = gram(view({sg(r_)}), view({sg(r_)}));
      for (int j = 0; j < kt; ++j) res_norm[j] = std::sqrt(g[j + static_cast<std::size_t>(j) * kt]);
    }
    for (int j = 0; j < kt; ++j) relres[j] = res_norm[j] / std::max(rep_.norm_estimate, kTinyDiag);
    for (int j = 0; j < kt; ++j) rep_.history.push_back({iter, j, relres[j], theta_[j]});
    if (obs) {
      host_x.resize(static_cast<std::size_t>(n_) * kt);
      CIEG_CUDA(cudaMemcpyAsync(host_x.data(), x_.p, sizeof(double) * host_x.size(), cudaMemcpyDeviceToHost,
                                ctx_->stream));
      CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
      obs(user, iter, host_x.data(), n_, static_cast<std::uint32_t>(kt), theta_.data(), relres.data());
    }
    bool all_converged = true;
    for (int j = 0; j < opt_.k_want; ++j) all_converged = all_converged && relres[j] <= opt_.tol;
    rep_.iterations = iter;
    if (all_converged) {
      rep_.converged = true;
      break;
    }
    if (iter >= opt_.max_iter) {
      rep_.converged = false;
      break;
    }

    const Block* wsource = &r_;
    if (prec_) {
      Clock c(ctx_, &rep_.timing_ms[kPrecond]);
      std::vector<double> ones(kt, 1.0);
      ShiftPlan plan = choose_shifts(theta_, res_norm, ones, relres, iter + 1, opt_.tol, opt_.precond_config);
      const bool engaged = std::any_of(plan.engage.begin(), plan.engage.end(), [](int b) { return b != 0; });
      if (!singular_) {
        CIEG_CUDA(cudaMalloc(&singular_, sizeof(int)));
        CIEG_CUDA(cudaMemsetAsync(singular_, 0, sizeof(int), ctx_->stream));
      }
      precond_apply(ctx_, prec_, r_.p, kt, plan, opt_.precond_config, wsrc_.p, singular_);
      wsrc_.w = kt;
      wsource = &wsrc_;
      if (engaged) ++rep_.counters[2];
    }
    std::vector<std::uint32_t> active;
    for (int j = 0; j < kt; ++j)
      if (relres[j] > opt_.tol) active.push_back(static_cast<std::uint32_t>(j));
    {
      Clock c(ctx_, &rep_.timing_ms[kOrtho]);
      gather_columns(ctx_, n_, wsource->p, wsource->w, active, w_.p);
      w_.w = static_cast<std::uint32_t>(active.size());
      View3 xp = view({sg(x_), sg(p_)});
      orthonormalize(w_, wtmp_, drop_tol, &xp);
    }
    ++rep_.counters[3];
    if (w_.w == 0) {
      rep_.converged = false;
      break;
    }
    spmm(w_, hw_);

    const int kw = static_cast<int>(w_.w);
    std::vector<double> evals;
    Mat evecs;
    int m = 0;
    {
      Clock c(ctx_, &rep_.timing_ms[kRR]);
      View3 y = view({sg(x_), sg(w_), sg(p_)});
      View3 hy = view({sg(hx_), sg(hw_), sg(hp_)});
      bool rescued = false;
      try {
        // the overlap check and Y^T HY are independent: one host round trip
        auto [overlap, yhy] = ops_.gram_pair(y, y, y, hy);
        const double dev = dev_from_identity(overlap, static_cast<int>(y.width));
        if (dev > 1e-8) fail(CIEG_ERR_INDEFINITE, "basis drift " + std::to_string(dev));
        eig_sym(yhy, static_cast<int>(y.width), evals, evecs);
      } catch (const Failure& f) {
        if (f.status != CIEG_ERR_INDEFINITE) throw;
        rescued = true;
      }
      if (rescued) {  // drop P and retry on [X W] (lobpcg.cpp:326-333)
        p_.w = hp_.w = 0;
        y = view({sg(x_), sg(w_)});
        hy = view({sg(hx_), sg(hw_)});
        eig_sym(gram(y, hy), static_cast<int>(y.width), evals, evecs);
      }
      m = static_cast<int>(y.width);
      const int kp_used = m - kt - kw;
      for (int j = 0; j < kt; ++j) theta_[j] = evals[j];
      rep_.norm_estimate =
          std::max({rep_.norm_estimate, std::fabs(evals[0]), std::fabs(evals[m - 1])});
      // [G | G0]: X' = Y G, P' = Y G0 with G0 = G without its X rows.
      Mat gg(static_cast<std::size_t>(m) * 2 * kt, 0.0);
      for (int c2 = 0; c2 < kt; ++c2)
        for (int i = 0; i < m; ++i) {
          const double v = evecs[i + static_cast<std::size_t>(c2) * m];
          gg[i + static_cast<std::size_t>(c2) * m] = v;
          if (i >= kt) gg[i + static_cast<std::size_t>(kt + c2) * m] = v;
        }
      (void)kp_used;
      combine(ctx_, n_, y, gg.data(), 2 * kt, out2(x2_.p, kt, p2_.p, kt), false);
      combine(ctx_, n_, hy, gg.data(), 2 * kt, out2(hx2_.p, kt, hp2_.p, kt), false);
      x2_.w = hx2_.w = p2_.w = hp2_.w = kt;
      std::swap(x_, x2_);
      std::swap(hx_, hx2_);
      std::swap(p_, p2_);
      std::swap(hp_, hp2_);
    }
    {
      Clock c(ctx_, &rep_.timing_ms[kOrtho]);
      // X guard (lobpcg.cpp:363-375): X^T X and clean_p's first X^T P from
      // one read of X and P
      Mat g_xp = gram(view({sg(x_), sg(p_)}), view({sg(x_), sg(p_)}));
      const int k2 = static_cast<int>(x_.w + p_.w);
      Mat xg(static_cast<std::size_t>(kt) * kt), xp(static_cast<std::size_t>(kt) * p_.w);
      for (int a = 0; a < kt; ++a) {
        for (int b = 0; b < kt; ++b) xg[a + static_cast<std::size_t>(b) * kt] = g_xp[a + static_cast<std::size_t>(b) * k2];
        for (std::uint32_t b = 0; b < p_.w; ++b)
          xp[a + static_cast<std::size_t>(b) * kt] = g_xp[a + static_cast<std::size_t>(kt + b) * k2];
      }
      bool rescaled = false;
      if (dev_from_identity(xg, kt) > 1e-12) {
        Mat rinv;
        if (llt_rinv(xg, kt, rinv)) {
          combine(ctx_, n_, view({sg(x_)}), rinv.data(), kt, out1(x_.p, kt), false);
          combine(ctx_, n_, view({sg(hx_)}), rinv.data(), kt, out1(hx_.p, kt), false);
          ++rep_.counters[3];
          rescaled = true;
        }
      }
      clean_p_block(drop_tol, rescaled ? Mat{} : xp);
    }
    ++rep_.counters[3];
  }

  rep_.k_want = static_cast<std::uint32_t>(opt_.k_want);
  rep_.kt = static_cast<std::uint32_t>(kt);
  rep_.n = n_;
  rep_.eigenvalues.assign(theta_.begin(), theta_.begin() + opt_.k_want);
  rep_.trial.resize(static_cast<std::size_t>(n_) * kt);
  CIEG_CUDA(cudaMemcpyAsync(rep_.trial.data(), x_.p, sizeof(double) * rep_.trial.size(), cudaMemcpyDeviceToHost,
                            ctx_->stream));
  int singular = 0;
  if (singular_) CIEG_CUDA(cudaMemcpyAsync(&singular, singular_, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx_->stream));
  for (int i = 0; i < singular; ++i)  // (the reference reports each one as it happens)
    std::fprintf(stderr, "ci-eigen: singular shifted tile block; passing residual through\n");
  clock_flush(ctx_);
  rep_.timing_ms[kTotal] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace
}  // namespace cieg

extern "C" {

void cieg_lobpcg_options_default(cieg_lobpcg_options* o) {
  if (!o) return;
  o->k_want = 8;
  o->tol = 1e-6;
  o->max_iter = 500;
  cieg_precond_config_default(&o->precond_config);
}

int cieg_lobpcg_solve(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                      const cieg_prec* prec, const cieg_lobpcg_options* opt, cieg_observer_fn observer,
                      void* observer_user, cieg_report** out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !x0_host || !opt || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_lobpcg_solve: null argument");
    if (prec && prec->dim != mat->row_hi - mat->row_lo)
      cieg::fail(CIEG_ERR_DIMENSION, "apply_preconditioner: tiles do not cover the basis");
    if (mat->row_lo != 0 || mat->row_hi != mat->dim)
      cieg::fail(CIEG_ERR_CONFIG, "cieg_lobpcg_solve needs the whole matrix; use cieg_lobpcg_solve_dist for a shard");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    auto rep = std::make_unique<cieg_report>();
    {
      cieg::Solver s(ctx, mat, prec, *opt, *rep);
      s.run(x0_host, kt, observer, observer_user);
    }
    *out = rep.release();
  });
}

int cieg_lobpcg_solve_dist(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                           const cieg_prec* prec, const cieg_lobpcg_options* opt, const cieg_dist_hooks* hooks,
                           cieg_report** out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !x0_host || !opt || !hooks || !out || !hooks->allreduce_sum || !hooks->allgather_rows)
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_lobpcg_solve_dist: null argument");
    if (prec && prec->dim != mat->row_hi - mat->row_lo)
      cieg::fail(CIEG_ERR_DIMENSION, "apply_preconditioner: tiles do not cover the basis");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    auto rep = std::make_unique<cieg_report>();
    {
      cieg::Solver s(ctx, mat, prec, *opt, *rep, hooks);
      s.run(x0_host, kt, nullptr, nullptr);
    }
    *out = rep.release();
  });
}

int cieg_lobpcg_solve_nccl(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                           const cieg_prec* prec, const cieg_lobpcg_options* opt, cieg_report** out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !x0_host || !opt || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_lobpcg_solve_nccl: null argument");
    if (!ctx->nccl) cieg::fail(CIEG_ERR_CONFIG, "cieg_lobpcg_solve_nccl: no NCCL communicator (cieg_ctx_nccl_init)");
    if (prec && prec->dim != mat->row_hi - mat->row_lo)
      cieg::fail(CIEG_ERR_DIMENSION, "apply_preconditioner: tiles do not cover the basis");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    auto rep = std::make_unique<cieg_report>();
    cieg::NcclSolve* ns = cieg::nccl_solve_begin(ctx, mat);
    cieg_dist_hooks hooks{ns, cieg::nccl_hook_allreduce, cieg::nccl_hook_gather, cieg::nccl_hook_reduce_partials};
    try {
      cieg::Solver s(ctx, mat, prec, *opt, *rep, &hooks);
      s.run(x0_host, kt, nullptr, nullptr);
    } catch (...) {
      cieg::nccl_solve_end(ns);
      throw;
    }
    cieg::nccl_solve_end(ns);
    *out = rep.release();
  });
}

int cieg_report_destroy(cieg_report* r) {
  delete r;
  return CIEG_OK;
}

int cieg_report_summary(const cieg_report* r, int* converged, int* iterations, double* norm_estimate,
                        uint32_t* k_want, uint32_t* kt, uint64_t* history_rows) {
  return cieg::guarded([&] {
    if (!r) cieg::fail(CIEG_ERR_ARGUMENT, "null report");
    if (converged) *converged = r->converged ? 1 : 0;
    if (iterations) *iterations = r->iterations;
    if (norm_estimate) *norm_estimate = r->norm_estimate;
    if (k_want) *k_want = r->k_want;
    if (kt) *kt = r->kt;
    if (history_rows) *history_rows = r->history.size();
  });
}

int cieg_report_counters(const cieg_report* r, uint64_t* c4) {
  return cieg::guarded([&] {
    if (!r || !c4) cieg::fail(CIEG_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 4; ++i) c4[i] = r->counters[i];
  });
}

int cieg_report_eigenvalues(const cieg_report* r, double* out) {
  return cieg::guarded([&] {
    if (!r || !out) cieg::fail(CIEG_ERR_ARGUMENT, "null argument");
    std::copy(r->eigenvalues.begin(), r->eigenvalues.end(), out);
  });
}

int cieg_report_trial_vectors(const cieg_report* r, double* out) {
  return cieg::guarded([&] {
    if (!r || !out) cieg::fail(CIEG_ERR_ARGUMENT, "null argument");
    std::copy(r->trial.begin(), r->trial.end(), out);
  });
}

int cieg_report_history(const cieg_report* r, int* it, int* col, double* relres, double* theta) {
  return cieg::guarded([&] {
    if (!r) cieg::fail(CIEG_ERR_ARGUMENT, "null report");
    for (std::size_t i = 0; i < r->history.size(); ++i) {
      if (it) it[i] = r->history[i].iteration;
      if (col) col[i] = r->history[i].column;
      if (relres) relres[i] = r->history[i].relres;
      if (theta) theta[i] = r->history[i].theta;
    }
  });
}

int cieg_report_timing(const cieg_report* r, double* ms7) {
  return cieg::guarded([&] {
    if (!r || !ms7) cieg::fail(CIEG_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 7; ++i) ms7[i] = r->timing_ms[i];
  });
}

/* ---- lobpcg.hpp public helpers ---------------------------------------- */

int cieg_orthonormalize(cieg_ctx* ctx, double* y_dev, uint32_t n, uint32_t k, double drop_tol,
                        const double* against_dev, uint32_t ka, uint32_t* k_out) {
  return cieg::guarded([&] {
    if (!ctx || !y_dev || !k_out || (ka && !against_dev))
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_orthonormalize: null argument");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    cieg::DevBuf scratch;
    cieg::Block v{y_dev, k, k};
    cieg::Block tmp{static_cast<double*>(scratch.get(sizeof(double) * std::max<std::size_t>(1, std::size_t(n) * k))),
                    0, k};
    const cieg::View3 ag = cieg::view({cieg::seg(against_dev, ka)});
    cieg::orthonormalize_dev(cieg::GramOps{ctx, n, nullptr}, v, tmp, drop_tol, ka ? &ag : nullptr);
    if (v.w && v.p != y_dev)
      CIEG_CUDA(cudaMemcpyAsync(y_dev, v.p, sizeof(double) * std::size_t(n) * v.w, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    *k_out = v.w;
  });
}

int cieg_rayleigh_ritz(cieg_ctx* ctx, const double* y_dev, const double* hy_dev, uint32_t n, uint32_t m,
                       uint32_t k_trial, double* theta_out, double* g_out) {
  return cieg::guarded([&] {
    if (!ctx || !y_dev || !hy_dev || !theta_out || !g_out)
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_rayleigh_ritz: null argument");
    if (k_trial > m) cieg::fail(CIEG_ERR_DIMENSION, "rayleigh_ritz: k_trial exceeds basis width");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const cieg::View3 y = cieg::view({cieg::seg(y_dev, m)}), hy = cieg::view({cieg::seg(hy_dev, m)});
    const int mm = static_cast<int>(m);
    cieg::Mat overlap = cieg::gram(ctx, n, y, y);
    const double dev = cieg::dev_from_identity(overlap, mm);
    if (dev > 1e-6)
      cieg::fail(CIEG_ERR_INDEFINITE, "basis overlap deviates from identity by " + std::to_string(dev));
    std::vector<double> evals;
    cieg::Mat evecs;
    cieg::eig_sym(cieg::gram(ctx, n, y, hy), mm, evals, evecs);
    for (uint32_t j = 0; j < k_trial; ++j) theta_out[j] = evals[j];
    std::copy(evecs.begin(), evecs.begin() + static_cast<std::size_t>(m) * k_trial, g_out);
  });
}

int cieg_residual_norms(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, uint32_t k, const double* theta,
                        double norm_est, double* out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !x_dev || !theta || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_residual_norms: null argument");
    if (mat->row_lo != 0 || mat->row_hi != mat->dim)
      cieg::fail(CIEG_ERR_CONFIG, "cieg_residual_norms needs the whole matrix (not a shard)");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const std::uint32_t n = mat->dim;
    cieg::DevBuf hx, r;
    auto* hxp = static_cast<double*>(hx.get(sizeof(double) * std::max<std::size_t>(1, std::size_t(n) * k)));
    auto* rp = static_cast<double*>(r.get(sizeof(double) * std::max<std::size_t>(1, std::size_t(n) * k)));
    // residual_norms (lobpcg.cpp:147-169): R = H X - X diag(theta), relative to est * |x_j|
    cieg::launch_spmm(ctx, mat, x_dev, k, hxp, k, k);
    cieg::residual(ctx, n, k, hxp, x_dev, theta, rp);
    const cieg::View3 rv = cieg::view({cieg::seg(rp, k)}), xv = cieg::view({cieg::seg(x_dev, k)});
    const cieg::Mat gr = cieg::gram(ctx, n, rv, rv), gx = cieg::gram(ctx, n, xv, xv);
    double est = norm_est;
    if (!(est > 0.0))
      for (uint32_t j = 0; j < k; ++j) est = std::max(est, std::fabs(theta[j]));
    for (uint32_t j = 0; j < k; ++j) {
      const double rn = std::sqrt(gr[j + static_cast<std::size_t>(k) * j]);
      const double xn = std::sqrt(gx[j + static_cast<std::size_t>(k) * j]);
      out[j] = rn / std::max(est * xn, cieg::kTinyDiag);
    }
  });
}

}  // extern "C"
