// report.hpp -- the solve report behind cieg_report (ci::SolveReport,
// proj/include/ci/lobpcg.hpp:27-60) shared by the LOBPCG (solver.cpp) and
// Lanczos (lanczos.cu) drivers, and the wall-clock phase timer.
#pragma once

#include <chrono>
#include <cstdint>
#include <vector>

#include "context.hpp"

struct cieg_report {
  std::vector<double> eigenvalues;
  std::vector<double> trial;  // n x kt row-major
  std::uint32_t n = 0, kt = 0, k_want = 0;
  struct Row {
    int iteration, column;
    double relres, theta;
  };
  std::vector<Row> history;
  std::uint64_t counters[4] = {0, 0, 0, 0};
  bool converged = false;
  int iterations = 0;
  double norm_estimate = 0.0;
  double timing_ms[7] = {0, 0, 0, 0, 0, 0, 0};
};

namespace cieg {

// Phase timer: CUDA events on the context's stream around the phase (device
// time from the phase's first to its last enqueued work, host gaps between
// them included); no host synchronisation -- clock_flush() adds the elapsed
// times to their slots, at the end of a solve.
inline cudaEvent_t clock_event(cieg_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  CIEG_CUDA(cudaEventCreate(&e));
  return e;
}
inline void clock_flush(cieg_ctx* ctx) {
  if (ctx->ev_pending.empty()) return;
  CIEG_CUDA(cudaEventSynchronize(ctx->ev_pending.back().b));
  for (const auto& r : ctx->ev_pending) {
    float ms = 0.0f;
    CIEG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    *r.slot += ms;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->ev_pending.clear();
}
// (a solve that ends by an exception drops its pending timers: their slots
// belong to a report that no longer exists)
inline void clock_discard(cieg_ctx* ctx) {
  for (const auto& r : ctx->ev_pending) {
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->ev_pending.clear();
}
struct Clock {
  cieg_ctx* ctx;
  double* slot;
  cudaEvent_t a;
  Clock(cieg_ctx* c, double* s) : ctx(c), slot(s), a(clock_event(c)) { CIEG_CUDA(cudaEventRecord(a, ctx->stream)); }
  ~Clock() {
    cudaEvent_t b = clock_event(ctx);
    cudaEventRecord(b, ctx->stream);
    ctx->ev_pending.push_back({a, b, slot});
    if (ctx->ev_pending.size() >= 4096) clock_flush(ctx);  // bound the pending list (a rare sync)
  }
};

enum Phase { kSpmm = 0, kRR = 1, kOrtho = 2, kPrecond = 3, kResid = 4, kOther = 5, kTotal = 6 };

}  // namespace cieg
