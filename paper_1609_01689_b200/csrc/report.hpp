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

struct Clock {
  cieg_ctx* ctx;
  double* slot;
  std::chrono::steady_clock::time_point t0;
  Clock(cieg_ctx* c, double* s) : ctx(c), slot(s), t0(std::chrono::steady_clock::now()) {}
  ~Clock() {
    cudaStreamSynchronize(ctx->stream);
    *slot += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

enum Phase { kSpmm = 0, kRR = 1, kOrtho = 2, kPrecond = 3, kResid = 4, kOther = 5, kTotal = 6 };

}  // namespace cieg
