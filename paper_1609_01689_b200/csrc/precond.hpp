// precond.hpp -- K5: the tile-diagonal preconditioner (ci::apply_preconditioner).
#pragma once

#include <cstdint>
#include <vector>

#include "context.hpp"

struct cieg_prec {
  cieg_ctx* ctx = nullptr;
  std::uint32_t dim = 0;
  std::uint32_t ngroups = 0;
  std::vector<std::uint32_t> bounds_host;
  std::vector<std::uint64_t> block_off_host;  // offsets (doubles) of each dense block
  std::uint32_t* bounds = nullptr;            // device
  std::uint64_t* block_off = nullptr;         // device
  double* blocks = nullptr;                   // device, column-major per group (fp64) ...
  float* blocks32 = nullptr;                  // ... or fp32 (blocks of an fp32 H; exact)
  std::uint32_t max_group = 0;
  ~cieg_prec();
};

namespace cieg {

struct ShiftPlan {
  std::vector<double> mu;
  std::vector<int> engage;
};

// ci::choose_shifts (proj/src/precond.cpp:13-55).
ShiftPlan choose_shifts(const std::vector<double>& theta, const std::vector<double>& res_norm,
                        const std::vector<double>& x_norm, const std::vector<double>& relres,
                        int iteration, double tol, const cieg_precond_config& cfg);

// W = apply_preconditioner(tiles, R, plan) on device (R, W row-major n x k,
// contiguous). Returns the number of singular-shift pass-throughs.
int precond_apply(cieg_ctx* ctx, const cieg_prec* prec, const double* r, std::uint32_t k,
                  const ShiftPlan& plan, const cieg_precond_config& cfg, double* w);

}  // namespace cieg
