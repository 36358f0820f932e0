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
  // group lists by size class for one small-block cutoff, kept on the device
  // (the partition is fixed per preconditioner and cutoff)
  mutable int lists_cutoff = -1;
  mutable std::vector<std::uint32_t> small_host, large_host;
  mutable std::uint32_t* lists = nullptr;  // small groups then large groups, + an int counter slot
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
// contiguous). Returns the number of singular-shift pass-throughs, reported on
// stderr like the reference -- unless singular_accum (a device counter) is
// given: then the count is added there with no host synchronisation (the
// caller reports it) and 0 is returned.
int precond_apply(cieg_ctx* ctx, const cieg_prec* prec, const double* r, std::uint32_t k,
                  const ShiftPlan& plan, const cieg_precond_config& cfg, double* w, int* singular_accum = nullptr);

}  // namespace cieg
