// generator.hpp -- shared pieces of the synthetic sector generator (host CSB
// in generator.cpp, device tile stream in gpugen.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "cieg_internal.hpp"

namespace cieg {

struct TileGrid {
  std::vector<std::uint32_t> start;         // tile t covers [start[t], start[t+1])
  std::vector<std::uint32_t> sector;        // sector of tile t
  std::vector<std::uint32_t> sector_start;  // sectors + 1
  std::uint32_t count() const { return static_cast<std::uint32_t>(sector.size()); }
};

TileGrid make_grid(const cieg_gen_params& p);
void validate(const cieg_gen_params& p);
double expected_nnz(const cieg_gen_params& p);
double avg_row_nnz(const cieg_gen_params& p);
std::uint64_t count_nnz(const cieg_gen_params& p);  // stored entries, counted without storage
double value_scale(const cieg_gen_params& p);  // 1 / sqrt(avg full-row off-diagonal count)
// kept column tiles J <= I of every tile row I (ascending; the diagonal last)
std::vector<std::vector<std::uint32_t>> kept_tiles(const cieg_gen_params& p, const TileGrid& g);

}  // namespace cieg
