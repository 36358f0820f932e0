// tiling.hpp -- host-side re-tiling of a flattened CsbMatrix into the device
// tile stream used by the SpMM kernels.
//
// Device format:
//   * rows are cut into panels of <= tile_edge rows (panel_start[npanels+1]);
//     panels follow group boundaries, so a device tile (PI, PJ) is the union
//     of whole reference tiles and keeps their density;
//   * one stored tile per nonzero (PI >= PJ) panel pair, entries as a packed
//     32-bit tile-local index plus the value (f32 or f64), tiles back to back
//     with 64-bit offsets, each list padded to a multiple of 4. The index
//     holds the entry's two shared-memory offsets, r*SA+perm(c) (low 16
//     bits) and c*SA+perm(r) (high 16 bits), SA = tile_edge + 8, perm pairing
//     the columns of consecutive k-steps, so the SpMM scatter is a single
//     store in either orientation;
//   * an owner work list per panel P: the tiles whose product lands in P's
//     rows -- (P, J) row parts, (I, P) transposed parts, (P, P) symmetric --
//     so one CTA computes all of Y[P] and writes it exactly once
//     (owner-computes; deterministic, no atomics).
#pragma once

#include <cstdint>
#include <vector>

#include "cieg_internal.hpp"

namespace cieg {

enum WorkKind : std::uint32_t { kRowPart = 0, kTransposed = 1, kDiagonal = 2 };

struct HostTiles {
  std::uint32_t dim = 0;
  std::uint32_t tile_edge = 0;
  int precision = 0;
  std::uint64_t nnz = 0;  // real entries (tile lists are padded to quads)
  std::vector<std::uint32_t> panel_start;      // npanels + 1
  std::vector<std::uint64_t> tile_off;         // ntiles + 1
  std::vector<std::uint32_t> tile_pi, tile_pj; // panel pair of each tile
  std::vector<std::uint32_t> idx;              // packed (r*SA+perm c) | (c*SA+perm r) << 16
  std::vector<float> val32;
  std::vector<double> val64;
  // owner work lists: items [work_off[P], work_off[P+1]) of (tile, other, kind)
  std::vector<std::uint32_t> work_off;
  std::vector<std::uint32_t> work_tile, work_other, work_kind;

  // Static per-CTA schedule for the persistent SpMM kernel (one CTA per SM):
  // CTA b runs sched[sched_off[b] .. sched_off[b+1]) in order.
  std::vector<std::uint32_t> sched_off;
  std::vector<std::uint32_t> sched;  // 8 words per item, see ItemDesc in spmm.cu
  // Single-pass schedule (full matrices only; empty for shards): one item
  // per stored tile, owned by its row panel. An off-diagonal item's
  // transposed product Aᵀ X_pi goes to partial slot = its item index; the
  // slots feeding block column Q are sp_col_items[sp_col_off[Q] .. sp_col_off[Q+1]).
  std::vector<std::uint32_t> sp_sched_off, sp_sched, sp_col_off, sp_col_items;
  // shards: first row of the transposed partials for rows of lower shards
  // (rows [sp_partial_lo, row_lo); = row_lo when there are none)
  std::uint32_t sp_partial_lo = 0;

  // owner rows of this (shard) tiling and the X rows its SpMM reads
  std::uint32_t row_lo = 0, row_hi = 0, halo_lo = 0, halo_hi = 0;

  std::uint32_t npanels() const { return static_cast<std::uint32_t>(panel_start.size() - 1); }
  std::uint64_t ntiles() const { return tile_pi.size(); }
};

// Panel plan from group bounds: groups larger than tile_edge are split into
// tile_edge chunks; consecutive groups are merged while the panel stays
// <= tile_edge and every merged group is smaller than tile_edge / 2 (small
// physics-style groups), otherwise each group is its own panel.
std::vector<std::uint32_t> plan_panels(std::uint32_t dim, const std::uint32_t* group_bounds,
                                       std::uint32_t ngroups, std::uint32_t tile_edge);
// The same plan with extra mandatory panel boundaries (e.g. the truncation
// levels of a multilevel guess, so their leading blocks are panel-aligned).
std::vector<std::uint32_t> plan_panels(std::uint32_t dim, const std::uint32_t* group_bounds,
                                       std::uint32_t ngroups, std::uint32_t tile_edge, const std::uint32_t* cuts,
                                       std::uint32_t ncuts);

void build_tiles(const cieg_csb_view& csb, const std::vector<std::uint32_t>& panels,
                 std::uint32_t tile_edge, HostTiles& out);

// Owner work lists of panels [p_lo, p_hi) from tiles sorted by (pi, pj).
void build_work_lists(HostTiles& t, std::uint32_t p_lo, std::uint32_t p_hi);

// Assign owner panels to `ctas` persistent CTAs (longest-first greedy on the
// entry count, ties by panel id, so the result is deterministic) and emit
// each CTA's item descriptors: {q0 lo/hi, q1 lo/hi, kind | first << 8 |
// last << 9 | owner rows << 16, other-panel start row, other-panel rows,
// owner start row} -- everything the consumer needs without a dependent load.
void build_schedule(HostTiles& t, std::uint32_t ctas);

// Keep only what owner rows [row_lo, row_hi) need (panel-aligned bounds):
// their work lists and the tiles those reference (re-indexed), and record the
// X halo. Other panels keep empty work lists.
void restrict_to_rows(HostTiles& t, std::uint32_t row_lo, std::uint32_t row_hi);

// Row partition over nranks at group boundaries balanced by the entries each
// owner streams (row part + transposed part); panel-expanded X halos.
void shard_plan(const cieg_csb_view& csb, const std::uint32_t* group_bounds, std::uint32_t ngroups,
                std::uint32_t tile_edge, std::uint32_t nranks, std::uint32_t* row_bounds,
                std::uint32_t* halo_lo, std::uint32_t* halo_hi);

}  // namespace cieg
