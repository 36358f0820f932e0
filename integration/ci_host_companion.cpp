// ci_host_companion.cpp -- the non-hot ci:: symbols that live in the
// reference translation units the drop-in replaces
// (proj/src/{csb,block_vectors,lobpcg}.cpp), restated on the host so that a
// build linking ci_gpu_dropin.cpp + this TU in place of
// proj/src/{csb,block_vectors,lobpcg,precond,lanczos}.cpp resolves every
// symbol the remaining reference TUs (basis, grouping, hamiltonian, guess,
// planner, config) and their callers (ci_eigen.cpp) use:
//   BlockVectors::select_columns / hcat / to_matrix / from_matrix
//     (block_vectors.hpp:41-46), assemble / matrix_stats / to_dense /
//     save_csb / load_csb (csb.hpp:75-106), write_history_csv
//     (lobpcg.hpp:102), and a weak extract_tile_diagonal (hamiltonian.hpp:65;
//     the strong one in hamiltonian.cpp wins when that TU is linked).
// Setup and I/O code: none of it is on the solver's hot path.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <ostream>
#include <string>
#include <vector>

#include "ci/block_vectors.hpp"
#include "ci/csb.hpp"
#include "ci/errors.hpp"
#include "ci/grouping.hpp"
#include "ci/hamiltonian.hpp"
#include "ci/lobpcg.hpp"

namespace ci {

// ---------------------------------------------------- block_vectors.hpp:41-46
BlockVectors BlockVectors::select_columns(const std::vector<std::uint32_t>& cols) const {
  const std::uint32_t k = static_cast<std::uint32_t>(cols.size());
  BlockVectors out(dim_, k);
  const double* src = values_.data();
  double* dst = out.values_.data();
  for (std::uint32_t i = 0; i < dim_; ++i, src += width_, dst += k)
    for (std::uint32_t c = 0; c < k; ++c) dst[c] = src[cols[c]];
  return out;
}

BlockVectors BlockVectors::hcat(const BlockVectors& a, const BlockVectors& b) {
  if (b.width_ == 0) return a;
  if (a.width_ == 0) return b;
  if (a.dim_ != b.dim_) throw DimensionMismatch("hcat: row counts differ");
  BlockVectors out(a.dim_, a.width_ + b.width_);
  for (std::uint32_t i = 0; i < a.dim_; ++i) {
    double* dst = out.row(i);
    dst = std::copy_n(a.row(i), a.width_, dst);
    std::copy_n(b.row(i), b.width_, dst);
  }
  return out;
}

Eigen::MatrixXd BlockVectors::to_matrix() const {
  Eigen::MatrixXd m(dim_, width_);
  double* col_major = m.data();
  for (std::uint32_t j = 0; j < width_; ++j)
    for (std::uint32_t i = 0; i < dim_; ++i) col_major[static_cast<std::size_t>(j) * dim_ + i] = at(i, j);
  return m;
}

BlockVectors BlockVectors::from_matrix(const Eigen::MatrixXd& m) {
  const auto rows = static_cast<std::uint32_t>(m.rows()), cols = static_cast<std::uint32_t>(m.cols());
  BlockVectors out(rows, cols);
  const double* col_major = m.data();
  for (std::uint32_t j = 0; j < cols; ++j)
    for (std::uint32_t i = 0; i < rows; ++i) out.at(i, j) = col_major[static_cast<std::size_t>(j) * rows + i];
  return out;
}

// ------------------------------------------------------------ csb.hpp:75-106
namespace {

struct Staged {
  std::uint16_t r, c;
  double v;
};

void store_block(std::vector<Staged>& st, CoordinateBlock& blk, Precision prec) {
  std::sort(st.begin(), st.end(), [](const Staged& a, const Staged& b) { return a.r < b.r || (a.r == b.r && a.c < b.c); });
  blk.rows.resize(st.size());
  blk.cols.resize(st.size());
  if (prec == Precision::Single)
    blk.values32.resize(st.size());
  else
    blk.values64.resize(st.size());
  for (std::size_t e = 0; e < st.size(); ++e) {
    blk.rows[e] = st[e].r;
    blk.cols[e] = st[e].c;
    if (prec == Precision::Single)
      blk.values32[e] = static_cast<float>(st[e].v);
    else
      blk.values64[e] = st[e].v;
  }
}

}  // namespace

// Evaluate the element function on every lower-triangle pair inside the
// nonzero tiles, one block row per OpenMP task; entries (row, col)-sorted
// per block. The optional audit scans the zero tiles for stray nonzeros.
CsbMatrix assemble(const TileMap& tiles, const CsbLayout& layout, const GroupPartition& partition,
                   const ElementFn& element, const AssembleOptions& options) {
  CsbMatrix h;
  h.layout = layout;
  h.precision = options.precision;
  h.dim = partition.dimension();
  h.groups = partition.group_count();
  h.nonzero_tiles = tiles.nonzero_tile_count();
  const std::uint32_t nb = layout.block_count();
  h.blocks.resize(static_cast<std::size_t>(nb) * (nb + 1) / 2);
  std::vector<std::vector<std::uint32_t>> row_groups(nb);
  for (std::uint32_t g = 0; g < partition.group_count(); ++g)
    row_groups[layout.block_of_state(partition.group_ranges[g].first)].push_back(g);
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t bi = 0; bi < static_cast<std::int64_t>(nb); ++bi) {
    const auto BI = static_cast<std::uint32_t>(bi);
    std::vector<std::vector<Staged>> staged(BI + 1);
    const std::uint32_t r0 = layout.block_boundaries[BI];
    for (std::uint32_t g : row_groups[BI]) {
      const auto [rs, re] = partition.group_ranges[g];
      for (std::uint32_t gc : tiles.cols_of_row[g]) {
        const auto [cs, ce] = partition.group_ranges[gc];
        const std::uint32_t BJ = layout.block_of_state(cs);
        const std::uint32_t c0 = layout.block_boundaries[BJ];
        for (std::uint32_t a = rs; a < re; ++a)
          for (std::uint32_t b = cs; b < std::min(ce, a + 1); ++b) {
            const double v = element(a, b);
            if (v != 0.0)
              staged[BJ].push_back({static_cast<std::uint16_t>(a - r0), static_cast<std::uint16_t>(b - c0), v});
          }
      }
    }
    for (std::uint32_t BJ = 0; BJ <= BI; ++BJ)
      if (!staged[BJ].empty()) store_block(staged[BJ], h.block(BI, BJ), options.precision);
  }
  h.nnz_lower = 0;
  for (const CoordinateBlock& b : h.blocks) h.nnz_lower += b.size();
  const bool audit = options.verify == AssembleOptions::Verify::On ||
                     (options.verify == AssembleOptions::Verify::Auto && h.dim <= 2000);
  if (audit) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
    for (std::int64_t g64 = 0; g64 < static_cast<std::int64_t>(partition.group_count()); ++g64) {
      const auto g = static_cast<std::uint32_t>(g64);
      const auto [rs, re] = partition.group_ranges[g];
      for (std::uint32_t gc = 0; gc <= g && !bad; ++gc) {
        if (tiles.is_nonzero(g, gc)) continue;
        const auto [cs, ce] = partition.group_ranges[gc];
        for (std::uint32_t a = rs; a < re && !bad; ++a)
          for (std::uint32_t b = cs; b < std::min(ce, a + 1) && !bad; ++b) bad |= element(a, b) != 0.0;
      }
    }
    if (bad)
      throw StructureViolation("provider yields a nonzero outside the nonzero tiles; body rank d is inconsistent");
  }
  return h;
}

MatrixStats matrix_stats(const CsbMatrix& h) {
  MatrixStats s;
  s.dim = h.dim;
  s.nnz_lower = h.nnz_lower;
  s.element_pairs = static_cast<std::uint64_t>(h.dim) * (h.dim + 1) / 2;
  s.element_sparsity = static_cast<double>(s.nnz_lower) / static_cast<double>(s.element_pairs);
  s.csb_blocks = h.block_count();
  s.groups = h.groups;
  s.nonzero_tiles = h.nonzero_tiles;
  s.tile_pairs_offdiag = h.groups * (h.groups - 1) / 2;
  s.tile_sparsity =
      s.tile_pairs_offdiag ? static_cast<double>(s.nonzero_tiles) / static_cast<double>(s.tile_pairs_offdiag) : 0.0;
  return s;
}

Eigen::MatrixXd to_dense(const CsbMatrix& h) {
  if (h.dim > 5000) throw DimensionMismatch("to_dense is a test oracle; dim > 5000");
  Eigen::MatrixXd d = Eigen::MatrixXd::Zero(h.dim, h.dim);
  const auto& bb = h.layout.block_boundaries;
  for (std::uint32_t bi = 0, id = 0; bi < h.block_count(); ++bi)
    for (std::uint32_t bj = 0; bj <= bi; ++bj, ++id) {
      const CoordinateBlock& b = h.blocks[id];
      for (std::size_t e = 0; e < b.size(); ++e) {
        const std::uint32_t r = bb[bi] + b.rows[e], c = bb[bj] + b.cols[e];
        d(r, c) = d(c, r) = h.value(id, e);
      }
    }
  return d;
}

namespace {

template <typename T>
void put(std::ostream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof v);
}
template <typename T>
T get(std::istream& is) {
  T v{};
  if (!is.read(reinterpret_cast<char*>(&v), sizeof v)) throw FormatError("truncated CSB file");
  return v;
}

}  // namespace

// CSB1: magic, u32 precision, u64 dim, u32 beta, u32 blocks, u64 nnz, u64
// groups, u64 nonzero tiles, u32 boundaries[blocks + 1], then per block (row
// major, lower triangle) u64 count and (u16 row, u16 col, value) records.
void save_csb(const CsbMatrix& h, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw FormatError("cannot open for writing: " + path);
  os.write("CSB1", 4);
  const bool single = h.precision == Precision::Single;
  put<std::uint32_t>(os, single ? 0u : 1u);
  put<std::uint64_t>(os, h.dim);
  put<std::uint32_t>(os, h.layout.beta);
  put<std::uint32_t>(os, h.block_count());
  put<std::uint64_t>(os, h.nnz_lower);
  put<std::uint64_t>(os, h.groups);
  put<std::uint64_t>(os, h.nonzero_tiles);
  for (std::uint32_t b : h.layout.block_boundaries) put<std::uint32_t>(os, b);
  std::vector<char> rec;
  for (const CoordinateBlock& b : h.blocks) {
    put<std::uint64_t>(os, b.size());
    const std::size_t w = 4 + (single ? 4 : 8);
    rec.resize(w * b.size());
    char* p = rec.data();
    for (std::size_t e = 0; e < b.size(); ++e, p += w) {
      std::memcpy(p, &b.rows[e], 2);
      std::memcpy(p + 2, &b.cols[e], 2);
      if (single)
        std::memcpy(p + 4, &b.values32[e], 4);
      else
        std::memcpy(p + 4, &b.values64[e], 8);
    }
    os.write(rec.data(), static_cast<std::streamsize>(rec.size()));
  }
  if (!os) throw FormatError("write failed: " + path);
}

CsbMatrix load_csb(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw FormatError("cannot open: " + path);
  char magic[4] = {};
  if (!is.read(magic, 4) || std::memcmp(magic, "CSB1", 4) != 0) throw FormatError("bad magic; not a CSB1 file: " + path);
  CsbMatrix h;
  const auto prec = get<std::uint32_t>(is);
  if (prec > 1) throw FormatError("bad precision tag");
  h.precision = prec == 0 ? Precision::Single : Precision::Double;
  h.dim = static_cast<std::uint32_t>(get<std::uint64_t>(is));
  h.layout.beta = get<std::uint32_t>(is);
  const auto nb = get<std::uint32_t>(is);
  const auto nnz = get<std::uint64_t>(is);
  h.groups = get<std::uint64_t>(is);
  h.nonzero_tiles = get<std::uint64_t>(is);
  h.layout.block_boundaries.resize(static_cast<std::size_t>(nb) + 1);
  for (auto& b : h.layout.block_boundaries) b = get<std::uint32_t>(is);
  if (h.layout.block_boundaries.front() != 0 || h.layout.block_boundaries.back() != h.dim)
    throw FormatError("inconsistent block boundaries");
  h.blocks.resize(static_cast<std::size_t>(nb) * (nb + 1) / 2);
  const std::size_t w = 4 + (prec == 0 ? 4 : 8);
  std::vector<char> rec;
  for (CoordinateBlock& b : h.blocks) {
    const auto n = get<std::uint64_t>(is);
    rec.resize(w * n);
    if (n && !is.read(rec.data(), static_cast<std::streamsize>(rec.size()))) throw FormatError("truncated CSB file");
    b.rows.resize(n);
    b.cols.resize(n);
    if (prec == 0)
      b.values32.resize(n);
    else
      b.values64.resize(n);
    const char* p = rec.data();
    for (std::uint64_t e = 0; e < n; ++e, p += w) {
      std::memcpy(&b.rows[e], p, 2);
      std::memcpy(&b.cols[e], p + 2, 2);
      if (prec == 0)
        std::memcpy(&b.values32[e], p + 4, 4);
      else
        std::memcpy(&b.values64[e], p + 4, 8);
    }
    h.nnz_lower += n;
  }
  if (h.nnz_lower != nnz) throw FormatError("entry count disagrees with header");
  return h;
}

// ----------------------------------------------------------- lobpcg.hpp:102
void write_history_csv(const SolveReport& report, std::ostream& os) {
  os << "iter,col,relres,theta\n";
  for (const HistoryRow& r : report.history) {
    char line[96];
    std::snprintf(line, sizeof line, "%d,%d,%.17g,%.17g\n", r.iteration, r.column, r.relres, r.theta);
    os << line;
  }
}

// ------------------------------------------------------- hamiltonian.hpp:65
// Weak: proj/src/hamiltonian.cpp's definition takes precedence when linked.
__attribute__((weak)) TileDiagonal extract_tile_diagonal(const CsbMatrix& h, const GroupPartition& partition) {
  TileDiagonal t;
  t.ranges = partition.group_ranges;
  for (const auto& [s, e] : partition.group_ranges) t.blocks.push_back(Eigen::MatrixXd::Zero(e - s, e - s));
  const auto& bb = h.layout.block_boundaries;
  for (std::uint32_t bi = 0; bi < h.block_count(); ++bi) {
    const std::uint32_t id = bi * (bi + 1) / 2 + bi;
    const CoordinateBlock& b = h.blocks[id];
    for (std::size_t e = 0; e < b.size(); ++e) {
      const std::uint32_t r = bb[bi] + b.rows[e], c = bb[bi] + b.cols[e];
      const std::uint32_t g = partition.group_of_state[r];
      if (partition.group_of_state[c] != g) continue;
      const std::uint32_t s = partition.group_ranges[g].first;
      t.blocks[g](r - s, c - s) = t.blocks[g](c - s, r - s) = h.value(id, e);
    }
  }
  return t;
}

}  // namespace ci
