// tiling.cpp -- see tiling.hpp.
#include "tiling.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>

namespace cieg {

std::vector<std::uint32_t> plan_panels(std::uint32_t dim, const std::uint32_t* gb,
                                       std::uint32_t ng, std::uint32_t te) {
  std::vector<std::uint32_t> p{0};
  if (!gb || ng == 0) {
    for (std::uint32_t r = te; r < dim; r += te) p.push_back(r);
    p.push_back(dim);
    return p;
  }
  if (gb[0] != 0 || gb[ng] != dim) fail(CIEG_ERR_DIMENSION, "group bounds do not cover [0, dim)");
  for (std::uint32_t g = 0; g < ng; ++g) {
    const std::uint32_t s = gb[g], e = gb[g + 1];
    if (e < s) fail(CIEG_ERR_FORMAT, "group bounds are not ascending");
    const std::uint32_t sz = e - s;
    if (sz == 0) continue;
    const bool small = sz < te / 2;
    const std::uint32_t cur = s - p.back();
    if (small && cur > 0 && cur + sz <= te) continue;  // merge into open panel
    if (s != p.back()) p.push_back(s);
    for (std::uint32_t r = s + te; r < e; r += te) p.push_back(r);
    if (!small) {
      if (e != p.back()) p.push_back(e);
    }
  }
  if (p.back() != dim) p.push_back(dim);
  return p;
}

void build_tiles(const cieg_csb_view& csb, const std::vector<std::uint32_t>& panels,
                 std::uint32_t te, HostTiles& out) {
  const std::uint32_t dim = csb.dim;
  const std::uint32_t nb = csb.nb;
  const std::uint32_t np = static_cast<std::uint32_t>(panels.size() - 1);
  if (csb.block_boundaries[0] != 0 || csb.block_boundaries[nb] != dim)
    fail(CIEG_ERR_FORMAT, "inconsistent block boundaries");
  for (std::uint32_t p = 0; p < np; ++p)
    if (panels[p + 1] <= panels[p] || panels[p + 1] - panels[p] > te)
      fail(CIEG_ERR_CONFIG, "panel plan violates the tile edge");

  const std::uint32_t sa = te + 8;
  const std::uint32_t sentinel = te | (te << 16);  // row 0, pad column te: never read
  // Within every 8 columns, k-step j's column 4j' + q and k-step j'+1's
  // column 4j' + 4 + q are stored side by side, so one 64-bit (fp32) or
  // 128-bit (fp64) shared load yields the A fragments of two k-steps.
  auto kperm = [](std::uint32_t k) { return (k & ~7u) | ((k & 3u) << 1) | ((k >> 2) & 1u); };
  std::vector<std::uint32_t> panel_of(dim);
  for (std::uint32_t p = 0; p < np; ++p)
    for (std::uint32_t r = panels[p]; r < panels[p + 1]; ++r) panel_of[r] = p;

  // Per panel row: entries bucketed by column panel.
  struct Bucket {
    std::uint32_t pj;
    std::vector<std::uint32_t> idx;
    std::vector<double> v;
  };
  std::vector<std::vector<Bucket>> rowtiles(np);
  const bool single = csb.precision == 0;
  const float* v32 = static_cast<const float*>(csb.values);
  const double* v64 = static_cast<const double*>(csb.values);

  // Block rows overlapping each panel.
#pragma omp parallel for schedule(dynamic, 4)
  for (std::int64_t p64 = 0; p64 < static_cast<std::int64_t>(np); ++p64) {
    const std::uint32_t P = static_cast<std::uint32_t>(p64);
    const std::uint32_t r0 = panels[P], r1 = panels[P + 1];
    std::vector<Bucket>& bk = rowtiles[P];
    std::vector<std::int64_t> slot;  // pj -> bucket index (sparse, via search)
    std::uint32_t bi = static_cast<std::uint32_t>(
        std::upper_bound(csb.block_boundaries, csb.block_boundaries + nb + 1, r0) -
        csb.block_boundaries) - 1;
    for (; bi < nb && csb.block_boundaries[bi] < r1; ++bi) {
      const std::uint32_t rb = csb.block_boundaries[bi];
      const std::uint64_t base = static_cast<std::uint64_t>(bi) * (bi + 1) / 2;
      for (std::uint32_t bj = 0; bj <= bi; ++bj) {
        const std::uint64_t e0 = csb.entry_offsets[base + bj], e1 = csb.entry_offsets[base + bj + 1];
        if (e0 == e1) continue;
        const std::uint32_t cb = csb.block_boundaries[bj];
        // entries sorted by row: restrict to rows [r0, r1)
        const std::uint16_t* rows = csb.rows;
        std::uint64_t lo = e0, hi = e1;
        if (r0 > rb) {
          const std::uint16_t key = static_cast<std::uint16_t>(r0 - rb);
          lo = static_cast<std::uint64_t>(std::lower_bound(rows + e0, rows + e1, key) - rows);
        }
        if (r1 < csb.block_boundaries[bi + 1]) {
          const std::uint16_t key = static_cast<std::uint16_t>(r1 - rb);
          hi = static_cast<std::uint64_t>(std::lower_bound(rows + lo, rows + e1, key) - rows);
        }
        for (std::uint64_t e = lo; e < hi; ++e) {
          const std::uint32_t a = rb + rows[e];
          const std::uint32_t b = cb + csb.cols[e];
          if (b > a) fail(CIEG_ERR_FORMAT, "entry above the diagonal in lower-triangle storage");
          const std::uint32_t pj = panel_of[b];
          Bucket* tb = nullptr;
          if (!bk.empty() && bk.back().pj == pj) {
            tb = &bk.back();
          } else {
            for (auto it = bk.rbegin(); it != bk.rend(); ++it)
              if (it->pj == pj) {
                tb = &*it;
                break;
              }
            if (!tb) {
              bk.push_back(Bucket{pj, {}, {}});
              tb = &bk.back();
            }
          }
          const std::uint32_t rl = a - r0, cl = b - panels[pj];
          // Packed tile-local index: the entry's shared-memory offset in the
          // row-part orientation (r * SA + perm(c)) and in the transposed one
          // (c * SA + perm(r)), SA = tile_edge + 8 (the kernels' padded row
          // stride, 8 mod 32 banks).
          tb->idx.push_back((rl * sa + kperm(cl)) | ((cl * sa + kperm(rl)) << 16));
          tb->v.push_back(single ? static_cast<double>(v32[e]) : v64[e]);
        }
      }
    }
    std::sort(bk.begin(), bk.end(), [](const Bucket& x, const Bucket& y) { return x.pj < y.pj; });
  }

  out = HostTiles{};
  out.dim = dim;
  out.tile_edge = te;
  out.precision = csb.precision;
  out.panel_start = panels;
  std::vector<std::uint64_t> tiles_before(np + 1, 0);
  for (std::uint32_t P = 0; P < np; ++P) tiles_before[P + 1] = tiles_before[P] + rowtiles[P].size();
  const std::uint64_t nt = tiles_before[np];
  out.tile_pi.resize(nt);
  out.tile_pj.resize(nt);
  out.tile_off.assign(nt + 1, 0);
  for (std::uint32_t P = 0; P < np; ++P)
    for (std::size_t k = 0; k < rowtiles[P].size(); ++k) {
      const std::uint64_t t = tiles_before[P] + k;
      out.tile_pi[t] = P;
      out.tile_pj[t] = rowtiles[P][k].pj;
      out.tile_off[t + 1] = rowtiles[P][k].idx.size();
    }
  // Each tile's entry list is padded to a multiple of 4 with sentinel entries
  // (value 0, offset = pad column te of row 0, which the consumers never
  // read) so the kernels stream it with 128-bit copies and scatter without
  // branches.
  out.nnz = 0;
  for (std::uint64_t t = 0; t < nt; ++t) {
    out.nnz += out.tile_off[t + 1];
    out.tile_off[t + 1] = (out.tile_off[t + 1] + 3) & ~std::uint64_t{3};
  }
  for (std::uint64_t t = 0; t < nt; ++t) out.tile_off[t + 1] += out.tile_off[t];
  const std::uint64_t slots = out.tile_off[nt];
  out.idx.assign(slots, sentinel);
  if (single)
    out.val32.assign(slots, 0.0f);
  else
    out.val64.assign(slots, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
  for (std::int64_t p64 = 0; p64 < static_cast<std::int64_t>(np); ++p64) {
    const std::uint32_t P = static_cast<std::uint32_t>(p64);
    for (std::size_t k = 0; k < rowtiles[P].size(); ++k) {
      Bucket& b = rowtiles[P][k];
      const std::uint64_t o = out.tile_off[tiles_before[P] + k];
      std::memcpy(out.idx.data() + o, b.idx.data(), b.idx.size() * sizeof(std::uint32_t));
      if (single)
        for (std::size_t e = 0; e < b.v.size(); ++e) out.val32[o + e] = static_cast<float>(b.v[e]);
      else
        std::memcpy(out.val64.data() + o, b.v.data(), b.v.size() * sizeof(double));
      std::vector<std::uint32_t>().swap(b.idx);
      std::vector<double>().swap(b.v);
    }
  }

  // Owner work lists: row parts and the diagonal tile of P (ascending J),
  // then transposed parts of tiles (I, P), I > P (ascending I).
  std::vector<std::vector<std::uint64_t>> trans(np);
  for (std::uint64_t t = 0; t < nt; ++t)
    if (out.tile_pi[t] != out.tile_pj[t]) trans[out.tile_pj[t]].push_back(t);
  out.work_off.assign(np + 1, 0);
  for (std::uint32_t P = 0; P < np; ++P)
    out.work_off[P + 1] = out.work_off[P] + static_cast<std::uint32_t>(rowtiles[P].size() + trans[P].size());
  const std::uint32_t nw = out.work_off[np];
  out.work_tile.resize(nw);
  out.work_other.resize(nw);
  out.work_kind.resize(nw);
  for (std::uint32_t P = 0; P < np; ++P) {
    std::uint32_t w = out.work_off[P];
    for (std::uint64_t t = tiles_before[P]; t < tiles_before[P + 1]; ++t, ++w) {
      out.work_tile[w] = static_cast<std::uint32_t>(t);
      out.work_other[w] = out.tile_pj[t];
      out.work_kind[w] = out.tile_pj[t] == P ? kDiagonal : kRowPart;
    }
    for (std::uint64_t t : trans[P]) {
      out.work_tile[w] = static_cast<std::uint32_t>(t);
      out.work_other[w] = out.tile_pi[t];
      out.work_kind[w] = kTransposed;
      ++w;
    }
  }
  if (nt >= (1ull << 32)) fail(CIEG_ERR_CONFIG, "tile count exceeds 2^32");
}

void build_schedule(HostTiles& t, std::uint32_t ctas) {
  const std::uint32_t np = t.npanels();
  ctas = std::max<std::uint32_t>(1, std::min<std::uint32_t>(ctas, np));
  // cost of a panel = entry quads of its work items + a fixed per-item charge
  std::vector<std::pair<std::uint64_t, std::uint32_t>> cost(np);
  for (std::uint32_t P = 0; P < np; ++P) {
    std::uint64_t c = 0;
    for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w) {
      const std::uint32_t tile = t.work_tile[w];
      c += (t.tile_off[tile + 1] - t.tile_off[tile]) / 4 + 256;
    }
    cost[P] = {c, P};
  }
  std::vector<std::uint32_t> order(np);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
    return cost[a].first > cost[b].first;
  });
  // min-heap of (load, cta)
  std::vector<std::pair<std::uint64_t, std::uint32_t>> heap;
  for (std::uint32_t b = 0; b < ctas; ++b) heap.push_back({0, b});
  auto cmp = [](const auto& x, const auto& y) { return x.first != y.first ? x.first > y.first : x.second > y.second; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  std::vector<std::vector<std::uint32_t>> panels_of(ctas);
  for (std::uint32_t P : order) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    auto& top = heap.back();
    panels_of[top.second].push_back(P);
    top.first += cost[P].first;
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  t.sched_off.assign(ctas + 1, 0);
  t.sched.clear();
  for (std::uint32_t b = 0; b < ctas; ++b) {
    std::sort(panels_of[b].begin(), panels_of[b].end());
    for (std::uint32_t P : panels_of[b]) {
      const std::uint32_t w0 = t.work_off[P], w1 = t.work_off[P + 1];
      if (w0 == w1) {  // empty panel: one no-op item so the owner still writes zeros
        const std::uint32_t d[8] = {0, 0, 0, 0, 3u | (1u << 8) | (1u << 9), t.panel_start[P],
                                    t.panel_start[P + 1] - t.panel_start[P], P};
        t.sched.insert(t.sched.end(), d, d + 8);
        continue;
      }
      for (std::uint32_t w = w0; w < w1; ++w) {
        const std::uint32_t tile = t.work_tile[w], other = t.work_other[w];
        const std::uint64_t q0 = t.tile_off[tile] / 4, q1 = t.tile_off[tile + 1] / 4;
        const std::uint32_t flags = t.work_kind[w] | ((w == w0) ? 1u << 8 : 0u) | ((w + 1 == w1) ? 1u << 9 : 0u);
        const std::uint32_t d[8] = {static_cast<std::uint32_t>(q0), static_cast<std::uint32_t>(q0 >> 32),
                                    static_cast<std::uint32_t>(q1), static_cast<std::uint32_t>(q1 >> 32),
                                    flags, t.panel_start[other], t.panel_start[other + 1] - t.panel_start[other], P};
        t.sched.insert(t.sched.end(), d, d + 8);
      }
    }
    t.sched_off[b + 1] = static_cast<std::uint32_t>(t.sched.size() / 8);
  }
}

}  // namespace cieg
