// tiling.cpp -- see tiling.hpp.
#include "tiling.hpp"
#include "tile_layout.h"

#include <algorithm>
#include <cstring>
#include <numeric>

namespace cieg {

std::vector<std::uint32_t> plan_panels(std::uint32_t dim, const std::uint32_t* gb,
                                       std::uint32_t ng, std::uint32_t te, const std::uint32_t* cuts,
                                       std::uint32_t ncuts) {
  std::vector<std::uint32_t> p = plan_panels(dim, gb, ng, te);
  // mandatory cuts only split panels, so every panel stays <= te
  for (std::uint32_t i = 0; i < ncuts; ++i) {
    if (cuts[i] == 0 || cuts[i] >= dim) continue;
    auto it = std::lower_bound(p.begin(), p.end(), cuts[i]);
    if (*it != cuts[i]) p.insert(it, cuts[i]);
  }
  return p;
}

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

  const int prec = csb.precision;
  const std::uint32_t sa = cieg_tl::stride(te, prec);  // tile_layout.h
  const std::uint32_t sentinel = te | (te << 16);  // row 0, pad column te: never read
  std::vector<std::uint32_t> panel_of(dim);
  for (std::uint32_t p = 0; p < np; ++p)
    for (std::uint32_t r = panels[p]; r < panels[p + 1]; ++r) panel_of[r] = p;

  // Per panel row: entries bucketed by column panel.
  struct Bucket {
    std::uint32_t pj;
    std::vector<std::uint32_t> idx;
    std::vector<double> v;
    std::vector<std::uint16_t> key;  // row-major position in the tile (canonical order)
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
              bk.push_back(Bucket{pj, {}, {}, {}});
              tb = &bk.back();
            }
          }
          const std::uint32_t rl = a - r0, cl = b - panels[pj];
          // Packed tile-local index: the entry's shared-memory offset in the
          // row-part orientation and in the transposed one (tile_layout.h).
          tb->idx.push_back(cieg_tl::pack(rl, cl, sa, prec));
          tb->key.push_back(static_cast<std::uint16_t>(rl * te + cl));
          tb->v.push_back(single ? static_cast<double>(v32[e]) : v64[e]);
        }
      }
    }
    std::sort(bk.begin(), bk.end(), [](const Bucket& x, const Bucket& y) { return x.pj < y.pj; });
    // canonical row-major entry order inside every tile (a panel may straddle
    // CSB blocks, which the walk above visits block by block): the GPU
    // generator emits the same order, and the bank-aware reorder (reorder.cu)
    // starts from it
    for (Bucket& b : bk) {
      if (!std::is_sorted(b.key.begin(), b.key.end())) {
        std::vector<std::uint32_t> ord(b.key.size());
        std::iota(ord.begin(), ord.end(), 0u);
        std::sort(ord.begin(), ord.end(), [&](std::uint32_t x, std::uint32_t y) { return b.key[x] < b.key[y]; });
        std::vector<std::uint32_t> idx(ord.size());
        std::vector<double> v(ord.size());
        for (std::size_t k = 0; k < ord.size(); ++k) {
          idx[k] = b.idx[ord[k]];
          v[k] = b.v[ord[k]];
        }
        b.idx.swap(idx);
        b.v.swap(v);
      }
      std::vector<std::uint16_t>().swap(b.key);
    }
  }

  out = HostTiles{};
  out.dim = dim;
  out.row_lo = 0;
  out.row_hi = dim;
  out.halo_lo = 0;
  out.halo_hi = dim;
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

  build_work_lists(out, 0, np);
  if (nt >= (1ull << 32)) fail(CIEG_ERR_CONFIG, "tile count exceeds 2^32");
}

namespace {

// Greedy longest-first assignment of owner panels [p_lo, p_hi) to CTAs and
// the per-CTA item lists. With single_pass the transposed items are left
// out (their product comes from the row-part item of the same tile).
void assign_items(const HostTiles& t, std::uint32_t ctas, std::uint32_t p_lo, std::uint32_t p_hi, bool single_pass,
                  std::vector<std::uint32_t>& sched_off, std::vector<std::uint32_t>& sched) {
  const std::uint32_t np = p_hi - p_lo;
  ctas = std::max<std::uint32_t>(1, std::min<std::uint32_t>(ctas, np));
  auto counted = [&](std::uint32_t w) { return !single_pass || t.work_kind[w] != kTransposed; };
  // cost of a panel = entry quads of its work items + a fixed per-item charge
  std::vector<std::pair<std::uint64_t, std::uint32_t>> cost(np);
  for (std::uint32_t i = 0; i < np; ++i) {
    const std::uint32_t P = p_lo + i;
    std::uint64_t c = 0;
    for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w) {
      if (!counted(w)) continue;
      const std::uint32_t tile = t.work_tile[w];
      c += (t.tile_off[tile + 1] - t.tile_off[tile]) / 4 + 256;
    }
    cost[i] = {c, P};
  }
  std::vector<std::uint32_t> order(np);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
    return cost[a].first > cost[b].first;
  });  // order holds local indices i; panel = p_lo + i
  // min-heap of (load, cta)
  std::vector<std::pair<std::uint64_t, std::uint32_t>> heap;
  for (std::uint32_t b = 0; b < ctas; ++b) heap.push_back({0, b});
  auto cmp = [](const auto& x, const auto& y) { return x.first != y.first ? x.first > y.first : x.second > y.second; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  std::vector<std::vector<std::uint32_t>> panels_of(ctas);
  for (std::uint32_t i : order) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    auto& top = heap.back();
    panels_of[top.second].push_back(p_lo + i);
    top.first += cost[i].first;
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  sched_off.assign(ctas + 1, 0);
  sched.clear();
  std::vector<std::uint32_t> ws;
  for (std::uint32_t b = 0; b < ctas; ++b) {
    std::sort(panels_of[b].begin(), panels_of[b].end());
    for (std::uint32_t P : panels_of[b]) {
      ws.clear();
      for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w)
        if (counted(w)) ws.push_back(w);
      const std::uint32_t prows = t.panel_start[P + 1] - t.panel_start[P];
      if (ws.empty()) {  // empty panel: one no-op item so the owner still writes zeros
        const std::uint32_t d[8] = {0, 0, 0, 0, 3u | (1u << 8) | (1u << 9) | (prows << 16), t.panel_start[P],
                                    prows, t.panel_start[P]};
        sched.insert(sched.end(), d, d + 8);
        continue;
      }
      for (std::size_t k = 0; k < ws.size(); ++k) {
        const std::uint32_t w = ws[k];
        const std::uint32_t tile = t.work_tile[w], other = t.work_other[w];
        const std::uint64_t q0 = t.tile_off[tile] / 4, q1 = t.tile_off[tile + 1] / 4;
        const std::uint32_t flags = t.work_kind[w] | (k == 0 ? 1u << 8 : 0u) | (k + 1 == ws.size() ? 1u << 9 : 0u) |
                                    (prows << 16);
        const std::uint32_t d[8] = {static_cast<std::uint32_t>(q0), static_cast<std::uint32_t>(q0 >> 32),
                                    static_cast<std::uint32_t>(q1), static_cast<std::uint32_t>(q1 >> 32),
                                    flags, t.panel_start[other], t.panel_start[other + 1] - t.panel_start[other],
                                    t.panel_start[P]};
        sched.insert(sched.end(), d, d + 8);
      }
    }
    sched_off[b + 1] = static_cast<std::uint32_t>(sched.size() / 8);
  }
}

}  // namespace

void build_schedule(HostTiles& t, std::uint32_t ctas) {
  // owner panels of this tiling (all of them unless restricted to a shard)
  const std::uint32_t p_lo = static_cast<std::uint32_t>(
      std::lower_bound(t.panel_start.begin(), t.panel_start.end(), t.row_lo) - t.panel_start.begin());
  const std::uint32_t p_hi = static_cast<std::uint32_t>(
      std::lower_bound(t.panel_start.begin(), t.panel_start.end(), t.row_hi) - t.panel_start.begin());
  assign_items(t, ctas, p_lo, p_hi, false, t.sched_off, t.sched);
  t.sp_sched_off.clear();
  t.sp_sched.clear();
  t.sp_col_off.clear();
  t.sp_col_items.clear();
  t.sp_partial_lo = t.row_lo;
  assign_items(t, ctas, p_lo, p_hi, true, t.sp_sched_off, t.sp_sched);
  // partial slots per block column, in item order (a fixed order: deterministic sums)
  const std::uint32_t np = t.npanels();
  const std::size_t nitems = t.sp_sched.size() / 8;
  std::vector<std::uint32_t> q_of(nitems, np);
  for (std::size_t i = 0; i < nitems; ++i) {
    const std::uint32_t* d = t.sp_sched.data() + 8 * i;
    if ((d[4] & 0xffu) != kRowPart) continue;
    q_of[i] = static_cast<std::uint32_t>(
        std::upper_bound(t.panel_start.begin(), t.panel_start.end(), d[5]) - t.panel_start.begin() - 1);
  }
  t.sp_col_off.assign(np + 1, 0);
  for (std::uint32_t qv : q_of)
    if (qv < np) {
      ++t.sp_col_off[qv + 1];
      t.sp_partial_lo = std::min(t.sp_partial_lo, t.panel_start[qv]);  // block columns below the shard
    }
  for (std::uint32_t Q = 0; Q < np; ++Q) t.sp_col_off[Q + 1] += t.sp_col_off[Q];
  t.sp_col_items.resize(t.sp_col_off[np]);
  std::vector<std::uint32_t> fill(t.sp_col_off.begin(), t.sp_col_off.end() - 1);
  for (std::size_t i = 0; i < nitems; ++i)
    if (q_of[i] < np) t.sp_col_items[fill[q_of[i]]++] = static_cast<std::uint32_t>(i);
}

void build_work_lists(HostTiles& out, std::uint32_t p_lo, std::uint32_t p_hi) {
  // Owner work lists for panels [p_lo, p_hi): row parts and the diagonal tile
  // of P (ascending J), then transposed parts of tiles (I, P), I > P
  // (ascending I). Tiles must be sorted by (pi, pj).
  const std::uint32_t np = static_cast<std::uint32_t>(out.panel_start.size() - 1);
  const std::uint64_t nt = out.tile_pi.size();
  std::vector<std::vector<std::uint32_t>> rowt(np), trans(np);
  for (std::uint64_t t = 0; t < nt; ++t) {
    const std::uint32_t pi = out.tile_pi[t], pj = out.tile_pj[t];
    if (pi >= p_lo && pi < p_hi) rowt[pi].push_back(static_cast<std::uint32_t>(t));
    if (pi != pj && pj >= p_lo && pj < p_hi) trans[pj].push_back(static_cast<std::uint32_t>(t));
  }
  out.work_off.assign(np + 1, 0);
  for (std::uint32_t P = 0; P < np; ++P)
    out.work_off[P + 1] = out.work_off[P] + static_cast<std::uint32_t>(rowt[P].size() + trans[P].size());
  const std::uint32_t nw = out.work_off[np];
  out.work_tile.resize(nw);
  out.work_other.resize(nw);
  out.work_kind.resize(nw);
  for (std::uint32_t P = 0; P < np; ++P) {
    std::uint32_t w = out.work_off[P];
    for (std::uint32_t t : rowt[P]) {
      out.work_tile[w] = t;
      out.work_other[w] = out.tile_pj[t];
      out.work_kind[w] = out.tile_pj[t] == P ? kDiagonal : kRowPart;
      ++w;
    }
    for (std::uint32_t t : trans[P]) {
      out.work_tile[w] = t;
      out.work_other[w] = out.tile_pi[t];
      out.work_kind[w] = kTransposed;
      ++w;
    }
  }
}

void restrict_to_rows(HostTiles& t, std::uint32_t row_lo, std::uint32_t row_hi) {
  const std::uint32_t np = t.npanels();
  const std::uint32_t p_lo = static_cast<std::uint32_t>(
      std::lower_bound(t.panel_start.begin(), t.panel_start.end(), row_lo) - t.panel_start.begin());
  const std::uint32_t p_hi = static_cast<std::uint32_t>(
      std::lower_bound(t.panel_start.begin(), t.panel_start.end(), row_hi) - t.panel_start.begin());
  if (p_lo > np || p_hi > np || t.panel_start[p_lo] != row_lo || t.panel_start[p_hi] != row_hi)
    fail(CIEG_ERR_CONFIG, "shard bounds are not panel boundaries");
  // tiles referenced by owned work items, in first-use order
  std::vector<std::int64_t> remap(t.ntiles(), -1);
  std::vector<std::uint64_t> keep;
  std::uint32_t hlo = row_lo, hhi = row_hi;
  for (std::uint32_t P = p_lo; P < p_hi; ++P)
    for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w) {
      const std::uint32_t tile = t.work_tile[w];
      if (remap[tile] < 0) {
        remap[tile] = static_cast<std::int64_t>(keep.size());
        keep.push_back(tile);
      }
      const std::uint32_t o = t.work_other[w];
      hlo = std::min(hlo, t.panel_start[o]);
      hhi = std::max(hhi, t.panel_start[o + 1]);
    }
  HostTiles r;
  r.dim = t.dim;
  r.tile_edge = t.tile_edge;
  r.precision = t.precision;
  r.panel_start = t.panel_start;
  r.tile_off.assign(1, 0);
  for (std::uint64_t k : keep) {
    r.tile_pi.push_back(t.tile_pi[k]);
    r.tile_pj.push_back(t.tile_pj[k]);
    r.tile_off.push_back(r.tile_off.back() + (t.tile_off[k + 1] - t.tile_off[k]));
  }
  const std::uint64_t slots = r.tile_off.back();
  r.idx.resize(slots);
  if (t.precision == 0)
    r.val32.resize(slots);
  else
    r.val64.resize(slots);
  r.nnz = 0;
#pragma omp parallel for schedule(dynamic, 64)
  for (std::int64_t j = 0; j < static_cast<std::int64_t>(keep.size()); ++j) {
    const std::uint64_t k = keep[j];
    const std::uint64_t n = t.tile_off[k + 1] - t.tile_off[k];
    std::memcpy(r.idx.data() + r.tile_off[j], t.idx.data() + t.tile_off[k], n * sizeof(std::uint32_t));
    if (t.precision == 0)
      std::memcpy(r.val32.data() + r.tile_off[j], t.val32.data() + t.tile_off[k], n * sizeof(float));
    else
      std::memcpy(r.val64.data() + r.tile_off[j], t.val64.data() + t.tile_off[k], n * sizeof(double));
  }
  for (std::uint64_t k : keep) {
    // count real (non-sentinel) entries
    const std::uint32_t te = t.tile_edge;
    const std::uint32_t sentinel = te | (te << 16);
    for (std::uint64_t e = t.tile_off[k]; e < t.tile_off[k + 1]; ++e) r.nnz += t.idx[e] != sentinel;
  }
  r.work_off.assign(np + 1, 0);
  for (std::uint32_t P = 0; P < np; ++P) {
    const std::uint32_t cnt = (P >= p_lo && P < p_hi) ? t.work_off[P + 1] - t.work_off[P] : 0;
    r.work_off[P + 1] = r.work_off[P] + cnt;
  }
  for (std::uint32_t P = p_lo; P < p_hi; ++P)
    for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w) {
      r.work_tile.push_back(static_cast<std::uint32_t>(remap[t.work_tile[w]]));
      r.work_other.push_back(t.work_other[w]);
      r.work_kind.push_back(t.work_kind[w]);
    }
  r.row_lo = row_lo;
  r.row_hi = row_hi;
  r.halo_lo = hlo;
  r.halo_hi = hhi;
  t = std::move(r);
}

void shard_plan(const cieg_csb_view& csb, const std::uint32_t* gb, std::uint32_t ng, std::uint32_t te,
                std::uint32_t nranks, std::uint32_t* row_bounds, std::uint32_t* halo_lo, std::uint32_t* halo_hi) {
  if (nranks == 0) fail(CIEG_ERR_CONFIG, "shard_plan: nranks must be positive");
  const std::uint32_t dim = csb.dim;
  // per-row streamed entries: row part + transposed part
  std::vector<std::uint64_t> cost(dim + 1, 0);
  const float* v32 = nullptr;
  (void)v32;
  for (std::uint32_t bi = 0; bi < csb.nb; ++bi) {
    const std::uint32_t rb = csb.block_boundaries[bi];
    for (std::uint32_t bj = 0; bj <= bi; ++bj) {
      const std::uint64_t b = static_cast<std::uint64_t>(bi) * (bi + 1) / 2 + bj;
      const std::uint32_t cb = csb.block_boundaries[bj];
      for (std::uint64_t e = csb.entry_offsets[b]; e < csb.entry_offsets[b + 1]; ++e) {
        const std::uint32_t r = rb + csb.rows[e], c = cb + csb.cols[e];
        ++cost[r];
        if (c != r) ++cost[c];
      }
    }
  }
  // candidate cut rows = the panel boundaries the shard upload will plan
  // (small groups merge into panels, so not every group boundary is one)
  std::vector<std::uint32_t> cuts;
  if (gb && ng) {
    if (gb[0] != 0 || gb[ng] != dim) fail(CIEG_ERR_DIMENSION, "group bounds do not cover [0, dim)");
    cuts = plan_panels(dim, gb, ng, te);
  } else {
    for (std::uint32_t r = 0; r <= dim; r += te) cuts.push_back(r);
    if (cuts.back() != dim) cuts.push_back(dim);
  }
  std::vector<std::uint64_t> pre(dim + 1, 0);
  for (std::uint32_t r = 0; r < dim; ++r) pre[r + 1] = pre[r] + cost[r];
  const std::uint64_t total = pre[dim];
  row_bounds[0] = 0;
  std::size_t ci = 0;
  for (std::uint32_t k = 1; k < nranks; ++k) {
    const long double target = static_cast<long double>(total) * k / nranks;
    while (ci + 1 < cuts.size() && pre[cuts[ci + 1]] <= target) ++ci;
    std::uint32_t cut = cuts[ci];
    if (ci + 1 < cuts.size() && (target - pre[cuts[ci]]) > (pre[cuts[ci + 1]] - target)) cut = cuts[ci + 1];
    cut = std::max(cut, row_bounds[k - 1]);
    row_bounds[k] = cut;
  }
  row_bounds[nranks] = dim;
  // halos from the device panel grid of a full tiling
  std::vector<std::uint32_t> panels = plan_panels(dim, gb, ng, te);
  HostTiles t;
  build_tiles(csb, panels, te, t);
  for (std::uint32_t k = 0; k < nranks; ++k) {
    const std::uint32_t lo = row_bounds[k], hi = row_bounds[k + 1];
    std::uint32_t hl = lo, hh = hi;
    for (std::uint32_t P = 0; P < t.npanels(); ++P) {
      if (t.panel_start[P] < lo || t.panel_start[P + 1] > hi) continue;
      for (std::uint32_t w = t.work_off[P]; w < t.work_off[P + 1]; ++w) {
        const std::uint32_t o = t.work_other[w];
        hl = std::min(hl, t.panel_start[o]);
        hh = std::max(hh, t.panel_start[o + 1]);
      }
    }
    halo_lo[k] = hl;
    halo_hi[k] = hh;
  }
}

}  // namespace cieg
