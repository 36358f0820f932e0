// gpugen.cu -- the BASELINE sector generator run on the GPU, writing the
// device tile stream of the SpMM directly: no host
// CSB, no host re-tiling. Same hash streams and portable Box-Muller as the
// host generator (gen_common.h), same panel plan, same entry order inside a
// tile (row-major), so the tile stream is bit-identical to
// cieg_matrix_upload(cieg_generate_csb(...)) -- checked by the GPU tests.
// Also builds the tile-diagonal preconditioner on the device from a matrix's
// diagonal tiles (ci::extract_tile_diagonal, hamiltonian.cpp:178-203).
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <string>
#include <numeric>

#include "context.hpp"
#include "device_common.cuh"
#include "tile_layout.h"
#include "gen_common.h"
#include "generator.hpp"
#include "precond.hpp"
#include "tiling.hpp"

namespace cieg {
namespace {

struct GenTile {
  std::uint32_t a0, nr;  // global first row / rows of panel PI
  std::uint32_t b0, nc;  // global first column / columns of panel PJ
  std::uint32_t diag;    // PI == PJ (lower part only, incl. the diagonal)
  std::uint32_t sector;  // sector of the rows (diagonal values), when not `general`
  std::uint32_t general; // a panel merges several generator tiles: per-entry tile lookup
};

struct GenArgs {
  const GenTile* tiles;
  std::uint64_t q_seed, v1_seed, v2_seed, d_seed;
  double q, scale;
  std::uint32_t sa, te;
  int precision;
  // generator tile grid, for `general` device tiles (small generator tiles
  // merged into one panel): tile starts (ntiles + 1), sectors, first kept-
  // candidate tile J0 of the band, and the tile-keep hash (generator.cpp:
  // kept_tiles)
  const std::uint32_t* tstart;
  const std::uint32_t* tsector;
  const std::uint32_t* tj0;
  std::uint32_t ntiles;
  std::uint64_t tile_seed;
  double p;
};

__device__ __forceinline__ std::uint32_t tile_of(const GenArgs& g, std::uint32_t r) {
  std::uint32_t lo = 0, hi = g.ntiles;  // largest t with tstart[t] <= r
  while (hi - lo > 1) {
    const std::uint32_t mid = (lo + hi) / 2;
    if (g.tstart[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool entry_exists(const GenArgs& g, const GenTile& t, std::uint32_t a, std::uint32_t b) {
  if (t.diag && b > a) return false;
  if (a == b) return true;
  if (t.general) {  // the generator tile pair of this entry must be kept
    const std::uint32_t I = tile_of(g, a), J = tile_of(g, b);
    if (I != J) {
      if (J > I || J < g.tj0[I]) return false;
      if (!(cieg_gen::unit_double(cieg_gen::hash3(g.tile_seed, I, J)) < g.p)) return false;
    }
  }
  return cieg_gen::unit_double(cieg_gen::hash3(g.q_seed, a, b)) < g.q;
}

__global__ void __launch_bounds__(256) gen_count_kernel(GenArgs g, std::uint32_t* counts) {
  const GenTile t = g.tiles[blockIdx.x];
  const std::uint32_t total = t.nr * t.nc;
  std::uint32_t cnt = 0;
  for (std::uint32_t e = threadIdx.x; e < total; e += blockDim.x) {
    const std::uint32_t r = e / t.nc, c = e - r * t.nc;
    cnt += entry_exists(g, t, t.a0 + r, t.b0 + c) ? 1u : 0u;
  }
  __shared__ std::uint32_t red[8];
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    std::uint32_t s = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
    counts[blockIdx.x] = s;
  }
}


// One CTA (128 threads, one column each) per tile, rows in order: entries are
// written row-major, exactly the order of the host CSB re-tiling.
template <typename V>
__global__ void __launch_bounds__(128) gen_fill_kernel(GenArgs g, const std::uint64_t* tile_off, std::uint32_t* idx,
                                                       V* val) {
  const GenTile t = g.tiles[blockIdx.x];
  __shared__ std::uint32_t wcount[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint32_t c = threadIdx.x;
  std::uint64_t pos = tile_off[blockIdx.x];
  for (std::uint32_t r = 0; r < t.nr; ++r) {
    const std::uint32_t a = t.a0 + r, b = t.b0 + c;
    const bool ex = c < t.nc && entry_exists(g, t, a, b);
    const unsigned ballot = __ballot_sync(0xffffffffu, ex);
    if (lane == 0) wcount[warp] = __popc(ballot);
    __syncthreads();
    std::uint32_t before = 0, rowtot = 0;
    for (int w = 0; w < 4; ++w) {
      if (w < warp) before += wcount[w];
      rowtot += wcount[w];
    }
    if (ex) {
      const std::uint64_t e = pos + before + __popc(ballot & ((1u << lane) - 1u));
      idx[e] = cieg_tl::pack(r, c, g.sa, g.precision);
      double v;
      if (a == b) {
        const double u = cieg_gen::unit_double(cieg_gen::hash3(g.d_seed, a, a));
        const std::uint32_t sec = t.general ? g.tsector[tile_of(g, a)] : t.sector;
        v = 10.0 * static_cast<double>(sec) + 4.0 * u - 2.0;
      } else {
        v = cieg_gen::normal_from(cieg_gen::hash3(g.v1_seed, a, b), cieg_gen::hash3(g.v2_seed, a, b)) * g.scale;
      }
      val[e] = static_cast<V>(v);
    }
    pos += rowtot;
    __syncthreads();
  }
}

__global__ void fill_u32(std::uint32_t* p, std::uint64_t n, std::uint32_t v) {
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

template <typename T>
T* dev_upload(const std::vector<T>& v) {
  T* d = nullptr;
  CIEG_CUDA(cudaMalloc(&d, std::max<std::size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) CIEG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

// The device tile edge of a generated matrix: the rule of cieg_matrix_upload
// (capi.cu: choose_tile_edge) on the generator's groups.
std::uint32_t generated_tile_edge(const cieg_gen_params& p, const TileGrid& grid, std::uint32_t te) {
  if (te == 0) {
    std::uint32_t mx = 0;
    for (std::uint32_t t = 0; t < grid.count(); ++t) mx = std::max(mx, grid.start[t + 1] - grid.start[t]);
    te = mx <= 64 ? 64 : 128;
  }
  if (p.precision == 1) te = 64;
  if (te != 64 && te != 128) fail(CIEG_ERR_CONFIG, "tile edge must be 64 or 128");
  return te;
}

cieg_mat* generate_device(cieg_ctx* ctx, const cieg_gen_params& p, std::uint32_t te, std::uint32_t row_lo,
                          std::uint32_t row_hi) {
  validate(p);
  if (row_hi == 0) row_hi = p.n;
  const TileGrid grid = make_grid(p);
  te = generated_tile_edge(p, grid, te);
  const std::uint32_t ng = grid.count();
  const std::vector<std::vector<std::uint32_t>> kept = kept_tiles(p, grid);
  const double scale = value_scale(p);

  HostTiles ht;
  ht.dim = p.n;
  ht.tile_edge = te;
  ht.precision = p.precision;
  ht.panel_start = plan_panels(p.n, grid.start.data(), ng, te);
  const std::uint32_t np = static_cast<std::uint32_t>(ht.panel_start.size() - 1);
  // generator tile -> its panel range [tpa, tpb): a chunked large tile spans
  // several panels; small tiles merged by the planner share one panel, whose
  // device tiles then decide per entry which generator tile pair it is in
  std::vector<std::uint32_t> tpa(ng), tpb(ng), tiles_in_panel(np, 0);
  for (std::uint32_t t = 0; t < ng; ++t) {
    const std::uint32_t r0 = grid.start[t], r1 = grid.start[t + 1];
    tpa[t] = static_cast<std::uint32_t>(std::upper_bound(ht.panel_start.begin(), ht.panel_start.end(), r0) -
                                        ht.panel_start.begin()) - 1;
    tpb[t] = static_cast<std::uint32_t>(std::lower_bound(ht.panel_start.begin(), ht.panel_start.end(), r1) -
                                        ht.panel_start.begin());
    for (std::uint32_t P = tpa[t]; P < tpb[t]; ++P) ++tiles_in_panel[P];
  }
  const std::uint32_t p_lo = static_cast<std::uint32_t>(
      std::lower_bound(ht.panel_start.begin(), ht.panel_start.end(), row_lo) - ht.panel_start.begin());
  const std::uint32_t p_hi = static_cast<std::uint32_t>(
      std::lower_bound(ht.panel_start.begin(), ht.panel_start.end(), row_hi) - ht.panel_start.begin());
  if (p_hi > np || ht.panel_start[p_lo] != row_lo || ht.panel_start[p_hi] != row_hi || row_lo >= row_hi)
    fail(CIEG_ERR_CONFIG, "shard rows are not panel boundaries");
  auto owned = [&](std::uint32_t P) { return P >= p_lo && P < p_hi; };

  struct Key {
    std::uint32_t pi, pj, I;
  };
  std::vector<Key> keys;
  for (std::uint32_t I = 0; I < ng; ++I)
    for (std::uint32_t J : kept[I])
      for (std::uint32_t PI = tpa[I]; PI < tpb[I]; ++PI)
        for (std::uint32_t PJ = tpa[J]; PJ < tpb[J]; ++PJ) {
          if (PJ > PI) continue;  // lower triangle of panels (diagonal tiles: lower part)
          if (!owned(PI) && !owned(PJ)) continue;
          keys.push_back({PI, PJ, I});
        }
  std::sort(keys.begin(), keys.end(), [](const Key& x, const Key& y) { return x.pi != y.pi ? x.pi < y.pi : x.pj < y.pj; });
  keys.erase(std::unique(keys.begin(), keys.end(), [](const Key& x, const Key& y) { return x.pi == y.pi && x.pj == y.pj; }),
             keys.end());
  const std::uint64_t nt = keys.size();
  std::vector<GenTile> gt(nt);
  ht.tile_pi.resize(nt);
  ht.tile_pj.resize(nt);
  for (std::uint64_t k = 0; k < nt; ++k) {
    const Key& q = keys[k];
    ht.tile_pi[k] = q.pi;
    ht.tile_pj[k] = q.pj;
    const std::uint32_t general = (tiles_in_panel[q.pi] > 1 || tiles_in_panel[q.pj] > 1) ? 1u : 0u;
    gt[k] = GenTile{ht.panel_start[q.pi], ht.panel_start[q.pi + 1] - ht.panel_start[q.pi], ht.panel_start[q.pj],
                    ht.panel_start[q.pj + 1] - ht.panel_start[q.pj], q.pi == q.pj ? 1u : 0u, grid.sector[q.I], general};
  }
  // band start J0 per tile row (generator.cpp: kept_tiles)
  std::vector<std::uint32_t> tj0(ng);
  for (std::uint32_t I = 0; I < ng; ++I) {
    const std::uint32_t sI = grid.sector[I];
    const std::uint32_t s_lo = sI >= p.band ? sI - p.band : 0;
    tj0[I] = static_cast<std::uint32_t>(std::lower_bound(grid.start.begin(), grid.start.end() - 1,
                                                         grid.sector_start[s_lo]) - grid.start.begin());
  }
  const cieg_gen::Seeds sd = cieg_gen::derive_seeds(p.seed);
  CIEG_CUDA(cudaSetDevice(ctx->device));
  GenTile* d_tiles = dev_upload(gt);
  std::uint32_t* d_tstart = dev_upload(grid.start);
  std::uint32_t* d_tsector = dev_upload(grid.sector);
  std::uint32_t* d_tj0 = dev_upload(tj0);
  std::uint32_t* d_counts = nullptr;
  CIEG_CUDA(cudaMalloc(&d_counts, std::max<std::uint64_t>(1, nt) * sizeof(std::uint32_t)));
  GenArgs ga{d_tiles, sd.q, sd.v1, sd.v2, sd.d, p.q, scale, cieg_tl::stride(te, p.precision), te, p.precision,
             d_tstart, d_tsector, d_tj0, ng, sd.tile, p.p};
  cieg_mat* m = nullptr;
  try {
    if (nt) {
      gen_count_kernel<<<static_cast<unsigned>(nt), 256, 0, ctx->stream>>>(ga, d_counts);
      CIEG_CUDA(cudaGetLastError());
      ++ctx->launches;
    }
    std::vector<std::uint32_t> counts(nt);
    if (nt) CIEG_CUDA(cudaMemcpyAsync(counts.data(), d_counts, nt * sizeof(std::uint32_t), cudaMemcpyDeviceToHost,
                                      ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    ht.tile_off.assign(nt + 1, 0);
    ht.nnz = 0;
    for (std::uint64_t k = 0; k < nt; ++k) {
      ht.nnz += counts[k];
      ht.tile_off[k + 1] = ht.tile_off[k] + ((counts[k] + 3u) & ~3u);
    }
    ht.row_lo = row_lo;
    ht.row_hi = row_hi;
    build_work_lists(ht, p_lo, p_hi);
    std::uint32_t hlo = row_lo, hhi = row_hi;
    for (std::uint32_t P = p_lo; P < p_hi; ++P)
      for (std::uint32_t w = ht.work_off[P]; w < ht.work_off[P + 1]; ++w) {
        hlo = std::min(hlo, ht.panel_start[ht.work_other[w]]);
        hhi = std::max(hhi, ht.panel_start[ht.work_other[w] + 1]);
      }
    ht.halo_lo = hlo;
    ht.halo_hi = hhi;
    build_schedule(ht, static_cast<std::uint32_t>(ctx->sm_count));

    m = new cieg_mat;
    m->ctx = ctx;
    m->dim = p.n;
    m->tile_edge = te;
    m->precision = p.precision;
    m->nnz = ht.nnz;
    m->npanels = np;
    m->ntiles = nt;
    m->row_lo = row_lo;
    m->row_hi = row_hi;
    m->halo_lo = hlo;
    m->halo_hi = hhi;
    m->panel_start_host = ht.panel_start;
    m->group_bounds_host.assign(grid.start.begin(), grid.start.end());
    m->panel_start = dev_upload(ht.panel_start);
    m->tile_off = dev_upload(ht.tile_off);
    m->tile_pi_host = ht.tile_pi;
    m->tile_pj_host = ht.tile_pj;
    m->tile_off_host = ht.tile_off;
    const std::uint64_t slots = ht.tile_off[nt];
    CIEG_CUDA(cudaMalloc(&m->idx, std::max<std::uint64_t>(1, slots) * sizeof(std::uint32_t)));
    CIEG_CUDA(cudaMalloc(&m->val, std::max<std::uint64_t>(1, slots) * (p.precision == 0 ? 4 : 8)));
    if (slots) {
      fill_u32<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(m->idx, slots, te | (te << 16));
      CIEG_CUDA(cudaMemsetAsync(m->val, 0, slots * (p.precision == 0 ? 4 : 8), ctx->stream));
      if (p.precision == 0)
        gen_fill_kernel<float><<<static_cast<unsigned>(nt), 128, 0, ctx->stream>>>(ga, m->tile_off, m->idx,
                                                                                   static_cast<float*>(m->val));
      else
        gen_fill_kernel<double><<<static_cast<unsigned>(nt), 128, 0, ctx->stream>>>(ga, m->tile_off, m->idx,
                                                                                    static_cast<double*>(m->val));
      CIEG_CUDA(cudaGetLastError());
      ctx->launches += 2;
    }
    upload_schedule(m, ht);
    m->tile_bytes = slots * (4 + (p.precision == 0 ? 4 : 8));
    order_tile_entries(ctx, m);
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFree(d_tiles);
    cudaFree(d_counts);
    cudaFree(d_tstart);
    cudaFree(d_tsector);
    cudaFree(d_tj0);
    delete m;
    throw;
  }
  cudaFree(d_tiles);
  cudaFree(d_counts);
  cudaFree(d_tstart);
  cudaFree(d_tsector);
  cudaFree(d_tj0);
  return m;
}

namespace {


struct DiagTile {
  std::uint64_t e0, e1;      // entry slots
  std::uint32_t a0, b0;      // global first row / column of the tile's panels
  std::uint32_t g_lo, g_hi;  // groups overlapping the row panel (g_hi exclusive)
};

// Scatter the tile's entries into their group's dense block, mirrored
// (ci::extract_tile_diagonal, hamiltonian.cpp:178-203). A panel may hold
// several small groups (merged generator tiles) or be part of one larger
// group: every entry looks up the groups of its row and its column and is
// kept only when both lie in the same group, indexed relative to it.
// Blocks are stored in the tile stream's own value type: fp32 values of an
// fp32 H widen to fp64 exactly when the preconditioner reads them.
__device__ __forceinline__ std::uint32_t group_of(const std::uint32_t* lb, std::uint32_t lo, std::uint32_t hi,
                                                  std::uint32_t row) {
  while (hi - lo > 1) {  // lb[lo] <= row < lb[hi]
    const std::uint32_t mid = (lo + hi) >> 1;
    if (lb[mid] <= row) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename V, typename B = V>
__global__ void diag_blocks_kernel(const DiagTile* dt, const std::uint32_t* idx, const V* val, std::uint32_t te,
                                   std::uint32_t row_lo, const std::uint32_t* lb, const std::uint64_t* off,
                                   std::uint32_t ngroups, B* blocks) {
  const DiagTile t = dt[blockIdx.x];
  for (std::uint64_t e = t.e0 + threadIdx.x; e < t.e1; e += blockDim.x) {
    const std::uint32_t o = idx[e] & 0xffffu;
    constexpr int prec = sizeof(V) == 4 ? 0 : 1;
    const std::uint32_t sa = cieg_tl::stride(te, prec);
    const std::uint32_t r = o / sa, pc = o - r * sa;
    if (pc >= te) continue;  // sentinel
    const std::uint32_t c = cieg_tl::unperm(pc, prec);
    const std::uint32_t ra = t.a0 + r - row_lo, cb = t.b0 + c - row_lo;  // shard-local row / column
    if (ra >= lb[ngroups] || cb >= lb[ngroups]) continue;
    const std::uint32_t g = group_of(lb, t.g_lo, t.g_hi + 1 > ngroups ? ngroups : t.g_hi + 1, ra);
    if (ra < lb[g] || ra >= lb[g + 1] || cb < lb[g] || cb >= lb[g + 1]) continue;  // cross-group coupling
    const std::uint32_t gn = lb[g + 1] - lb[g], ia = ra - lb[g], ib = cb - lb[g];
    const B v = static_cast<B>(val[e]);
    blocks[off[g] + ia + static_cast<std::uint64_t>(ib) * gn] = v;
    blocks[off[g] + ib + static_cast<std::uint64_t>(ia) * gn] = v;
  }
}

}  // namespace

cieg_prec* precond_from_matrix(cieg_ctx* ctx, const cieg_mat* m) {
  if (m->group_bounds_host.empty() || m->tile_pi_host.empty())
    fail(CIEG_ERR_CONFIG, "precond_from_matrix needs a matrix made by cieg_generate_device");
  const std::vector<std::uint32_t>& gb = m->group_bounds_host;
  const std::uint32_t ng = static_cast<std::uint32_t>(gb.size() - 1);
  std::uint32_t g0 = 0;
  while (g0 < ng && gb[g0] < m->row_lo) ++g0;
  std::uint32_t g1 = g0;
  while (g1 < ng && gb[g1 + 1] <= m->row_hi) ++g1;
  const std::uint32_t lng = g1 - g0;
  std::vector<std::uint32_t> lb(lng + 1);
  for (std::uint32_t g = 0; g <= lng; ++g) lb[g] = gb[g0 + g] - m->row_lo;
  std::vector<std::uint64_t> off(lng + 1, 0);
  for (std::uint32_t g = 0; g < lng; ++g) {
    const std::uint64_t sz = lb[g + 1] - lb[g];
    off[g + 1] = off[g] + sz * sz;
  }
  // groups overlapping every owned panel: [gfirst, glast]
  const std::vector<std::uint32_t>& ps = m->panel_start_host;
  std::vector<std::int64_t> gfirst(m->npanels, -1), glast(m->npanels, -1);
  for (std::uint32_t P = 0, g = 0; P < m->npanels; ++P) {
    if (ps[P] < m->row_lo || ps[P + 1] > m->row_hi) continue;
    const std::uint32_t a = ps[P] - m->row_lo, b = ps[P + 1] - m->row_lo;
    while (g < lng && lb[g + 1] <= a) ++g;
    if (g >= lng) continue;
    std::uint32_t h = g;
    while (h + 1 < lng && lb[h + 1] < b) ++h;
    gfirst[P] = g;
    glast[P] = h;
  }
  std::vector<DiagTile> dts;
  for (std::uint64_t t = 0; t < m->ntiles; ++t) {
    const std::uint32_t pi = m->tile_pi_host[t], pj = m->tile_pj_host[t];
    if (gfirst[pi] < 0 || gfirst[pj] < 0) continue;
    if (glast[pi] < gfirst[pj] || glast[pj] < gfirst[pi]) continue;  // no group shared by the two panels
    dts.push_back(DiagTile{m->tile_off_host[t], m->tile_off_host[t + 1], ps[pi], ps[pj],
                           static_cast<std::uint32_t>(gfirst[pi]), static_cast<std::uint32_t>(glast[pi])});
  }
  auto* pr = new cieg_prec;
  try {
    pr->ctx = ctx;
    pr->dim = m->row_hi - m->row_lo;
    pr->ngroups = lng;
    pr->bounds_host = lb;
    pr->block_off_host = off;
    for (std::uint32_t g = 0; g < lng; ++g) pr->max_group = std::max(pr->max_group, lb[g + 1] - lb[g]);
    pr->bounds = dev_upload(lb);
    pr->block_off = dev_upload(off);
    // storage: an fp32 H's blocks are stored in fp32 -- exact (the values
    // are fp32) and half the bytes the FOM products stream at every Krylov
    // step; CIEG_PREC_STORAGE=fp64 keeps fp64 blocks (results identical)
    bool f32 = false;
    if (m->precision == 0) {
      f32 = true;
      if (const char* e = std::getenv("CIEG_PREC_STORAGE")) f32 = std::string(e) != "fp64";
    }
    const std::size_t vb = f32 ? sizeof(float) : sizeof(double);
    void* blocks = nullptr;
    CIEG_CUDA(cudaMalloc(&blocks, vb * std::max<std::uint64_t>(1, off[lng])));
    if (f32)
      pr->blocks32 = static_cast<float*>(blocks);
    else
      pr->blocks = static_cast<double*>(blocks);
    CIEG_CUDA(cudaMemsetAsync(blocks, 0, vb * off[lng], ctx->stream));
    if (!dts.empty()) {
      DiagTile* d = dev_upload(dts);
      if (f32)
        diag_blocks_kernel<float><<<static_cast<unsigned>(dts.size()), 256, 0, ctx->stream>>>(
            d, m->idx, static_cast<const float*>(m->val), m->tile_edge, m->row_lo, pr->bounds, pr->block_off, lng,
            pr->blocks32);
      else if (m->precision == 0)
        diag_blocks_kernel<float, double><<<static_cast<unsigned>(dts.size()), 256, 0, ctx->stream>>>(
            d, m->idx, static_cast<const float*>(m->val), m->tile_edge, m->row_lo, pr->bounds, pr->block_off, lng,
            pr->blocks);
      else
        diag_blocks_kernel<double><<<static_cast<unsigned>(dts.size()), 256, 0, ctx->stream>>>(
            d, m->idx, static_cast<const double*>(m->val), m->tile_edge, m->row_lo, pr->bounds, pr->block_off, lng,
            pr->blocks);
      CIEG_CUDA(cudaGetLastError());
      ++ctx->launches;
      CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(d);
    }
  } catch (...) {
    delete pr;
    throw;
  }
  return pr;
}

}  // namespace cieg

extern "C" {

int cieg_generated_panels(const cieg_gen_params* prm, uint32_t tile_edge, uint32_t* panel_start, uint32_t cap,
                          uint32_t* npanels) {
  return cieg::guarded([&] {
    if (!prm || !npanels) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_generated_panels: null argument");
    cieg::validate(*prm);
    const cieg::TileGrid grid = cieg::make_grid(*prm);
    const std::uint32_t te = cieg::generated_tile_edge(*prm, grid, tile_edge);
    const std::vector<std::uint32_t> ps = cieg::plan_panels(prm->n, grid.start.data(), grid.count(), te);
    *npanels = static_cast<uint32_t>(ps.size() - 1);
    if (panel_start) {
      if (cap < ps.size()) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_generated_panels: buffer too small");
      std::copy(ps.begin(), ps.end(), panel_start);
    }
  });
}

int cieg_generate_device(cieg_ctx* ctx, const cieg_gen_params* prm, uint32_t tile_edge, uint32_t row_lo,
                         uint32_t row_hi, cieg_mat** out) {
  return cieg::guarded([&] {
    if (!ctx || !prm || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_generate_device: null argument");
    *out = cieg::generate_device(ctx, *prm, tile_edge, row_lo, row_hi);
  });
}

int cieg_precond_from_matrix(cieg_ctx* ctx, const cieg_mat* mat, cieg_prec** out) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_precond_from_matrix: null argument");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    *out = cieg::precond_from_matrix(ctx, mat);
  });
}

int cieg_matrix_groups(const cieg_mat* mat, const uint32_t** bounds, uint32_t* ngroups) {
  return cieg::guarded([&] {
    if (!mat || !bounds || !ngroups) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_matrix_groups: null argument");
    *bounds = mat->group_bounds_host.data();
    *ngroups = mat->group_bounds_host.empty() ? 0 : static_cast<uint32_t>(mat->group_bounds_host.size() - 1);
  });
}

// Copy the device tile stream back (tests: bit-identity with the host path).
int cieg_matrix_export(const cieg_mat* m, uint64_t* tile_off, uint32_t* tile_pi, uint32_t* tile_pj, uint32_t* idx,
                       void* val) {
  return cieg::guarded([&] {
    if (!m) cieg::fail(CIEG_ERR_ARGUMENT, "null matrix");
    std::vector<std::uint64_t> to(m->ntiles + 1);
    CIEG_CUDA(cudaMemcpy(to.data(), m->tile_off, to.size() * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
    if (tile_off) std::memcpy(tile_off, to.data(), to.size() * sizeof(std::uint64_t));
    if (tile_pi && !m->tile_pi_host.empty()) std::memcpy(tile_pi, m->tile_pi_host.data(), m->ntiles * 4);
    if (tile_pj && !m->tile_pj_host.empty()) std::memcpy(tile_pj, m->tile_pj_host.data(), m->ntiles * 4);
    const std::uint64_t slots = to.back();
    if (idx && slots) CIEG_CUDA(cudaMemcpy(idx, m->idx, slots * 4, cudaMemcpyDeviceToHost));
    if (val && slots) CIEG_CUDA(cudaMemcpy(val, m->val, slots * (m->precision == 0 ? 4 : 8), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
