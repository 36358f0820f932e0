// reorder.cu -- bank-aware ordering of the entries inside every tile.
//
// The SpMM producer warps (spmm.cu) place a tile's entries into the dense
// shared-memory tile with one 32-bit (fp32) or 64-bit (fp64) store per entry:
// the entries of a 128-entry block (32 quads from the tile start) go out as
// four warp-wide stores, store x taking entry 4l + x from lane l. Row-major
// entry order makes those stores conflict heavily, above all in the
// transposed orientation (all entries of a row share a bank there). The
// order of entries inside a tile is free, so at upload every tile is
// re-ordered once:
//   1. first-fit edge colouring of the bipartite multigraph (own-row bank,
//      transposed bank) in row-major entry order: every colour is a set of
//      entries that is bank-conflict-free in BOTH orientations (capacity 32
//      banks for fp32; 16 for fp64, whose 64-bit stores go out in half-warps);
//   2. colours are laid out by size (largest first, then colour index) and
//      the resulting sequence is dealt to the lane/store positions.
// Fully deterministic (the colouring is sequential per tile), so a host
// upload and the GPU generator produce the same tile stream. A permutation
// within each tile: tile_off, the schedule and the packed offsets are
// unchanged. One warp per tile.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cieg_internal.hpp"
#include "context.hpp"

namespace cieg {
namespace {

constexpr int kWarps = 4;            // tiles per CTA
constexpr int kMaxColors = 1024;     // > 2 * max bank degree of a 128 x 128 tile's colouring
constexpr int kWarpSmem = kMaxColors * (4 + 4 + 2 + 2);

struct ReorderArgs {
  const std::uint64_t* tile_off;
  std::uint64_t t0, t1;   // tiles of this chunk
  std::uint64_t e_base;   // first entry slot of the chunk
  const std::uint32_t* idx;
  const void* val;
  std::uint32_t* out_idx;  // chunk-local
  void* out_val;
  std::uint32_t* scratch;  // chunk-local: colour | rank << 16 per entry
  int nbanks;              // 32 (fp32) or 16 (fp64)
  int vbytes;
};

__device__ __forceinline__ std::uint64_t slot_of(std::uint64_t j, std::uint64_t n) {
  const std::uint64_t b = j >> 7, jj = j & 127;
  const std::uint64_t lanes = std::min<std::uint64_t>(32, (n - 128 * b) >> 2);
  return 128 * b + 4 * (jj % lanes) + jj / lanes;
}

__global__ void __launch_bounds__(32 * kWarps) reorder_kernel(const ReorderArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint64_t t = a.t0 + static_cast<std::uint64_t>(blockIdx.x) * kWarps + warp;
  if (t >= a.t1) return;
  unsigned char* base = smem + static_cast<std::size_t>(warp) * kWarpSmem;
  std::uint32_t* ulo = reinterpret_cast<std::uint32_t*>(base);
  std::uint32_t* uhi = ulo + kMaxColors;
  std::uint16_t* start = reinterpret_cast<std::uint16_t*>(uhi + kMaxColors);
  std::uint16_t* csize = start + kMaxColors;
  for (int k = lane; k < kMaxColors; k += 32) {
    ulo[k] = 0;
    uhi[k] = 0;
    csize[k] = 0;
  }
  __syncwarp();
  const std::uint64_t e0 = a.tile_off[t], e1 = a.tile_off[t + 1];
  const std::uint64_t n = e1 - e0;
  const std::uint32_t cap = static_cast<std::uint32_t>(a.nbanks);
  const std::uint32_t bmask = cap - 1;
  int ncol = 0, first_open = 0;
  // 1. first-fit colouring in entry order
  for (std::uint64_t c0 = 0; c0 < n; c0 += 32) {
    const std::uint64_t e = c0 + lane;
    const std::uint32_t mine = e < n ? a.idx[e0 + e] : 0u;
    std::uint32_t res = 0;
    const int cnt = static_cast<int>(std::min<std::uint64_t>(32, n - c0));
    for (int s = 0; s < cnt; ++s) {
      const std::uint32_t id = __shfl_sync(0xffffffffu, mine, s);
      const std::uint32_t bl = (id & 0xffffu) & bmask, bh = (id >> 16) & bmask;
      int k = -1;
      for (int cb = first_open & ~31; cb < ncol; cb += 32) {
        const int kk = cb + lane;
        const bool fr = kk < ncol && !((ulo[kk] >> bl) & 1u) && !((uhi[kk] >> bh) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, fr);
        if (bal) {
          k = cb + __ffs(bal) - 1;
          break;
        }
      }
      if (k < 0) k = ncol < kMaxColors ? ncol++ : kMaxColors - 1;  // last colour: overflow bin
      std::uint32_t r = 0;
      if (lane == 0) {
        ulo[k] |= 1u << bl;
        uhi[k] |= 1u << bh;
        r = csize[k];
        csize[k] = static_cast<std::uint16_t>(r + 1);
      }
      r = __shfl_sync(0xffffffffu, r, 0);
      __syncwarp();
      if (lane == 0)
        while (first_open < ncol && csize[first_open] >= cap) ++first_open;
      first_open = __shfl_sync(0xffffffffu, first_open, 0);
      if (lane == s) res = static_cast<std::uint32_t>(k) | (r << 16);
    }
    if (e < n) a.scratch[e0 - a.e_base + e] = res;
  }
  __syncwarp();
  // 2. colour starts: by size descending, then colour index
  std::uint32_t off = 0;
  for (int sz = static_cast<int>(cap); sz >= 1; --sz) {
    for (int cb = 0; cb < ncol; cb += 32) {
      const int k = cb + lane;
      const bool p = k < ncol && (sz == static_cast<int>(cap) ? csize[k] >= cap : csize[k] == sz);
      const unsigned bal = __ballot_sync(0xffffffffu, p);
      if (p) {
        const std::uint32_t before = __popc(bal & ((1u << lane) - 1u));
        start[k] = static_cast<std::uint16_t>(off + before * sz);
      }
      // the overflow colour can exceed cap: it is laid out last-in-class with its true size
      std::uint32_t add = 0;
      if (p) add = (sz == static_cast<int>(cap)) ? csize[k] : static_cast<std::uint32_t>(sz);
      for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
      off += add;
    }
  }
  __syncwarp();
  // 3. permute (out of place, chunk-local)
  for (std::uint64_t e = lane; e < n; e += 32) {
    const std::uint32_t w = a.scratch[e0 - a.e_base + e];
    const std::uint64_t j = start[w & 0xffffu] + (w >> 16);
    const std::uint64_t dst = e0 - a.e_base + slot_of(j, n);
    a.out_idx[dst] = a.idx[e0 + e];
    if (a.vbytes == 4)
      static_cast<float*>(a.out_val)[dst] = static_cast<const float*>(a.val)[e0 + e];
    else
      static_cast<double*>(a.out_val)[dst] = static_cast<const double*>(a.val)[e0 + e];
  }
}

}  // namespace

void order_tile_entries(cieg_ctx* ctx, cieg_mat* m) {
  if (m->ntiles == 0) return;
  const std::vector<std::uint64_t>& to = m->tile_off_host;
  const std::uint64_t slots = to.back();
  const int vb = m->precision == 0 ? 4 : 8;
  const std::uint64_t chunk = std::min<std::uint64_t>(slots, 1ull << 26);
  std::uint32_t* out_idx = nullptr;
  void* out_val = nullptr;
  std::uint32_t* scratch = nullptr;
  CIEG_CUDA(cudaMalloc(&out_idx, chunk * 4));
  CIEG_CUDA(cudaMalloc(&out_val, chunk * vb));
  CIEG_CUDA(cudaMalloc(&scratch, chunk * 4));
  const int smem = kWarps * kWarpSmem;
  CIEG_CUDA(cudaFuncSetAttribute(reorder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  try {
    for (std::uint64_t t0 = 0; t0 < m->ntiles;) {
      std::uint64_t t1 = t0;
      while (t1 < m->ntiles && to[t1 + 1] - to[t0] <= chunk) ++t1;
      if (t1 == t0) fail(CIEG_ERR_CONFIG, "tile larger than the reorder chunk");
      ReorderArgs args{m->tile_off, t0, t1, to[t0], m->idx, m->val, out_idx, out_val, scratch,
                       m->precision == 0 ? 32 : 16, vb};
      const unsigned grid = static_cast<unsigned>((t1 - t0 + kWarps - 1) / kWarps);
      reorder_kernel<<<grid, 32 * kWarps, smem, ctx->stream>>>(args);
      CIEG_CUDA(cudaGetLastError());
      ++ctx->launches;
      const std::uint64_t ne = to[t1] - to[t0];
      CIEG_CUDA(cudaMemcpyAsync(m->idx + to[t0], out_idx, ne * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      CIEG_CUDA(cudaMemcpyAsync(static_cast<char*>(m->val) + to[t0] * vb, out_val, ne * vb,
                                cudaMemcpyDeviceToDevice, ctx->stream));
      t0 = t1;
    }
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFree(out_idx);
    cudaFree(out_val);
    cudaFree(scratch);
    throw;
  }
  cudaFree(out_idx);
  cudaFree(out_val);
  cudaFree(scratch);
}

}  // namespace cieg
