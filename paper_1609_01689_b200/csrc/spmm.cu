// spmm.cu -- K1: fused symmetric SpMM  U = (L + L^T - diag L) X  from the
// stored lower triangle, replacing ci::spmm (proj/src/csb.cpp:118-193).
//
// Design:
//   * owner-computes: CTA P owns output panel P and walks its work list (row
//     parts of tiles (P, J), transposed parts of tiles (I, P), the symmetric
//     diagonal tile). Each Y row is reduced by exactly one CTA in a fixed
//     order and written once: no atomics, no zero-fill, bitwise
//     deterministic. The price is that every off-diagonal tile is streamed
//     twice (once per owner); at m >= 8 the kernel is FP64-bound, so the extra
//     bytes hide under the math.
//   * each tile's packed (row | col << 16, value) list is scattered into a
//     dense shared-memory tile (transposed on the fly for transposed parts, so
//     the inner loop is uniform), the partner panel's X slab is staged in
//     shared memory, and the panel product runs on the FP64 tensor pipe
//     (DMMA m8n8k4). fp32 values are promoted to fp64 exactly on load, the
//     products and sums are fp64 (the reference's precision contract,
//     csb.hpp:79-82).
//   * padding is chosen for conflict-free fragment loads: A row stride
//     TD+4 words (4i+j bank pattern), X slab row stride 8*NT+4 doubles.
#include <algorithm>
#include <cstdint>

#include "context.hpp"
#include "device_common.cuh"

namespace cieg {
namespace {

template <typename V>
struct ValTraits;
template <>
struct ValTraits<float> {
  static constexpr int kPad = 4;  // words
};
template <>
struct ValTraits<double> {
  static constexpr int kPad = 4;  // doubles (S = TD + 4 = 4 mod 16)
};

struct SpmmArgs {
  const std::uint32_t* panel_start;
  const std::uint32_t* work_off;
  const std::uint32_t* work_tile;
  const std::uint32_t* work_other;
  const std::uint32_t* work_kind;
  const std::uint64_t* tile_off;
  const std::uint32_t* idx;
  const void* val;
  const double* x;
  double* y;
  std::uint32_t ldx, ldy, mcols;
};

template <typename V, int TD, int NT>
struct SpmmShape {
  static constexpr int kThreads = TD * 2;  // TD/16 warps, 2 m-tiles each
  static constexpr int kSA = TD + ValTraits<V>::kPad;
  static constexpr int kSX = 8 * NT + 4;
  static constexpr std::size_t kTileBytes = sizeof(V) * TD * kSA;
  static constexpr std::size_t kSlabBytes = sizeof(double) * TD * kSX;
  static constexpr std::size_t kSmem = kTileBytes + kSlabBytes;
};

template <typename V, int TD, int NT>
__global__ void __launch_bounds__(TD * 2) spmm_owner_kernel(SpmmArgs a) {
  using S = SpmmShape<V, TD, NT>;
  extern __shared__ __align__(16) unsigned char smem[];
  V* As = reinterpret_cast<V*>(smem);
  double* xs = reinterpret_cast<double*>(smem + S::kTileBytes);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const std::uint32_t P = blockIdx.x;
  const std::uint32_t r0 = a.panel_start[P];
  const std::uint32_t prow = a.panel_start[P + 1] - r0;
  const V* val = static_cast<const V*>(a.val);

  // clear the dense tile once (16-byte stores)
  {
    float4* p = reinterpret_cast<float4*>(As);
    const int n4 = static_cast<int>(S::kTileBytes / 16);
    for (int i = tid; i < n4; i += S::kThreads) p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }

  double acc[2][NT][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;

  const int m_base = warp * 16;
  const bool warp_live = m_base < static_cast<int>(prow);
  const std::uint32_t w0 = a.work_off[P], w1 = a.work_off[P + 1];
  __syncthreads();

  for (std::uint32_t w = w0; w < w1; ++w) {
    const std::uint32_t tile = a.work_tile[w];
    const std::uint32_t other = a.work_other[w];
    const std::uint32_t kind = a.work_kind[w];
    const std::uint32_t o0 = a.panel_start[other];
    const int orow = static_cast<int>(a.panel_start[other + 1] - o0);

    // X slab of the partner panel, zero padded to TD x 8NT.
    for (int e = tid; e < TD * 8 * NT; e += S::kThreads) {
      const int k = e / (8 * NT), t = e - k * (8 * NT);
      double v = 0.0;
      if (k < orow && t < static_cast<int>(a.mcols))
        v = __ldg(a.x + static_cast<std::size_t>(o0 + k) * a.ldx + t);
      xs[k * S::kSX + t] = v;
    }
    // scatter the tile's entries into the dense tile as [m][k]
    const std::uint64_t e0 = a.tile_off[tile], e1 = a.tile_off[tile + 1];
    for (std::uint64_t e = e0 + tid; e < e1; e += S::kThreads) {
      const std::uint32_t id = __ldg(a.idx + e);
      const V v = val[e];
      const std::uint32_t r = id & 0xffffu, c = id >> 16;
      if (kind == 1u) {
        As[c * S::kSA + r] = v;
      } else {
        As[r * S::kSA + c] = v;
        if (kind == 2u) As[c * S::kSA + r] = v;
      }
    }
    __syncthreads();

    if (warp_live) {
      const int ksteps = (orow + 3) >> 2;
      const V* arow0 = As + (m_base + g) * S::kSA + q;
      const V* arow1 = arow0 + 8 * S::kSA;
      const double* xb = xs + q * S::kSX + g;
#pragma unroll 4
      for (int ks = 0; ks < ksteps; ++ks) {
        const double a0 = static_cast<double>(arow0[4 * ks]);
        const double a1 = static_cast<double>(arow1[4 * ks]);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double b = xb[4 * ks * S::kSX + 8 * n];
          dmma_8x8x4(acc[0][n][0], acc[0][n][1], a0, b);
          dmma_8x8x4(acc[1][n][0], acc[1][n][1], a1, b);
        }
      }
    }
    __syncthreads();
    // clear the entries just used
    for (std::uint64_t e = e0 + tid; e < e1; e += S::kThreads) {
      const std::uint32_t id = __ldg(a.idx + e);
      const std::uint32_t r = id & 0xffffu, c = id >> 16;
      if (kind == 1u) {
        As[c * S::kSA + r] = V(0);
      } else {
        As[r * S::kSA + c] = V(0);
        if (kind == 2u) As[c * S::kSA + r] = V(0);
      }
    }
    __syncthreads();
  }

  if (!warp_live) return;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int row = m_base + 8 * j + g;
    if (row >= static_cast<int>(prow)) continue;
    double* yr = a.y + static_cast<std::size_t>(r0 + row) * a.ldy;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = 8 * n + 2 * q;
      if (c < static_cast<int>(a.mcols)) yr[c] = acc[j][n][0];
      if (c + 1 < static_cast<int>(a.mcols)) yr[c + 1] = acc[j][n][1];
    }
  }
}

template <typename V, int TD, int NT>
void launch_variant(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args) {
  using S = SpmmShape<V, TD, NT>;
  auto kern = spmm_owner_kernel<V, TD, NT>;
  static bool configured = false;  // per-variant attribute (process-wide)
  if (!configured) {
    CIEG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(S::kSmem)));
    configured = true;
  }
  kern<<<m->npanels, S::kThreads, S::kSmem, ctx->stream>>>(args);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

template <typename V, int TD>
void dispatch_nt(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args, std::uint32_t mc) {
  if (mc <= 8)
    launch_variant<V, TD, 1>(ctx, m, args);
  else if (mc <= 16)
    launch_variant<V, TD, 2>(ctx, m, args);
  else if (mc <= 32)
    launch_variant<V, TD, 4>(ctx, m, args);
  else
    launch_variant<V, TD, 8>(ctx, m, args);
}

}  // namespace

void launch_spmm(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                 std::uint32_t ldy, std::uint32_t mcols) {
  if (mcols == 0 || m->dim == 0) return;
  for (std::uint32_t c0 = 0; c0 < mcols; c0 += 64) {
    const std::uint32_t mc = std::min<std::uint32_t>(64, mcols - c0);
    SpmmArgs args{m->panel_start, m->work_off, m->work_tile, m->work_other, m->work_kind,
                  m->tile_off,    m->idx,      m->val,       x + c0,        y + c0,
                  ldx,            ldy,         mc};
    if (m->precision == 0) {
      if (m->tile_edge == 64)
        dispatch_nt<float, 64>(ctx, m, args, mc);
      else
        dispatch_nt<float, 128>(ctx, m, args, mc);
    } else {
      if (m->tile_edge == 64)
        dispatch_nt<double, 64>(ctx, m, args, mc);
      else
        dispatch_nt<double, 128>(ctx, m, args, mc);
    }
  }
}

}  // namespace cieg
