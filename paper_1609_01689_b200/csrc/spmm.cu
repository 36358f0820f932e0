// spmm.cu -- K1: fused symmetric SpMM  U = (L + L^T - diag L) X  from the
// stored lower triangle, replacing ci::spmm (proj/src/csb.cpp:118-193).
//
// Design:
//   * owner-computes: output panel P is reduced by exactly one CTA, walking
//     P's work list -- row parts of tiles (P, J), transposed parts of tiles
//     (I, P), the symmetric diagonal tile -- in a fixed order, and written
//     once: no atomics, no zero-fill, bitwise deterministic run to run. Every
//     off-diagonal tile is therefore streamed twice (once per owner); at
//     m >= 8 the kernel is FP64-bound, so the extra bytes hide under the math.
//   * persistent, warp-specialised CTA (one per SM): 4 producer warps clear a
//     dense shared-memory tile, scatter the next work item's packed
//     (row | col << 16, value) entries into it -- transposed on the fly for
//     transposed parts, mirrored for the diagonal tile, so the consumer loop
//     is uniform -- and stage the partner panel's X slab; 4 consumer warps run
//     the panel product on the FP64 tensor pipe (DMMA m8n8k4) out of the other
//     buffer. The two stages hand buffers over with named barriers
//     (FULL/EMPTY per buffer), so scatter latency hides behind the DMMAs.
//   * fp32 values are promoted to fp64 exactly on fragment load (F2F runs on
//     its own unit, measured not to slow DMMA); products and sums are fp64,
//     the reference's precision contract (csb.hpp:79-82).
//   * padding makes fragment loads conflict-free: tile row stride TD+4 words
//     (bank 4g+q), X slab row stride 8*NT+4 doubles.
#include <algorithm>
#include <cstdint>

#include "context.hpp"
#include "device_common.cuh"

namespace cieg {
namespace {

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
  std::uint32_t ldx, ldy, mcols, npanels;
};

constexpr int kProducerWarps = 4;
constexpr int kConsumerWarps = 4;
constexpr int kThreads = 32 * (kProducerWarps + kConsumerWarps);
constexpr int kProducerThreads = 32 * kProducerWarps;
// named barrier ids (0 is __syncthreads)
constexpr int kBarFull0 = 1, kBarEmpty0 = 3, kBarProducers = 5;

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <typename V, int TD, int NT>
struct Shape {
  static constexpr int kSA = TD + 4;              // words (f32) or doubles (f64); S = 4 mod 16
  static constexpr int kSX = 8 * NT + 4;          // doubles
  static constexpr int kMT = TD / 8 / kConsumerWarps;  // m-tiles per consumer warp
  static constexpr std::size_t kTileBytes = sizeof(V) * TD * kSA;
  static constexpr std::size_t kSlabBytes = sizeof(double) * TD * kSX;
  static constexpr std::size_t kSmem = 2 * (kTileBytes + kSlabBytes);
};

constexpr int kQuads = 4;  // entry quads per producer thread per batch

template <typename V>
struct Quad;
template <>
struct Quad<float> {
  uint4 id;
  float4 v;
};
template <>
struct Quad<double> {
  uint4 id;
  double2 v0, v1;
};

struct Item {
  std::uint32_t kind, o0;
  int orow;
  std::uint64_t q0, q1;  // entry quads [q0, q1)
};

__device__ __forceinline__ void fetch_item(const SpmmArgs& a, std::uint32_t w, Item& it) {
  const std::uint32_t tile = __ldg(a.work_tile + w);
  const std::uint32_t other = __ldg(a.work_other + w);
  it.kind = __ldg(a.work_kind + w);
  it.o0 = __ldg(a.panel_start + other);
  it.orow = static_cast<int>(__ldg(a.panel_start + other + 1) - it.o0);
  it.q0 = __ldg(a.tile_off + tile) >> 2;
  it.q1 = __ldg(a.tile_off + tile + 1) >> 2;
}

__device__ __forceinline__ void load_quad(const SpmmArgs& a, const float* val, std::uint64_t q, Quad<float>& o) {
  o.id = __ldg(reinterpret_cast<const uint4*>(a.idx) + q);
  o.v = __ldg(reinterpret_cast<const float4*>(val) + q);
}
__device__ __forceinline__ void load_quad(const SpmmArgs& a, const double* val, std::uint64_t q, Quad<double>& o) {
  o.id = __ldg(reinterpret_cast<const uint4*>(a.idx) + q);
  o.v0 = __ldg(reinterpret_cast<const double2*>(val) + 2 * q);
  o.v1 = __ldg(reinterpret_cast<const double2*>(val) + 2 * q + 1);
}

template <typename V>
__device__ __forceinline__ void load_batch(const SpmmArgs& a, const V* val, const Item& it, std::uint64_t qb, int pt,
                                           Quad<V> (&out)[kQuads]) {
#pragma unroll
  for (int j = 0; j < kQuads; ++j) {
    const std::uint64_t q = qb + pt + j * kProducerThreads;
    if (q < it.q1)
      load_quad(a, val, q, out[j]);
    else
      out[j].id = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  }
}

template <int TD, int NT, int kPer>
__device__ __forceinline__ void load_slab(const SpmmArgs& a, const Item& it, int pt, double (&xv)[kPer]) {
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = pt + j * kProducerThreads;
    const int k = e / (8 * NT), t = e - k * (8 * NT);
    xv[j] = (k < it.orow && t < static_cast<int>(a.mcols)) ? __ldg(a.x + static_cast<std::size_t>(it.o0 + k) * a.ldx + t)
                                                            : 0.0;
  }
}

template <typename V, int SA>
__device__ __forceinline__ void put(V* A, std::uint32_t kind, std::uint32_t id, V v) {
  if (id == 0xffffffffu) return;
  const std::uint32_t r = id & 0xffffu, c = id >> 16;
  if (kind == 1u) {
    A[c * SA + r] = v;
  } else {
    A[r * SA + c] = v;
    if (kind == 2u) A[c * SA + r] = v;
  }
}

template <typename V, int SA>
__device__ __forceinline__ void scatter(V* A, std::uint32_t kind, const Quad<float> (&b)[kQuads]) {
#pragma unroll
  for (int j = 0; j < kQuads; ++j) {
    put<float, SA>(A, kind, b[j].id.x, b[j].v.x);
    put<float, SA>(A, kind, b[j].id.y, b[j].v.y);
    put<float, SA>(A, kind, b[j].id.z, b[j].v.z);
    put<float, SA>(A, kind, b[j].id.w, b[j].v.w);
  }
}
template <typename V, int SA>
__device__ __forceinline__ void scatter(V* A, std::uint32_t kind, const Quad<double> (&b)[kQuads]) {
#pragma unroll
  for (int j = 0; j < kQuads; ++j) {
    put<double, SA>(A, kind, b[j].id.x, b[j].v0.x);
    put<double, SA>(A, kind, b[j].id.y, b[j].v0.y);
    put<double, SA>(A, kind, b[j].id.z, b[j].v1.x);
    put<double, SA>(A, kind, b[j].id.w, b[j].v1.y);
  }
}

template <typename V, int TD, int NT>
__global__ void __launch_bounds__(kThreads, 1) spmm_ws_kernel(const SpmmArgs a) {
  using S = Shape<V, TD, NT>;
  extern __shared__ __align__(16) unsigned char smem[];
  auto tile_buf = [&](int b) { return reinterpret_cast<V*>(smem + b * S::kTileBytes); };
  auto slab_buf = [&](int b) { return reinterpret_cast<double*>(smem + 2 * S::kTileBytes + b * S::kSlabBytes); };
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const V* val = static_cast<const V*>(a.val);

  // Total work items of this CTA (to balance the EMPTY barrier arrivals).
  std::uint32_t total = 0;
  for (std::uint32_t P = blockIdx.x; P < a.npanels; P += gridDim.x) total += a.work_off[P + 1] - a.work_off[P];

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producer
    // Software-pipelined: the next batch of entry quads (or the first batch
    // of the next work item plus its X slab) is in flight while the current
    // batch is scattered.
    const int pt = tid;  // 0 .. 127
    constexpr int kSlabElems = TD * 8 * NT;
    constexpr int kPer = kSlabElems / kProducerThreads;
    std::uint32_t P = blockIdx.x;
    if (P >= a.npanels) return;
    std::uint32_t w = a.work_off[P];
    while (w >= a.work_off[P + 1]) {
      P += gridDim.x;
      if (P >= a.npanels) return;
      w = a.work_off[P];
    }
    auto advance = [&]() -> bool {
      ++w;
      while (w >= a.work_off[P + 1]) {
        P += gridDim.x;
        if (P >= a.npanels) return false;
        w = a.work_off[P];
      }
      return true;
    };
    Item it, nit;
    fetch_item(a, w, it);
    Quad<V> cur[kQuads], nxt[kQuads];
    load_batch(a, val, it, it.q0, pt, cur);
    double xv[kPer];
    load_slab<TD, NT, kPer>(a, it, pt, xv);
    int buf = 0;
    for (;;) {
      bar_sync(kBarEmpty0 + buf, kThreads);
      V* A = tile_buf(buf);
      {
        float4* p4 = reinterpret_cast<float4*>(A);
        constexpr int n4 = static_cast<int>(S::kTileBytes / 16);
#pragma unroll 4
        for (int i = pt; i < n4; i += kProducerThreads) p4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      double* X = slab_buf(buf);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int e = pt + j * kProducerThreads;
        const int k = e / (8 * NT), t = e - k * (8 * NT);
        X[k * S::kSX + t] = xv[j];
      }
      bar_sync(kBarProducers, kProducerThreads);  // clear before scatter
      bool next_exists = false;
      for (std::uint64_t qb = it.q0;; qb += kQuads * kProducerThreads) {
        const std::uint64_t qn = qb + kQuads * kProducerThreads;
        const bool more = qn < it.q1;
        if (more) {
          load_batch(a, val, it, qn, pt, nxt);
        } else {
          next_exists = advance();
          if (next_exists) {
            fetch_item(a, w, nit);
            load_batch(a, val, nit, nit.q0, pt, nxt);
          }
        }
        scatter<V, S::kSA>(A, it.kind, cur);
#pragma unroll
        for (int j = 0; j < kQuads; ++j) cur[j] = nxt[j];
        if (!more) break;
      }
      bar_arrive(kBarFull0 + buf, kThreads);
      buf ^= 1;
      if (!next_exists) break;
      it = nit;
      load_slab<TD, NT, kPer>(a, it, pt, xv);
    }
  } else {
    // ------------------------------------------------------------ consumer
    const int cw = warp - kProducerWarps;
    const int g = lane >> 2, q = lane & 3;
    const int m_base = cw * 8 * S::kMT;
    bar_arrive(kBarEmpty0 + 0, kThreads);
    bar_arrive(kBarEmpty0 + 1, kThreads);
    int buf = 0;
    std::uint32_t done = 0;
    for (std::uint32_t P = blockIdx.x; P < a.npanels; P += gridDim.x) {
      const std::uint32_t r0 = __ldg(a.panel_start + P);
      const int prow = static_cast<int>(__ldg(a.panel_start + P + 1) - r0);
      double acc[S::kMT][NT][2];
#pragma unroll
      for (int j = 0; j < S::kMT; ++j)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
      const bool live = m_base < prow;
      for (std::uint32_t w = a.work_off[P]; w < a.work_off[P + 1]; ++w) {
        const std::uint32_t other = __ldg(a.work_other + w);
        const int orow = static_cast<int>(__ldg(a.panel_start + other + 1) - __ldg(a.panel_start + other));
        bar_sync(kBarFull0 + buf, kThreads);
        if (live) {
          const V* A = tile_buf(buf) + (m_base + g) * S::kSA + q;
          const double* xb = slab_buf(buf) + q * S::kSX + g;
          const int ksteps = (orow + 3) >> 2;
#pragma unroll 2
          for (int ks = 0; ks < ksteps; ++ks) {
            double af[S::kMT];
#pragma unroll
            for (int j = 0; j < S::kMT; ++j) af[j] = static_cast<double>(A[j * 8 * S::kSA + 4 * ks]);
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const double b = xb[4 * ks * S::kSX + 8 * n];
#pragma unroll
              for (int j = 0; j < S::kMT; ++j) dmma_8x8x4(acc[j][n][0], acc[j][n][1], af[j], b);
            }
          }
        }
        ++done;
        if (done + 2 <= total) bar_arrive(kBarEmpty0 + buf, kThreads);
        buf ^= 1;
      }
      if (live) {
#pragma unroll
        for (int j = 0; j < S::kMT; ++j) {
          const int row = m_base + 8 * j + g;
          if (row >= prow) continue;
          double* yr = a.y + static_cast<std::size_t>(r0 + row) * a.ldy;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int c = 8 * n + 2 * q;
            if (c + 1 < static_cast<int>(a.mcols)) {
              yr[c] = acc[j][n][0];
              yr[c + 1] = acc[j][n][1];
            } else if (c < static_cast<int>(a.mcols)) {
              yr[c] = acc[j][n][0];
            }
          }
        }
      }
    }
  }
}

template <typename V, int TD, int NT>
void launch_variant(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args) {
  using S = Shape<V, TD, NT>;
  auto kern = spmm_ws_kernel<V, TD, NT>;
  CIEG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::kSmem)));
  int per_sm = 0;
  CIEG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, S::kSmem));
  per_sm = std::max(1, per_sm);
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(m->npanels, static_cast<std::uint64_t>(per_sm) * ctx->sm_count));
  kern<<<grid, kThreads, S::kSmem, ctx->stream>>>(args);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

template <typename V, int TD>
void dispatch_nt(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args, std::uint32_t mc) {
  if (mc <= 8)
    launch_variant<V, TD, 1>(ctx, m, args);
  else
    launch_variant<V, TD, 2>(ctx, m, args);
}

}  // namespace

void launch_spmm(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                 std::uint32_t ldy, std::uint32_t mcols) {
  if (mcols == 0 || m->dim == 0) return;
  for (std::uint32_t c0 = 0; c0 < mcols; c0 += 16) {
    const std::uint32_t mc = std::min<std::uint32_t>(16, mcols - c0);
    SpmmArgs args{m->panel_start, m->work_off, m->work_tile, m->work_other, m->work_kind,
                  m->tile_off,    m->idx,      m->val,       x + c0,        y + c0,
                  ldx,            ldy,         mc,           m->npanels};
    if (m->precision == 0) {
      if (m->tile_edge == 64)
        dispatch_nt<float, 64>(ctx, m, args, mc);
      else
        dispatch_nt<float, 128>(ctx, m, args, mc);
    } else {  // fp64 values: 64-row tiles (a 128-row fp64 tile pair exceeds shared memory)
      dispatch_nt<double, 64>(ctx, m, args, mc);
    }
  }
}

}  // namespace cieg
