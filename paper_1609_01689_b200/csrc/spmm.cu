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
//   * persistent, warp-specialised CTA (one per SM). 8 producer warps stream
//     the work items' packed entry lists with 128-bit loads into a register
//     double buffer (the next 4096-entry batch is in flight while the current
//     one is placed), clear a dense shared-memory tile and scatter the
//     entries into it with one store each -- the 32-bit index carries the
//     entry's offset in both orientations (row part / transposed part), the
//     diagonal tile is mirrored -- and stage the partner panel's X slab,
//     prefetched one item ahead in registers. 8 consumer warps run the panel
//     product on the FP64 tensor pipe (DMMA m8n8k4) out of the other tile
//     buffer. Producer and consumers hand the two buffers over with named
//     barriers (FULL/EMPTY per buffer).
//   * fp32 values are promoted to fp64 exactly on fragment load (F2F runs on
//     its own unit, measured not to slow DMMA); products and sums are fp64,
//     the reference's precision contract (csb.hpp:79-82).
//   * fragment loads are conflict-free and wide (tile_layout.h): fp32 tile
//     columns are interleaved in 16-column groups with row stride TD+16, so
//     one float4 per lane yields the A fragments of 4 k-steps (fp64: stride
//     TD+8, one double2 = 2 k-steps); the X slab stores the two n-tiles'
//     columns side by side, so one double2 yields both B fragments of a
//     k-step. The consumer double-buffers fragments across groups of 4
//     k-steps so loads and conversions overlap the previous group's DMMAs.
//   * scatter stores are (nearly) bank-conflict-free: reorder.cu orders every
//     tile's entries at upload so each warp-wide store hits distinct banks in
//     both orientations; only the TD data columns of a tile are zeroed.
//   * the next item's entry stream is bulk-prefetched into L2
//     (cp.async.bulk.prefetch.L2) a whole item ahead of the register batches.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cstdint>

#include "context.hpp"
#include "device_common.cuh"
#include "tile_layout.h"

namespace cieg {
namespace {

struct SpmmArgs {
  const std::uint32_t* panel_start;
  const std::uint32_t* work_off;
  const std::uint32_t* work_tile;
  const std::uint32_t* work_other;
  const std::uint32_t* work_kind;
  const std::uint32_t* sched_off;
  const uint4* sched;  // 2 x uint4 per item
  const std::uint64_t* tile_off;
  const std::uint32_t* idx;
  const void* val;
  const double* x;
  double* y;
  std::uint32_t ldx, ldy, mcols, npanels;
  std::uint32_t row_base;  // first owner row of a shard (U is written shard-local)
  unsigned* nonfinite;     // = launch_id when an X value is Inf/NaN (staged as 0; fixed up after the launch)
  unsigned launch_id;      // per-launch tag: no reset of the flag between launches
  double* partial;         // single pass: Aᵀ X_pi of item i at partial + i * TD * mcols (row-major, ld mcols)
};

constexpr int kProducerWarps = 8;
constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (kProducerWarps + kConsumerWarps);
constexpr int kProducerThreads = 32 * kProducerWarps;
constexpr int kGroupWarps = kProducerWarps / 2;        // two producer groups (alternating items)
constexpr int kGroupThreads = 32 * kGroupWarps;
constexpr int kConsumerThreads = 32 * kConsumerWarps;
constexpr int kQuads = 4;                                  // entry quads per producer thread per batch
constexpr int kChunkQuads = kQuads * kProducerThreads;     // 1024 quads = 4096 entries per batch
constexpr int kGroupChunkQuads = kQuads * kGroupThreads;  // per producer group
// named barrier ids (0 is __syncthreads)
constexpr int kBarProducers = 5, kBarProducers0 = 5;  // producer groups: 5, 6
constexpr int kBarConsumers = 7;  // single pass: the consumers' owner-slab refresh

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Tile-buffer hand-off over shared-memory mbarriers: FULL[b] completes when
// every thread of the filling producer group has arrived (release: its
// shared stores are visible to the waiters), EMPTY[b] when every consumer
// warp has released the buffer. Each consumer warp waits on FULL on its own
// -- no barrier makes the consumer warps meet at every item, so one warp's
// DMMAs keep the pipe busy while another crosses the item boundary.
// Fill u of a buffer waits for EMPTY parity (u & 1) ^ 1 (fill 0 passes at
// once) and is consumed at FULL parity u & 1.
__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
  const std::uint32_t addr = smem_addr(b);
  std::uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}
// consumer warp: release a tile buffer (after the warp's last read of it)
__device__ __forceinline__ void release_buffer(std::uint64_t* empty, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
}
template <typename V, int TD, int NT>
struct Shape {
  static constexpr int kSA = sizeof(V) == 4 ? TD + 16 : TD + 8;  // row stride (elements), tile_layout.h
  static constexpr int kSX = 8 * NT + 4;                // doubles
  static constexpr int kMT = TD / 8 / kConsumerWarps;   // m-tiles per consumer warp
  static constexpr std::size_t kTileBytes = ((sizeof(V) * TD * kSA + 15) / 16) * 16;
  static constexpr std::size_t kSlabBytes = sizeof(double) * TD * kSX;
  static constexpr std::size_t kSmem = 2 * (kTileBytes + kSlabBytes);
  static constexpr std::size_t kSmemSP = kSmem + kSlabBytes;  // + the owner panel's X slab
  static constexpr int kSlabPer = TD * 8 * NT / kProducerThreads;  // slab doubles per producer thread
  static constexpr int kSlabPerG = TD * 8 * NT / kGroupThreads;    // ... per producer-group thread
};

struct Item {
  std::uint64_t q0, q1;  // entry quads [q0, q1)
  std::uint32_t flags;   // kind | first << 8 | last << 9 | owner rows << 16
  std::uint32_t o0;      // partner panel start row
  int orow;              // partner panel rows
  std::uint32_t r0;      // owner panel start row
  __device__ __forceinline__ std::uint32_t kind() const { return flags & 0xffu; }
  __device__ __forceinline__ bool first() const { return (flags >> 8) & 1u; }
  __device__ __forceinline__ bool last() const { return (flags >> 9) & 1u; }
  __device__ __forceinline__ int prow() const { return static_cast<int>(flags >> 16); }
};

__device__ __forceinline__ Item load_item(const SpmmArgs& a, std::uint32_t i) {
  const uint4 u = __ldg(a.sched + 2 * static_cast<std::size_t>(i));
  const uint4 v = __ldg(a.sched + 2 * static_cast<std::size_t>(i) + 1);
  Item it;
  it.q0 = (static_cast<std::uint64_t>(u.y) << 32) | u.x;
  it.q1 = (static_cast<std::uint64_t>(u.w) << 32) | u.z;
  it.flags = v.x;
  it.o0 = v.y;
  it.orow = static_cast<int>(v.z);
  it.r0 = v.w;
  return it;
}

template <typename V, int TD, int NT>
__device__ __forceinline__ void load_slab(const SpmmArgs& a, const Item& it, int pt,
                                          double (&xv)[Shape<V, TD, NT>::kSlabPer]) {
#pragma unroll
  for (int j = 0; j < Shape<V, TD, NT>::kSlabPer; ++j) {
    const int e = pt + j * kProducerThreads;
    const int k = e / (8 * NT), t = e - k * (8 * NT);
    xv[j] = (k < it.orow && t < static_cast<int>(a.mcols)) ? __ldg(a.x + static_cast<std::size_t>(it.o0 + k) * a.ldx + t)
                                                            : 0.0;
  }
}

// Bulk L2 prefetch of a byte range (no registers, no shared memory): keeps
// the DRAM stream of the items ahead in flight while the producer warps'
// register batches only see L2 latency.
__device__ __forceinline__ void prefetch_l2(const void* p, std::uint64_t bytes) {
  const std::uint64_t a0 = reinterpret_cast<std::uint64_t>(p) & ~15ull;
  const std::uint64_t a1 = (reinterpret_cast<std::uint64_t>(p) + bytes + 15) & ~15ull;
  for (std::uint64_t a = a0; a < a1; a += (1u << 20)) {
    const std::uint32_t n = static_cast<std::uint32_t>(a1 - a < (1u << 20) ? a1 - a : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
  }
}

template <typename V>
__device__ __forceinline__ void prefetch_item(const SpmmArgs& a, const Item& it) {
  const std::uint64_t nq = it.q1 - it.q0;
  if (nq) {
    prefetch_l2(a.idx + 4 * it.q0, 16 * nq);
    prefetch_l2(static_cast<const V*>(a.val) + 4 * it.q0, 4 * sizeof(V) * nq);
  }
  if (it.orow) prefetch_l2(a.x + static_cast<std::size_t>(it.o0) * a.ldx, sizeof(double) * it.orow * a.ldx);
}

template <typename V, int TD, int NT>
__device__ __forceinline__ void load_slab_g(const SpmmArgs& a, const Item& it, int pt,
                                            double (&xv)[Shape<V, TD, NT>::kSlabPerG]) {
#pragma unroll
  for (int j = 0; j < Shape<V, TD, NT>::kSlabPerG; ++j) {
    const int e = pt + j * kGroupThreads;
    const int k = e / (8 * NT), t = e - k * (8 * NT);
    xv[j] = (k < it.orow && t < static_cast<int>(a.mcols)) ? __ldg(a.x + static_cast<std::size_t>(it.o0 + k) * a.ldx + t)
                                                            : 0.0;
  }
}

template <int KIND, typename V>
__device__ __forceinline__ void put(V* A, std::uint32_t id, V v) {
  if (KIND == 1) {
    A[id >> 16] = v;
  } else {
    A[id & 0xffffu] = v;
    if (KIND == 2) A[id >> 16] = v;
  }
}

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
constexpr std::uint32_t kNoQuad = 0xffffffffu;  // marks an empty batch slot (never a real index)

__device__ __forceinline__ void load_quad(const SpmmArgs& a, const float* val, std::uint64_t q, Quad<float>& o) {
  o.id = __ldg(reinterpret_cast<const uint4*>(a.idx) + q);
  o.v = __ldg(reinterpret_cast<const float4*>(val) + q);
}
__device__ __forceinline__ void load_quad(const SpmmArgs& a, const double* val, std::uint64_t q, Quad<double>& o) {
  o.id = __ldg(reinterpret_cast<const uint4*>(a.idx) + q);
  o.v0 = __ldg(reinterpret_cast<const double2*>(val) + 2 * q);
  o.v1 = __ldg(reinterpret_cast<const double2*>(val) + 2 * q + 1);
}

template <int KIND>
__device__ __forceinline__ void put4(float* A, const Quad<float>& b) {
  put<KIND>(A, b.id.x, b.v.x);
  put<KIND>(A, b.id.y, b.v.y);
  put<KIND>(A, b.id.z, b.v.z);
  put<KIND>(A, b.id.w, b.v.w);
}
template <int KIND>
__device__ __forceinline__ void put4(double* A, const Quad<double>& b) {
  put<KIND>(A, b.id.x, b.v0.x);
  put<KIND>(A, b.id.y, b.v0.y);
  put<KIND>(A, b.id.z, b.v1.x);
  put<KIND>(A, b.id.w, b.v1.y);
}

// Single pass, consumer warp cw: the transposed product D = Aᵀ X_P of an
// off-diagonal item for tile columns [8 MT cw, 8 MT (cw + 1)) (D rows),
// k over the tile rows, from the shared tile read column-wise, and its store
// to the item's partial slot. fp32, 2 m-tiles: lane g takes columns
// c0 = 16 cw + (g & 3) + 8 (g >> 2) and c0 + 4, adjacent in the permuted
// row (tile_layout.h), so one float2 carries both m-tiles' A fragments.
template <typename V, int TD, int NT>
__device__ __forceinline__ void transposed_product(const SpmmArgs& a, const V* T, const double* oslab, std::uint32_t i,
                                                   const Item& it, int cw, int lane) {
  using S = Shape<V, TD, NT>;
  constexpr int MT = S::kMT;
  constexpr bool kPair = sizeof(V) == 4 && MT == 2;
  const int g = lane >> 2, q = lane & 3;
  const int prec = sizeof(V) == 4 ? 0 : 1;
  int col[MT], pos[MT];
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    col[j] = kPair ? 16 * cw + (g & 3) + 8 * (g >> 2) + 4 * j : 8 * MT * cw + 8 * j + g;
    pos[j] = static_cast<int>(cieg_tl::perm(static_cast<std::uint32_t>(col[j]), prec));
  }
  double acc[MT][NT][2];
#pragma unroll
  for (int j = 0; j < MT; ++j)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
  const V* A = T + q * S::kSA;
  const double* xb = oslab + q * S::kSX + (NT == 2 ? 2 * g : g);
  // all TD/4 k-steps, fully unrolled (tile and slab rows >= prow are zero):
  // measured faster than a prow-bounded loop (cfg2 m = 8: 2.99 vs 3.13 ms)
#pragma unroll
  for (int s = 0; s < TD / 4; ++s) {
    double fa[MT], fb[NT];
    const V* Ar = A + 4 * s * S::kSA;
    if constexpr (kPair) {
      const float2 v2 = *reinterpret_cast<const float2*>(Ar + pos[0]);
      fa[0] = static_cast<double>(v2.x);
      fa[1] = static_cast<double>(v2.y);
    } else {
#pragma unroll
      for (int j = 0; j < MT; ++j) fa[j] = static_cast<double>(Ar[pos[j]]);
    }
    const double* xr = xb + 4 * s * S::kSX;
    if constexpr (NT == 2) {
      const double2 v2 = *reinterpret_cast<const double2*>(xr);
      fb[0] = v2.x;
      fb[1] = v2.y;
    } else {
      fb[0] = xr[0];
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < MT; ++j) dmma_8x8x4(acc[j][n][0], acc[j][n][1], fa[j], fb[n]);
  }
  const int mc = static_cast<int>(a.mcols);
  double* out = a.partial + static_cast<std::size_t>(i) * TD * mc;
#pragma unroll
  for (int j = 0; j < MT; ++j) {
    if (col[j] >= it.orow) continue;
    double* o = out + static_cast<std::size_t>(col[j]) * mc;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = 8 * n + 2 * q;
      if (c < mc) o[c] = acc[j][n][0];
      if (c + 1 < mc) o[c + 1] = acc[j][n][1];
    }
  }
}

// Single pass at m <= 2 (SCM = m): a scalar FP64 consumer. The n8 DMMA
// would spend 4-8x the useful flops on one or two columns; here every
// consumer warp reads its TD / 8 tile rows once per item (one vector load
// per row covers the row: PPL positions per lane) and forms both products
// from the same registers: the row part into per-lane partials that persist
// over the owner's items (lane-reduced in a fixed xor tree at the owner's
// end), the transposed part against the owner slab (per-lane partials over
// the warp's rows, combined across warps in warp order through shared
// memory). Deterministic. Positions are the permuted tile columns
// (tile_layout.h), so the partner slab is read at unperm(position).
template <typename V, int TD, int NT, int SCM>
__device__ __forceinline__ void scalar_consumer(const SpmmArgs& a, unsigned char* smem, std::uint64_t* hand,
                                                std::uint32_t i_beg, std::uint32_t i_end, int cw, int lane, int tid) {
  using S = Shape<V, TD, NT>;
  constexpr int RPW = TD / kConsumerWarps;  // tile rows per consumer warp
  constexpr int PPL = TD / 32;              // tile positions per lane
  constexpr int prec = sizeof(V) == 4 ? 0 : 1;
  using VecT = typename std::conditional<sizeof(V) * PPL == 16, typename std::conditional<sizeof(V) == 4, float4, double2>::type, float2>::type;
  static_assert(sizeof(VecT) == sizeof(V) * PPL, "one vector load per row and lane");
  double* oslab = reinterpret_cast<double*>(smem + 2 * S::kTileBytes + 2 * S::kSlabBytes);
  double* red = oslab + TD * S::kSX;  // [kConsumerWarps][TD][SCM]
  const int p0 = PPL * lane;
  int col[PPL];
#pragma unroll
  for (int k = 0; k < PPL; ++k) col[k] = static_cast<int>(cieg_tl::unperm(static_cast<std::uint32_t>(p0 + k), prec));
  const int r_base = cw * RPW;
  const int mc = static_cast<int>(a.mcols);
  int buf = 0;
  double racc[RPW][SCM];
  Item it = load_item(a, i_beg);
  for (std::uint32_t i = i_beg; i < i_end; ++i) {
    const Item nit = (i + 1 < i_end) ? load_item(a, i + 1) : it;
    if (it.first()) {
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
        for (int j = 0; j < SCM; ++j) racc[rr][j] = 0.0;
      bar_sync(kBarConsumers, kConsumerThreads);  // every warp is done with the previous owner's slab
      bool bad = false;
      for (int e = tid - kProducerThreads; e < TD * 8 * NT; e += kConsumerThreads) {
        const int k = e / (8 * NT), t = e - k * (8 * NT);
        double v = (k < it.prow() && t < mc) ? __ldg(a.x + static_cast<std::size_t>(it.r0 + k) * a.ldx + t) : 0.0;
        if (!isfinite(v)) {  // staged as 0; nonfinite_fix_kernel adds its terms
          v = 0.0;
          bad = true;
        }
        oslab[k * S::kSX + t] = v;
      }
      if (bad) *a.nonfinite = a.launch_id;
      bar_sync(kBarConsumers, kConsumerThreads);
    }
    mbar_wait(&hand[buf], ((i - i_beg) >> 1) & 1u);
    const V* A = reinterpret_cast<const V*>(smem + buf * S::kTileBytes);
    const double* X = reinterpret_cast<const double*>(smem + 2 * S::kTileBytes + buf * S::kSlabBytes);
    const bool trans = it.kind() == 0u;
    double xq[PPL][SCM], tacc[PPL][SCM];
#pragma unroll
    for (int k = 0; k < PPL; ++k)
#pragma unroll
      for (int j = 0; j < SCM; ++j) {
        xq[k][j] = X[col[k] * S::kSX + j];
        tacc[k][j] = 0.0;
      }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
      const int r = r_base + rr;
      const VecT vv = *reinterpret_cast<const VecT*>(A + r * S::kSA + p0);
      const V* av = reinterpret_cast<const V*>(&vv);
      double ad[PPL];
#pragma unroll
      for (int k = 0; k < PPL; ++k) ad[k] = static_cast<double>(av[k]);
#pragma unroll
      for (int k = 0; k < PPL; ++k)
#pragma unroll
        for (int j = 0; j < SCM; ++j) racc[rr][j] = fma(ad[k], xq[k][j], racc[rr][j]);
      if (trans) {
#pragma unroll
        for (int j = 0; j < SCM; ++j) {
          const double xp = oslab[r * S::kSX + j];
#pragma unroll
          for (int k = 0; k < PPL; ++k) tacc[k][j] = fma(ad[k], xp, tacc[k][j]);
        }
      }
    }
    release_buffer(&hand[2 + buf], lane);
    buf ^= 1;
    if (trans) {
#pragma unroll
      for (int k = 0; k < PPL; ++k)
#pragma unroll
        for (int j = 0; j < SCM; ++j) red[(cw * TD + col[k]) * SCM + j] = tacc[k][j];
      bar_sync(kBarConsumers, kConsumerThreads);
      double* out = a.partial + static_cast<std::size_t>(i) * TD * mc;
      for (int e = tid - kProducerThreads; e < TD * SCM; e += kConsumerThreads) {
        const int c = e / SCM, j = e - c * SCM;
        if (c >= it.orow || j >= mc) continue;
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) sum += red[(w * TD + c) * SCM + j];
        out[c * mc + j] = sum;
      }
      bar_sync(kBarConsumers, kConsumerThreads);  // red free for the next item
    }
    if (it.last()) {
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
        for (int j = 0; j < SCM; ++j) {
          const double v = warp_sum(racc[rr][j]);
          const int r = r_base + rr;
          if (lane == 0 && r < it.prow() && j < mc)
            a.y[static_cast<std::size_t>(it.r0 - a.row_base + r) * a.ldy + j] = v;
        }
    }
    it = nit;
  }
}

// SP = false: owner-computes -- an off-diagonal tile is streamed twice, once
// per owner panel (row part into P, transposed part into Q), each output
// row summed in registers by its owner. SP = true: single pass -- one item
// per stored tile; the consumers also form Aᵀ X_P from the same shared tile
// (X_P, the owner panel's slab, staged once per owner) and store it to the
// item's partial slot, added to block column Q by sp_reduce_kernel in a
// fixed order. Both are deterministic.
template <typename V, int TD, int NT, bool SP, int SCM = 0>
__global__ void __launch_bounds__(kThreads, 1) spmm_ws_kernel(const SpmmArgs a) {
  using S = Shape<V, TD, NT>;
  extern __shared__ __align__(16) unsigned char smem[];
  auto tile_buf = [&](int b) { return reinterpret_cast<V*>(smem + b * S::kTileBytes); };
  auto slab_buf = [&](int b) { return reinterpret_cast<double*>(smem + 2 * S::kTileBytes + b * S::kSlabBytes); };
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  const std::uint32_t i_beg = a.sched_off[blockIdx.x], i_end = a.sched_off[blockIdx.x + 1];
  const std::uint32_t total = i_end - i_beg;
  if (total == 0) return;
  // Producer layout: with one n-tile (m <= 8) the consumers are quick and the
  // producers' per-item memory round trips dominate, so two producer groups
  // fill alternating items concurrently; with two n-tiles the DMMA work per
  // item (128-row tiles) covers them and one 8-warp group (twice the
  // placement rate) wins.
  constexpr bool kTwoGroups = NT == 1 || TD == 64;  // 64-row tiles: little DMMA work per item
  __shared__ __align__(8) std::uint64_t hand[4];     // FULL[0..1], EMPTY[0..1]
  if (tid == 0) {
    constexpr unsigned kFill = kTwoGroups ? kGroupThreads : kProducerThreads;
    mbar_init(&hand[0], kFill);
    mbar_init(&hand[1], kFill);
    mbar_init(&hand[2], kConsumerWarps);
    mbar_init(&hand[3], kConsumerWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp < kProducerWarps && !kTwoGroups) {
    // ------------------------------------------------------------ producer
    // Register double buffer: the next batch of entry quads (or the first
    // batch of the next work item) is in flight while the current batch is
    // placed; item descriptors are prefetched two items ahead and the next
    // item's X slab a whole item ahead.
    const int pt = tid;  // 0 .. 255
    const V* val = static_cast<const V*>(a.val);
    auto load_batch = [&](const Item& it, std::uint64_t qb, Quad<V>(&out)[kQuads]) {
#pragma unroll
      for (int j = 0; j < kQuads; ++j) {
        const std::uint64_t q = qb + pt + static_cast<std::uint64_t>(j) * kProducerThreads;
        if (q < it.q1)
          load_quad(a, val, q, out[j]);
        else
          out[j].id.x = kNoQuad;
      }
    };
    Item cur = load_item(a, i_beg);
    Item nxt = (i_beg + 1 < i_end) ? load_item(a, i_beg + 1) : cur;
    // qb carries each item's first batch across the item boundary: it is
    // moved to qa only after the tile is cleared, so its memory round trip
    // overlaps the clearing and the slab store instead of stalling them.
    Quad<V> qa[kQuads], qb[kQuads];
    load_batch(cur, cur.q0, qb);
    double xv[S::kSlabPer];
    load_slab<V, TD, NT>(a, cur, pt, xv);
    bool nonfinite = false;
    int buf = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i) {
      const bool has_next = i + 1 < i_end;
      // the item after this one: its entries (and X slab) are bulk-prefetched
      // into L2 a whole item ahead of the register batches (measured best at
      // distance 1; deeper prefetch loses)
      if (pt == 0 && has_next) prefetch_item<V>(a, nxt);
      mbar_wait(&hand[2 + buf], (((i - i_beg) >> 1) & 1u) ^ 1u);
      V* A = tile_buf(buf);
      {
        // zero the TD data columns of every row (the pad columns are never read)
        float4* p4 = reinterpret_cast<float4*>(A);
        constexpr int kRow4 = TD * static_cast<int>(sizeof(V)) / 16, kStride4 = S::kSA * static_cast<int>(sizeof(V)) / 16;
#pragma unroll 4
        for (int k = pt; k < TD * kRow4; k += kProducerThreads)
          p4[(k / kRow4) * kStride4 + k % kRow4] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      double* X = slab_buf(buf);
#pragma unroll
      for (int j = 0; j < S::kSlabPer; ++j) {
        const int e = pt + j * kProducerThreads;
        const int k = e / (8 * NT), t = e - k * (8 * NT);
        // A non-finite X value would meet the dense tile's explicit zeros
        // (0 * Inf = NaN) where the reference multiplies stored entries
        // only: it is staged as 0 and nonfinite_fix_kernel adds its terms.
        // (Checked here, a whole item after the load was issued.)
        const bool bad = !isfinite(xv[j]);
        const double v = bad ? 0.0 : xv[j];
        nonfinite |= bad;
        // NT == 2: columns g and 8 + g side by side (one 128-bit B load)
        X[k * S::kSX + (NT == 2 ? 2 * (t & 7) + (t >> 3) : t)] = v;
      }
      if (has_next) load_slab<V, TD, NT>(a, nxt, pt, xv);
      const Item after = (i + 2 < i_end) ? load_item(a, i + 2) : nxt;
      bar_sync(kBarProducers, kProducerThreads);  // clear before scatter
      const std::uint32_t kind = cur.kind();
#pragma unroll
      for (int j = 0; j < kQuads; ++j) qa[j] = qb[j];
      for (std::uint64_t q = cur.q0;; q += kChunkQuads) {
        const bool more = q + kChunkQuads < cur.q1;
        if (more)
          load_batch(cur, q + kChunkQuads, qb);
        else if (has_next)
          load_batch(nxt, nxt.q0, qb);
#pragma unroll
        for (int j = 0; j < kQuads; ++j) {
          if (qa[j].id.x == kNoQuad) continue;
          if (kind == 0u)
            put4<0>(A, qa[j]);
          else if (kind == 1u)
            put4<1>(A, qa[j]);
          else if (kind == 2u)
            put4<2>(A, qa[j]);
        }
        if (!more) break;
#pragma unroll
        for (int j = 0; j < kQuads; ++j) qa[j] = qb[j];
      }
      mbar_arrive(&hand[buf]);
      buf ^= 1;
      cur = nxt;
      nxt = after;
    }
    if (nonfinite) *a.nonfinite = a.launch_id;
  } else if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    // Two producer groups of 4 warps fill alternating items -- group G the
    // items i_beg + G, i_beg + G + 2, ... into tile buffer G -- so one
    // group's per-item memory round trips overlap the other's. Within a
    // group: a register double buffer (the next batch of entry quads, or the
    // first batch of the group's next item, is in flight while the current
    // batch is placed), item descriptors two group-items ahead, the next
    // group-item's X slab staged a whole item ahead.
    const int grp = warp / kGroupWarps;
    const int pt = tid - grp * kGroupThreads;  // 0 .. 127
    const V* val = static_cast<const V*>(a.val);
    auto load_batch = [&](const Item& it, std::uint64_t qb, Quad<V>(&out)[kQuads]) {
#pragma unroll
      for (int j = 0; j < kQuads; ++j) {
        const std::uint64_t q = qb + pt + static_cast<std::uint64_t>(j) * kGroupThreads;
        if (q < it.q1)
          load_quad(a, val, q, out[j]);
        else
          out[j].id.x = kNoQuad;
      }
    };
    const std::uint32_t i0 = i_beg + grp;
    if (i0 < i_end) {
      Item cur = load_item(a, i0);
      Item nxt = (i0 + 2 < i_end) ? load_item(a, i0 + 2) : cur;
      Quad<V> qa[kQuads], qb[kQuads];  // qb: the item's first batch, as above
      load_batch(cur, cur.q0, qb);
      double xv[S::kSlabPerG];
      load_slab_g<V, TD, NT>(a, cur, pt, xv);
      bool nonfinite = false;
      const int buf = grp;
      for (std::uint32_t i = i0; i < i_end; i += 2) {
        const bool has_next = i + 2 < i_end;
        // the group's next item: entries and X slab bulk-prefetched into L2
        if (pt == 0 && has_next) prefetch_item<V>(a, nxt);
        mbar_wait(&hand[2 + buf], (((i - i0) >> 1) & 1u) ^ 1u);
        V* A = tile_buf(buf);
        {
          // zero the TD data columns of every row (the pad columns are never read)
          float4* p4 = reinterpret_cast<float4*>(A);
          constexpr int kRow4 = TD * static_cast<int>(sizeof(V)) / 16, kStride4 = S::kSA * static_cast<int>(sizeof(V)) / 16;
#pragma unroll 4
          for (int k = pt; k < TD * kRow4; k += kGroupThreads)
            p4[(k / kRow4) * kStride4 + k % kRow4] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double* X = slab_buf(buf);
#pragma unroll
        for (int j = 0; j < S::kSlabPerG; ++j) {
          const int e = pt + j * kGroupThreads;
          const int k = e / (8 * NT), t = e - k * (8 * NT);
          // A non-finite X value would meet the dense tile's explicit zeros
          // (0 * Inf = NaN) where the reference multiplies stored entries
          // only: it is staged as 0 and nonfinite_fix_kernel adds its terms.
          // (Checked here, a whole item after the load was issued.)
          const bool bad = !isfinite(xv[j]);
          const double v = bad ? 0.0 : xv[j];
          nonfinite |= bad;
          // NT == 2: columns g and 8 + g side by side (one 128-bit B load)
          X[k * S::kSX + (NT == 2 ? 2 * (t & 7) + (t >> 3) : t)] = v;
        }
        if (has_next) load_slab_g<V, TD, NT>(a, nxt, pt, xv);
        const Item after = (i + 4 < i_end) ? load_item(a, i + 4) : nxt;
        bar_sync(kBarProducers0 + grp, kGroupThreads);  // zeroing done before any scatter
        const std::uint32_t kind = cur.kind();
#pragma unroll
        for (int j = 0; j < kQuads; ++j) qa[j] = qb[j];
        for (std::uint64_t q = cur.q0;; q += kGroupChunkQuads) {
          const bool more = q + kGroupChunkQuads < cur.q1;
          if (more)
            load_batch(cur, q + kGroupChunkQuads, qb);
          else if (has_next)
            load_batch(nxt, nxt.q0, qb);
#pragma unroll
          for (int j = 0; j < kQuads; ++j) {
            if (qa[j].id.x == kNoQuad) continue;
            if (kind == 0u)
              put4<0>(A, qa[j]);
            else if (kind == 1u)
              put4<1>(A, qa[j]);
            else if (kind == 2u)
              put4<2>(A, qa[j]);
          }
          if (!more) break;
#pragma unroll
          for (int j = 0; j < kQuads; ++j) qa[j] = qb[j];
        }
        mbar_arrive(&hand[buf]);
        cur = nxt;
        nxt = after;
      }
      if (nonfinite) *a.nonfinite = a.launch_id;
    }
  } else if constexpr (SCM > 0) {
    scalar_consumer<V, TD, NT, SCM>(a, smem, hand, i_beg, i_end, warp - kProducerWarps, lane, tid);
  } else {
    // ------------------------------------------------------------ consumer
    const int cw = warp - kProducerWarps;
    const int g = lane >> 2, q = lane & 3;
    const int m_base = cw * 8 * S::kMT;
    double* oslab = reinterpret_cast<double*>(smem + 2 * S::kTileBytes + 2 * S::kSlabBytes);  // SP only
    int buf = 0;
    double acc[S::kMT][NT][2];
    Item it = load_item(a, i_beg);
    for (std::uint32_t i = i_beg; i < i_end; ++i) {
      const Item nit = (i + 1 < i_end) ? load_item(a, i + 1) : it;
      if (it.first()) {
#pragma unroll
        for (int j = 0; j < S::kMT; ++j)
#pragma unroll
          for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
        if constexpr (SP) {
          // the owner panel's X rows, for the transposed products of its items
          bar_sync(kBarConsumers, kConsumerThreads);  // every warp is done with the previous owner's slab
          bool bad = false;
          for (int e = tid - kProducerThreads; e < TD * 8 * NT; e += kConsumerThreads) {
            const int k = e / (8 * NT), t = e - k * (8 * NT);
            double v = (k < it.prow() && t < static_cast<int>(a.mcols))
                           ? __ldg(a.x + static_cast<std::size_t>(it.r0 + k) * a.ldx + t)
                           : 0.0;
            if (!isfinite(v)) {  // staged as 0; nonfinite_fix_kernel adds its terms
              v = 0.0;
              bad = true;
            }
            oslab[k * S::kSX + (NT == 2 ? 2 * (t & 7) + (t >> 3) : t)] = v;
          }
          if (bad) *a.nonfinite = a.launch_id;
          bar_sync(kBarConsumers, kConsumerThreads);
        }
      }
      const std::uint32_t r0 = it.r0;
      const int prow = it.prow();
      const bool live = m_base < prow;
      mbar_wait(&hand[buf], ((i - i_beg) >> 1) & 1u);
      if (live) {
        // Rows >= orow of the slab and of the tile are zero: all TD/4
        // k-steps run, in groups of 4 (two interleaved k-step pairs), with
        // the next group's fragments loaded and converted while the current
        // group's DMMAs issue.
        // fp32: one float4 = the A fragments of the group's 4 k-steps;
        // fp64: two double2 (tile_layout.h). NT == 2: one double2 = both
        // n-tiles' B fragments of a k-step.
        const V* A = tile_buf(buf) + (m_base + g) * S::kSA + (sizeof(V) == 4 ? 4 : 2) * q;
        const double* xb = slab_buf(buf) + q * S::kSX + (NT == 2 ? 2 * g : g);
        double af[2][4][S::kMT], bf[2][4][NT];
        auto load_group = [&](int grp, double (&fa)[4][S::kMT], double (&fb)[4][NT]) {
#pragma unroll
          for (int j = 0; j < S::kMT; ++j) {
            if constexpr (sizeof(V) == 4) {
              const float4 v4 = *reinterpret_cast<const float4*>(A + j * 8 * S::kSA + 16 * grp);
              fa[0][j] = static_cast<double>(v4.x);
              fa[1][j] = static_cast<double>(v4.y);
              fa[2][j] = static_cast<double>(v4.z);
              fa[3][j] = static_cast<double>(v4.w);
            } else {
#pragma unroll
              for (int p = 0; p < 2; ++p) {
                const double2 v2 = *reinterpret_cast<const double2*>(A + j * 8 * S::kSA + 8 * (2 * grp + p));
                fa[2 * p][j] = v2.x;
                fa[2 * p + 1][j] = v2.y;
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* xr = xb + 4 * (4 * grp + u) * S::kSX;
            if constexpr (NT == 2) {
              const double2 v2 = *reinterpret_cast<const double2*>(xr);
              fb[u][0] = v2.x;
              fb[u][1] = v2.y;
            } else {
#pragma unroll
              for (int n = 0; n < NT; ++n) fb[u][n] = xr[8 * n];
            }
          }
        };
        auto mma_group = [&](const double (&fa)[4][S::kMT], const double (&fb)[4][NT]) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
              for (int j = 0; j < S::kMT; ++j) dmma_8x8x4(acc[j][n][0], acc[j][n][1], fa[u][j], fb[u][n]);
        };
        constexpr int kGroups = TD / 16;
        if constexpr (sizeof(V) == 4) {
          // A fragments held raw (float4 per m-tile) and widened right before
          // their DMMAs: the conversions no longer wait on the next group's
          // loads ahead of the current group's DMMAs
          float4 ar[2][S::kMT];
          auto load_raw = [&](int grp, float4 (&o)[S::kMT], double (&fb)[4][NT]) {
#pragma unroll
            for (int j = 0; j < S::kMT; ++j) o[j] = *reinterpret_cast<const float4*>(A + j * 8 * S::kSA + 16 * grp);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double* xr = xb + 4 * (4 * grp + u) * S::kSX;
              if constexpr (NT == 2) {
                const double2 v2 = *reinterpret_cast<const double2*>(xr);
                fb[u][0] = v2.x;
                fb[u][1] = v2.y;
              } else {
#pragma unroll
                for (int n = 0; n < NT; ++n) fb[u][n] = xr[8 * n];
              }
            }
          };
          auto mma_raw = [&](const float4 (&o)[S::kMT], const double (&fb)[4][NT]) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              double fa[S::kMT];
#pragma unroll
              for (int j = 0; j < S::kMT; ++j)
                fa[j] = static_cast<double>(u == 0 ? o[j].x : u == 1 ? o[j].y : u == 2 ? o[j].z : o[j].w);
#pragma unroll
              for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int j = 0; j < S::kMT; ++j) dmma_8x8x4(acc[j][n][0], acc[j][n][1], fa[j], fb[u][n]);
            }
          };
          load_raw(0, ar[0], bf[0]);
#pragma unroll 1
          for (int grp = 0; grp < kGroups; grp += 2) {
            load_raw(grp + 1, ar[1], bf[1]);
            mma_raw(ar[0], bf[0]);
            if (grp + 2 < kGroups) load_raw(grp + 2, ar[0], bf[0]);
            mma_raw(ar[1], bf[1]);
          }
        } else {
          load_group(0, af[0], bf[0]);
#pragma unroll 1
          for (int grp = 0; grp < kGroups; grp += 2) {
            load_group(grp + 1, af[1], bf[1]);
            mma_group(af[0], bf[0]);
            if (grp + 2 < kGroups) load_group(grp + 2, af[0], bf[0]);
            mma_group(af[1], bf[1]);
          }
        }
      }
      if constexpr (SP) {
        if (it.kind() == 0u && m_base < it.orow) transposed_product<V, TD, NT>(a, tile_buf(buf), oslab, i, it, cw, lane);
      }
      release_buffer(&hand[2 + buf], lane);
      buf ^= 1;
      if (it.last() && live) {
#pragma unroll
        for (int j = 0; j < S::kMT; ++j) {
          const int row = m_base + 8 * j + g;
          if (row >= prow) continue;
          double* yr = a.y + static_cast<std::size_t>(r0 - a.row_base + row) * a.ldy;
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
      it = nit;
    }
  }
}

// Exact terms of non-finite X values (rare; exits at once when K1 saw none):
// for every Inf/NaN x[j][c] on the shard's halo rows, every stored entry in
// row or column j adds h * x[j][c] to the owner output it feeds -- the same
// owner-computes terms K1 would have produced, now without the dense
// tile's zeros. Inf/NaN absorb, so the non-finite results do not depend on
// the order of the (atomic) additions.
template <typename V>
__global__ void nonfinite_fix_kernel(const SpmmArgs a, std::uint32_t te, int precision, std::uint32_t p_lo,
                                     std::uint32_t p_hi, std::uint32_t halo_lo, std::uint32_t halo_hi, int force) {
  // force: a single-pass shard -- terms of another shard's tiles reach this
  // shard's rows through its partials, so K1's flag here does not see them
  if (!force && *a.nonfinite != a.launch_id) return;
  const std::uint32_t sa = cieg_tl::stride(te, precision);
  const V* val = static_cast<const V*>(a.val);
  const std::uint64_t total = static_cast<std::uint64_t>(halo_hi - halo_lo) * a.mcols;
  for (std::uint64_t e = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; e < total;
       e += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint32_t j = halo_lo + static_cast<std::uint32_t>(e / a.mcols);
    const std::uint32_t c = static_cast<std::uint32_t>(e % a.mcols);
    const double xv = a.x[static_cast<std::size_t>(j) * a.ldx + c];
    if (isfinite(xv)) continue;
    std::uint32_t lo = 0, hi = a.npanels;  // panel of row j
    while (hi - lo > 1) {
      const std::uint32_t mid = (lo + hi) / 2;
      if (a.panel_start[mid] <= j) lo = mid; else hi = mid;
    }
    const std::uint32_t pjx = lo;
    for (std::uint32_t P = p_lo; P < p_hi; ++P)
      for (std::uint32_t w = a.work_off[P]; w < a.work_off[P + 1]; ++w) {
        const std::uint32_t o = a.work_other[w], kind = a.work_kind[w];
        if (P != pjx && o != pjx) continue;
        const std::uint32_t pi = kind == 1 ? o : P, pj = kind == 0 ? o : P;
        const std::uint32_t r0 = a.panel_start[pi], q0 = a.panel_start[pj];
        const std::uint32_t t = a.work_tile[w];
        for (std::uint64_t q = a.tile_off[t]; q < a.tile_off[t + 1]; ++q) {
          const std::uint32_t off = a.idx[q] & 0xffffu;
          const std::uint32_t r = off / sa, pc = off - r * sa;
          if (pc >= te) continue;  // padding
          const std::uint32_t gr = r0 + r, gc = q0 + cieg_tl::unperm(pc, precision);
          const double h = static_cast<double>(val[q]);
          // kind 0: Y[gr] += h x[gc]; kind 1: Y[gc] += h x[gr]; kind 2: both (gr != gc)
          if (kind != 1 && gc == j) atomicAdd(&a.y[static_cast<std::size_t>(gr - a.row_base) * a.ldy + c], h * xv);
          if (kind != 0 && gr == j && (kind == 1 || gr != gc))
            atomicAdd(&a.y[static_cast<std::size_t>(gc - a.row_base) * a.ldy + c], h * xv);
        }
      }
  }
}

// Single pass: Y[rows of Q] += sum of the partial slots of block column Q,
// in the fixed slot order of sp_col_items (deterministic). One CTA per panel.
// On a shard, block columns below the owned rows (q0 < row_lo) belong to
// lower shards: their sums go to yhalo (rows from part_lo) for the
// point-to-point reduction to their owners (dist.py).
__global__ void sp_reduce_kernel(const double* partial, const std::uint32_t* col_off, const std::uint32_t* col_items,
                                 const std::uint32_t* panel_start, double* y, std::uint32_t ldy, std::uint32_t mcols,
                                 std::uint32_t td, std::uint32_t row_lo, double* yhalo, std::uint32_t ldh,
                                 std::uint32_t part_lo) {
  const std::uint32_t Q = blockIdx.x;
  const std::uint32_t k0 = col_off[Q], k1 = col_off[Q + 1];
  if (k0 == k1) return;
  const std::uint32_t q0 = panel_start[Q], rows = panel_start[Q + 1] - q0;
  const bool own = q0 >= row_lo;
  for (std::uint32_t e = threadIdx.x; e < rows * mcols; e += blockDim.x) {
    const std::uint32_t r = e / mcols, c = e - r * mcols;
    double sum = 0.0;
    for (std::uint32_t k = k0; k < k1; ++k)
      sum += partial[(static_cast<std::size_t>(col_items[k]) * td + r) * mcols + c];
    if (own)
      y[static_cast<std::size_t>(q0 + r - row_lo) * ldy + c] += sum;
    else
      yhalo[static_cast<std::size_t>(q0 + r - part_lo) * ldh + c] = sum;
  }
}

template <typename V, int TD, int NT, bool SP, int SCM = 0>
void launch_variant(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args) {
  using S = Shape<V, TD, NT>;
  constexpr std::size_t smem =
      (SP ? S::kSmemSP : S::kSmem) + sizeof(double) * kConsumerWarps * TD * SCM;  // SCM: warp partials
  static_assert(smem <= 227 * 1024, "shared memory budget");
  auto kern = spmm_ws_kernel<V, TD, NT, SP, SCM>;
  CIEG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<SP ? m->sp_ctas : m->sched_ctas, kThreads, smem, ctx->stream>>>(args);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

template <typename V, int TD>
void dispatch_nt(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args, std::uint32_t mc, bool sp) {
  if (sp) {
    if (mc == 1)
      launch_variant<V, TD, 1, true, 1>(ctx, m, args);
    else if (mc == 2)
      launch_variant<V, TD, 1, true, 2>(ctx, m, args);
    else if (mc <= 8)
      launch_variant<V, TD, 1, true>(ctx, m, args);
    else
      launch_variant<V, TD, 2, true>(ctx, m, args);
  } else {
    if (mc <= 8)
      launch_variant<V, TD, 1, false>(ctx, m, args);
    else
      launch_variant<V, TD, 2, false>(ctx, m, args);
  }
}

// K1 mode (cieg_ctx_set_spmm_mode; else CIEG_SPMM_MODE=owner|single; else
// auto): single pass for block widths <= kSinglePassMaxCols on full
// (unsharded) matrices, owner-computes otherwise. Measured on config 2
// (profiles/README.md): single pass 2.14 / 2.99 / 5.03 ms at m = 1 / 8 / 16
// (scalar consumer at m <= 2) vs owner-computes 3.65 / 3.71 / 4.72 ms.
}  // namespace

bool single_pass_fits(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc) {
  const std::size_t need = sizeof(double) * static_cast<std::size_t>(m->sp_items) * m->tile_edge * mc;
  if (need <= ctx->scratch_partial.bytes) return true;
  std::size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  return need <= free_b / 4;
}

bool single_pass_default(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc) {
  if (!single_pass_rule(ctx, m, mc)) return false;
  const int mode = ctx->spmm_mode;
  // auto (and env-selected) mode: owner-computes when the partials would crowd HBM
  return mode == CIEG_SPMM_SINGLE_PASS || single_pass_fits(ctx, m, mc);
}

bool single_pass_rule(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc) {
  static const int env_mode = [] {
    const char* e = std::getenv("CIEG_SPMM_MODE");
    if (e && std::strcmp(e, "owner") == 0) return static_cast<int>(CIEG_SPMM_OWNER);
    if (e && std::strcmp(e, "single") == 0) return static_cast<int>(CIEG_SPMM_SINGLE_PASS);
    if (e && std::strcmp(e, "sliced") == 0) return static_cast<int>(CIEG_SPMM_SLICED);
    return static_cast<int>(CIEG_SPMM_AUTO);
  }();
  if (!m->sp_sched) return false;
  const int mode = ctx->spmm_mode >= 0 ? ctx->spmm_mode : env_mode;
  if (mode == CIEG_SPMM_SLICED) return !sliced_supported(m);  // (the DMMA single pass where sliced cannot run)
  if (mode != CIEG_SPMM_AUTO) return mode == CIEG_SPMM_SINGLE_PASS;
  return mc <= kSinglePassMaxCols;
}

int effective_mode(const cieg_ctx* ctx) {
  static const int env_mode = [] {
    const char* e = std::getenv("CIEG_SPMM_MODE");
    if (e && std::strcmp(e, "owner") == 0) return static_cast<int>(CIEG_SPMM_OWNER);
    if (e && std::strcmp(e, "single") == 0) return static_cast<int>(CIEG_SPMM_SINGLE_PASS);
    if (e && std::strcmp(e, "sliced") == 0) return static_cast<int>(CIEG_SPMM_SLICED);
    return static_cast<int>(CIEG_SPMM_AUTO);
  }();
  return ctx->spmm_mode >= 0 ? ctx->spmm_mode : env_mode;
}

int spmm_effective_mode(cieg_ctx* ctx, cieg_mat* m, std::uint32_t mc) {
  const bool shard = m->row_lo != 0 || m->row_hi != m->dim;
  if (!shard && sliced_rule(ctx, m, mc) && sliced_ready(ctx, m)) return CIEG_SPMM_SLICED;
  if (!shard && single_pass_default(ctx, m, mc)) return CIEG_SPMM_SINGLE_PASS;
  return CIEG_SPMM_OWNER;
}

bool sliced_rule(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc) {
  if (!sliced_supported(m)) return false;
  const int mode = effective_mode(ctx);
  if (mode == CIEG_SPMM_SLICED) return true;
  if (mode != CIEG_SPMM_AUTO) return false;
  return mc >= kSlicedMinCols;
}


// The non-finite flag: zeroed once when allocated; each K1 launch tags it
// with its own launch id, so it never needs a reset (launch ids start at 1).
unsigned* nonfinite_flag(cieg_ctx* ctx) {
  const bool fresh = ctx->scratch_flag.bytes == 0;
  auto* f = static_cast<unsigned*>(ctx->scratch_flag.get(sizeof(unsigned)));
  if (fresh) CIEG_CUDA(cudaMemsetAsync(f, 0, sizeof(unsigned), ctx->stream));
  return f;
}

namespace {
// the Inf/NaN fix-up of the K1 launch described by args (exits at once when
// that launch's flag is clear; forced on a single-pass shard)
void launch_nonfinite_fix_args(cieg_ctx* ctx, const cieg_mat* m, const SpmmArgs& args, bool force) {
  // owned panels of this (shard) matrix
  const auto& ps = m->panel_start_host;
  const std::uint32_t p_lo = static_cast<std::uint32_t>(std::lower_bound(ps.begin(), ps.end(), m->row_lo) - ps.begin());
  const std::uint32_t p_hi = static_cast<std::uint32_t>(std::lower_bound(ps.begin(), ps.end(), m->row_hi) - ps.begin());
  const int prec = m->precision;
  if (prec == 0)
    nonfinite_fix_kernel<float><<<ctx->sm_count, 256, 0, ctx->stream>>>(args, m->tile_edge, prec, p_lo, p_hi,
                                                                        m->halo_lo, m->halo_hi, force ? 1 : 0);
  else
    nonfinite_fix_kernel<double><<<ctx->sm_count, 256, 0, ctx->stream>>>(args, m->tile_edge, prec, p_lo, p_hi,
                                                                         m->halo_lo, m->halo_hi, force ? 1 : 0);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

SpmmArgs make_args(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y, std::uint32_t ldy,
                   std::uint32_t mc, unsigned launch_id) {
  return SpmmArgs{m->panel_start,
                  m->work_off,
                  m->work_tile,
                  m->work_other,
                  m->work_kind,
                  m->sched_off,
                  reinterpret_cast<const uint4*>(m->sched),
                  m->tile_off,
                  m->idx,
                  m->val,
                  x,
                  y,
                  ldx,
                  ldy,
                  mc,
                  m->npanels,
                  m->row_lo,
                  nonfinite_flag(ctx),
                  launch_id,
                  nullptr};
}
}  // namespace

void launch_nonfinite_fix(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                          std::uint32_t ldy, std::uint32_t mc, unsigned launch_id) {
  launch_nonfinite_fix_args(ctx, m, make_args(ctx, m, x, ldx, y, ldy, mc, launch_id), false);
}

void launch_spmm(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                 std::uint32_t ldy, std::uint32_t mcols, double* yhalo, std::uint32_t ldh, bool shard_single_pass) {
  if (mcols == 0 || m->dim == 0) return;
  const bool shard = m->row_lo != 0 || m->row_hi != m->dim;
  const bool shard_sp = shard && shard_single_pass;
  if (shard_sp && !m->sp_sched) fail(CIEG_ERR_CONFIG, "single-pass SpMM: the shard has no single-pass schedule");
  if (shard_sp && !yhalo && m->row_lo > m->sp_partial_lo) fail(CIEG_ERR_ARGUMENT, "single-pass SpMM: null partial buffer");
  if (shard_sp && m->row_lo > m->sp_partial_lo)  // rows without partials read as zero
    CIEG_CUDA(cudaMemset2DAsync(yhalo, sizeof(double) * ldh, 0, sizeof(double) * mcols, m->row_lo - m->sp_partial_lo,
                                ctx->stream));
  for (std::uint32_t c0 = 0; c0 < mcols; c0 += 16) {
    const std::uint32_t mc = std::min<std::uint32_t>(16, mcols - c0);
    SpmmArgs args = make_args(ctx, m, x + c0, ldx, y + c0, ldy, mc, ++ctx->spmm_launch_id);
    const bool sliced = !shard && sliced_rule(ctx, m, mc) && sliced_ready(ctx, const_cast<cieg_mat*>(m));
    const bool sp = !sliced && (shard ? shard_sp : single_pass_default(ctx, m, mc));
    if (sp) {
      args.sched_off = m->sp_sched_off;
      args.sched = reinterpret_cast<const uint4*>(m->sp_sched);
      args.partial = static_cast<double*>(
          ctx->scratch_partial.get(sizeof(double) * std::max<std::size_t>(1, std::size_t(m->sp_items) * m->tile_edge * mc)));
    }
    if (sliced) {
      launch_spmm_sliced(ctx, const_cast<cieg_mat*>(m), x + c0, ldx, y + c0, ldy, mc, args.nonfinite, args.launch_id);
    } else if (m->precision == 0) {
      if (m->tile_edge == 64)
        dispatch_nt<float, 64>(ctx, m, args, mc, sp);
      else
        dispatch_nt<float, 128>(ctx, m, args, mc, sp);
    } else {  // fp64 values: 64-row tiles (a 128-row fp64 tile pair exceeds shared memory)
      dispatch_nt<double, 64>(ctx, m, args, mc, sp);
    }
    if (sp) {
      sp_reduce_kernel<<<m->npanels, 256, 0, ctx->stream>>>(args.partial, m->sp_col_off, m->sp_col_items,
                                                            m->panel_start, y + c0, ldy, mc, m->tile_edge, m->row_lo,
                                                            shard_sp && yhalo ? yhalo + c0 : nullptr, ldh, m->sp_partial_lo);
      CIEG_CUDA(cudaGetLastError());
      ++ctx->launches;
    }
    if (sliced) launch_sliced_tiny_fix(ctx, m, x + c0, ldx, y + c0, ldy, mc);
    launch_nonfinite_fix_args(ctx, m, args, shard_sp);
  }
}

}  // namespace cieg
