// umma.cuh -- the few tcgen05 (5th-generation tensor core) primitives K1's
// integer-slice path uses (spmm_i8.cu): shared-memory matrix descriptors for
// the no-swizzle canonical layouts, the kind::i8 instruction descriptor,
// TMEM allocation, MMA issue/commit and TMEM -> register loads. sm_100a only.
//
// Canonical no-swizzle layouts (8-bit elements): a "core matrix" is 8 rows x
// 16 bytes, stored as 128 contiguous bytes.
//   K-major operand  (rows = M or N, 16 K bytes per core row):
//     LBO = byte stride between core matrices adjacent in K,
//     SBO = byte stride between core matrices adjacent in M/N (8-row groups).
//   MN-major operand (16 M/N bytes per core row, 8 K per core matrix):
//     LBO = byte stride between core matrices adjacent in K (8-K groups),
//     SBO = byte stride between core matrices adjacent in M/N (16-byte chunks).
// A tile stored as 8-row x 16-column core matrices is therefore the K-major
// A of H*X (M = tile row, K = tile column) and, with LBO/SBO swapped, the
// MN-major A of H^T*X (M = tile column, K = tile row): one shared-memory copy
// serves both orientations of a stored tile.
#pragma once

#include <cstdint>

namespace cieg {
namespace umma {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start
// address, LBO, SBO (all >> 4), version 1 (bits 46-47), no swizzle.
__device__ __forceinline__ std::uint64_t sdesc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return static_cast<std::uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<std::uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<std::uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::i8, S32 accumulate: a/b signed (1) or
// unsigned (0), a/b MN-major (1) or K-major (0), shape M x N.
__host__ __device__ constexpr std::uint32_t idesc_i8(int a_signed, int b_signed, int a_mn, int b_mn, int m, int n) {
  return (2u << 4) | (static_cast<std::uint32_t>(a_signed) << 7) | (static_cast<std::uint32_t>(b_signed) << 10) |
         (static_cast<std::uint32_t>(a_mn) << 15) | (static_cast<std::uint32_t>(b_mn) << 16) |
         (static_cast<std::uint32_t>(n >> 3) << 17) | (static_cast<std::uint32_t>(m >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]; issued by one thread.
__device__ __forceinline__ void mma_i8(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                       std::uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// The same issued by one elected lane of a converged warp: every lane runs
// the issue loop with warp-uniform descriptors (kept in uniform registers, no
// per-MMA waterfall), one lane executes the MMA.
__device__ __forceinline__ void mma_i8_warp(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                            std::uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.b32 p, %4, 0;\n elect.sync _|q, 0xffffffff;\n"
      " @q tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_warp(std::uint64_t* mbar) {
  asm volatile(
      "{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n"
      " @q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(mbar))
      : "memory");
}

// Arrive on an mbarrier once every MMA issued so far by this thread completes.
__device__ __forceinline__ void commit(std::uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

// TMEM allocation by one full warp; the base address is written to *slot.
template <int kCols>
__device__ __forceinline__ void tmem_alloc(std::uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_free(std::uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(kCols) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes -> 16 registers.
__device__ __forceinline__ void ld16(std::uint32_t taddr, std::int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
// 8 consecutive 32-bit TMEM columns of this warp's 32 lanes -> 8 registers.
__device__ __forceinline__ void ld8(std::uint32_t taddr, std::int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes <- 0
__device__ __forceinline__ void st16_zero(std::uint32_t taddr) {
  const std::uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(z)
      : "memory");
}
// 8 consecutive 32-bit TMEM columns of this warp's 32 lanes <- 0
__device__ __forceinline__ void st8_zero(std::uint32_t taddr) {
  const std::uint32_t z = 0;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(z) : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }


// ---- mbarriers and bulk (TMA-engine) copies ---------------------------------
__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// arrive and add `bytes` to the transaction count the phase waits for
__device__ __forceinline__ void mbar_arrive_tx(std::uint64_t* b, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
  const std::uint32_t a = smem_u32(b);
  std::uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// the same, backing off with nanosleep between polls: for warps that wait
// long (epilogue, producers), so their polling does not compete with the
// tensor core's shared-memory operand reads
__device__ __forceinline__ void mbar_wait_sleep(std::uint64_t* b, unsigned parity, unsigned ns = 128) {
  const std::uint32_t a = smem_u32(b);
  std::uint32_t ok = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}
// global -> shared bulk copy (bytes % 16 == 0, both ends 16-byte aligned),
// completing `bytes` transactions on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// the same with an L2 cache-policy hint (createpolicy_evict_first): streamed
// data that should not displace the L2-resident working set
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar,
                                              std::uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ std::uint64_t createpolicy_evict_first() {
  std::uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ std::uint64_t createpolicy_evict_last() {
  std::uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_l2(const void* p, std::uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace umma
}  // namespace cieg
