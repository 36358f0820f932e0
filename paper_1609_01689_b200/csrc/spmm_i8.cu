// spmm_i8.cu -- K1 on the 5th-generation tensor cores: the fused symmetric
// SpMM U = (L + L^T - diag L) X of ci::spmm (proj/src/csb.cpp:118-193) for an
// fp32 H, computed exactly in integer arithmetic by slicing (Ozaki scheme)
// and run as tcgen05.mma kind::i8 with int32 accumulators in TMEM.
//
// Why: fp64 X makes K1 FP64-bound on the DMMA pipe (37 TF/s; dense 128 x 128
// tiles at the generator's 40 % in-tile density issue 2.5x the useful flops,
// so the DMMA floor on config 2 at m = 16 is 3.46 ms = 31 % of HBM). The int8
// tensor cores run ~120x that rate, so the same dense-tile products fit under
// the HBM time once both operands are exact integer slices:
//   * H: every stored value h of row r is a_int * 2^(e_r - 39) with
//     |a_int| < 2^39 (e_r = exponent of the largest |h| touching index r, as
//     row or column), so a_int is exact for every entry within 2^-16 of its
//     row maximum and rounded at 2^-40 of it below that; a_int is split into
//     five 8-bit slices, top signed, four unsigned (two's complement bytes).
//     The diagonal is not sliced (its d_r x_r is added in fp64), so e_r is
//     the off-diagonal scale of the row.
//     Built once per matrix on the device (records_kernel): one 8-byte record
//     per stored entry = its position in the 128 x 128 core-matrix tile layout
//     (umma.cuh) + the five slice bytes -- the same 8 bytes per entry as the
//     fp32 value + packed index of the DMMA stream.
//   * X: per 128-row panel and column, x = x_int * 2^(ex - 54), |x_int| <= 2^54,
//     as seven balanced signed 8-bit digits (digitize_kernel, every call). For
//     the transposed product the row scale 2^e_r is folded into X first, so
//     one slice tile serves H X (K-major A) and H^T X (MN-major A).
//   * the product a_int x_int = sum_d D_d 2^(8 (10 - d)), D_d = sum_{s+t=d}
//     A_s X_t: one MMA per H slice s computes all its diagonals at once (B =
//     digits 0 .. 6-s, D columns from 16 s), diagonals d <= 6 are kept (the
//     dropped terms are below 2^-52 of max|a| max|x| per product), each D_d is
//     an exact int32 over the 128-long tile dot product, and the epilogue
//     recombines sum_d D_d 2^(-8 d) in fp64 and scales by 2^(e_r + ex - 13).
// The result agrees with the fp64 reference to rounding (tests compare at
// 1e-13 relative), but its rounding is not the DMMA kernels': this mode is
// selected per width (cieg_ctx_set_spmm_mode, CIEG_SPMM_SLICED).
//
// Schedule: the single-pass item list (tiling.cpp): one item per stored tile
// of its row panel, items of an owner panel consecutive. The row part
// accumulates in fp64 registers of the owner's epilogue warps and is written
// once; the transposed part goes to the item's partial slot, added to its
// block column by sp_reduce_kernel in a fixed order (spmm.cu) -- no atomics,
// deterministic. Diagonal tiles are stored mirrored (both triangles) and use
// the row part only.
//
// CTA (one per SM, 512 threads):
//   warp 0      TMEM allocation; one lane issues the MMAs (40 per tile)
//   warps 1-7   producers: zero a slice buffer, scatter the item's records
//               (5 byte stores each, bank-ordered at build), bulk-copy the X
//               digit slabs (cp.async.bulk, mbarrier complete_tx)
//   warps 8-11  row epilogue (TMEM lanes = tile rows): recombine, accumulate
//   warps 12-15 transposed epilogue (TMEM lanes = tile columns): partials
// Two slice buffers, two owner slabs, two TMEM accumulator stages, all handed
// over with mbarriers (tcgen05.commit for the MMA side).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>

#include "context.hpp"
#include "tile_layout.h"
#include "umma.cuh"

namespace cieg {

constexpr int kTD = 128;                   // tile edge (fp32 H panels)
constexpr int kAS = 5;                     // H slices
constexpr int kXD = 7;                     // X digits = diagonals kept
constexpr int kNB = 16 * kXD;              // B rows per slab (digit-major, 16 columns each)
constexpr int kPlane = kTD * kTD;          // bytes per H slice plane
constexpr int kPlanes = kAS * kPlane;      // 81920
constexpr int kSlab = kNB * kTD;           // 14336: X digits of one panel
constexpr int kSlabBytes = kSlab + 64;     // + 16 int32 exponents
constexpr int kStageCols = 2 * kNB;        // TMEM columns per accumulator stage (row + transposed)
constexpr int kThreads = 512;
constexpr int kProducers = 7 * 32;         // warps 1..7
constexpr std::uint16_t kNoEntry = 0xffff;

struct OzItem {
  std::uint64_t rec0;   // first record
  std::uint32_t nrec;   // records (even; sentinels included)
  std::uint32_t flags;  // kind | first << 8 | last << 9 | owner rows << 16
  std::uint32_t owner, partner;  // panel indices
  std::uint32_t r0;     // owner start row
  std::uint32_t orow;   // partner rows
};
static_assert(sizeof(OzItem) == 32, "item descriptor");

struct SlicedPlan {
  OzItem* items = nullptr;
  std::uint32_t* cta_off = nullptr;
  uint2* rec = nullptr;
  int* rowexp = nullptr;
  float* diag = nullptr;  // stored diagonal of H (applied in fp64, not sliced)
  std::uint8_t* xd = nullptr;                 // per-call digit slabs, npanels * kSlabBytes
  std::uint8_t* xt = nullptr;
  std::uint64_t nrec = 0;
  bool finite = true;  // every stored value finite (else the DMMA kernels run)
  ~SlicedPlan() {
    cudaFree(items);
    cudaFree(cta_off);
    cudaFree(rec);
    cudaFree(rowexp);
    cudaFree(diag);
    cudaFree(xd);
    cudaFree(xt);
  }
};

namespace {

__host__ __device__ __forceinline__ std::uint32_t off_a(std::uint32_t r, std::uint32_t c) {
  return (r >> 3) * 1024u + (c >> 4) * 128u + (r & 7u) * 16u + (c & 15u);
}
__host__ __device__ __forceinline__ std::uint32_t off_b(std::uint32_t n, std::uint32_t k) {
  return (n >> 3) * 1024u + (k >> 4) * 128u + (n & 7u) * 16u + (k & 15u);
}

// exponent E with |v| < 2^E (frexp), for finite nonzero v
__device__ __forceinline__ int exp_of(double v) { return ilogb(v) + 1; }

// 2^e as a double (normal range; exact)
__device__ __forceinline__ double pow2(int e) {
  if (e >= -1022 && e <= 1023) return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
  return ldexp(1.0, e);
}

// exact int32 -> double without the conversion unit: 2^52 + 2^31 + v
__device__ __forceinline__ double i2d(std::int32_t v) {
  return __hiloint2double(0x43300000, static_cast<int>(static_cast<unsigned>(v) ^ 0x80000000u)) -
         4503601774854144.0;
}

// ---------------------------------------------------------------- build time

// e_r: the largest exponent of any stored off-diagonal |h| in row r or
// column r. The diagonal -- typically the dominant entry of a CI row (the
// unperturbed energies) -- is not sliced: the row epilogue adds d_r x_r in
// fp64, so e_r follows the off-diagonal scale and the five slices hold every
// off-diagonal value within 2^-16 of it exactly.
__global__ void rowexp_kernel(const std::uint64_t* tile_off, const std::uint32_t* tile_pi,
                              const std::uint32_t* tile_pj, const std::uint32_t* panel_start,
                              const std::uint32_t* idx, const float* val, int* emax, unsigned* bad) {
  const std::uint64_t t = blockIdx.x;
  const std::uint32_t sa = cieg_tl::stride(kTD, 0);
  const std::uint32_t a0 = panel_start[tile_pi[t]], b0 = panel_start[tile_pj[t]];
  for (std::uint64_t e = tile_off[t] + threadIdx.x; e < tile_off[t + 1]; e += blockDim.x) {
    const std::uint32_t o = idx[e] & 0xffffu, r = o / sa, pc = o - r * sa;
    if (pc >= kTD) continue;
    const float h = val[e];
    if (!isfinite(h)) *bad = 1u;
    const std::uint32_t gr = a0 + r, gc = b0 + cieg_tl::unperm(pc, 0);
    if (h == 0.0f || !isfinite(h) || gr == gc) continue;  // the diagonal is applied in fp64 (epilogue)
    const int E = ilogbf(h) + 1 + 2048;
    atomicMax(&emax[gr], E);
    atomicMax(&emax[gc], E);
  }
}

__device__ __forceinline__ uint2 make_record(float h, int er, std::uint32_t pos) {
  // a_int = h 2^(39 - e_r), |a_int| < 2^39; two's complement bytes
  const long long a = __double2ll_rn(ldexp(static_cast<double>(h), 39 - er));
  const unsigned long long u = static_cast<unsigned long long>(a);
  const std::uint32_t d0 = static_cast<std::uint32_t>(a >> 32) & 0xffu;  // signed top byte
  const std::uint32_t d1 = static_cast<std::uint32_t>(u >> 24) & 0xffu;
  const std::uint32_t d2 = static_cast<std::uint32_t>(u >> 16) & 0xffu;
  const std::uint32_t d3 = static_cast<std::uint32_t>(u >> 8) & 0xffu;
  const std::uint32_t d4 = static_cast<std::uint32_t>(u) & 0xffu;
  return make_uint2(pos | (d0 << 16) | (d1 << 24), d2 | (d3 << 8) | (d4 << 16));
}

// One CTA per single-pass item: the item's entries as slice records, the
// mirrored twin of every strictly lower entry of a diagonal tile, in an order
// where every 32 consecutive records hit 32 distinct shared-memory banks of
// the slice planes (bank = 4 (r & 7) + (c & 15) / 4): records are ranked
// within their bank and emitted rank-major.
__global__ void records_kernel(const OzItem* items, const std::uint32_t* sp_sched, const std::uint32_t* idx,
                               const float* val, const int* rowexp, uint2* rec, float* diag_out) {
  __shared__ unsigned cnt[32], cnt2[32];
  const std::uint32_t i = blockIdx.x;
  const OzItem it = items[i];
  const std::uint32_t* d = sp_sched + 8ull * i;
  const std::uint64_t q0 = (static_cast<std::uint64_t>(d[1]) << 32) | d[0];
  const std::uint64_t q1 = (static_cast<std::uint64_t>(d[3]) << 32) | d[2];
  const bool diag = (it.flags & 0xffu) == 2u;
  float* dg = diag_out;
  const std::uint32_t sa = cieg_tl::stride(kTD, 0);
  if (threadIdx.x < 32) cnt[threadIdx.x] = cnt2[threadIdx.x] = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (std::uint64_t e = 4 * q0 + threadIdx.x; e < 4 * q1; e += blockDim.x) {
      const std::uint32_t o = idx[e] & 0xffffu, r = o / sa, pc = o - r * sa;
      if (pc >= kTD) continue;
      const std::uint32_t c = cieg_tl::unperm(pc, 0);
      const float h = val[e];
      if (diag && r == c) {
        if (pass == 0) dg[it.r0 + r] = h;
        continue;
      }
      for (int twin = 0; twin < (diag ? 2 : 1); ++twin) {
        const std::uint32_t rr = twin ? c : r, cc = twin ? r : c;
        const std::uint32_t pos = off_a(rr, cc);
        const std::uint32_t bank = (pos >> 2) & 31u;
        if (pass == 0) {
          atomicAdd(&cnt[bank], 1u);
          continue;
        }
        const unsigned rank = atomicAdd(&cnt2[bank], 1u);
        unsigned out = 0;
        for (int b = 0; b < 32; ++b) out += min(cnt[b], rank) + ((static_cast<unsigned>(b) < bank && cnt[b] > rank) ? 1u : 0u);
        rec[it.rec0 + out] = make_record(h, rowexp[it.r0 + rr], pos);
      }
    }
    __syncthreads();
  }
  unsigned total = 0;
  for (int b = 0; b < 32; ++b) total += cnt[b];
  for (std::uint32_t k = total + threadIdx.x; k < it.nrec; k += blockDim.x) rec[it.rec0 + k] = make_uint2(kNoEntry, 0);
}

// ----------------------------------------------------------------- per call

// X digits of one panel: B-operand slabs for the row part (x) and the
// transposed part (x 2^e_r), seven balanced digits per value, plus the
// per-column exponents. Non-finite values are staged as 0 (flag set; the
// caller's fix-up adds their exact terms).
__global__ void __launch_bounds__(128) digitize_kernel(const double* x, std::uint32_t ldx, std::uint32_t mc,
                                                       const std::uint32_t* panel_start, const int* rowexp,
                                                       std::uint8_t* xd, std::uint8_t* xt, unsigned* nonfinite,
                                                       unsigned launch_id) {
  __shared__ __align__(16) std::uint8_t sd[2][kSlab];
  __shared__ int wmax[2][4][16];
  __shared__ int cmax[2][16];
  const std::uint32_t P = blockIdx.x, p0 = panel_start[P], rows = panel_start[P + 1] - p0;
  const int r = threadIdx.x, w = r >> 5, lane = r & 31;
  const int er = r < static_cast<int>(rows) ? rowexp[p0 + r] : 0;
  double xv[16];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    double v = (r < static_cast<int>(rows) && j < static_cast<int>(mc)) ? x[static_cast<std::size_t>(p0 + r) * ldx + j] : 0.0;
    if (!isfinite(v)) {
      v = 0.0;
      bad = true;
    }
    xv[j] = v;
    int E = v != 0.0 ? exp_of(v) : INT_MIN / 4, Ep = v != 0.0 ? E + er : INT_MIN / 4;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      E = max(E, __shfl_xor_sync(0xffffffffu, E, s));
      Ep = max(Ep, __shfl_xor_sync(0xffffffffu, Ep, s));
    }
    if (lane == 0) {
      wmax[0][w][j] = E;
      wmax[1][w][j] = Ep;
    }
  }
  if (bad) *nonfinite = launch_id;
  __syncthreads();
  if (r < 32) {
    const int k = r >> 4, j = r & 15;
    int m = max(max(wmax[k][0][j], wmax[k][1][j]), max(wmax[k][2][j], wmax[k][3][j]));
    cmax[k][j] = m < INT_MIN / 8 ? 0 : m;  // all-zero column: exponent 0, digits 0
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      long long v = __double2ll_rn(ldexp(xv[j], (k ? er : 0) + 54 - cmax[k][j]));
      int dig[kXD];
#pragma unroll
      for (int t = kXD - 1; t > 0; --t) {
        int dd = static_cast<int>(v & 0xff);
        dd = dd >= 128 ? dd - 256 : dd;
        dig[t] = dd;
        v = (v - dd) >> 8;
      }
      dig[0] = static_cast<int>(v);
#pragma unroll
      for (int t = 0; t < kXD; ++t) sd[k][off_b(16 * t + j, r)] = static_cast<std::uint8_t>(dig[t]);
    }
  __syncthreads();
  const uint4* s0 = reinterpret_cast<const uint4*>(sd[0]);
  const uint4* s1 = reinterpret_cast<const uint4*>(sd[1]);
  uint4* g0 = reinterpret_cast<uint4*>(xd + static_cast<std::size_t>(P) * kSlabBytes);
  uint4* g1 = reinterpret_cast<uint4*>(xt + static_cast<std::size_t>(P) * kSlabBytes);
  for (int e = r; e < kSlab / 16; e += 128) {
    g0[e] = s0[e];
    g1[e] = s1[e];
  }
  if (r < 16) {
    reinterpret_cast<int*>(xd + static_cast<std::size_t>(P) * kSlabBytes + kSlab)[r] = cmax[0][r];
    reinterpret_cast<int*>(xt + static_cast<std::size_t>(P) * kSlabBytes + kSlab)[r] = cmax[1][r];
  }
}

struct SlicedArgs {
  const OzItem* items;
  const std::uint32_t* cta_off;
  const uint2* rec;
  const std::uint8_t* xd;
  const std::uint8_t* xt;
  const int* rowexp;
  const float* diag;
  const double* x;  // the call's X (the diagonal term d_r x_r)
  double* y;
  double* partial;
  std::uint32_t ldx, ldy, mc, row_base;
};

struct Smem {
  std::uint8_t planes[2][kPlanes];
  std::uint8_t xd[2][kSlabBytes];
  std::uint8_t xt[2][kSlabBytes];
  std::uint64_t full_a[2], empty_a[2], full_t[2], empty_t[2], acc_full[2], acc_empty[2];
  std::uint32_t tmem;
};

__device__ __forceinline__ void scatter(std::uint8_t* pl, std::uint32_t x, std::uint32_t y) {
  const std::uint32_t pos = x & 0xffffu;
  if (pos >= static_cast<std::uint32_t>(kPlane)) return;
  pl[pos] = static_cast<std::uint8_t>(x >> 16);
  pl[pos + kPlane] = static_cast<std::uint8_t>(x >> 24);
  pl[pos + 2 * kPlane] = static_cast<std::uint8_t>(y);
  pl[pos + 3 * kPlane] = static_cast<std::uint8_t>(y >> 8);
  pl[pos + 4 * kPlane] = static_cast<std::uint8_t>(y >> 16);
}

// sum_d D_d 2^(-8 d) over the kXD diagonal blocks at TMEM column col0 of this
// warp's 32 lanes (Horner from the lowest diagonal; fp64, one rounding per step)
__device__ __forceinline__ void recombine(std::uint32_t taddr, double (&v)[16]) {
  std::int32_t hi[16], lo[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = 0.0;
#pragma unroll
  for (int d = kXD - 1; d >= 1; d -= 2) {
    umma::ld16(taddr + 16 * d, hi);
    umma::ld16(taddr + 16 * (d - 1), lo);
    umma::ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = fma(v[j], 0x1p-8, i2d(hi[j]));
      v[j] = fma(v[j], 0x1p-8, i2d(lo[j]));
    }
  }
  if constexpr (kXD % 2 == 1) {
    umma::ld16(taddr, lo);
    umma::ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fma(v[j], 0x1p-8, i2d(lo[j]));
  }
}

__global__ void __launch_bounds__(kThreads, 1) spmm_sliced_kernel(const SlicedArgs a) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::uint32_t i_beg = a.cta_off[blockIdx.x], i_end = a.cta_off[blockIdx.x + 1];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&S.full_a[b], kProducers + 1);
      umma::mbar_init(&S.empty_a[b], 1);
      umma::mbar_init(&S.full_t[b], 1);
      umma::mbar_init(&S.empty_t[b], 1);
      umma::mbar_init(&S.acc_full[b], 1);
      umma::mbar_init(&S.acc_empty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc<512>(&S.tmem);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const std::uint32_t tbase = S.tmem;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issue
    std::uint32_t k = 0, owners = 0;
    int o = 0;
    const std::uint32_t pa[2] = {umma::smem_u32(S.planes[0]), umma::smem_u32(S.planes[1])};
    const std::uint32_t pb[2] = {umma::smem_u32(S.xd[0]), umma::smem_u32(S.xd[1])};
    const std::uint32_t pt[2] = {umma::smem_u32(S.xt[0]), umma::smem_u32(S.xt[1])};
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      if ((it.flags >> 8) & 1u) {
        o = owners & 1;
        umma::mbar_wait(&S.full_t[o], (owners >> 1) & 1u);
        ++owners;
      }
      umma::mbar_wait(&S.full_a[b], (k >> 1) & 1u);
      umma::mbar_wait(&S.acc_empty[b], ((k >> 1) & 1u) ^ 1u);
      umma::fence_after();
      if (lane == 0) {
        const std::uint32_t d_row = tbase + b * kStageCols, d_tr = d_row + kNB;
        const bool trans = (it.flags & 0xffu) == 0u;
#pragma unroll
        for (int s = 0; s < kAS; ++s) {
          const int n = 16 * (kXD - s);
          const std::uint32_t id_row = umma::idesc_i8(s == 0, 1, 0, 0, 128, n);
          const std::uint32_t id_tr = umma::idesc_i8(s == 0, 1, 1, 0, 128, n);
          const std::uint32_t ap = pa[b] + s * kPlane;
#pragma unroll
          for (int ks = 0; ks < kTD / 32; ++ks) {
            umma::mma_i8(d_row + 16 * s, umma::sdesc(ap + 256 * ks, 128, 1024), umma::sdesc(pb[b] + 256 * ks, 128, 1024),
                         id_row, (s | ks) != 0);
            if (trans)
              umma::mma_i8(d_tr + 16 * s, umma::sdesc(ap + 4096 * ks, 1024, 128),
                           umma::sdesc(pt[o] + 256 * ks, 128, 1024), id_tr, (s | ks) != 0);
          }
        }
        umma::commit(&S.empty_a[b]);
        umma::commit(&S.acc_full[b]);
        if ((it.flags >> 9) & 1u) umma::commit(&S.empty_t[o]);
      }
      __syncwarp();
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ producers
    const int pt = tid - 32;
    std::uint32_t k = 0, owners = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      if ((it.flags >> 8) & 1u) {
        const int o = owners & 1;
        if (pt == 0) {
          umma::mbar_wait(&S.empty_t[o], ((owners >> 1) & 1u) ^ 1u);
          umma::mbar_arrive_tx(&S.full_t[o], kSlabBytes);
          umma::bulk_g2s(S.xt[o], a.xt + static_cast<std::size_t>(it.owner) * kSlabBytes, kSlabBytes, &S.full_t[o]);
        }
        ++owners;
      }
      umma::mbar_wait(&S.empty_a[b], ((k >> 1) & 1u) ^ 1u);
      if (pt == 0) {
        umma::mbar_arrive_tx(&S.full_a[b], kSlabBytes);
        umma::bulk_g2s(S.xd[b], a.xd + static_cast<std::size_t>(it.partner) * kSlabBytes, kSlabBytes, &S.full_a[b]);
        if (i + 1 < i_end) {  // next item's records into L2 while this one is placed
          const OzItem nx = a.items[i + 1];
          const std::uint8_t* p = reinterpret_cast<const std::uint8_t*>(a.rec + nx.rec0);
          for (std::uint32_t off = 0; off < 8u * nx.nrec; off += 1u << 16)
            umma::prefetch_l2(p + off, min(1u << 16, 8u * nx.nrec - off));
        }
      }
      uint4* z = reinterpret_cast<uint4*>(S.planes[b]);
      for (int e = pt; e < kPlanes / 16; e += kProducers) z[e] = make_uint4(0, 0, 0, 0);
      asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
      const uint4* src = reinterpret_cast<const uint4*>(a.rec + it.rec0);
      const std::uint32_t nq = it.nrec >> 1;
      std::uint8_t* pl = S.planes[b];
      for (std::uint32_t q = pt; q < nq; q += 4 * kProducers) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = q + u * kProducers < nq ? __ldg(src + q + u * kProducers) : make_uint4(kNoEntry, 0, kNoEntry, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          scatter(pl, v[u].x, v[u].y);
          scatter(pl, v[u].z, v[u].w);
        }
      }
      umma::fence_async_smem();
      umma::mbar_arrive(&S.full_a[b]);
    }
  } else if (warp < 12) {
    // ------------------------------------------------- row-part epilogue
    const int q = warp - 8, r = 32 * q + lane;
    const std::uint32_t lanes = static_cast<std::uint32_t>(32 * q) << 16;
    double yacc[16];
    int er = 0;
    std::uint32_t k = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      const int prow = static_cast<int>(it.flags >> 16);
      if ((it.flags >> 8) & 1u) {
#pragma unroll
        for (int j = 0; j < 16; ++j) yacc[j] = 0.0;
        er = r < prow ? a.rowexp[it.r0 + r] : 0;
      }
      umma::mbar_wait(&S.acc_full[b], (k >> 1) & 1u);
      umma::fence_after();
      double v[16];
      recombine(tbase + lanes + b * kStageCols, v);
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&S.acc_empty[b]);
      const int* ex = reinterpret_cast<const int*>(a.xd + static_cast<std::size_t>(it.partner) * kSlabBytes + kSlab);
#pragma unroll
      for (int j = 0; j < 16; ++j) yacc[j] = fma(v[j], pow2(er + __ldg(ex + j) - 13), yacc[j]);
      if ((it.flags & 0xffu) == 2u && r < prow) {  // d_r x_r in fp64 (Inf/NaN x: the caller's fix-up adds it)
        const double dr = static_cast<double>(a.diag[it.r0 + r]);
        const double* xr = a.x + static_cast<std::size_t>(it.r0 + r) * a.ldx;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double xv = j < static_cast<int>(a.mc) ? xr[j] : 0.0;
          yacc[j] = fma(dr, isfinite(xv) ? xv : 0.0, yacc[j]);
        }
      }
      if (((it.flags >> 9) & 1u) && r < prow) {
        double* yr = a.y + static_cast<std::size_t>(it.r0 + r - a.row_base) * a.ldy;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < static_cast<int>(a.mc)) yr[j] = yacc[j];
      }
    }
  } else {
    // ------------------------------------------ transposed-part epilogue
    const int q = warp - 12, c = 32 * q + lane;
    const std::uint32_t lanes = static_cast<std::uint32_t>(32 * q) << 16;
    std::uint32_t k = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      const bool trans = (it.flags & 0xffu) == 0u;
      umma::mbar_wait(&S.acc_full[b], (k >> 1) & 1u);
      umma::fence_after();
      double v[16];
      if (trans) recombine(tbase + lanes + b * kStageCols + kNB, v);
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&S.acc_empty[b]);
      if (trans && c < static_cast<int>(it.orow)) {
        const int* ex = reinterpret_cast<const int*>(a.xt + static_cast<std::size_t>(it.owner) * kSlabBytes + kSlab);
        double* out = a.partial + (static_cast<std::size_t>(i) * kTD + c) * a.mc;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < static_cast<int>(a.mc)) out[j] = v[j] * pow2(__ldg(ex + j) - 13);
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tbase);
}

template <typename T>
T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  CIEG_CUDA(cudaMalloc(&d, sizeof(T) * std::max<std::size_t>(1, v.size())));
  if (!v.empty()) CIEG_CUDA(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return d;
}

std::uint32_t panel_of(const std::vector<std::uint32_t>& ps, std::uint32_t row) {
  return static_cast<std::uint32_t>(std::upper_bound(ps.begin(), ps.end(), row) - ps.begin() - 1);
}

SlicedPlan* build_plan(cieg_ctx* ctx, cieg_mat* m) {
  const std::uint32_t nitems = m->sp_items;
  std::vector<std::uint32_t> sched(8ull * nitems), cta_off(m->sp_ctas + 1);
  CIEG_CUDA(cudaMemcpy(sched.data(), m->sp_sched, sizeof(std::uint32_t) * sched.size(), cudaMemcpyDeviceToHost));
  CIEG_CUDA(cudaMemcpy(cta_off.data(), m->sp_sched_off, sizeof(std::uint32_t) * cta_off.size(), cudaMemcpyDeviceToHost));
  const auto& ps = m->panel_start_host;
  std::vector<OzItem> items(nitems);
  std::uint64_t total = 0;
  for (std::uint32_t i = 0; i < nitems; ++i) {
    const std::uint32_t* d = sched.data() + 8ull * i;
    const std::uint64_t q0 = (static_cast<std::uint64_t>(d[1]) << 32) | d[0];
    const std::uint64_t q1 = (static_cast<std::uint64_t>(d[3]) << 32) | d[2];
    const std::uint32_t kind = d[4] & 0xffu;
    OzItem& it = items[i];
    it.flags = d[4];
    it.r0 = d[7];
    it.orow = d[6];
    it.owner = panel_of(ps, d[7]);
    it.partner = panel_of(ps, d[5]);
    it.rec0 = total;
    std::uint64_t n = 4 * (q1 - q0) * (kind == 2 ? 2 : 1);
    n += n & 1;
    it.nrec = static_cast<std::uint32_t>(n);
    total += n;
  }
  auto* pl = new SlicedPlan;
  try {
    pl->nrec = total;
    pl->items = upload(items);
    pl->cta_off = upload(cta_off);
    CIEG_CUDA(cudaMalloc(&pl->rec, sizeof(uint2) * std::max<std::uint64_t>(1, total)));
    const std::uint32_t rows = ps.back() + kTD;
    CIEG_CUDA(cudaMalloc(&pl->rowexp, sizeof(int) * rows));
    CIEG_CUDA(cudaMalloc(&pl->diag, sizeof(float) * rows));
    CIEG_CUDA(cudaMemsetAsync(pl->diag, 0, sizeof(float) * rows, ctx->stream));
    CIEG_CUDA(cudaMemsetAsync(pl->rowexp, 0, sizeof(int) * rows, ctx->stream));
    std::uint32_t *tpi = upload(m->tile_pi_host), *tpj = upload(m->tile_pj_host);
    unsigned* bad = upload(std::vector<unsigned>{0u});
    if (m->ntiles)
      rowexp_kernel<<<static_cast<unsigned>(m->ntiles), 256, 0, ctx->stream>>>(
          m->tile_off, tpi, tpj, m->panel_start, m->idx, static_cast<const float*>(m->val), pl->rowexp, bad);
    CIEG_CUDA(cudaGetLastError());
    // stored as e_r (the kernel kept E + 2048; rows without entries -> 0, no record uses them)
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int> eh(rows);
    CIEG_CUDA(cudaMemcpy(eh.data(), pl->rowexp, sizeof(int) * rows, cudaMemcpyDeviceToHost));
    for (int& e : eh) e = e > 0 ? e - 2048 : 0;
    CIEG_CUDA(cudaMemcpy(pl->rowexp, eh.data(), sizeof(int) * rows, cudaMemcpyHostToDevice));
    unsigned bad_h = 0;
    CIEG_CUDA(cudaMemcpy(&bad_h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost));
    cudaFree(bad);
    pl->finite = bad_h == 0;
    std::uint32_t* dsched = m->sp_sched;
    if (nitems)
      records_kernel<<<nitems, 256, 0, ctx->stream>>>(pl->items, dsched, m->idx, static_cast<const float*>(m->val),
                                                      pl->rowexp, pl->rec, pl->diag);
    CIEG_CUDA(cudaGetLastError());
    ctx->launches += 2;
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(tpi);
    cudaFree(tpj);
    CIEG_CUDA(cudaMalloc(&pl->xd, static_cast<std::size_t>(m->npanels) * kSlabBytes));
    CIEG_CUDA(cudaMalloc(&pl->xt, static_cast<std::size_t>(m->npanels) * kSlabBytes));
  } catch (...) {
    delete pl;
    throw;
  }
  return pl;
}

}  // namespace

bool sliced_supported(const cieg_mat* m) {
  return m->precision == 0 && m->tile_edge == kTD && m->sp_sched != nullptr && m->row_lo == 0 &&
         m->row_hi == m->dim && (!m->sliced || m->sliced->finite);
}

bool sliced_ready(cieg_ctx* ctx, cieg_mat* m) {
  if (!sliced_supported(m)) return false;
  if (!m->sliced) m->sliced = build_plan(ctx, m);
  return m->sliced->finite;
}

void destroy_sliced(cieg_mat* m) {
  delete m->sliced;
  m->sliced = nullptr;
}

void launch_spmm_sliced(cieg_ctx* ctx, cieg_mat* m, const double* x, std::uint32_t ldx, double* y, std::uint32_t ldy,
                        std::uint32_t mc, double* partial, unsigned* nonfinite, unsigned launch_id) {
  if (!sliced_ready(ctx, m))
    fail(CIEG_ERR_CONFIG, "sliced SpMM needs an unsharded fp32 matrix with 128-row panels and finite values");
  if (mc == 0 || mc > 16) fail(CIEG_ERR_ARGUMENT, "sliced SpMM: 1..16 columns per launch");
  SlicedPlan* pl = m->sliced;
  digitize_kernel<<<m->npanels, 128, 0, ctx->stream>>>(x, ldx, mc, m->panel_start, pl->rowexp, pl->xd, pl->xt,
                                                       nonfinite, launch_id);
  CIEG_CUDA(cudaGetLastError());
  SlicedArgs args{pl->items, pl->cta_off, pl->rec, pl->xd, pl->xt, pl->rowexp, pl->diag, x, y, partial,
                  ldx, ldy, mc, m->row_lo};
  constexpr std::size_t smem = sizeof(Smem) + 1024;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  CIEG_CUDA(cudaFuncSetAttribute(spmm_sliced_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  spmm_sliced_kernel<<<m->sp_ctas, kThreads, smem, ctx->stream>>>(args);
  CIEG_CUDA(cudaGetLastError());
  ctx->launches += 2;
}

}  // namespace cieg
