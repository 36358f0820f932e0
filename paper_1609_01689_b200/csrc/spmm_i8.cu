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
//   * H: every stored value h of row r is a_int * 2^(e_r - 38) with
//     |a_int| < 2^38 (e_r = exponent of the largest |h| touching index r, as
//     row or column), so a_int is exact for every entry within 2^-15 of its
//     row maximum and rounded at 2^-39 of it below that; a_int is split into
//     five balanced signed 8-bit digits.
//     The diagonal is not sliced (its d_r x_r is added in fp64), so e_r is
//     the off-diagonal scale of the row.
//     Built once per matrix on the device: records_kernel writes one 8-byte
//     record per stored entry (its position in the 128 x 128 core-matrix tile
//     layout of umma.cuh + the five slice bytes), dense_kernel scatters them
//     into every item's five dense slice planes (5 x 16 KB, zeros included)
//     and the records are dropped. Entries too small for their row's slices
//     go to an fp64 list (tiny_fix_kernel), so every stored value enters
//     exactly.
//   * X: per 128-row panel and column, x = x_int * 2^(ex - 54), |x_int| <= 2^54,
//     as seven balanced signed 8-bit digits (digitize_kernel, every call). For
//     the transposed product the row scale 2^e_r is folded into X first, so
//     one slice tile serves H X (K-major A) and H^T X (MN-major A).
//   * the product a_int x_int = sum_d D_d 2^(8 (10 - d)), D_d = sum_{s+t=d}
//     A_s X_t: one MMA per H slice s computes all its diagonals at once (B =
//     digits 0 .. min(6, 7-s), D columns from 16 s), diagonals d <= 7 are kept
//     (the dropped terms are below 2^-58 of max|a| max|x| per product), each
//     D_d is an exact int32 over the 128-long tile dot product; the epilogue
//     recombines the diagonals exactly in int64 (two groups of four, joined
//     in fp64 with one rounding).
//   * Y: every contribution to a panel's rows -- the owner's row part (kept in
//     fp64 registers over the owner's items) and the transposed parts of the
//     tiles below it -- is converted to fixed point (int64, units of
//     2^(escale - 62), escale a bound on |Y| per (panel, column) set every
//     call by scales_kernel from the neighbours' X exponents) and added to
//     yint with 64-bit integer reds: exact, so the sum does not depend on the
//     order of the additions -- deterministic without slots, tickets or a
//     second reduction pass. yint_to_y_kernel converts (one rounding), adds the
//     diagonal term d_r x_r in fp64 and clears yint for the next call.
// The result agrees with the fp64 reference to rounding (tests compare at
// 1e-13 relative), but its rounding is not the DMMA kernels': this mode is
// selected per width (cieg_ctx_set_spmm_mode, CIEG_SPMM_SLICED).
//
// Schedule: the single-pass item list (tiling.cpp), one item per stored tile
// of its row panel, items of an owner panel consecutive; owner panels dealt
// to the CTAs in ascending order (least-loaded CTA first), so the grid sweeps
// the matrix front to back. Diagonal tiles are stored mirrored (both
// triangles) and use the row part only.
//
// CTA (one per SM, 18 warps):
//   warp 0      TMEM allocation; one lane issues the MMAs (40 per tile)
//   warp 1      one lane issues the bulk copies (cp.async.bulk, mbarrier
//               complete_tx): the item's planes (evict-first), the partner's
//               and the owner's X digit slabs (evict-last), their exponents
//   warps 2-17  epilogue, four per TMEM lane quarter: row part columns 0-7 /
//               8-15, transposed part columns 0-7 / 8-15
// Two plane buffers, two owner slabs, two TMEM accumulator stages, all handed
// over with mbarriers (tcgen05.commit for the MMA side).
//
// The host call (sliced_spmm_host, ci::spmm's path in the drop-in) runs the
// same kernels over chunks of owner panels, pipelined with the upload of X
// and the download of U (see there).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <vector>

#include "context.hpp"
#include "tile_layout.h"
#include "umma.cuh"

namespace cieg {

constexpr int kTD = 128;                   // tile edge (fp32 H panels)
constexpr int kAS = 5;                     // H slices
constexpr int kXD = 7;                     // X digits
constexpr int kDiag = 8;                   // accumulated diagonals d = s + t (d <= 7 kept)
constexpr int kNB = 16 * kXD;              // B rows per slab (digit-major, 16 columns each)
constexpr int kND = 16 * kDiag;            // TMEM columns per orientation
constexpr int kPlane = kTD * kTD;          // bytes per H slice plane
constexpr int kPlanes = kAS * kPlane;      // 81920
constexpr int kSlab = kNB * kTD;           // 14336: X digits of one panel
constexpr int kSlabBytes = kSlab + 64;     // + 16 int32 exponents
constexpr int kStageCols = 2 * kND;        // TMEM columns per accumulator stage (row + transposed)
constexpr std::uint16_t kNoEntry = 0xffff;
// Sparse lowest slice: digit 4 (weight 2^0) is non-zero only for entries below
// 2^-7 of their row scale -- ~2 % of the generator's entries -- so its plane is
// kept as a per-item list (position | digit << 16, at most kL4Cap entries) and
// scattered into a zero plane in shared memory by the copy warp instead of
// being streamed dense (64.5 KB per item instead of 80 KB). A matrix with a
// fuller lowest slice keeps the five dense planes.
constexpr int kL4Cap = 512;

struct OzItem {
  std::uint64_t rec0;   // first record
  std::uint32_t nrec;   // records (a multiple of 64; sentinels included)
  std::uint32_t flags;  // kind | first << 8 | last << 9 | owner rows << 16
  std::uint32_t owner, partner;  // panel indices
  std::uint32_t r0;     // owner start row
  std::uint32_t orow;   // partner rows
  std::uint32_t slot;   // the item's index in the single-pass schedule (its partial slot)
  std::uint32_t pad;
};
static_assert(sizeof(OzItem) == 40, "item descriptor");

struct SlicedPlan {
  OzItem* items = nullptr;
  std::uint32_t* cta_off = nullptr;
  uint2* rec = nullptr;
  std::uint8_t* dense = nullptr;  // every item's dense slice planes (five, or four with the sparse lowest slice), TMA-loaded
  std::uint32_t* list4 = nullptr;  // sparse lowest slice: kL4Cap entries per item (OzItem.pad = the item's count)
  bool sparse4 = false;
  int* rowexp = nullptr;
  float* diag = nullptr;  // stored diagonal of H (applied in fp64, not sliced)
  std::uint8_t* xd = nullptr;                 // per-call digit slabs, npanels * kSlabBytes
  std::uint8_t* xt = nullptr;
  // tiny entries (not exactly sliceable) as CSR over output rows, fp64
  std::uint32_t ntiny_rows = 0;
  std::uint32_t *tiny_rows = nullptr, *tiny_off = nullptr, *tiny_in = nullptr;
  double* tiny_val = nullptr;
  // Fixed-point accumulation of every contribution to a panel's rows (the
  // row part and the transposed parts), int64, exact and order-independent:
  // yint[Q][row quarter][column][32 rows] in units of 2^(escale[Q][column] - 62). The scales
  // are bounds on |Y| per (panel, column), set every call from the X digit
  // exponents of the panel's neighbours (scales_kernel).
  long long* yint = nullptr;
  int* escale = nullptr;
  std::uint32_t* nb_off = nullptr;  // per panel: neighbours (P | 1 << 31 for a transposed contributor)
  std::uint32_t* nb = nullptr;
  int* erq = nullptr;  // per panel: max row scale e_r of its rows
  int* edq = nullptr;  // per panel: max exponent of its stored diagonal
  std::uint64_t nrec = 0;
  std::uint32_t ctas = 0;
  // host copies for the chunked host call (sliced_spmm_host): the items'
  // owner panels in schedule order, the CTA ranges, the tiny rows, and per
  // panel the prefix maximum of its highest neighbour panel (a panel's
  // scales need the digits of all its neighbours; its rows are final once
  // every owner up to that neighbour has run)
  std::vector<std::uint32_t> item_owner_host, cta_off_host, tiny_rows_host, nb_prefix_max;
  struct Chunks {
    std::uint32_t want = 0;            // the chunk count asked for (cache key)
    std::vector<std::uint32_t> panel;  // chunk c = owner panels [panel[c], panel[c + 1])
    std::uint32_t* cta_lim = nullptr;  // device [(chunks + 1) * ctas]: CTA b runs items [c * ctas + b], [(c + 1) * ctas + b])
  };
  std::vector<Chunks> chunkings;
  bool usable = true;  // every stored value finite and the planes fit (else the DMMA kernels run)
  ~SlicedPlan() {
    for (auto& c : chunkings) cudaFree(c.cta_lim);
    cudaFree(items);
    cudaFree(cta_off);
    cudaFree(rec);
    cudaFree(dense);
    cudaFree(list4);
    cudaFree(rowexp);
    cudaFree(diag);
    cudaFree(xd);
    cudaFree(xt);
    cudaFree(tiny_rows);
    cudaFree(tiny_off);
    cudaFree(tiny_in);
    cudaFree(tiny_val);
    cudaFree(yint);
    cudaFree(escale);
    cudaFree(nb_off);
    cudaFree(nb);
    cudaFree(erq);
    cudaFree(edq);
  }
};

namespace {

__host__ __device__ __forceinline__ std::uint32_t off_a(std::uint32_t r, std::uint32_t c) {
  return (r >> 3) * 1024u + (c >> 4) * 128u + (r & 7u) * 16u + (c & 15u);
}
__host__ __device__ __forceinline__ std::uint32_t off_b(std::uint32_t n, std::uint32_t k) {
  return (n >> 3) * 1024u + (k >> 4) * 128u + (n & 7u) * 16u + (k & 15u);
}

// 2^e as a double, exact and branchless for |e| <= 2044 (a product of two
// normal powers of two; subnormal results are exact too)
__device__ __forceinline__ double pow2(int e) {
  e = max(-2044, min(2044, e));
  const int h = e >> 1;
  return __longlong_as_double(static_cast<long long>(h + 1023) << 52) *
         __longlong_as_double(static_cast<long long>(e - h + 1023) << 52);
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
  // a_int = h 2^(38 - e_r), |a_int| < 2^38, as five balanced base-256 digits
  // (all signed: no cancellation between diagonals in the fp64 recombination)
  // via the carry-free bias: bytes of (a_int + B) ^ B, B = 0x8080808080
  constexpr long long kBias = 0x8080808080ll;
  const long long a = __double2ll_rn(ldexp(static_cast<double>(h), 38 - er));
  const unsigned long long u = static_cast<unsigned long long>((a + kBias) ^ kBias);
  const std::uint32_t d0 = static_cast<std::uint32_t>(u >> 32) & 0xffu;  // weight 2^32
  const std::uint32_t d1 = static_cast<std::uint32_t>(u >> 24) & 0xffu;
  const std::uint32_t d2 = static_cast<std::uint32_t>(u >> 16) & 0xffu;
  const std::uint32_t d3 = static_cast<std::uint32_t>(u >> 8) & 0xffu;
  const std::uint32_t d4 = static_cast<std::uint32_t>(u) & 0xffu;
  return make_uint2(pos | (d0 << 16) | (d1 << 24), d2 | (d3 << 8) | (d4 << 16));
}

// Producer lane l of a warp loads the 16-byte pair of records (2 (32 w + l),
// 2 (32 w + l) + 1) and stores the first of every pair in one warp-wide
// pass, the second in the next: so rank-major record k = 64 w + 32 h + l is
// kept at 64 w + 2 l + h, and each pass stores 32 consecutive ranks.
__device__ __forceinline__ unsigned interleave(unsigned k) { return (k & ~63u) | ((k & 31u) << 1) | ((k >> 5) & 1u); }

// One CTA per single-pass item: the item's entries as slice records, the
// mirrored twin of every strictly lower entry of a diagonal tile, in an order
// where every 32 consecutive records hit 32 distinct shared-memory banks of
// the slice planes (bank = 4 (r & 7) + (c & 15) / 4): records are ranked
// within their bank and emitted rank-major.
// An entry is sliced only when its a_int is exact (|h| >= 2^(e_r - 15) for
// a normal fp32 h); the few smaller ones go to the tiny list instead (output
// row, input row, value), added in fp64 after the SpMM (tiny_fix_kernel), so
// every stored value enters the product exactly.
struct Tiny {
  std::uint32_t out, in;
  double v;
};

__device__ __forceinline__ bool sliceable(float h, int er) {
  const double s = ldexp(static_cast<double>(h), 38 - er);
  return s == rint(s);
}

__global__ void records_kernel(const OzItem* items, const std::uint32_t* sp_sched, const std::uint32_t* idx,
                               const float* val, const int* rowexp, const std::uint32_t* panel_start, uint2* rec,
                               float* diag_out, Tiny* tiny, unsigned* ntiny, unsigned tiny_cap) {
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
        const int er = rowexp[it.r0 + rr];
        if (!sliceable(h, er)) {
          if (pass == 1) {
            const std::uint32_t gr = it.r0 + rr, gc = (diag ? it.r0 : panel_start[it.partner]) + cc;
            const unsigned t = atomicAdd(ntiny, diag ? 1u : 2u);
            if (t + 1 < tiny_cap) {
              tiny[t] = Tiny{gr, gc, static_cast<double>(h)};
              if (!diag) tiny[t + 1] = Tiny{gc, gr, static_cast<double>(h)};
            }
          }
          continue;
        }
        const std::uint32_t pos = off_a(rr, cc);
        const std::uint32_t bank = (pos >> 2) & 31u;
        if (pass == 0) {
          atomicAdd(&cnt[bank], 1u);
          continue;
        }
        const unsigned rank = atomicAdd(&cnt2[bank], 1u);
        unsigned k = 0;  // rank-major position
        for (int b = 0; b < 32; ++b) k += min(cnt[b], rank) + ((static_cast<unsigned>(b) < bank && cnt[b] > rank) ? 1u : 0u);
        rec[it.rec0 + interleave(k)] = make_record(h, er, pos);
      }
    }
    __syncthreads();
  }
  unsigned total = 0;
  for (int b = 0; b < 32; ++b) total += cnt[b];
  for (std::uint32_t k = total + threadIdx.x; k < it.nrec; k += blockDim.x)
    rec[it.rec0 + interleave(k)] = make_uint2(kNoEntry, 0);  // (nrec is a multiple of 64)
}

// Dense mode: every item's records scattered once into its five slice planes
// in HBM (kPlanes bytes per item, zeros included), so the SpMM streams them
// with bulk copies instead of scattering records every call.
__global__ void dense_kernel(const OzItem* items, const uint2* rec, std::uint8_t* dense, int nplanes) {
  const std::uint32_t i = blockIdx.x;
  const OzItem it = items[i];
  std::uint8_t* d = dense + static_cast<std::size_t>(i) * nplanes * kPlane;
  uint4* d4 = reinterpret_cast<uint4*>(d);
  for (int u = threadIdx.x; u < nplanes * kPlane / 16; u += blockDim.x) d4[u] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  for (std::uint32_t k = threadIdx.x; k < it.nrec; k += blockDim.x) {
    const uint2 r = rec[it.rec0 + k];
    const std::uint32_t pos = r.x & 0xffffu;
    if (pos >= static_cast<std::uint32_t>(kPlane)) continue;
    d[pos] = static_cast<std::uint8_t>(r.x >> 16);
    d[pos + kPlane] = static_cast<std::uint8_t>(r.x >> 24);
    d[pos + 2 * kPlane] = static_cast<std::uint8_t>(r.y);
    d[pos + 3 * kPlane] = static_cast<std::uint8_t>(r.y >> 8);
    if (nplanes == kAS) d[pos + 4 * kPlane] = static_cast<std::uint8_t>(r.y >> 16);
  }
}

// The lowest slice of every item as a list (position | digit << 16; the order
// within an item does not matter: positions are distinct). The item's count
// goes to its descriptor; *over is set when an item exceeds kL4Cap.
__global__ void list4_kernel(OzItem* items, const uint2* rec, std::uint32_t* list4, unsigned* over) {
  __shared__ unsigned cnt;
  const std::uint32_t i = blockIdx.x;
  const OzItem it = items[i];
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  std::uint32_t* l = list4 + static_cast<std::size_t>(i) * kL4Cap;
  for (std::uint32_t k = threadIdx.x; k < it.nrec; k += blockDim.x) {
    const uint2 r = rec[it.rec0 + k];
    const std::uint32_t pos = r.x & 0xffffu, d4 = (r.y >> 16) & 0xffu;
    if (pos >= static_cast<std::uint32_t>(kPlane) || d4 == 0) continue;
    const unsigned t = atomicAdd(&cnt, 1u);
    if (t < static_cast<unsigned>(kL4Cap)) l[t] = pos | (d4 << 16);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    items[i].pad = min(cnt, static_cast<unsigned>(kL4Cap));
    if (cnt > static_cast<unsigned>(kL4Cap)) *over = 1u;
  }
}

// ----------------------------------------------------------------- per call

// x = M 2^q with M a 53-bit integer (exact decomposition of a finite double)
__device__ __forceinline__ void decompose(double x, long long& m, int& q) {
  const long long bits = __double_as_longlong(x);
  const int eb = static_cast<int>((bits >> 52) & 0x7ff);
  const long long mant = bits & ((1ll << 52) - 1);
  m = eb ? (mant | (1ll << 52)) : mant;
  q = (eb ? eb : 1) - 1075;
  if (bits < 0) m = -m;
}
// round(M 2^(q + s)) for |M 2^(q+s)| <= 2^54, integer arithmetic only
__device__ __forceinline__ long long scaled(long long m, int sh) {
  if (sh >= 0) return m << sh;
  if (sh < -62) return 0;
  const long long a = m < 0 ? -m : m;
  const long long r = (a + (1ll << (-sh - 1))) >> -sh;
  return m < 0 ? -r : r;
}
// exponent E with |x| < 2^E for M 2^q (M != 0)
__device__ __forceinline__ int exp_mq(long long m, int q) {
  const long long a = m < 0 ? -m : m;
  return 64 - __clzll(a) + q;
}

// X digits of one panel: B-operand slabs for the row part (x) and the
// transposed part (x 2^e_r), seven balanced digits per value, plus the
// per-column exponents, in integer arithmetic on the bit patterns. Thread
// (column j, row group g) handles rows 4 (g + 16 u) .. +3, u = 0..1, so each
// digit of four consecutive rows is one 32-bit shared store. Non-finite
// values are staged as 0 (flag set; the caller's fix-up adds their exact
// terms).
__global__ void __launch_bounds__(256, 4) digitize_kernel(const double* x, std::uint32_t ldx, std::uint32_t mc,
                                                       const std::uint32_t* panel_start, const int* rowexp,
                                                       std::uint8_t* xd, std::uint8_t* xt, unsigned* nonfinite,
                                                       unsigned launch_id, std::uint32_t p_base) {
  __shared__ __align__(16) std::uint8_t sd[2][kSlab];
  __shared__ int wmax[2][8][16];
  __shared__ int cmax[2][16];
  const std::uint32_t P = blockIdx.x + p_base, p0 = panel_start[P], rows = panel_start[P + 1] - p0;
  const int tid = threadIdx.x, j = tid & 15, g = tid >> 4;
  long long mv[8];
  int qv[8], er[8];
  int E = INT_MIN / 4, Ep = INT_MIN / 4;
  bool bad = false;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = 4 * (g + 16 * u) + v, e = 4 * u + v;
      const bool in = r < static_cast<int>(rows);
      double xv = (in && j < static_cast<int>(mc)) ? x[static_cast<std::size_t>(p0 + r) * ldx + j] : 0.0;
      er[e] = in ? rowexp[p0 + r] : 0;
      if (!isfinite(xv)) {
        xv = 0.0;
        bad = true;
      }
      decompose(xv, mv[e], qv[e]);
      if (mv[e] != 0) {
        const int ee = exp_mq(mv[e], qv[e]);
        E = max(E, ee);
        Ep = max(Ep, ee + er[e]);
      }
    }
  if (bad) *nonfinite = launch_id;
  E = max(E, __shfl_xor_sync(0xffffffffu, E, 16));
  Ep = max(Ep, __shfl_xor_sync(0xffffffffu, Ep, 16));
  if ((tid & 31) < 16) {
    wmax[0][tid >> 5][j] = E;
    wmax[1][tid >> 5][j] = Ep;
  }
  __syncthreads();
  if (tid < 32) {
    const int k = tid >> 4, jj = tid & 15;
    int m = wmax[k][0][jj];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = max(m, wmax[k][w][jj]);
    cmax[k][jj] = m < INT_MIN / 8 ? 0 : m;  // all-zero column: exponent 0, digits 0
  }
  __syncthreads();
  // Balanced base-256 digits without carries: x_int + sum_t 128 256^t has
  // the plain bytes X_t + 128, so the digit bytes (two's complement) are the
  // bytes of (x_int + B) ^ B, B = 0x80808080808080; byte t weighs 256^t
  // (digit index 6 - t). Four rows' bytes of one digit -> one word (PRMT).
  constexpr long long kBias = 0x0080808080808080ll;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int cm = cmax[k][j];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      std::uint32_t lo[4], hi[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int e = 4 * u + v;
        const long long w = (scaled(mv[e], qv[e] + (k ? er[e] : 0) + 54 - cm) + kBias) ^ kBias;
        lo[v] = static_cast<std::uint32_t>(w);
        hi[v] = static_cast<std::uint32_t>(w >> 32);
      }
#pragma unroll
      for (int t = 0; t < kXD; ++t) {  // byte t of the values = digit kXD - 1 - t
        const std::uint32_t* src = t < 4 ? lo : hi;
        const std::uint32_t sel = static_cast<std::uint32_t>(t & 3) | (static_cast<std::uint32_t>(4 + (t & 3)) << 4);
        const std::uint32_t p01 = __byte_perm(src[0], src[1], sel), p23 = __byte_perm(src[2], src[3], sel);
        *reinterpret_cast<std::uint32_t*>(&sd[k][off_b(16 * (kXD - 1 - t) + j, 4 * (g + 16 * u))]) =
            __byte_perm(p01, p23, 0x5410);
      }
    }
  }
  __syncthreads();
  const uint4* s0 = reinterpret_cast<const uint4*>(sd[0]);
  const uint4* s1 = reinterpret_cast<const uint4*>(sd[1]);
  uint4* g0 = reinterpret_cast<uint4*>(xd + static_cast<std::size_t>(P) * kSlabBytes);
  uint4* g1 = reinterpret_cast<uint4*>(xt + static_cast<std::size_t>(P) * kSlabBytes);
  for (int e = tid; e < kSlab / 16; e += 256) {
    g0[e] = s0[e];
    g1[e] = s1[e];
  }
  if (tid < 16) {
    reinterpret_cast<int*>(xd + static_cast<std::size_t>(P) * kSlabBytes + kSlab)[tid] = cmax[0][tid];
    reinterpret_cast<int*>(xt + static_cast<std::size_t>(P) * kSlabBytes + kSlab)[tid] = cmax[1][tid];
  }
}

// Per (panel, column) bound exponents of Y: |y| < 2^escale. Every
// contribution to a row of Q is below 2^(e + 7) -- a row part of tile (Q, P):
// e = max e_r (rows of Q) + ex_P (|h| < 2^e_r, |x_P| < 2^ex_P, 128 terms);
// a transposed part of tile (P, Q): e = ex'_P (|x_P 2^e_r| < 2^ex'_P) -- and
// there are cnt of them, so escale = max + ceil(log2(cnt + 1)) + 1 bounds
// their sum. (The diagonal d_r x_r is not in yint: yint_to_y_kernel adds it
// in fp64, so a row's own diagonal never sets its panel's scale.)
__global__ void scales_kernel(const std::uint32_t* nb_off, const std::uint32_t* nb, const int* erq, const int* edq,
                              const std::uint8_t* xd, const std::uint8_t* xt, int* escale, std::uint32_t q_base) {
  const std::uint32_t Q = blockIdx.x + q_base;
  const int j = threadIdx.x;
  if (j >= 16) return;
  auto xe = [&](const std::uint8_t* slabs, std::uint32_t P) {
    return reinterpret_cast<const int*>(slabs + static_cast<std::size_t>(P) * kSlabBytes + kSlab)[j];
  };
  int e = INT_MIN / 4;
  std::uint32_t cnt = 1;
  for (std::uint32_t t = nb_off[Q]; t < nb_off[Q + 1]; ++t, ++cnt) {
    const std::uint32_t v = nb[t], P = v & 0x7fffffffu;
    e = max(e, (v >> 31) ? xe(xt, P) + 7 : erq[Q] + xe(xd, P) + 7);
  }
  (void)edq;               // (the diagonal term is added in fp64 after the conversion)
  if (e < -1000) e = 0;  // no contribution at all
  escale[Q * 16 + j] = e + (32 - __clz(cnt + 1)) + 1;
}

// Y = yint 2^(escale - 62) (one rounding, deterministic) + D X for the
// columns of this call; yint is zeroed for the next call.
__global__ void __launch_bounds__(256) yint_to_y_kernel(long long* yint, const int* escale,
                                                       const std::uint32_t* panel_start, const float* diag,
                                                       const double* x, std::uint32_t ldx, double* y, std::uint32_t ldy,
                                                       std::uint32_t mc, std::uint32_t row_base, std::uint32_t q_base) {
  __shared__ double t[16][kTD + 1];  // [column][row], transposed through shared memory
  __shared__ double sc[16];
  const std::uint32_t Q = blockIdx.x + q_base;
  const std::uint32_t q0 = panel_start[Q], rows = panel_start[Q + 1] - q0;
  long long* yi = yint + static_cast<std::size_t>(Q) * kTD * 16;
  const int tid = threadIdx.x;
  if (tid < 16) sc[tid] = pow2(escale[Q * 16 + tid] - 62);
  long long v[kTD * 16 / 256];
#pragma unroll
  for (int u = 0; u < kTD * 16 / 256; ++u) v[u] = __ldcg(yi + tid + 256 * u);  // coalesced
#pragma unroll
  for (int u = 0; u < kTD * 16 / 256; ++u) __stcg(yi + tid + 256 * u, 0ll);   // cleared for the next call
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kTD * 16 / 256; ++u) {  // yint is [row quarter][column][32 rows]
    const int e = tid + 256 * u, c = (e >> 5) & 15, r = ((e >> 9) << 5) | (e & 31);
    t[c][r] = __ll2double_rn(v[u]) * sc[c];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kTD * 16 / 256; ++u) {  // Y rows: coalesced writes
    const int e = tid + 256 * u, r = e >> 4, c = e & 15;
    if (r < static_cast<int>(rows) && c < static_cast<int>(mc)) {
      // + d_r x_r in fp64 (Inf/NaN x: the caller's fix-up adds it)
      const double xv = x[static_cast<std::size_t>(q0 + r) * ldx + c];
      y[static_cast<std::size_t>(q0 + r - row_base) * ldy + c] =
          fma(static_cast<double>(diag[q0 + r]), isfinite(xv) ? xv : 0.0, t[c][r]);
    }
  }
}

struct SlicedArgs {
  const OzItem* items;
  const std::uint32_t* cta_beg;  // per CTA: its items [cta_beg[b], cta_end[b]) of this launch
  const std::uint32_t* cta_end;
  const std::uint8_t* dense;  // every item's dense slice planes (five, or four + list4)
  const std::uint32_t* list4;
  const std::uint8_t* xd;
  const std::uint8_t* xt;
  const int* rowexp;
  const float* diag;
  const double* x;  // the call's X (the diagonal term d_r x_r)
  long long* yint;     // fixed-point Y, [panel][row quarter][column][32 rows], units 2^(escale - 62)
  const int* escale;   // [panel][column]
  std::uint32_t ldx, mc;
  long long* trace;  // debug timeline (CIEG_SLICED_TRACE): CTA 0, 16 clock64 slots per item
  int ablate;        // timing-only (CIEG_SLICED_ABLATE, results invalid): 1 no transposed reduction, 2 planes of item 0 only
};

// (slabs hold the digits only -- every operand starts on a 1024-byte
// boundary: whole 128-byte core matrices; the column exponents are staged
// separately)
struct Smem {
  std::uint8_t planes[2][kPlanes];
  std::uint8_t xd[2][kSlab];
  std::uint8_t xt[2][kSlab];  // the owner panels' slabs (the next owner's is loaded while the current one's items run)
  // the slabs' column exponents, staged with them (4 deep: an epilogue reads
  // an item's exponents before it releases the item's accumulator stage)
  int xd_exp[4][16];
  int xt_exp[4][16];
  std::uint32_t list4[4][kL4Cap];  // sparse lowest slice: the lists of four consecutive items (bulk-copy targets, 16-byte aligned)
  std::uint64_t full_a[2], empty_a[2], full_t[2], empty_t[2], acc_full[2], acc_empty[2];
  std::uint64_t full_l[4];
  std::uint32_t tmem;
};

// exact int64 -> double for |v| < 2^51 (the 2^52 + 2^51 bias; no conversion unit)
__device__ __forceinline__ double l2d(long long v) {
  return __longlong_as_double(v + 0x4338000000000000ll) - 6755399441055744.0;
}

// sum_d D_d 2^(24 - 8 d) over the kDiag diagonal blocks at TMEM address taddr
// (8 columns of this warp's 32 lanes): the diagonals are combined exactly in
// int64 in two groups of four (|D_d| < 2^24, so each group is below 2^49) and
// the two groups are joined in fp64 with a single rounding.
template <typename Release>
__device__ __forceinline__ void recombine8(std::uint32_t taddr, double (&v)[8], Release release) {
  static_assert(kDiag == 8, "two groups of four diagonals");
  std::int32_t d0[8], d1[8], d2[8], d3[8];
  long long hi[8];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    umma::ld8(taddr + 16 * (4 * g), d0);
    umma::ld8(taddr + 16 * (4 * g + 1), d1);
    umma::ld8(taddr + 16 * (4 * g + 2), d2);
    umma::ld8(taddr + 16 * (4 * g + 3), d3);
    umma::ld_wait();
    if (g == 1) release();  // every diagonal is in registers: the accumulator stage goes back before the arithmetic
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const long long w = static_cast<long long>(d3[j]) + (static_cast<long long>(d2[j]) << 8) +
                          (static_cast<long long>(d1[j]) << 16) + (static_cast<long long>(d0[j]) << 24);
      if (g == 0)
        hi[j] = w;
      else
        v[j] = fma(l2d(w), 0x1p-32, l2d(hi[j]));
    }
  }
}

// ---- fixed-point accumulation into yint: 64-bit integer adds in L2
// (red.global.add.u64 -- exact, so the result does not depend on their order)
// v 2^e rounded to the nearest integer (|result| < 2^62 by the scale bounds)
__device__ __forceinline__ long long fixp(double v, int e) { return __double2ll_rn(v * pow2(e)); }

#define TRACE(item, slot, cond)                                                                      \
  do {                                                                                               \
    if (a.trace && blockIdx.x == 0 && (cond) && (item) - i_beg < 256)                                \
      a.trace[((item) - i_beg) * 16 + (slot)] = clock64();                                           \
  } while (0)

// CTA: 18 warps (one per SM). Warp 0 issues the MMAs, warp 1 the bulk copies;
// warps 2..17 are the epilogue, four per TMEM lane quarter (warp & 3):
// row part columns 0-7 / 8-15, transposed part columns 0-7 / 8-15.
constexpr int kWarps = 18;
constexpr int kThreads = 32 * kWarps;
constexpr int kEpiWarps = 16;

template <bool S4>
__global__ void __launch_bounds__(kThreads, 1) spmm_sliced_kernel(const SlicedArgs a) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::uint32_t i_beg = a.cta_beg[blockIdx.x], i_end = a.cta_end[blockIdx.x];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&S.full_a[b], S4 ? 2 : 1);  // the copies' expect_tx arrival (+ the scattered lowest slice)
      umma::mbar_init(&S.empty_a[b], 1);

      umma::mbar_init(&S.acc_full[b], 1);
      umma::mbar_init(&S.acc_empty[b], kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&S.full_t[b], 1);
      umma::mbar_init(&S.empty_t[b], 1);
    }
    for (int b = 0; b < 4; ++b) umma::mbar_init(&S.full_l[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (S4) {  // the lowest-slice planes start as zeros (each item's entries are scattered in and wiped again)
    for (int b = 0; b < 2; ++b) {
      uint4* z = reinterpret_cast<uint4*>(S.planes[b] + (kAS - 1) * kPlane);
      for (int u = tid; u < kPlane / 16; u += kThreads) z[u] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc<512>(&S.tmem);
  umma::fence_before();
  __syncthreads();
  // Diagonal kDiag - 1 is first written by slice 1 (slice 0's MMA covers
  // d < kXD only), so it accumulates onto TMEM that must start at zero: each
  // epilogue warp clears its 8 columns of it in both stages here and again
  // after reading a stage.
  const int eq = warp & 3, role = (warp - 2) >> 2, orient = role >> 1, half = role & 1;
  const std::uint32_t ecol = (static_cast<std::uint32_t>(32 * eq) << 16) + orient * kND + 8 * half;
  if (warp >= 2) {
    umma::fence_after();
    umma::st8_zero(S.tmem + ecol + 16 * (kDiag - 1));
    umma::st8_zero(S.tmem + ecol + kStageCols + 16 * (kDiag - 1));
    umma::st_wait();
    umma::fence_before();
  }
  __syncthreads();
  umma::fence_after();
  const std::uint32_t tbase = S.tmem;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issue
    // The whole warp runs the issue loop converged, descriptors are
    // warp-uniform (base descriptor + constant offsets, in uniform
    // registers), one elected lane executes each tcgen05.mma.
    std::uint32_t k = 0, owners = 0;
    const std::uint64_t a_k0 = umma::sdesc(umma::smem_u32(S.planes[0]), 128, 1024);   // A K-major (H X)
    const std::uint64_t a_mn0 = umma::sdesc(umma::smem_u32(S.planes[0]), 1024, 128);  // A MN-major (H^T X)
    const std::uint64_t b_d0 = umma::sdesc(umma::smem_u32(S.xd[0]), 128, 1024);
    const std::uint64_t b_t0 = umma::sdesc(umma::smem_u32(S.xt[0]), 128, 1024);
    int o = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      TRACE(i, 0, lane == 0);
      umma::mbar_wait(&S.full_a[b], (k >> 1) & 1u);
      TRACE(i, 1, lane == 0);
      umma::mbar_wait(&S.acc_empty[b], ((k >> 1) & 1u) ^ 1u);
      TRACE(i, 2, lane == 0);
      umma::fence_after();
      const std::uint32_t d_row = tbase + b * kStageCols, d_tr = d_row + kND;
      const bool trans = (it.flags & 0xffu) == 0u;
      // descriptor start-address field: (byte offset) >> 4, no carry out of 14 bits
      const std::uint64_t ab = static_cast<std::uint64_t>(b * (kPlanes >> 4));
      const std::uint64_t bd = b_d0 + static_cast<std::uint64_t>(b * (kSlab >> 4));
      // row part first: at an owner's first item it covers the owner slab's load
      // (CIEG_ABLATE_ROW_MMA / CIEG_ABLATE_TRANS_MMA: timing-only builds without one orientation's MMAs)
#pragma unroll 1
#ifdef CIEG_ABLATE_ROW_MMA
      for (int s = 0; s < 0; ++s) {
#else
      for (int s = 0; s < kAS; ++s) {
#endif
        const int n = 16 * min(kXD, kDiag - s);  // digits t with s + t < kDiag
        const std::uint32_t id_row = umma::idesc_i8(1, 1, 0, 0, 128, n);  // balanced digits: all signed
#pragma unroll
        for (int ks = 0; ks < kTD / 32; ++ks)
          umma::mma_i8_warp(d_row + 16 * s, a_k0 + ab + ((s * kPlane + 256 * ks) >> 4), bd + ((256 * ks) >> 4), id_row,
                            (s | ks) != 0);
      }
      if ((it.flags >> 8) & 1u) {
        o = owners & 1;
        umma::mbar_wait(&S.full_t[o], (owners >> 1) & 1u);
        ++owners;
        umma::fence_after();
      }
      const std::uint64_t bt = b_t0 + static_cast<std::uint64_t>(o * (kSlab >> 4));
#ifdef CIEG_ABLATE_TRANS_MMA
      if (false) {
#else
      if (trans) {
#endif
#pragma unroll 1
        for (int s = 0; s < kAS; ++s) {
          const int n = 16 * min(kXD, kDiag - s);
          const std::uint32_t id_tr = umma::idesc_i8(1, 1, 1, 0, 128, n);
#pragma unroll
          for (int ks = 0; ks < kTD / 32; ++ks)
            umma::mma_i8_warp(d_tr + 16 * s, a_mn0 + ab + ((s * kPlane + 4096 * ks) >> 4), bt + ((256 * ks) >> 4),
                              id_tr, (s | ks) != 0);
        }
      }
      umma::commit_warp(&S.empty_a[b]);
      umma::commit_warp(&S.acc_full[b]);
      if ((it.flags >> 9) & 1u) umma::commit_warp(&S.empty_t[o]);
      TRACE(i, 3, lane == 0);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ bulk-copy issue
    // One lane streams each item's five slice planes (built once per matrix;
    // evict-first, so the X digit slabs of the sector band stay in L2) and
    // the partner's X digit slab into a free buffer; the owner's slab when a
    // new owner panel starts.
    std::uint32_t k = 0, owners = 0;
    const std::uint64_t stream = umma::createpolicy_evict_first();
    // the X digit slabs are re-read by every item of the sector band: keep them
    const std::uint64_t keep = umma::createpolicy_evict_last();
    constexpr int kDense = S4 ? kAS - 1 : kAS;  // planes streamed dense
    // sparse lowest slice: item k's list sits in ring slot k & 3 (requested one
    // item ahead); n4 of items k, k - 1, k - 2
    std::uint32_t n4 = 0, n4_p1 = 0, n4_p2 = 0;
    auto list_bytes = [](std::uint32_t n) { return std::max<std::uint32_t>(16u, (4u * n + 15u) & ~15u); };
    auto request_list = [&](std::uint32_t i, std::uint32_t kk, std::uint32_t n) {
      umma::mbar_arrive_tx(&S.full_l[kk & 3], list_bytes(n));
      umma::bulk_g2s(S.list4[kk & 3], a.list4 + static_cast<std::size_t>((a.ablate & 2) ? 0 : i) * kL4Cap,
                     list_bytes(n), &S.full_l[kk & 3]);
    };
    if (S4 && i_beg < i_end) {
      n4 = a.items[i_beg].pad;
      if (lane == 0) request_list(i_beg, 0, n4);
    }
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      TRACE(i, 8, lane == 0);
      if (((it.flags >> 8) & 1u) && lane == 0) {  // (the owner before last read this buffer until empty_t)
        const int o = owners & 1;
        umma::mbar_wait(&S.empty_t[o], ((owners >> 1) & 1u) ^ 1u);
        umma::mbar_arrive_tx(&S.full_t[o], kSlab + 64);
        const std::uint8_t* src = a.xt + static_cast<std::size_t>(it.owner) * kSlabBytes;
        umma::bulk_g2s_hint(S.xt[o], src, kSlab, &S.full_t[o], keep);
        umma::bulk_g2s(S.xt_exp[owners & 3], src + kSlab, 64, &S.full_t[o]);
      }
      if ((it.flags >> 8) & 1u) ++owners;
      if (S4 || lane == 0) umma::mbar_wait(&S.empty_a[b], ((k >> 1) & 1u) ^ 1u);
      TRACE(i, 4, lane == 0);
      if (lane == 0) {
        umma::mbar_arrive_tx(&S.full_a[b], kSlab + 64 + kDense * kPlane);
        const std::uint8_t* xsrc = a.xd + static_cast<std::size_t>(it.partner) * kSlabBytes;
        umma::bulk_g2s_hint(S.xd[b], xsrc, kSlab, &S.full_a[b], keep);
        umma::bulk_g2s(S.xd_exp[k & 3], xsrc + kSlab, 64, &S.full_a[b]);
        const std::uint8_t* src = a.dense + static_cast<std::size_t>((a.ablate & 2) ? 0 : i) * (kDense * kPlane);
#pragma unroll 1
        for (int s = 0; s < kDense; ++s)
          umma::bulk_g2s_hint(S.planes[b] + s * kPlane, src + s * kPlane, kPlane, &S.full_a[b], stream);
      }
      if (S4) {
        std::uint8_t* p4 = S.planes[b] + (kAS - 1) * kPlane;
        // wipe the entries of the item that used this buffer last (k - 2)
        if (k >= 2)
          for (std::uint32_t e = lane; e < n4_p2; e += 32) p4[S.list4[(k - 2) & 3][e] & 0xffffu] = 0;
        __syncwarp();
        // request the next item's list (its ring slot held item k - 3's, wiped one item ago)
        std::uint32_t n4_next = 0;
        if (i + 1 < i_end) {
          n4_next = a.items[i + 1].pad;
          if (lane == 0) request_list(i + 1, k + 1, n4_next);
        }
        umma::mbar_wait(&S.full_l[k & 3], (k >> 2) & 1u);
        for (std::uint32_t e = lane; e < n4; e += 32) {
          const std::uint32_t v = S.list4[k & 3][e];
          p4[v & 0xffffu] = static_cast<std::uint8_t>(v >> 16);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> the tensor core's reads
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(&S.full_a[b]);
        n4_p2 = n4_p1;
        n4_p1 = n4;
        n4 = n4_next;
      }
      TRACE(i, 7, lane == 0);
    }
  } else if (orient == 0) {
    // ------------------------------------------------- row-part epilogue
    // (TMEM lanes = tile rows; 8 of the 16 columns per warp)
    const int r = 32 * eq + lane, j0 = 8 * half;
    double yacc[8];
    int er = 0, osc[8];
    std::uint32_t k = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      const int prow = static_cast<int>(it.flags >> 16);
      if ((it.flags >> 8) & 1u) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          yacc[j] = 0.0;
          osc[j] = __ldg(a.escale + it.owner * 16 + j0 + j);
        }
        er = r < prow ? a.rowexp[it.r0 + r] : 0;
      }
      TRACE(i, 9, lane == 0 && warp == 4);
      umma::mbar_wait(&S.acc_full[b], (k >> 1) & 1u);
      TRACE(i, 11, lane == 0 && warp == 4);
      umma::fence_after();
      int ex[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) ex[j] = S.xd_exp[k & 3][j0 + j];
      double v[8];
      recombine8(tbase + ecol + b * kStageCols, v, [&] {
        umma::st8_zero(tbase + ecol + b * kStageCols + 16 * (kDiag - 1));
        umma::st_wait();
        umma::fence_before();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(&S.acc_empty[b]);
        TRACE(i, 12, lane == 0 && warp == 4);
      });
      TRACE(i, 13, lane == 0 && warp == 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) yacc[j] = fma(v[j], pow2(er + ex[j] - 36), yacc[j]);
      TRACE(i, 10, lane == 0 && warp == 4);
      if (((it.flags >> 9) & 1u) && r < prow) {  // the owner's row part, in fixed point, added to yint
        unsigned long long* yr = reinterpret_cast<unsigned long long*>(a.yint) +
                                 static_cast<std::size_t>(it.owner) * kTD * 16 + eq * 512 + j0 * 32 + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          atomicAdd(yr + j * 32, static_cast<unsigned long long>(fixp(yacc[j], 62 - osc[j])));
      }
    }
  } else {
    // ------------------------------------------ transposed-part epilogue
    // (TMEM lanes = tile columns; 8 of the 16 columns per warp): the item's
    // contribution to its partner panel, in fixed point, added to yint with
    // coalesced 64-bit integer reds from the registers.
    const int c = 32 * eq + lane, j0 = 8 * half;
    std::uint32_t k = 0, owners = 0;
    for (std::uint32_t i = i_beg; i < i_end; ++i, ++k) {
      const OzItem it = a.items[i];
      const int b = k & 1;
      const bool trans = (it.flags & 0xffu) == 0u;
      if ((it.flags >> 8) & 1u) ++owners;
      int psc[8];
      if (trans) {
#pragma unroll
        for (int j = 0; j < 8; ++j) psc[j] = __ldg(a.escale + it.partner * 16 + j0 + j);
      }
      umma::mbar_wait(&S.acc_full[b], (k >> 1) & 1u);
      TRACE(i, 14, lane == 0 && warp == 12);
      umma::fence_after();
      int ex[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) ex[j] = S.xt_exp[(owners - 1) & 3][j0 + j];
      double v[8];
      auto release = [&] {
        umma::fence_before();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(&S.acc_empty[b]);
        TRACE(i, 15, lane == 0 && warp == 12);
      };
      if (trans) {
        recombine8(tbase + ecol + b * kStageCols, v, [&] {
          umma::st8_zero(tbase + ecol + b * kStageCols + 16 * (kDiag - 1));
          umma::st_wait();
          release();
        });
      } else {
        release();
      }
      if (!trans || (a.ablate & 1)) continue;
      if (c < static_cast<int>(it.orow)) {  // the contribution to the partner's rows, in fixed point
        unsigned long long* yr = reinterpret_cast<unsigned long long*>(a.yint) +
                                 static_cast<std::size_t>(it.partner) * kTD * 16 + eq * 512 + j0 * 32 + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          atomicAdd(yr + j * 32, static_cast<unsigned long long>(fixp(v[j], ex[j] - 36 + 62 - psc[j])));
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
  std::vector<std::uint32_t> sp(8ull * nitems);
  CIEG_CUDA(cudaMemcpy(sp.data(), m->sp_sched, sizeof(std::uint32_t) * sp.size(), cudaMemcpyDeviceToHost));
  const auto& ps = m->panel_start_host;
  // The single-pass items grouped by owner panel (a panel's items are
  // consecutive in the single-pass schedule), re-dealt in ascending panel
  // order, each panel to the least-loaded CTA (cost: a per-item charge +
  // a little per record): every CTA walks ascending panels and the grid sweeps the matrix
  // front to back, so the partner panels' X digit slabs of concurrent items
  // lie within one sector band and stay in L2.
  struct Run {
    std::uint32_t panel, first, count;
    std::uint64_t cost;
  };
  std::vector<Run> runs;
  for (std::uint32_t i = 0; i < nitems; ++i) {
    const std::uint32_t* d = sp.data() + 8ull * i;
    const std::uint32_t owner = panel_of(ps, d[7]);
    const std::uint64_t q0 = (static_cast<std::uint64_t>(d[1]) << 32) | d[0];
    const std::uint64_t q1 = (static_cast<std::uint64_t>(d[3]) << 32) | d[2];
    // (dense mode: every item streams the same plane bytes and MMA work)
    const std::uint64_t c = (4 * (q1 - q0) * ((d[4] & 0xffu) == 2u ? 2 : 1)) / 8 + 8192;
    if (runs.empty() || runs.back().panel != owner || ((d[4] >> 8) & 1u)) runs.push_back(Run{owner, i, 0, 0});
    ++runs.back().count;
    runs.back().cost += c;
  }
  std::stable_sort(runs.begin(), runs.end(), [](const Run& x, const Run& y) { return x.panel < y.panel; });
  const std::uint32_t ctas =
      std::max<std::uint32_t>(1, std::min<std::uint32_t>(m->sp_ctas, static_cast<std::uint32_t>(runs.size())));
  std::vector<std::pair<std::uint64_t, std::uint32_t>> heap;
  for (std::uint32_t b = 0; b < ctas; ++b) heap.push_back({0, b});
  auto cmp = [](const auto& x, const auto& y) { return x.first != y.first ? x.first > y.first : x.second > y.second; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  std::vector<std::vector<std::uint32_t>> runs_of(ctas);
  for (std::uint32_t r = 0; r < runs.size(); ++r) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    runs_of[heap.back().second].push_back(r);
    heap.back().first += runs[r].cost;
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  std::vector<std::uint32_t> order;  // new item -> single-pass item
  order.reserve(nitems);
  std::vector<std::uint32_t> cta_off(ctas + 1, 0);
  for (std::uint32_t b = 0; b < ctas; ++b) {
    for (std::uint32_t r : runs_of[b])
      for (std::uint32_t i = runs[r].first; i < runs[r].first + runs[r].count; ++i) order.push_back(i);
    cta_off[b + 1] = static_cast<std::uint32_t>(order.size());
  }
  std::vector<std::uint32_t> sched(8ull * nitems);  // the descriptors in the new order (records_kernel)
  for (std::uint32_t i = 0; i < nitems; ++i)
    std::copy(sp.begin() + 8ull * order[i], sp.begin() + 8ull * order[i] + 8, sched.begin() + 8ull * i);
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
    it.slot = order[i];
    it.pad = 0;
    it.rec0 = total;
    std::uint64_t n = 4 * (q1 - q0) * (kind == 2 ? 2 : 1);
    n = (n + 63) & ~63ull;  // whole 64-record interleave chunks
    it.nrec = static_cast<std::uint32_t>(n);
    total += n;
  }
  auto* pl = new SlicedPlan;
  try {
    pl->nrec = total;
    pl->items = upload(items);
    pl->ctas = ctas;
    pl->cta_off = upload(cta_off);
    pl->cta_off_host = cta_off;
    pl->item_owner_host.resize(nitems);
    for (std::uint32_t i = 0; i < nitems; ++i) pl->item_owner_host[i] = items[i].owner;
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
    std::vector<char> e_valid(rows);
    for (std::uint32_t r = 0; r < rows; ++r) e_valid[r] = eh[r] > 0;
    for (int& e : eh) e = e > 0 ? e - 2048 : 0;
    CIEG_CUDA(cudaMemcpy(pl->rowexp, eh.data(), sizeof(int) * rows, cudaMemcpyHostToDevice));
    unsigned bad_h = 0;
    CIEG_CUDA(cudaMemcpy(&bad_h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost));
    cudaFree(bad);
    pl->usable = bad_h == 0;
    std::uint32_t* dsched = upload(sched);
    const unsigned tiny_cap = static_cast<unsigned>(std::min<std::uint64_t>(1u << 30, m->nnz / 512 + 4096));
    Tiny* tiny = nullptr;
    CIEG_CUDA(cudaMalloc(&tiny, sizeof(Tiny) * tiny_cap));
    unsigned* ntiny = upload(std::vector<unsigned>{0u});
    if (nitems)
      records_kernel<<<nitems, 256, 0, ctx->stream>>>(pl->items, dsched, m->idx, static_cast<const float*>(m->val),
                                                      pl->rowexp, m->panel_start, pl->rec, pl->diag, tiny, ntiny,
                                                      tiny_cap);
    CIEG_CUDA(cudaGetLastError());
    unsigned nt = 0;
    CIEG_CUDA(cudaMemcpyAsync(&nt, ntiny, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (nt + 1 >= tiny_cap) {
      pl->usable = false;  // too many unsliceable entries: this matrix runs the fp64 DMMA kernels
    } else if (nt) {
      std::vector<Tiny> th(nt);
      CIEG_CUDA(cudaMemcpy(th.data(), tiny, sizeof(Tiny) * nt, cudaMemcpyDeviceToHost));
      std::sort(th.begin(), th.end(), [](const Tiny& a, const Tiny& b) { return a.out < b.out || (a.out == b.out && a.in < b.in); });
      std::vector<std::uint32_t> rows, off{0}, in(nt);
      std::vector<double> v(nt);
      for (unsigned t = 0; t < nt; ++t) {
        if (t == 0 || th[t].out != th[t - 1].out) {
          if (t) off.push_back(t);
          rows.push_back(th[t].out);
        }
        in[t] = th[t].in;
        v[t] = th[t].v;
      }
      off.push_back(nt);
      pl->ntiny_rows = static_cast<std::uint32_t>(rows.size());
      pl->tiny_rows = upload(rows);
      pl->tiny_rows_host = rows;
      pl->tiny_off = upload(off);
      pl->tiny_in = upload(in);
      pl->tiny_val = upload(v);
    }
    cudaFree(tiny);
    cudaFree(ntiny);
    cudaFree(dsched);
    ctx->launches += 2;
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(tpi);
    cudaFree(tpj);
    CIEG_CUDA(cudaMalloc(&pl->xd, static_cast<std::size_t>(m->npanels) * kSlabBytes));
    CIEG_CUDA(cudaMalloc(&pl->xt, static_cast<std::size_t>(m->npanels) * kSlabBytes));
    // The lowest slice as per-item lists when every item's fits (else five
    // dense planes; CIEG_SLICED_DENSE5=1 forces that).
    std::size_t free_b = 0, total_b = 0;
    static const bool dense5 = [] {
      const char* e = std::getenv("CIEG_SLICED_DENSE5");
      return e && std::atoi(e) != 0;
    }();
    if (nitems && pl->usable && !dense5 &&
        cudaMalloc(&pl->list4, sizeof(std::uint32_t) * kL4Cap * static_cast<std::size_t>(nitems)) == cudaSuccess) {
      unsigned* over = upload(std::vector<unsigned>{0u});
      list4_kernel<<<nitems, 256, 0, ctx->stream>>>(pl->items, pl->rec, pl->list4, over);
      CIEG_CUDA(cudaGetLastError());
      unsigned over_h = 0;
      CIEG_CUDA(cudaMemcpyAsync(&over_h, over, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
      CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(over);
      ++ctx->launches;
      pl->sparse4 = over_h == 0;
      if (!pl->sparse4) {
        cudaFree(pl->list4);
        pl->list4 = nullptr;
      }
    } else {
      cudaGetLastError();
      pl->list4 = nullptr;
    }
    // The dense slice planes of every item (16 KB each: 10 bytes per stored
    // entry with four planes at the generator's 40 % tile density) when they
    // fit in three quarters of the free memory; the records are dropped once
    // scattered. Otherwise the matrix keeps the fp64 DMMA kernels.
    const int nplanes = pl->sparse4 ? kAS - 1 : kAS;
    const std::size_t dense_bytes = static_cast<std::size_t>(nitems) * nplanes * kPlane;
    if (nitems && pl->usable && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && dense_bytes <= free_b / 4 * 3 &&
        cudaMalloc(&pl->dense, dense_bytes) == cudaSuccess) {
      dense_kernel<<<nitems, 256, 0, ctx->stream>>>(pl->items, pl->rec, pl->dense, nplanes);
      CIEG_CUDA(cudaGetLastError());
      CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
      ++ctx->launches;
    } else {
      cudaGetLastError();  // (a failed allocation: the DMMA kernels run)
      pl->dense = nullptr;
      pl->usable = false;
    }
    cudaFree(pl->rec);
    pl->rec = nullptr;
    if (pl->usable) {
      // neighbour lists and per-panel row / diagonal exponents (host)
      const std::uint32_t np = m->npanels;
      std::vector<std::vector<std::uint32_t>> nbs(np);
      for (const OzItem& it : items) {
        const std::uint32_t kind = it.flags & 0xffu;
        if (kind == 0u) {
          nbs[it.owner].push_back(it.partner);
          nbs[it.partner].push_back(it.owner | 0x80000000u);
        } else if (kind == 2u) {
          nbs[it.owner].push_back(it.owner);
        }
      }
      std::vector<std::uint32_t> off(np + 1, 0), flat;
      pl->nb_prefix_max.assign(np, 0);
      for (std::uint32_t q = 0; q < np; ++q) {
        flat.insert(flat.end(), nbs[q].begin(), nbs[q].end());
        off[q + 1] = static_cast<std::uint32_t>(flat.size());
        std::uint32_t hi = q;
        for (std::uint32_t v : nbs[q]) hi = std::max(hi, v & 0x7fffffffu);
        pl->nb_prefix_max[q] = q ? std::max(hi, pl->nb_prefix_max[q - 1]) : hi;
      }
      std::vector<float> dh(rows);
      CIEG_CUDA(cudaMemcpy(dh.data(), pl->diag, sizeof(float) * rows, cudaMemcpyDeviceToHost));
      std::vector<int> erq(np, INT_MIN / 4), edq(np, INT_MIN / 4);
      for (std::uint32_t q = 0; q < np; ++q)
        for (std::uint32_t r = ps[q]; r < ps[q + 1]; ++r) {
          if (e_valid[r]) erq[q] = std::max(erq[q], eh[r]);
          if (dh[r] != 0.0f) edq[q] = std::max(edq[q], std::ilogb(dh[r]) + 1);
        }
      pl->nb_off = upload(off);
      pl->nb = upload(flat);
      pl->erq = upload(erq);
      pl->edq = upload(edq);
      CIEG_CUDA(cudaMalloc(&pl->escale, sizeof(int) * np * 16));
      CIEG_CUDA(cudaMalloc(&pl->yint, sizeof(long long) * np * kTD * 16));
      CIEG_CUDA(cudaMemset(pl->yint, 0, sizeof(long long) * np * kTD * 16));
    }
  } catch (...) {
    delete pl;
    throw;
  }
  return pl;
}

// y[out] += sum h x[in] over the tiny entries of each output row (fixed
// order; non-finite x are left to the caller's non-finite fix-up).
__global__ void tiny_fix_kernel(const std::uint32_t* rows, const std::uint32_t* off, const std::uint32_t* in,
                                const double* val, std::uint32_t t_lo, std::uint32_t t_hi, const double* x,
                                std::uint32_t ldx, double* y, std::uint32_t ldy, std::uint32_t mc,
                                std::uint32_t row_base) {
  const std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  const std::uint32_t t = t_lo + (e >> 4), j = e & 15u;
  if (t >= t_hi || j >= mc) return;
  double s = 0.0;
  for (std::uint32_t k = off[t]; k < off[t + 1]; ++k) {
    const double xv = x[static_cast<std::size_t>(in[k]) * ldx + j];
    s = fma(val[k], isfinite(xv) ? xv : 0.0, s);
  }
  y[static_cast<std::size_t>(rows[t] - row_base) * ldy + j] += s;
}

}  // namespace

void launch_sliced_tiny_fix(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                            std::uint32_t ldy, std::uint32_t mc) {
  const SlicedPlan* pl = m->sliced;
  if (!pl || pl->ntiny_rows == 0) return;
  const std::uint32_t threads = pl->ntiny_rows * 16;
  tiny_fix_kernel<<<(threads + 255) / 256, 256, 0, ctx->stream>>>(pl->tiny_rows, pl->tiny_off, pl->tiny_in,
                                                                  pl->tiny_val, 0, pl->ntiny_rows, x, ldx, y, ldy, mc,
                                                                  m->row_lo);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

bool sliced_supported(const cieg_mat* m) {
  return m->precision == 0 && m->tile_edge == kTD && m->sp_sched != nullptr && m->row_lo == 0 &&
         m->row_hi == m->dim && (!m->sliced || m->sliced->usable);
}

bool sliced_ready(cieg_ctx* ctx, cieg_mat* m) {
  if (!sliced_supported(m)) return false;
  if (!m->sliced) m->sliced = build_plan(ctx, m);
  return m->sliced->usable;
}

void destroy_sliced(cieg_mat* m) {
  delete m->sliced;
  m->sliced = nullptr;
}

namespace {

void launch_digitize(cieg_ctx* ctx, const cieg_mat* m, SlicedPlan* pl, const double* x, std::uint32_t ldx,
                     std::uint32_t mc, unsigned* nonfinite, unsigned launch_id, std::uint32_t p_lo, std::uint32_t p_hi) {
  if (p_hi <= p_lo) return;
  digitize_kernel<<<p_hi - p_lo, 256, 0, ctx->stream>>>(x, ldx, mc, m->panel_start, pl->rowexp, pl->xd, pl->xt,
                                                        nonfinite, launch_id, p_lo);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

void launch_scales(cieg_ctx* ctx, SlicedPlan* pl, std::uint32_t q_lo, std::uint32_t q_hi) {
  if (q_hi <= q_lo) return;
  scales_kernel<<<q_hi - q_lo, 32, 0, ctx->stream>>>(pl->nb_off, pl->nb, pl->erq, pl->edq, pl->xd, pl->xt, pl->escale,
                                                     q_lo);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

// the main kernel over the items [beg[b], end[b]) of every CTA b
void launch_main(cieg_ctx* ctx, SlicedPlan* pl, const double* x, std::uint32_t ldx, std::uint32_t mc,
                 const std::uint32_t* beg, const std::uint32_t* end, long long* trace) {
  SlicedArgs args{pl->items, beg, end, pl->dense, pl->list4, pl->xd, pl->xt, pl->rowexp, pl->diag, x,
                  pl->yint,  pl->escale, ldx, mc, trace, 0};
  static const int ablate = [] {
    const char* e = std::getenv("CIEG_SLICED_ABLATE");
    return e ? std::atoi(e) : 0;
  }();
  args.ablate = ablate;
  constexpr std::size_t smem = sizeof(Smem) + 1024;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static const bool attr_set = [] {
    CIEG_CUDA(cudaFuncSetAttribute(spmm_sliced_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    CIEG_CUDA(cudaFuncSetAttribute(spmm_sliced_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    return true;
  }();
  (void)attr_set;
  if (pl->sparse4)
    spmm_sliced_kernel<true><<<pl->ctas, kThreads, smem, ctx->stream>>>(args);
  else
    spmm_sliced_kernel<false><<<pl->ctas, kThreads, smem, ctx->stream>>>(args);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

void launch_convert(cieg_ctx* ctx, const cieg_mat* m, SlicedPlan* pl, const double* x, std::uint32_t ldx, double* y,
                    std::uint32_t ldy, std::uint32_t mc, std::uint32_t q_lo, std::uint32_t q_hi) {
  if (q_hi <= q_lo) return;
  yint_to_y_kernel<<<q_hi - q_lo, 256, 0, ctx->stream>>>(pl->yint, pl->escale, m->panel_start, pl->diag, x, ldx, y,
                                                         ldy, mc, m->row_lo, q_lo);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

// the tiny-entry terms of the output rows [r_lo, r_hi)
void launch_tiny_rows(cieg_ctx* ctx, const cieg_mat* m, const SlicedPlan* pl, const double* x, std::uint32_t ldx,
                      double* y, std::uint32_t ldy, std::uint32_t mc, std::uint32_t r_lo, std::uint32_t r_hi) {
  const auto& tr = pl->tiny_rows_host;
  const std::uint32_t t_lo = static_cast<std::uint32_t>(std::lower_bound(tr.begin(), tr.end(), r_lo) - tr.begin());
  const std::uint32_t t_hi = static_cast<std::uint32_t>(std::lower_bound(tr.begin(), tr.end(), r_hi) - tr.begin());
  if (t_hi <= t_lo) return;
  const std::uint32_t threads = (t_hi - t_lo) * 16;
  tiny_fix_kernel<<<(threads + 255) / 256, 256, 0, ctx->stream>>>(pl->tiny_rows, pl->tiny_off, pl->tiny_in,
                                                                  pl->tiny_val, t_lo, t_hi, x, ldx, y, ldy, mc,
                                                                  m->row_lo);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

// Owner panels cut into chunks of about equal rows -- `want` of them over the
// matrix, the last quarter of the rows in half-size chunks (what is still to
// do once the last rows of X have arrived -- the band's kernels and the
// download of the rows that were waiting for them -- shrinks with the chunk
// size there); per chunk and CTA the item range (a CTA's items ascend by owner
// panel). Cached per `want`.
const SlicedPlan::Chunks& chunking(const cieg_mat* m, SlicedPlan* pl, std::uint32_t want) {
  const auto& ps = m->panel_start_host;
  const std::uint32_t np = m->npanels;
  want = std::max<std::uint32_t>(1, std::min(want, np));
  for (const auto& c : pl->chunkings)
    if (c.want == want) return c;
  SlicedPlan::Chunks ch;
  ch.want = want;
  ch.panel.push_back(0);
  // cuts in units of 1 / (2 want) of the rows: pairs of units up to 3/4, single units after
  for (std::uint32_t u = 1; u < 2 * want; ++u) {
    const bool tail = 4ull * u > 6ull * want;  // u / (2 want) > 3/4
    if (!tail && (u & 1u)) continue;
    const std::uint32_t row = static_cast<std::uint32_t>(static_cast<std::uint64_t>(m->dim) * u / (2ull * want));
    const std::uint32_t p = std::max(ch.panel.back(), panel_of(ps, row));
    if (p > ch.panel.back() && p < np) ch.panel.push_back(p);
  }
  ch.panel.push_back(np);
  const std::uint32_t nchunks = static_cast<std::uint32_t>(ch.panel.size() - 1);
  const std::uint32_t ctas = pl->ctas;
  std::vector<std::uint32_t> lim(static_cast<std::size_t>(nchunks + 1) * ctas);
  for (std::uint32_t b = 0; b < ctas; ++b) {
    const auto first = pl->item_owner_host.begin() + pl->cta_off_host[b];
    const auto last = pl->item_owner_host.begin() + pl->cta_off_host[b + 1];
    for (std::uint32_t c = 0; c <= nchunks; ++c)
      lim[static_cast<std::size_t>(c) * ctas + b] =
          static_cast<std::uint32_t>(std::lower_bound(first, last, ch.panel[c]) - pl->item_owner_host.begin());
  }
  ch.cta_lim = upload(lim);
  pl->chunkings.push_back(std::move(ch));
  return pl->chunkings.back();
}

}  // namespace

void launch_spmm_sliced(cieg_ctx* ctx, cieg_mat* m, const double* x, std::uint32_t ldx, double* y, std::uint32_t ldy,
                        std::uint32_t mc, unsigned* nonfinite, unsigned launch_id) {
  if (!sliced_ready(ctx, m))
    fail(CIEG_ERR_CONFIG, "sliced SpMM needs an unsharded fp32 matrix with 128-row panels and finite values");
  if (mc == 0 || mc > 16) fail(CIEG_ERR_ARGUMENT, "sliced SpMM: 1..16 columns per launch");
  SlicedPlan* pl = m->sliced;
  launch_digitize(ctx, m, pl, x, ldx, mc, nonfinite, launch_id, 0, m->npanels);
  launch_scales(ctx, pl, 0, m->npanels);
  static const char* trace_path = std::getenv("CIEG_SLICED_TRACE");
  long long* trace = nullptr;
  if (trace_path) {
    CIEG_CUDA(cudaMalloc(&trace, sizeof(long long) * 256 * 16));
    CIEG_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * 256 * 16, ctx->stream));
  }
  launch_main(ctx, pl, x, ldx, mc, pl->cta_off, pl->cta_off + 1, trace);
  if (trace) {  // debug: dump CTA 0's timeline
    std::vector<long long> h(256 * 16);
    CIEG_CUDA(cudaMemcpyAsync(h.data(), trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(trace);
    if (FILE* f = std::fopen(trace_path, "wb")) {
      std::fwrite(h.data(), sizeof(long long), h.size(), f);
      std::fclose(f);
    }
  }
  launch_convert(ctx, m, pl, x, ldx, y, ldy, mc, 0, m->npanels);
}

// ---- ci::spmm's host call on the sliced kernel, pipelined over row chunks.
//
// The stored triangle couples an owner panel P only to partner panels Q <= P,
// and the schedule sweeps the owner panels front to back. So the call is cut
// into chunks of owner panels: while chunk c's rows of X are on the wire
// (upload stream), the digits of the chunks before it are formed, every panel
// whose neighbours are all digitized gets its fixed-point scales, every chunk
// whose panels all have scales runs the main kernel, every panel whose
// contributing owners have all run is converted to fp64 and its rows of U go
// home on the download stream. Upload, kernels and download overlap; the
// fixed-point accumulation does not depend on the order of the additions, so
// the result is bitwise that of the one-launch call. For the block-banded
// sector matrices a panel's neighbours lie within +-2 sectors, so U trails X
// by about that band; for a matrix without such structure the pipeline
// degenerates to upload, compute, download.
//
// Pageable host buffers (the std::vector inside ci::BlockVectors) stream
// through pinned rings in both directions: the calling thread copies X into
// the upload ring, a helper thread (capi.cu) copies finished pieces of U out of
// the download ring, half the OpenMP threads each.
bool sliced_spmm_host(cieg_ctx* ctx, cieg_mat* m, const double* x_host, double* y_host, std::uint32_t mc,
                      bool x_pinned, bool y_pinned) {
  const bool shard = m->row_lo != 0 || m->row_hi != m->dim;
  if (shard || mc == 0 || mc > 16 || !sliced_rule(ctx, m, mc) || !sliced_ready(ctx, m)) return false;
  static const bool off = [] {
    const char* e = std::getenv("CIEG_HOST_PIPELINE");
    return e && std::atoi(e) == 0;
  }();
  if (off) return false;
  SlicedPlan* pl = m->sliced;
  const auto& ps = m->panel_start_host;
  const std::uint32_t np = m->npanels, n = m->dim;
  const std::size_t row_bytes = sizeof(double) * mc;
  constexpr std::size_t kChunkBytes = 8u << 20;  // ring slot size = upload chunk bound
  const std::size_t xbytes = static_cast<std::size_t>(n) * row_bytes;
  // about 16 MB of X per chunk, at most 32 chunks (measured on config 2: 16 chunks 7.9 ms, 32 8.0 ms, 48 8.3 ms
  // on pinned buffers; CIEG_HOST_CHUNKS overrides)
  std::uint32_t want = static_cast<std::uint32_t>(std::min<std::size_t>(32, (xbytes + kChunkBytes) / (2 * kChunkBytes)));
  if (const char* e = std::getenv("CIEG_HOST_CHUNKS")) want = static_cast<std::uint32_t>(std::max(1, std::atoi(e)));
  const auto& ch = chunking(m, pl, want);
  const std::uint32_t nch = static_cast<std::uint32_t>(ch.panel.size() - 1);
  double* dx = static_cast<double*>(ctx->scratch_x.get(xbytes));
  double* dy = static_cast<double*>(ctx->scratch_y.get(xbytes));
  if (!ctx->pipe_up) CIEG_CUDA(cudaStreamCreateWithFlags(&ctx->pipe_up, cudaStreamNonBlocking));
  if (!ctx->pipe_down) CIEG_CUDA(cudaStreamCreateWithFlags(&ctx->pipe_down, cudaStreamNonBlocking));
  std::size_t ev_next = 0;
  auto event = [&]() {
    if (ev_next == ctx->pipe_ev.size()) {
      cudaEvent_t e = nullptr;
      CIEG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->pipe_ev.push_back(e);
    }
    return ctx->pipe_ev[ev_next++];
  };
  constexpr int kUpSlots = 4, kDownSlots = 8;
  char* up_ring = x_pinned ? nullptr : static_cast<char*>(ctx->pinned_stage.get(kUpSlots * kChunkBytes));
  char* down_ring = y_pinned ? nullptr : static_cast<char*>(ctx->pinned_stage_down.get(kDownSlots * kChunkBytes));
  unsigned* flag = nonfinite_flag(ctx);
  const unsigned launch_id = ++ctx->spmm_launch_id;

  // nothing may touch dx / dy before the work already queued on the context stream
  cudaEvent_t e0 = event();
  CIEG_CUDA(cudaEventRecord(e0, ctx->stream));
  CIEG_CUDA(cudaStreamWaitEvent(ctx->pipe_up, e0, 0));
  CIEG_CUDA(cudaStreamWaitEvent(ctx->pipe_down, e0, 0));

  // host-side time split of the call (CIEG_HOST_TRACE=1: printed to stderr)
  static const bool host_trace = std::getenv("CIEG_HOST_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  double t_copy = 0, t_upwait = 0, t_downwait = 0, t_enqueue = 0;
  const auto t_begin = clk::now();
  auto since = [](clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); };
  // downloads in ring slots are copied out by the helper thread, in order
  const std::size_t jobs0 = y_pinned ? 0 : copier_submitted(ctx);
  std::size_t issued = 0;
  try {
  // rows [r_lo, r_hi) of U, ready on the context stream -> host
  auto download = [&](std::uint32_t r_lo, std::uint32_t r_hi) {
    if (r_hi <= r_lo) return;
    cudaEvent_t ready = event();
    CIEG_CUDA(cudaEventRecord(ready, ctx->stream));
    CIEG_CUDA(cudaStreamWaitEvent(ctx->pipe_down, ready, 0));
    const std::size_t b0 = r_lo * row_bytes, b1 = r_hi * row_bytes;
    if (y_pinned) {
      CIEG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(y_host) + b0, reinterpret_cast<const char*>(dy) + b0, b1 - b0,
                                cudaMemcpyDeviceToHost, ctx->pipe_down));
      return;
    }
    for (std::size_t o = b0; o < b1; o += kChunkBytes) {
      const std::size_t len = std::min(kChunkBytes, b1 - o);
      if (issued >= static_cast<std::size_t>(kDownSlots)) {  // the slot's last piece is home
        const auto t0 = clk::now();
        copier_wait(ctx, jobs0 + issued - kDownSlots + 1);
        t_downwait += since(t0);
      }
      char* slot = down_ring + (issued % kDownSlots) * kChunkBytes;
      CIEG_CUDA(cudaMemcpyAsync(slot, reinterpret_cast<const char*>(dy) + o, len, cudaMemcpyDeviceToHost, ctx->pipe_down));
      cudaEvent_t done = event();
      CIEG_CUDA(cudaEventRecord(done, ctx->pipe_down));
      copier_submit(ctx, done, reinterpret_cast<char*>(y_host) + o, slot, len);
      ++issued;
    }
  };

  const auto& pm = pl->nb_prefix_max;
  auto below = [&](std::uint32_t lim) {  // panels whose neighbours all lie below lim
    return lim >= np ? np : static_cast<std::uint32_t>(std::lower_bound(pm.begin(), pm.end(), lim) - pm.begin());
  };
  std::uint32_t scaled = 0, next_chunk = 0, computed = 0, converted = 0;
  std::vector<cudaEvent_t> up_done(kUpSlots, nullptr);
  std::size_t up_count = 0;
  for (std::uint32_t c = 0; c < nch; ++c) {
    const std::uint32_t p_lo = ch.panel[c], p_hi = ch.panel[c + 1];
    if (p_hi <= p_lo) continue;
    const std::size_t b0 = ps[p_lo] * row_bytes, b1 = (p_hi == np ? n : ps[p_hi]) * row_bytes;
    if (x_pinned) {
      CIEG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dx) + b0, reinterpret_cast<const char*>(x_host) + b0, b1 - b0,
                                cudaMemcpyHostToDevice, ctx->pipe_up));
    } else {
      for (std::size_t o = b0; o < b1; o += kChunkBytes) {
        const std::size_t len = std::min(kChunkBytes, b1 - o);
        const int s = static_cast<int>(up_count++ % kUpSlots);
        auto t0 = clk::now();
        if (up_done[s]) CIEG_CUDA(cudaEventSynchronize(up_done[s]));
        t_upwait += since(t0);
        t0 = clk::now();
        host_copy_in(up_ring + s * kChunkBytes, reinterpret_cast<const char*>(x_host) + o, len, !y_pinned);
        t_copy += since(t0);
        CIEG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dx) + o, up_ring + s * kChunkBytes, len,
                                  cudaMemcpyHostToDevice, ctx->pipe_up));
        up_done[s] = event();
        CIEG_CUDA(cudaEventRecord(up_done[s], ctx->pipe_up));
      }
    }
    const auto t_enq = clk::now();
    cudaEvent_t uploaded = event();
    CIEG_CUDA(cudaEventRecord(uploaded, ctx->pipe_up));
    CIEG_CUDA(cudaStreamWaitEvent(ctx->stream, uploaded, 0));
    launch_digitize(ctx, m, pl, dx, mc, mc, flag, launch_id, p_lo, p_hi);
    const std::uint32_t s_hi = below(p_hi);
    launch_scales(ctx, pl, scaled, s_hi);
    scaled = std::max(scaled, s_hi);
    while (next_chunk < nch && ch.panel[next_chunk + 1] <= scaled) {
      if (ch.panel[next_chunk + 1] > ch.panel[next_chunk])
        launch_main(ctx, pl, dx, mc, mc, ch.cta_lim + static_cast<std::size_t>(next_chunk) * pl->ctas,
                    ch.cta_lim + static_cast<std::size_t>(next_chunk + 1) * pl->ctas, nullptr);
      computed = ch.panel[++next_chunk];
    }
    const std::uint32_t y_hi = below(computed);
    if (y_hi > converted) {
      const std::uint32_t r_lo = ps[converted], r_hi = y_hi == np ? n : ps[y_hi];
      launch_convert(ctx, m, pl, dx, mc, dy, mc, mc, converted, y_hi);
      launch_tiny_rows(ctx, m, pl, dx, mc, dy, mc, mc, r_lo, r_hi);
      download(r_lo, r_hi);
      converted = y_hi;
    }
    t_enqueue += since(t_enq);
  }
  const double t_loop = since(t_begin);
  if (converted != np || next_chunk != nch) fail(CIEG_ERR_CUDA, "sliced host pipeline: incomplete schedule");
  // Inf/NaN in X (staged as zeros): the rare path -- the exact stored-entry
  // terms are added on the device and U is downloaded again, whole
  unsigned* flag_host = static_cast<unsigned*>(ctx->pinned_small.get(256));
  CIEG_CUDA(cudaMemcpyAsync(flag_host, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  if (!y_pinned) copier_wait(ctx, jobs0 + issued);
  CIEG_CUDA(cudaStreamSynchronize(ctx->pipe_down));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*flag_host == launch_id) {
    launch_nonfinite_fix(ctx, m, dx, mc, dy, mc, mc, launch_id);
    download(0, n);
    if (!y_pinned) copier_wait(ctx, jobs0 + issued);
    CIEG_CUDA(cudaStreamSynchronize(ctx->pipe_down));
  }
  if (host_trace)
    std::fprintf(stderr, "sliced_spmm_host: %u chunks, loop %.3f ms (copy-in %.3f, upload-slot waits %.3f, enqueue incl. "
                 "download-slot waits %.3f / %.3f), total %.3f ms\n", nch, t_loop, t_copy, t_upwait, t_enqueue, t_downwait,
                 since(t_begin));
  } catch (...) {
    if (!y_pinned) copier_drain(ctx);  // no copy into the caller's U after the call has failed
    throw;
  }
  return true;
}

}  // namespace cieg
