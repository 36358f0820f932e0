// blockvec.cu -- K2/K3/K4: the tall-skinny LOBPCG block kernels.
//
//   K2 gram     : L^T R over column-concatenated views ([X W P] without the
//                 hcat copies), FP64 tensor pipe (DMMA m8n8k4), each warp
//                 streams a contiguous row range, warp/block/grid partials are
//                 reduced in a fixed order (deterministic, like the
//                 reference's fixed panel order, block_vectors.cpp:74-85).
//   K3 combine  : out = [out] + [Y1 Y2 Y3] G with up to two output blocks, so
//                 X' = XG1 + WG2 + PG3 and P' = WG2 + PG3 come out of one pass
//                 (lobpcg.cpp:341-361); row-local, so it may run in place.
//                 Replaces linear_combination / add_linear_combination
//                 (block_vectors.cpp:101-160).
//   K4 residual : R = HX - X Theta (lobpcg.cpp:256-261).
#include <algorithm>
#include <cstring>

#include "blockvec.hpp"
#include "device_common.cuh"

namespace cieg {
namespace {

constexpr int kGramWarps = 8;

template <int MT, int NT>
struct GramUnroll {
  static constexpr int kU = (MT + NT) <= 4 ? 8 : ((MT + NT) <= 8 ? 4 : ((MT + NT) <= 10 ? 2 : 1));
};

// SYM (L and R the same view, MT == NT): the B fragments are the A
// fragments and only tiles nt >= mt are computed; the reduction mirrors the
// rest (tile (n, m) is the exact transpose of tile (m, n): same products,
// same accumulation order).
template <int MT, int NT, bool SYM = false>
__global__ void __launch_bounds__(32 * kGramWarps) gram_kernel(View3 L, View3 R, std::uint32_t n,
                                                               std::uint32_t rows_per_warp,
                                                               double* partials) {
  constexpr int MA = 8 * MT, NB = 8 * NT;
  constexpr int U = SYM ? GramUnroll<MT, 0>::kU : GramUnroll<MT, NT>::kU;  // SYM loads A only
  __shared__ double red[MA * NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;

  const double* pa[MT];
  std::uint32_t la[MT];
  const double* pb[NT];
  std::uint32_t lb[NT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    std::uint32_t c = 8 * mt + g;
    pa[mt] = nullptr;
    la[mt] = 0;
    for (int s = 0; s < L.nseg; ++s) {
      if (c < L.s[s].w) {
        pa[mt] = L.s[s].p + c;
        la[mt] = L.s[s].ld;
        break;
      }
      c -= L.s[s].w;
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    std::uint32_t c = 8 * nt + g;
    pb[nt] = nullptr;
    lb[nt] = 0;
    if (SYM) continue;
    for (int s = 0; s < R.nseg; ++s) {
      if (c < R.s[s].w) {
        pb[nt] = R.s[s].p + c;
        lb[nt] = R.s[s].ld;
        break;
      }
      c -= R.s[s].w;
    }
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  const std::uint64_t gw = static_cast<std::uint64_t>(blockIdx.x) * kGramWarps + warp;
  const std::uint64_t r0 = gw * rows_per_warp;
  const std::uint64_t r1 = std::min<std::uint64_t>(n, r0 + rows_per_warp);
  // U k-steps (4 rows each) of fragments are loaded before their DMMAs issue
  for (std::uint64_t i0 = r0; i0 < r1; i0 += 4 * U) {
    double a[U][MT], b[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const std::uint64_t i = i0 + 4 * u + q;
      const bool ok = i < r1;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[u][mt] = (ok && pa[mt]) ? __ldg(pa[mt] + i * la[mt]) : 0.0;
      if (!SYM) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[u][nt] = (ok && pb[nt]) ? __ldg(pb[nt] + i * lb[nt]) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (SYM && nt < mt) continue;
          dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[u][mt], SYM ? a[u][nt] : b[u][nt]);
        }
  }

  // warps fold their partials into one buffer in warp order (deterministic)
  for (int w = 0; w < kGramWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (SYM && nt < mt) continue;
          const int row = 8 * mt + g, col = 8 * nt + 2 * q;
          if (w == 0) {
            red[row * NB + col] = acc[mt][nt][0];
            red[row * NB + col + 1] = acc[mt][nt][1];
          } else {
            red[row * NB + col] += acc[mt][nt][0];
            red[row * NB + col + 1] += acc[mt][nt][1];
          }
        }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < MA * NB; e += 32 * kGramWarps)
    partials[static_cast<std::size_t>(blockIdx.x) * MA * NB + e] = red[e];
}

// out[a + kx*b] (column major) = sum over block partials: one warp per
// element, lane-strided partial sums then a fixed xor tree (deterministic).
__global__ void gram_reduce_kernel(const double* partials, int nblocks, int MA, int NB, int kx,
                                   int ky, int sym, double* out) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= kx * ky) return;
  int a = e % kx, b = e / kx;
  if (sym && (a >> 3) > (b >> 3)) {  // lower tile: read the mirrored upper entry
    const int t = a;
    a = b;
    b = t;
  }
  double s = 0.0;
  for (int k = lane; k < nblocks; k += 32) s += partials[static_cast<std::size_t>(k) * MA * NB + a * NB + b];
  s = warp_sum(s);
  if (lane == 0) out[e] = s;
}

template <int MT, int NT>
void launch_gram(cieg_ctx* ctx, std::uint32_t n, const View3& L, const View3& R, int blocks,
                 std::uint32_t rpw, double* partials) {
  gram_kernel<MT, NT><<<blocks, 32 * kGramWarps, 0, ctx->stream>>>(L, R, n, rpw, partials);
}

template <int MT>
void launch_gram_sym(cieg_ctx* ctx, std::uint32_t n, const View3& L, int blocks, std::uint32_t rpw,
                     double* partials) {
  gram_kernel<MT, MT, true><<<blocks, 32 * kGramWarps, 0, ctx->stream>>>(L, L, n, rpw, partials);
}

bool same_view(const View3& a, const View3& b) {
  if (a.nseg != b.nseg || a.width != b.width) return false;
  for (int s = 0; s < a.nseg; ++s)
    if (a.s[s].p != b.s[s].p || a.s[s].ld != b.s[s].ld || a.s[s].w != b.s[s].w) return false;
  return true;
}

using GramLauncher = void (*)(cieg_ctx*, std::uint32_t, const View3&, const View3&, int,
                              std::uint32_t, double*);

template <int MT, int... NTs>
constexpr GramLauncher pick_nt(int nt, std::integer_sequence<int, NTs...>) {
  GramLauncher table[] = {&launch_gram<MT, NTs + 1>...};
  return table[nt - 1];
}

GramLauncher gram_launcher(int mt, int nt) {
  using S = std::make_integer_sequence<int, 6>;
  switch (mt) {
    case 1: return pick_nt<1>(nt, S{});
    case 2: return pick_nt<2>(nt, S{});
    case 3: return pick_nt<3>(nt, S{});
    case 4: return pick_nt<4>(nt, S{});
    case 5: return pick_nt<5>(nt, S{});
    default: return pick_nt<6>(nt, S{});
  }
}

// ---------------------------------------------------------------- combine
constexpr int kCombineMaxG = 3712;  // doubles carried as a kernel parameter (<= 32 KB)

struct CombineParams {
  View3 in;
  Out2 out;
  std::uint32_t n, kin, kout;
  int accumulate;
  const double* g_dev;  // used when kin*kout > kCombineMaxG
  View3 L;              // fused Gram L^T out (combine_gram; unused for SYM)
  double* partials;     // fused Gram: per-CTA partials (8 LT x 8 OT)
  double g[kCombineMaxG];
};

constexpr int kCombineWarps = 8;

// LT > 0 fuses a Gram of the freshly computed output into the pass:
// L^T out (L a view over the same rows, LT = ceil(L.width / 8)) or, SYM,
// out^T out (upper tiles; mirrored by gram_reduce_kernel). Each warp stages
// its 8 output rows in shared memory to re-read them in fragment layout;
// per-warp partials are folded in warp order, per-CTA partials reduced in a
// fixed order (deterministic).
// Resident blocks per SM the register budget is capped for: the narrow
// variants are latency-bound streams and gain from occupancy (ncu, config 4).
// (0 = no constraint: the compiler's own register choice)
constexpr int combine_min_blocks(int ot, int lt, int ks) { return lt == 0 && ot <= 2 && ks <= 4 ? 4 : 0; }

template <int OT, int LT = 0, bool SYM = false, int KS = 12>
__global__ void __launch_bounds__(32 * kCombineWarps, combine_min_blocks(OT, LT, KS))
    combine_kernel(const __grid_constant__ CombineParams p) {
  constexpr int SG = 8 * OT + 4;
  constexpr int SO = 8 * OT + 4;  // staged output row stride
  extern __shared__ double gs[];  // [padded kin rows][SG] | LT: [warps][8][SO] | fold [8 LT][8 OT]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const double* gsrc = p.g_dev ? p.g_dev : p.g;

  // Stage G per segment with rows padded to a multiple of 4 (zero pad).
  int poff[3];
  {
    int off = 0, src = 0;
    for (int s = 0; s < p.in.nseg; ++s) {
      poff[s] = off;
      const int w = static_cast<int>(p.in.s[s].w), wp = (w + 3) & ~3;
      for (int e = threadIdx.x; e < wp * SG; e += blockDim.x) {
        const int k = e / SG, c = e - k * SG;
        gs[(off + k) * SG + c] =
            (k < w && c < static_cast<int>(p.kout)) ? gsrc[(src + k) + static_cast<std::size_t>(c) * p.kin] : 0.0;
      }
      off += wp;
      src += w;
    }
  }
  __syncthreads();
  int gsrows = 0;
  for (int s = 0; s < p.in.nseg; ++s) gsrows += (static_cast<int>(p.in.s[s].w) + 3) & ~3;
  double* ostage = gs + (gsrows > 4 ? gsrows : 4) * SG + warp * 8 * SO;
  constexpr int LTX = LT > 0 ? LT : 1;
  double gacc[LTX][OT][2];
  const double* pl[LTX];
  std::uint32_t ll[LTX];
  if constexpr (LT > 0) {
#pragma unroll
    for (int lt = 0; lt < LT; ++lt) {
#pragma unroll
      for (int nt = 0; nt < OT; ++nt) gacc[lt][nt][0] = gacc[lt][nt][1] = 0.0;
      pl[lt] = nullptr;
      ll[lt] = 0;
      if (!SYM) {
        std::uint32_t c = 8 * lt + g;
        for (int s = 0; s < p.L.nseg; ++s) {
          if (c < p.L.s[s].w) {
            pl[lt] = p.L.s[s].p + c;
            ll[lt] = p.L.s[s].ld;
            break;
          }
          c -= p.L.s[s].w;
        }
      }
    }
  }

  const std::uint64_t ngroups = (p.n + 7) / 8;
  // A fragments of a group of 8 rows, every segment at once (KS k-steps per
  // segment): thread (g, q) holds Y[row i0 + g][4 ks + q] of segment s.
  auto load_a = [&](std::uint64_t grp, double (&a)[3][KS]) {
    const std::uint64_t arow = grp * 8 + g;
    const bool rok = arow < p.n;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (s >= p.in.nseg) break;
      const double* base = p.in.s[s].p + arow * p.in.s[s].ld;
      const std::uint32_t w = p.in.s[s].w;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const std::uint32_t k = 4 * ks + q;
        a[s][ks] = (rok && k < w) ? base[k] : 0.0;
      }
    }
  };
  auto process = [&](std::uint64_t grp, const double (&a)[3][KS]) {
    const std::uint64_t i0 = grp * 8;
    double acc[OT][2];
    // C fragment rows i0 + g, columns 8 nt + 2q (+1)
    const std::uint64_t crow = i0 + g;
#pragma unroll
    for (int nt = 0; nt < OT; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = 0.0;
        const std::uint32_t c = 8 * nt + 2 * q + h;
        if (p.accumulate && crow < p.n && c < p.kout) {
          if (c < p.out.w0)
            v = p.out.o0[crow * p.out.ld0 + c];
          else
            v = p.out.o1[crow * p.out.ld1 + (c - p.out.w0)];
        }
        acc[nt][h] = v;
      }
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      if (s >= p.in.nseg) break;
      const int ksteps = static_cast<int>((p.in.s[s].w + 3) / 4);
      const double* gsb = gs + (poff[s] + q) * SG + g;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        if (ks >= ksteps) break;
#pragma unroll
        for (int nt = 0; nt < OT; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], a[s][ks], gsb[4 * ks * SG + 8 * nt]);
      }
    }
    if (crow < p.n) {
#pragma unroll
      for (int nt = 0; nt < OT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const std::uint32_t c = 8 * nt + 2 * q + h;
          if (c >= p.kout) continue;
          if (c < p.out.w0)
            p.out.o0[crow * p.out.ld0 + c] = acc[nt][h];
          else
            p.out.o1[crow * p.out.ld1 + (c - p.out.w0)] = acc[nt][h];
        }
    }
    if constexpr (LT > 0) {
      // stage the 8 output rows (zero beyond n / kout), then accumulate
      // L^T out over them: two k-steps of 4 rows
#pragma unroll
      for (int nt = 0; nt < OT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const std::uint32_t c = 8 * nt + 2 * q + h;
          ostage[g * SO + 8 * nt + 2 * q + h] = (crow < p.n && c < p.kout) ? acc[nt][h] : 0.0;
        }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 4 * u + q;
        const std::uint64_t row = i0 + r;
        double bfr[OT], afr[LTX];
#pragma unroll
        for (int nt = 0; nt < OT; ++nt) bfr[nt] = ostage[r * SO + 8 * nt + g];
#pragma unroll
        for (int lt = 0; lt < LT; ++lt)
          afr[lt] = SYM ? ostage[r * SO + 8 * lt + g] : ((row < p.n && pl[lt]) ? __ldg(pl[lt] + row * ll[lt]) : 0.0);
#pragma unroll
        for (int lt = 0; lt < LT; ++lt)
#pragma unroll
          for (int nt = 0; nt < OT; ++nt) {
            if (SYM && nt < lt) continue;
            dmma_8x8x4(gacc[lt][nt][0], gacc[lt][nt][1], afr[lt], bfr[nt]);
          }
      }
      __syncwarp();
    }
    };
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kCombineWarps;
  std::uint64_t grp = static_cast<std::uint64_t>(blockIdx.x) * kCombineWarps + warp;
  for (; grp < ngroups; grp += stride) {
    double a[3][KS];
    load_a(grp, a);
    process(grp, a);
  }
  if constexpr (LT > 0) {
    constexpr int MA = 8 * LT, NB = 8 * OT;
    double* red = gs + (gsrows > 4 ? gsrows : 4) * SG + kCombineWarps * 8 * SO;
    for (int w = 0; w < kCombineWarps; ++w) {
      if (warp == w) {
#pragma unroll
        for (int lt = 0; lt < LT; ++lt)
#pragma unroll
          for (int nt = 0; nt < OT; ++nt) {
            if (SYM && nt < lt) continue;
            const int row = 8 * lt + g, col = 8 * nt + 2 * q;
            if (w == 0) {
              red[row * NB + col] = gacc[lt][nt][0];
              red[row * NB + col + 1] = gacc[lt][nt][1];
            } else {
              red[row * NB + col] += gacc[lt][nt][0];
              red[row * NB + col + 1] += gacc[lt][nt][1];
            }
          }
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < MA * NB; e += 32 * kCombineWarps)
      p.partials[static_cast<std::size_t>(blockIdx.x) * MA * NB + e] = red[e];
  }
}

template <int OT, int LT = 0, bool SYM = false>
void launch_combine(cieg_ctx* ctx, const CombineParams& prm, int blocks) {
  constexpr int SG = 8 * OT + 4, SO = 8 * OT + 4;
  int rows = 0;
  for (int s = 0; s < prm.in.nseg; ++s) rows += (static_cast<int>(prm.in.s[s].w) + 3) & ~3;
  std::size_t smem = sizeof(double) * static_cast<std::size_t>(std::max(rows, 4)) * SG;
  if (LT > 0) smem += sizeof(double) * (static_cast<std::size_t>(kCombineWarps) * 8 * SO + 64 * LT * OT);
  // KS: k-steps per input segment (4 covers the <= 16-wide LOBPCG blocks)
  bool narrow = true;
  for (int s = 0; s < prm.in.nseg; ++s) narrow = narrow && prm.in.s[s].w <= 16;
  auto kern = narrow ? combine_kernel<OT, LT, SYM, 4> : combine_kernel<OT, LT, SYM, 12>;
  if (smem > 48 * 1024)
    CIEG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<blocks, 32 * kCombineWarps, smem, ctx->stream>>>(prm);
}

// ---------------------------------------------------------------- residual
// Index arithmetic in the element type I: 32-bit when the block has fewer
// than 2^32 elements (config 4: 8e7), which keeps the per-element column
// division off the 64-bit emulation path.
template <typename I>
__global__ void residual_kernel(I total, std::uint32_t k, const double* __restrict__ hx,
                                const double* __restrict__ x, const double* __restrict__ theta,
                                double* __restrict__ r) {
  for (I e = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<I>(gridDim.x) * blockDim.x) {
    const std::uint32_t j = static_cast<std::uint32_t>(e % k);
    r[e] = hx[e] - theta[j] * x[e];
  }
}

template <typename I>
__global__ void gather_kernel(I n, std::uint32_t ksrc, const double* __restrict__ src, std::uint32_t kd,
                              const std::uint32_t* __restrict__ cols, double* __restrict__ dst) {
  const I total = n * kd;
  for (I e = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<I>(gridDim.x) * blockDim.x) {
    const I i = e / kd;
    const std::uint32_t j = static_cast<std::uint32_t>(e - i * kd);
    dst[e] = __ldg(src + static_cast<std::size_t>(i) * ksrc + cols[j]);
  }
}

// Streaming elementwise kernels: 8 resident 256-thread blocks per SM (full
// occupancy) keep enough loads in flight for HBM.
int elementwise_grid(cieg_ctx* ctx, std::uint64_t total) {
  const std::uint64_t want = (total + 255) / 256;
  return static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, 8ull * ctx->sm_count)));
}

int grid_for(cieg_ctx* ctx, std::uint64_t work, int per_block) {
  const std::uint64_t want = (work + per_block - 1) / per_block;
  return static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, 4ull * ctx->sm_count)));
}

}  // namespace

namespace {

// Enqueue one Gram (partial kernel + fixed-order reduction) writing kx x ky
// doubles to dout; `part` selects a private region of the partials scratch
// so two Grams can be in flight before one D2H.
int enqueue_gram(cieg_ctx* ctx, std::uint32_t n, const View3& L, const View3& R, double* partials, double* dout) {
  const std::uint32_t kx = L.width, ky = R.width;
  const int MT = static_cast<int>((kx + 7) / 8), NT = static_cast<int>((ky + 7) / 8);
  // fixed decomposition: rows_per_warp multiple of 4, at most 4 blocks per SM
  const int max_blocks = 4 * ctx->sm_count;
  std::uint64_t rpw = (static_cast<std::uint64_t>(n) + max_blocks * kGramWarps - 1) / (max_blocks * kGramWarps);
  rpw = std::max<std::uint64_t>(64, (rpw + 3) & ~3ull);
  const int blocks = static_cast<int>(std::max<std::uint64_t>(1, (n + rpw * kGramWarps - 1) / (rpw * kGramWarps)));
  const int MA = 8 * MT, NB = 8 * NT;
  const bool sym = same_view(L, R);  // X^T X: upper tiles only, mirrored
  if (sym) {
    switch (MT) {
      case 1: launch_gram_sym<1>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
      case 2: launch_gram_sym<2>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
      case 3: launch_gram_sym<3>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
      case 4: launch_gram_sym<4>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
      case 5: launch_gram_sym<5>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
      default: launch_gram_sym<6>(ctx, n, L, blocks, static_cast<std::uint32_t>(rpw), partials); break;
    }
  } else {
    gram_launcher(MT, NT)(ctx, n, L, R, blocks, static_cast<std::uint32_t>(rpw), partials);
  }
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
  const int e = static_cast<int>(kx * ky);
  gram_reduce_kernel<<<(e + 3) / 4, 128, 0, ctx->stream>>>(partials, blocks, MA, NB, static_cast<int>(kx),
                                                                static_cast<int>(ky), sym ? 1 : 0, dout);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
  return e;
}

std::size_t gram_partials_doubles(cieg_ctx* ctx, std::uint32_t n) {
  const int max_blocks = 4 * ctx->sm_count;
  (void)n;
  return static_cast<std::size_t>(max_blocks) * 48 * 48 + 64;
}

}  // namespace

std::vector<double> gram(cieg_ctx* ctx, std::uint32_t n, const View3& L, const View3& R) {
  const std::uint32_t kx = L.width, ky = R.width;
  std::vector<double> out(static_cast<std::size_t>(kx) * ky, 0.0);
  if (kx == 0 || ky == 0) return out;
  if (kx > 48 || ky > 48) fail(CIEG_ERR_CONFIG, "gram: block width above 48");
  double* partials = static_cast<double*>(ctx->scratch_red.get(sizeof(double) * gram_partials_doubles(ctx, n)));
  double* dout = static_cast<double*>(ctx->scratch_small.get(sizeof(double) * 2 * 48 * 48));
  const int e = static_cast<int>(kx * ky);
  if (n > 0)
    enqueue_gram(ctx, n, L, R, partials, dout);
  else
    CIEG_CUDA(cudaMemsetAsync(dout, 0, sizeof(double) * e, ctx->stream));
  if (n == 0 && !nccl_active(ctx)) return out;
  if (nccl_active(ctx)) nccl_allreduce_sum(ctx, dout, static_cast<std::size_t>(e));  // sharded: sum over ranks
  double* pin = static_cast<double*>(ctx->pinned_small.get(sizeof(double) * 2 * 48 * 48));
  CIEG_CUDA(cudaMemcpyAsync(pin, dout, sizeof(double) * e, cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(out.data(), pin, sizeof(double) * e);
  return out;
}

// Two independent Grams with one D2H and one synchronisation.
std::pair<std::vector<double>, std::vector<double>> gram_pair(cieg_ctx* ctx, std::uint32_t n, const View3& L1,
                                                              const View3& R1, const View3& L2, const View3& R2) {
  if (L1.width == 0 || R1.width == 0 || L2.width == 0 || R2.width == 0 || n == 0)
    return {gram(ctx, n, L1, R1), gram(ctx, n, L2, R2)};
  if (L1.width > 48 || R1.width > 48 || L2.width > 48 || R2.width > 48)
    fail(CIEG_ERR_CONFIG, "gram: block width above 48");
  const std::size_t pd = gram_partials_doubles(ctx, n);
  double* partials = static_cast<double*>(ctx->scratch_red.get(sizeof(double) * 2 * pd));
  double* dout = static_cast<double*>(ctx->scratch_small.get(sizeof(double) * 2 * 48 * 48));
  const int e1 = enqueue_gram(ctx, n, L1, R1, partials, dout);
  const int e2 = enqueue_gram(ctx, n, L2, R2, partials + pd, dout + e1);
  if (nccl_active(ctx)) nccl_allreduce_sum(ctx, dout, static_cast<std::size_t>(e1 + e2));
  double* pin = static_cast<double*>(ctx->pinned_small.get(sizeof(double) * 2 * 48 * 48));
  CIEG_CUDA(cudaMemcpyAsync(pin, dout, sizeof(double) * (e1 + e2), cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<double> a(pin, pin + e1), b(pin + e1, pin + e1 + e2);
  return {std::move(a), std::move(b)};
}


namespace {

// Shared parameter setup of combine / combine_gram (G as a kernel parameter
// when it fits, else staged in device scratch).
CombineParams& setup_combine(cieg_ctx* ctx, std::uint32_t n, const View3& in, const double* g_host,
                             std::uint32_t kout, const Out2& out, bool accumulate) {
  static thread_local CombineParams prm;  // ~30 KB: keep off the stack
  const std::uint32_t kin = in.width;
  prm.in = in;
  prm.out = out;
  prm.n = n;
  prm.kin = kin;
  prm.kout = kout;
  prm.accumulate = accumulate ? 1 : 0;
  prm.L = View3{};
  prm.partials = nullptr;
  const std::size_t ng = static_cast<std::size_t>(kin) * kout;
  if (ng <= static_cast<std::size_t>(kCombineMaxG)) {
    std::memcpy(prm.g, g_host, sizeof(double) * ng);
    prm.g_dev = nullptr;
  } else {
    double* d = static_cast<double*>(ctx->scratch_small.get(sizeof(double) * ng));
    // (a copy from pageable memory returns once the source is staged: no
    // synchronisation needed before the caller reuses g_host)
    CIEG_CUDA(cudaMemcpyAsync(d, g_host, sizeof(double) * ng, cudaMemcpyHostToDevice, ctx->stream));
    prm.g_dev = d;
  }
  return prm;
}

}  // namespace

void combine(cieg_ctx* ctx, std::uint32_t n, const View3& in, const double* g_host, std::uint32_t kout,
             const Out2& out, bool accumulate) {
  if (n == 0 || kout == 0) return;
  if (kout > 48) fail(CIEG_ERR_CONFIG, "combine: output width above 48");
  for (int k = 0; k < in.nseg; ++k)
    if (in.s[k].w > 48) fail(CIEG_ERR_CONFIG, "combine: input segment wider than 48");
  if (out.w0 + out.w1 != kout) fail(CIEG_ERR_DIMENSION, "combine: output split mismatch");
  const std::uint32_t kin = in.width;
  if (kin == 0) {
    if (!accumulate) {  // Y * G with an empty Y is a zero block
      for (int k = 0; k < 2; ++k) {
        double* o = k == 0 ? out.o0 : out.o1;
        const std::uint32_t w = k == 0 ? out.w0 : out.w1, ld = k == 0 ? out.ld0 : out.ld1;
        if (!o || w == 0) continue;
        CIEG_CUDA(cudaMemset2DAsync(o, ld * sizeof(double), 0, w * sizeof(double), n, ctx->stream));
      }
    }
    return;
  }
  CombineParams& prm = setup_combine(ctx, n, in, g_host, kout, out, accumulate);
  const int OT = static_cast<int>((kout + 7) / 8);
  const int blocks = grid_for(ctx, (n + 7) / 8, kCombineWarps * 4);
  switch (OT) {
    case 1: launch_combine<1>(ctx, prm, blocks); break;
    case 2: launch_combine<2>(ctx, prm, blocks); break;
    case 3: launch_combine<3>(ctx, prm, blocks); break;
    case 4: launch_combine<4>(ctx, prm, blocks); break;
    case 5: launch_combine<5>(ctx, prm, blocks); break;
    default: launch_combine<6>(ctx, prm, blocks); break;
  }
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

namespace {

template <int OT, int... LTs>
void launch_fused_lt(cieg_ctx* ctx, const CombineParams& prm, int blocks, int lt, std::integer_sequence<int, LTs...>) {
  using L = void (*)(cieg_ctx*, const CombineParams&, int);
  L table[] = {&launch_combine<OT, LTs + 1, false>...};
  table[lt - 1](ctx, prm, blocks);
}

void launch_fused(cieg_ctx* ctx, const CombineParams& prm, int blocks, int ot, int lt, bool sym) {
  using S = std::make_integer_sequence<int, 4>;
  if (sym) {
    switch (ot) {
      case 1: launch_combine<1, 1, true>(ctx, prm, blocks); break;
      case 2: launch_combine<2, 2, true>(ctx, prm, blocks); break;
      case 3: launch_combine<3, 3, true>(ctx, prm, blocks); break;
      default: launch_combine<4, 4, true>(ctx, prm, blocks); break;
    }
    return;
  }
  switch (ot) {
    case 1: launch_fused_lt<1>(ctx, prm, blocks, lt, S{}); break;
    case 2: launch_fused_lt<2>(ctx, prm, blocks, lt, S{}); break;
    case 3: launch_fused_lt<3>(ctx, prm, blocks, lt, S{}); break;
    default: launch_fused_lt<4>(ctx, prm, blocks, lt, S{}); break;
  }
}

}  // namespace

std::vector<double> combine_gram(cieg_ctx* ctx, std::uint32_t n, const View3& in, const double* g_host,
                                 std::uint32_t kout, const Out2& out, bool accumulate, const View3* L) {
  const std::uint32_t kx = L ? L->width : kout;
  const int OT = static_cast<int>((kout + 7) / 8), LT = static_cast<int>((kx + 7) / 8);
  const bool fusable = n > 0 && kout > 0 && in.width > 0 && kx > 0 && OT <= 4 && LT <= 4;
  if (!fusable) {  // the two passes separately
    combine(ctx, n, in, g_host, kout, out, accumulate);
    const View3 ov = view({Seg{out.o0, out.ld0, out.w0}, Seg{out.o1, out.ld1, out.w1}});
    return gram(ctx, n, L ? *L : ov, ov);
  }
  for (int k = 0; k < in.nseg; ++k)
    if (in.s[k].w > 48) fail(CIEG_ERR_CONFIG, "combine: input segment wider than 48");
  if (out.w0 + out.w1 != kout) fail(CIEG_ERR_DIMENSION, "combine: output split mismatch");
  CombineParams& prm = setup_combine(ctx, n, in, g_host, kout, out, accumulate);
  const int blocks = grid_for(ctx, (n + 7) / 8, kCombineWarps * 4);
  const int MA = 8 * (L ? LT : OT), NB = 8 * OT;
  prm.L = L ? *L : View3{};
  prm.partials = static_cast<double*>(ctx->scratch_red.get(sizeof(double) * blocks * MA * NB + 64));
  launch_fused(ctx, prm, blocks, OT, LT, L == nullptr);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
  double* dout = static_cast<double*>(ctx->scratch_small.get(sizeof(double) * 48 * 48));
  const int e = static_cast<int>(kx * kout);
  gram_reduce_kernel<<<(e + 3) / 4, 128, 0, ctx->stream>>>(prm.partials, blocks, MA, NB, static_cast<int>(kx),
                                                                static_cast<int>(kout), L ? 0 : 1, dout);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
  std::vector<double> res(static_cast<std::size_t>(e));
  if (nccl_active(ctx)) nccl_allreduce_sum(ctx, dout, static_cast<std::size_t>(e));  // sharded: sum over ranks
  double* pin = static_cast<double*>(ctx->pinned_small.get(sizeof(double) * 48 * 48));
  CIEG_CUDA(cudaMemcpyAsync(pin, dout, sizeof(double) * e, cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(res.data(), pin, sizeof(double) * e);
  return res;
}

void residual(cieg_ctx* ctx, std::uint32_t n, std::uint32_t k, const double* hx, const double* x,
              const double* theta_host, double* r) {
  if (n == 0 || k == 0) return;
  double* th = static_cast<double*>(ctx->scratch_small.get(sizeof(double) * 64));
  // theta travels through a small pinned staging copy, ordered on the stream
  double* pin = static_cast<double*>(ctx->pinned_small.get(sizeof(double) * 48 * 48));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(pin, theta_host, sizeof(double) * k);
  CIEG_CUDA(cudaMemcpyAsync(th, pin, sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
  const std::uint64_t total = static_cast<std::uint64_t>(n) * k;
  if (total < (1ull << 32))
    residual_kernel<std::uint32_t><<<elementwise_grid(ctx, total), 256, 0, ctx->stream>>>(
        static_cast<std::uint32_t>(total), k, hx, x, th, r);
  else
    residual_kernel<std::uint64_t><<<elementwise_grid(ctx, total), 256, 0, ctx->stream>>>(total, k, hx, x, th, r);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

void gather_columns(cieg_ctx* ctx, std::uint32_t n, const double* src, std::uint32_t ksrc,
                    const std::vector<std::uint32_t>& cols, double* dst) {
  const std::uint32_t kd = static_cast<std::uint32_t>(cols.size());
  if (n == 0 || kd == 0) return;
  std::uint32_t* dc = static_cast<std::uint32_t*>(ctx->scratch_small.get(sizeof(std::uint32_t) * 64 + 64));
  std::uint32_t* pin = static_cast<std::uint32_t*>(ctx->pinned_small.get(sizeof(double) * 48 * 48));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(pin, cols.data(), sizeof(std::uint32_t) * kd);
  CIEG_CUDA(cudaMemcpyAsync(dc, pin, sizeof(std::uint32_t) * kd, cudaMemcpyHostToDevice, ctx->stream));
  const std::uint64_t total = static_cast<std::uint64_t>(n) * kd;
  if (total < (1ull << 32))
    gather_kernel<std::uint32_t><<<elementwise_grid(ctx, total), 256, 0, ctx->stream>>>(n, ksrc, src, kd, dc, dst);
  else
    gather_kernel<std::uint64_t><<<elementwise_grid(ctx, total), 256, 0, ctx->stream>>>(n, ksrc, src, kd, dc, dst);
  CIEG_CUDA(cudaGetLastError());
  ++ctx->launches;
}

}  // namespace cieg

// ------------------------------------------------------------------ C ABI
extern "C" {

int cieg_block_inner(cieg_ctx* ctx, uint32_t n, const double* x_dev, uint32_t kx, const double* y_dev,
                     uint32_t ky, double* out_host) {
  return cieg::guarded([&] {
    if (!ctx || (!out_host && kx && ky)) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_block_inner: null argument");
    auto g = cieg::gram(ctx, n, cieg::view({cieg::seg(x_dev, kx)}), cieg::view({cieg::seg(y_dev, ky)}));
    std::memcpy(out_host, g.data(), sizeof(double) * g.size());
  });
}

int cieg_linear_combination(cieg_ctx* ctx, uint32_t n, const double* y_dev, uint32_t kin,
                            const double* g_host, uint32_t kout, double* out_dev) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_linear_combination: null context");
    if (y_dev == out_dev && kin != kout)
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_linear_combination: in-place needs equal widths");
    cieg::combine(ctx, n, cieg::view({cieg::seg(y_dev, kin)}), g_host, kout, cieg::out1(out_dev, kout), false);
  });
}

int cieg_add_linear_combination(cieg_ctx* ctx, uint32_t n, double* y_dev, uint32_t ky, const double* x_dev,
                                uint32_t kx, const double* g_host) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_add_linear_combination: null context");
    cieg::combine(ctx, n, cieg::view({cieg::seg(x_dev, kx)}), g_host, ky, cieg::out1(y_dev, ky), true);
  });
}

int cieg_column_norms(cieg_ctx* ctx, uint32_t n, const double* x_dev, uint32_t k, double* out_host) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_column_norms: null context");
    auto v = cieg::view({cieg::seg(x_dev, k)});
    auto g = cieg::gram(ctx, n, v, v);
    for (uint32_t j = 0; j < k; ++j) out_host[j] = std::sqrt(g[j + static_cast<std::size_t>(k) * j]);
  });
}

}  // extern "C"
