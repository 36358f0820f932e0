// umma_i8_probe.cu -- bring-up and throughput check of the tcgen05 kind::i8
// pattern K1's integer-slice path uses (paper_1609_01689_b200/csrc/umma.cuh):
// one 128x128 int8 tile in 8x16 core matrices read as a K-major A (H X) and
// as an MN-major A (H^T X), five A slices (top signed, lower unsigned)
// against seven signed X-digit blocks with the diagonal window (slice s:
// N = 16 (7 - s), D columns from 16 s). Checks every accumulator against the
// host, then times the per-tile MMA sequence.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1609_01689_b200/csrc -o umma_i8_probe umma_i8_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "umma.cuh"

using namespace cieg;

constexpr int kS = 5, kD = 7, kNB = 16 * kD;
constexpr int kPlane = 128 * 128;
constexpr int kBBytes = kNB * 128;

__host__ __device__ inline int offA(int r, int c) { return (r >> 3) * 1024 + (c >> 4) * 128 + (r & 7) * 16 + (c & 15); }
__host__ __device__ inline int offB(int n, int k) { return (n >> 3) * 1024 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15); }

// the sliced kernel's compact (rolled) issue loop
__device__ __noinline__ void issue_tile_rolled(std::uint32_t tmem, std::uint32_t a0, std::uint32_t b0, std::uint32_t bt0) {
#pragma unroll 1
  for (int s = 0; s < kS; ++s) {
    const int n = 16 * (kD - s);
    const std::uint32_t a = a0 + s * kPlane;
    const std::uint32_t id_row = umma::idesc_i8(s == 0, 1, 0, 0, 128, n);
    const std::uint32_t id_tr = umma::idesc_i8(s == 0, 1, 1, 0, 128, n);
#pragma unroll 1
    for (int ks = 0; ks < 4; ++ks) {
      umma::mma_i8(tmem + 16 * s, umma::sdesc(a + ks * 256, 128, 1024), umma::sdesc(b0 + ks * 256, 128, 1024), id_row,
                   s > 0 || ks > 0);
      umma::mma_i8(tmem + kNB + 16 * s, umma::sdesc(a + ks * 4096, 1024, 128), umma::sdesc(bt0 + ks * 256, 128, 1024),
                   id_tr, s > 0 || ks > 0);
    }
  }
}

// one tile: row part into columns [0, 112), transposed part into [112, 224)
__device__ void issue_tile(std::uint32_t tmem, std::uint32_t a0, std::uint32_t b0, std::uint32_t bt0) {
  // (tmem may carry a stage offset)
  for (int s = 0; s < kS; ++s) {
    const int n = 16 * (kD - s);
    const std::uint32_t a = a0 + s * kPlane;
    const std::uint32_t id_row = umma::idesc_i8(s == 0, 1, 0, 0, 128, n);
    const std::uint32_t id_tr = umma::idesc_i8(s == 0, 1, 1, 0, 128, n);
    for (int ks = 0; ks < 4; ++ks) {
      umma::mma_i8(tmem + 16 * s, umma::sdesc(a + ks * 256, 128, 1024), umma::sdesc(b0 + ks * 256, 128, 1024), id_row,
                   s > 0 || ks > 0);
      umma::mma_i8(tmem + kNB + 16 * s, umma::sdesc(a + ks * 4096, 1024, 128), umma::sdesc(bt0 + ks * 256, 128, 1024),
                   id_tr, s > 0 || ks > 0);
    }
  }
}

// mode: what the extra warps (blockDim > 128) do while the MMAs of the timed
// stream run -- 0 idle, 1 poll the stream's mbarrier (try_wait loop),
// 2 byte stores into a scratch shared buffer, 3 tcgen05.ld of the other
// TMEM half
__global__ void __launch_bounds__(512, 1) probe(const std::int8_t* gA, const std::int8_t* gB, const std::int8_t* gBt,
                                                std::int32_t* out, int reps, long long* cycles, int mode, int issue_mode) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  __shared__ __align__(8) std::uint64_t bar;
  __shared__ __align__(8) std::uint64_t sbar[2];
  __shared__ std::uint32_t tbase;
  std::uint8_t* sA = smem;
  std::uint8_t* sB = smem + kS * kPlane;
  std::uint8_t* sBt = sB + kBBytes;
  std::uint8_t* scratch = sBt + kBBytes;  // 32 KB
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid >= 128) {  // extra warps: interference during the timed stream
    __syncthreads();  // setup
    __syncthreads();  // checked tile done
    unsigned x = tid * 2654435761u;
    for (int it = 0;; ++it) {
      std::uint32_t ok = 0;
      asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok)
                   : "r"(umma::smem_u32(&bar)), "r"(1u));
      if (ok) break;
      if (mode == 1) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; }" ::"r"(umma::smem_u32(&bar)), "r"(1u));
      } else if (mode == 2) {
        for (int u = 0; u < 64; ++u) {
          x = x * 1664525u + 1013904223u;
          scratch[(x >> 8) & 32767] = static_cast<std::uint8_t>(x);
        }
      } else if (mode == 3) {
        std::int32_t v[16];
        umma::ld16(tbase + (static_cast<std::uint32_t>(32 * (warp & 3)) << 16) + 256 + 16 * (it & 7), v);
        umma::ld_wait();
        if (v[0] == 0x7fffffff) scratch[0] = 1;
      } else {
        __nanosleep(1000);
      }
    }
    __syncthreads();
    return;
  }
  for (int i = tid; i < kS * kPlane; i += 128) sA[i] = gA[i];
  for (int i = tid; i < kBBytes; i += 128) {
    sB[i] = gB[i];
    sBt[i] = gBt[i];
  }
  if (warp == 0) umma::tmem_alloc<512>(&tbase);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_u32(&sbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_u32(&sbar[1])));
  }
  umma::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const std::uint32_t tmem = tbase;
  const std::uint32_t a0 = umma::smem_u32(sA), b0 = umma::smem_u32(sB), bt0 = umma::smem_u32(sBt);
  auto wait_bar = [&](unsigned ph) {
    std::uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok)
                   : "r"(umma::smem_u32(&bar)), "r"(ph));
  };
  // the checked tile
  if (tid == 0) {
    issue_tile(tmem, a0, b0, bt0);
    umma::commit(&bar);
  }
  __syncwarp();
  wait_bar(0);
  umma::fence_after();
  for (int c0 = 0; c0 < 2 * kNB; c0 += 16) {
    std::int32_t v[16];
    umma::ld16(tmem + (static_cast<std::uint32_t>(32 * warp) << 16) + c0, v);
    umma::ld_wait();
    if (blockIdx.x == 0)
      for (int j = 0; j < 16; ++j) out[(32 * warp + (tid & 31)) * (2 * kNB) + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  // the timed stream: reps tiles issued back to back, one commit
  long long t0 = clock64(), t1;
  if (tid == 0) {
    if (issue_mode == 0) {
      for (int rep = 0; rep < reps; ++rep) issue_tile(tmem, a0, b0, bt0);
    } else {
      // issue_mode 1: a tcgen05.commit to a per-stage mbarrier after every tile;
      // issue_mode 2: also alternate two TMEM stages and wait for the commit of
      // tile k-2 before issuing tile k (the sliced kernel's hand-off)
      for (int rep = 0; rep < reps; ++rep) {
        const int st = rep & 1;
        if (issue_mode >= 2 && rep >= 2) {
          std::uint32_t ok = 0;
          while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(ok)
                         : "r"(umma::smem_u32(&sbar[st])), "r"(static_cast<unsigned>(((rep - 2) >> 1) & 1)));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (issue_mode == 3)
          issue_tile_rolled(tmem + st * 224, a0, b0, bt0);
        else
          issue_tile(tmem + (issue_mode == 2 ? st * 224 : 0), a0, b0, bt0);
        umma::commit(&sbar[st]);
      }
    }
    umma::commit(&bar);
  }
  __syncwarp();
  wait_bar(1);
  t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tmem);
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 2000;
  const int ctas = argc > 2 ? atoi(argv[2]) : 1;
  const int extra = argc > 3 ? atoi(argv[3]) : 0;  // extra warps
  const int mode = argc > 4 ? atoi(argv[4]) : 0;
  const int issue_mode = argc > 5 ? atoi(argv[5]) : 0;
  std::mt19937 rng(7);
  std::vector<std::int8_t> A(kS * kPlane), B(kBBytes), Bt(kBBytes);
  std::vector<int> a_val(kS * 128 * 128), b_val(kNB * 128), bt_val(kNB * 128);
  for (int s = 0; s < kS; ++s)
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        int v = s == 0 ? static_cast<int>(rng() % 256) - 128 : static_cast<int>(rng() % 256);  // s8 / u8
        if (rng() % 10 < 6) v = 0;  // 40 % dense
        a_val[(s * 128 + r) * 128 + c] = v;
        A[s * kPlane + offA(r, c)] = static_cast<std::int8_t>(v);
      }
  for (int n = 0; n < kNB; ++n)
    for (int k = 0; k < 128; ++k) {
      const int v = static_cast<int>(rng() % 256) - 128, w = static_cast<int>(rng() % 256) - 128;
      b_val[n * 128 + k] = v;
      bt_val[n * 128 + k] = w;
      B[offB(n, k)] = static_cast<std::int8_t>(v);
      Bt[offB(n, k)] = static_cast<std::int8_t>(w);
    }
  std::int8_t *dA, *dB, *dBt;
  std::int32_t* dOut;
  long long* dCyc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dBt, Bt.size());
  cudaMalloc(&dOut, sizeof(std::int32_t) * 128 * 2 * kNB);
  cudaMalloc(&dCyc, sizeof(long long));
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dBt, Bt.data(), Bt.size(), cudaMemcpyHostToDevice);
  const int smem = kS * kPlane + 2 * kBBytes + 32768;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<ctas, 128 + 32 * extra, smem>>>(dA, dB, dBt, dOut, reps, dCyc, mode, issue_mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("FAIL launch: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<std::int32_t> out(128 * 2 * kNB);
  long long cyc = 0;
  cudaMemcpy(out.data(), dOut, sizeof(std::int32_t) * out.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dCyc, sizeof(long long), cudaMemcpyDeviceToHost);
  long long bad = 0, first = -1;
  for (int m = 0; m < 128; ++m)
    for (int d = 0; d < kD; ++d)
      for (int j = 0; j < 16; ++j) {
        long long row = 0, tr = 0;
        for (int s = 0; s <= d && s < kS; ++s) {
          const int n = 16 * (d - s) + j;
          for (int k = 0; k < 128; ++k) {
            row += static_cast<long long>(a_val[(s * 128 + m) * 128 + k]) * b_val[n * 128 + k];
            tr += static_cast<long long>(a_val[(s * 128 + k) * 128 + m]) * bt_val[n * 128 + k];
          }
        }
        const std::int32_t gr = out[m * 2 * kNB + 16 * d + j], gt = out[m * 2 * kNB + kNB + 16 * d + j];
        if (gr != row || gt != tr) {
          if (first < 0) {
            first = m * 1000 + d * 100 + j;
            printf("mismatch m=%d d=%d j=%d: row %d vs %lld, trans %d vs %lld\n", m, d, j, gr, row, gt, tr);
          }
          ++bad;
        }
      }
  const double per_tile = static_cast<double>(cyc) / reps;
  printf("%s: %lld mismatches of %d; %.0f cycles per tile (40 MMAs, floor 1600) [ctas %d, extra warps %d, mode %d, issue %d]\n",
         bad ? "FAIL" : "PASS", bad, 128 * kD * 16, per_tile, ctas, extra, mode, issue_mode);
  return bad ? 1 : 0;
}
