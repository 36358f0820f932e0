// stream_probe.cu -- is K1's producer stream limited by per-SM outstanding
// L1 misses? Streams 52 KB chunks at scattered offsets (the K1 item pattern)
// with one persistent 256-thread CTA per SM, three ways:
//   regs : register double buffer, 4 x 128-bit loads per thread per batch (K1 today)
//   tma  : cp.async.bulk into a shared-memory ring of S x 16 KB stages (mbarrier)
//   lin  : plain grid-stride 128-bit streaming read (the HBM ceiling)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int kThreads = 256;
constexpr int kChunk = 52 * 1024;  // bytes per item
constexpr int kStage = 16 * 1024;  // bytes per TMA stage

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kThreads, 1) regs_kernel(const uint4* buf, const uint64_t* offs, int items_per_cta,
                                                           uint32_t* out) {
  const uint64_t* my = offs + static_cast<uint64_t>(blockIdx.x) * items_per_cta;
  uint32_t acc = 0;
  constexpr int kQ = 4, kBatch = kQ * kThreads;          // quads per batch
  constexpr int kQuadsPerItem = kChunk / 16;              // 3328
  uint4 qa[kQ], qb[kQ];
  auto load = [&](int item, int q0, uint4 (&o)[kQ]) {
#pragma unroll
    for (int j = 0; j < kQ; ++j) {
      const int q = q0 + threadIdx.x + j * kThreads;
      o[j] = q < kQuadsPerItem ? __ldg(buf + my[item] / 16 + q) : make_uint4(0, 0, 0, 0);
    }
  };
  load(0, 0, qa);
  for (int it = 0; it < items_per_cta; ++it) {
    for (int q0 = 0;; q0 += kBatch) {
      const bool more = q0 + kBatch < kQuadsPerItem;
      if (more)
        load(it, q0 + kBatch, qb);
      else if (it + 1 < items_per_cta)
        load(it + 1, 0, qb);
#pragma unroll
      for (int j = 0; j < kQ; ++j) acc ^= qa[j].x ^ qa[j].y ^ qa[j].z ^ qa[j].w;
#pragma unroll
      for (int j = 0; j < kQ; ++j) qa[j] = qb[j];
      if (!more) break;
    }
  }
  out[blockIdx.x * kThreads + threadIdx.x] = acc;
}

template <int S>
__global__ void __launch_bounds__(kThreads, 1) tma_kernel(const uint8_t* buf, const uint64_t* offs, int items_per_cta,
                                                          uint32_t* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[S];
  const uint64_t* my = offs + static_cast<uint64_t>(blockIdx.x) * items_per_cta;
  constexpr int kStagesPerItem = (kChunk + kStage - 1) / kStage;  // 4 (last one partial)
  const int total = items_per_cta * kStagesPerItem;
  auto stage_bytes = [&](int k) {
    const int part = k % kStagesPerItem;
    return part + 1 < kStagesPerItem ? kStage : kChunk - part * kStage;
  };
  auto issue = [&](int k) {  // thread 0: copy stage k of the sequence into slot k % S
    const int slot = k % S;
    const int item = k / kStagesPerItem, part = k % kStagesPerItem;
    const uint32_t bytes = static_cast<uint32_t>(stage_bytes(k));
    const uint32_t mb = smem_addr(&full[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(smem + slot * kStage)),
        "l"(buf + my[item] + static_cast<uint64_t>(part) * kStage), "r"(bytes), "r"(mb)
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < S && k < total; ++k) issue(k);
  uint32_t acc = 0;
  for (int k = 0; k < total; ++k) {
    const int slot = k % S;
    const uint32_t parity = (k / S) & 1;
    const uint32_t mb = smem_addr(&full[slot]);
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(mb), "r"(parity)
          : "memory");
    const uint4* st = reinterpret_cast<const uint4*>(smem + slot * kStage);
    const int nq = stage_bytes(k) / 16;
    for (int q = threadIdx.x; q < nq; q += kThreads) {
      const uint4 v = st[q];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncthreads();  // slot consumed
    if (threadIdx.x == 0 && k + S < total) issue(k + S);
  }
  out[blockIdx.x * kThreads + threadIdx.x] = acc;
}

__global__ void lin_kernel(const uint4* buf, uint64_t nq, uint32_t* out) {
  uint32_t acc = 0;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq; q += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(buf + q);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 6400ull << 20;  // 6.4 GB, like K1's stored stream
  uint8_t* buf = nullptr;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  const int items_per_cta = static_cast<int>((2 * bytes) / kChunk / sms);  // 2 x the buffer, like owner-computes
  std::vector<uint64_t> offs(static_cast<size_t>(items_per_cta) * sms);
  std::mt19937_64 rng(1);
  for (auto& o : offs) o = (rng() % ((bytes - kChunk) / 16)) * 16;
  uint64_t* d_offs = nullptr;
  cudaMalloc(&d_offs, offs.size() * 8);
  cudaMemcpy(d_offs, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice);
  uint32_t* out = nullptr;
  cudaMalloc(&out, 1 << 24);
  const double streamed = double(items_per_cta) * sms * kChunk;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char* name, double b, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("%-10s %8.3f ms  %8.1f GB/s  (%s)\n", name, ms, b / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  report("lin", double(bytes), [&] { lin_kernel<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out); });
  report("regs", streamed, [&] {
    regs_kernel<<<sms, kThreads>>>(reinterpret_cast<const uint4*>(buf), d_offs, items_per_cta, out);
  });
  cudaFuncSetAttribute(tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStage);
  cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStage);
  cudaFuncSetAttribute(tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kStage);
  report("tma S=2", streamed, [&] { tma_kernel<2><<<sms, kThreads, 2 * kStage>>>(buf, d_offs, items_per_cta, out); });
  report("tma S=4", streamed, [&] { tma_kernel<4><<<sms, kThreads, 4 * kStage>>>(buf, d_offs, items_per_cta, out); });
  report("tma S=8", streamed, [&] { tma_kernel<8><<<sms, kThreads, 8 * kStage>>>(buf, d_offs, items_per_cta, out); });
  return 0;
}
