// Are DMMA (FP64 tensor) and DFMA (FP64 vector) separate pipes? Run both in one kernel.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dfma_loop(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, 1.0);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mode 0: all dmma; 1: all dfma; 2: half warps dmma, half dfma
__global__ void k_mix(double* out, int it_mma, int it_fma, int mode) {
  int w = threadIdx.x / 32;
  bool do_mma = mode == 0 || (mode == 2 && (w & 1));
  if (do_mma) dmma_loop(out, it_mma); else dfma_loop(out, it_fma, 0.999);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 4, threads = 512;
  // per warp: dmma iteration = 8*256*2 flop*... per-thread view: 8 dmma * 512 flop / 32 = 128 flop/thread/iter
  // dfma iteration: 32 fma = 64 flop/thread/iter -> use it_fma = 2*it_mma for equal flops
  int itm = 2048, itf = 4096;
  float ms;
  for (int mode = 0; mode < 3; ++mode) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); k_mix<<<blocks, threads>>>(out, itm, itf, mode); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = (double)blocks * threads * 128.0 * itm;   // equal flops per thread in all modes
    printf("mode %d (%s): %.3f ms  %.2f TFLOP/s\n", mode, mode == 0 ? "dmma" : mode == 1 ? "dfma" : "half/half", ms, flops / ms / 1e9);
  }
  return 0;
}
