// Does F2F.F64.F32 share the FP64 (DMMA) pipe? Half the warps run DMMA, half run F2F.
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
__device__ __forceinline__ void f2f_loop(double* out, int iters, float f0) {
  float f[8];
  unsigned long long acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = f0 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double d;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[j]));
      acc ^= __double_as_longlong(d);
      f[j] = __int_as_float(__float_as_int(f[j]) + 1);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (double)acc;
}
__global__ void k(double* out, int itm, int itf, int mode) {
  int w = threadIdx.x / 32;
  if (mode == 0) dmma_loop(out, itm);
  else if (mode == 1) f2f_loop(out, itf, threadIdx.x);
  else { if (w & 1) dmma_loop(out, itm); else f2f_loop(out, itf, threadIdx.x); }
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 4, threads = 512;
  float ms;
  for (int mode = 0; mode < 3; ++mode) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); k<<<blocks, threads>>>(out, 2048, 2048, mode); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("mode %d (%s): %.3f ms\n", mode, mode == 0 ? "all dmma" : mode == 1 ? "all f2f" : "half dmma / half f2f", ms);
  }
  return 0;
}
