// DMMA throughput vs resident warps per SM scheduler (independent accumulators).
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps : {1, 2, 3, 4, 8}) {
    int threads = 32 * 4 * wps;  // 4 schedulers
    int iters = 4096;
    float ms;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); k<4><<<p.multiProcessorCount, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double fl = 2.0 * 256 * 4 * (double)iters * (threads / 32) * p.multiProcessorCount;
    float ms8;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); k<8><<<p.multiProcessorCount, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms8, e0, e1);
    }
    printf("warps/scheduler %d: 4 acc %.2f TF/s   8 acc %.2f TF/s\n", wps, fl / ms / 1e9, 2 * fl / ms8 / 1e9);
  }
  return 0;
}
