// Microbenchmark: FP64 vector vs DMMA throughput, predicated DFMA, red.f64.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void k_dfma(double* out, int iters, double a) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
      x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}

// predicated DFMA: predicate warp-uniform false for half of the FMAs
__global__ void k_dfma_pred(double* out, int iters, double a, unsigned mask) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    unsigned m = mask ^ (unsigned)i;   // runtime, warp-uniform
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      unsigned mm = m >> (u*4);
      if (mm & 1) x0 = fma(x0, a, 1.0);
      if (mm & 2) x1 = fma(x1, a, 1.0);
      if (mm & 4) x2 = fma(x2, a, 1.0);
      if (mm & 8) x3 = fma(x3, a, 1.0);
      if (mm & 1) x4 = fma(x4, a, 1.0);
      if (mm & 2) x5 = fma(x5, a, 1.0);
      if (mm & 4) x6 = fma(x6, a, 1.0);
      if (mm & 8) x7 = fma(x7, a, 1.0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_f2f(double* out, const float* in, int iters) {
  float f = in[threadIdx.x];
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    float g = f + (float)i;
    s0 += (double)g; s1 += (double)(g*2.f); s2 += (double)(g*3.f); s3 += (double)(g*4.f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0+s1+s2+s3;
}

__global__ void k_red(double* y, size_t n, int iters) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  unsigned long long h = tid * 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < iters; ++i) {
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    size_t idx = (h % (n / 16)) * 16 + (threadIdx.x & 15);   // 16 consecutive doubles per half-warp
    atomicAdd(y + idx, 1.0);
  }
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  float* fin; CK(cudaMalloc(&fin, 4096)); CK(cudaMemset(fin, 0, 4096));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(out, iters, 0.999); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * blocks * threads * (double)iters * 64;
    printf("DFMA: %.3f ms  %.2f TFLOP/s\n", ms, fl / ms / 1e9);
  }
  for (unsigned mask : {0xFFFFFFFFu, 0x55555555u, 0x11111111u, 0u}) {
    cudaEventRecord(e0); k_dfma_pred<<<blocks, threads>>>(out, iters, 0.999, mask); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA pred mask %08x: %.3f ms (per 64 slots)\n", mask, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * (blocks * threads / 32);
    printf("DMMA m8n8k4: %.3f ms  %.2f TFLOP/s\n", ms, fl / ms / 1e9);
  }
  cudaEventRecord(e0); k_f2f<<<blocks, threads>>>(out, fin, iters * 4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("F2F+DADD: %.3f ms  %.2f Gconv/s\n", ms, 4.0 * blocks * threads * iters * 4 / ms / 1e6);
  size_t n = 32ull << 20; double* y; CK(cudaMalloc(&y, n * 8)); CK(cudaMemset(y, 0, n * 8));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_red<<<blocks, threads>>>(y, n, 256); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("red.f64 (16-contig groups): %.3f ms  %.2f Gred/s\n", ms, (double)blocks * threads * 256 / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
