// Does a guard-false DFMA cost FP64 pipe time? (warp-uniform vs per-lane predicates)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_pred(double* out, int iters, double a, unsigned seed) {
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = threadIdx.x + j;
  unsigned h = seed;
  for (int i = 0; i < iters; ++i) {
    h = h * 1664525u + 1013904223u;                 // warp-uniform LCG
    unsigned m;
    if (MODE == 0) m = 0xFFFFFFFFu;                 // all true
    else if (MODE == 1) m = 0u;                     // all false (uniform)
    else if (MODE == 2) m = h;                      // ~50% uniform
    else m = h ^ (threadIdx.x * 0x9E3779B9u);       // per-lane ~50%
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      unsigned mm = m >> (g * 8);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
                     "and.b32 t, %1, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
                     "@p fma.rn.f64 %0, %0, %2, 0d3FF0000000000000;\n\t}"
                     : "+d"(acc[j]) : "r"(mm), "d"(a), "n"(1 << (0)));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same, but predicates computed once per 16 FMAs (lower issue overhead).
template <int MODE>
__global__ void k_pred2(double* out, int iters, double a, unsigned seed) {
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = threadIdx.x + j;
  unsigned h = seed;
  for (int i = 0; i < iters; ++i) {
    h = h * 1664525u + 1013904223u;
    unsigned m;
    if (MODE == 0) m = 0xFFFFFFFFu;
    else if (MODE == 1) m = 0u;
    else if (MODE == 2) m = h;
    else m = h ^ (threadIdx.x * 0x9E3779B9u);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      unsigned mm = (m >> (g * 4)) & 1u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %16, 0;\n\t"
                   "@p fma.rn.f64 %0, %0, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %1, %1, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %2, %2, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %3, %3, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %4, %4, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %5, %5, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %6, %6, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %7, %7, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %8, %8, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %9, %9, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %10, %10, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %11, %11, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %12, %12, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %13, %13, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %14, %14, %17, 0d3FF0000000000000;\n\t"
                   "@p fma.rn.f64 %15, %15, %17, 0d3FF0000000000000;\n\t}"
                   : "+d"(acc[0]), "+d"(acc[1]), "+d"(acc[2]), "+d"(acc[3]), "+d"(acc[4]), "+d"(acc[5]),
                     "+d"(acc[6]), "+d"(acc[7]), "+d"(acc[8]), "+d"(acc[9]), "+d"(acc[10]), "+d"(acc[11]),
                     "+d"(acc[12]), "+d"(acc[13]), "+d"(acc[14]), "+d"(acc[15])
                   : "r"(mm), "d"(a));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// smem-operand sparse-style: per step, LDS.64 one operand then DFMA (8 B/FMA)
__global__ void k_lds_dfma(double* out, int iters) {
  __shared__ double xs[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = i * 1e-3;
  __syncthreads();
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0;
  unsigned h = threadIdx.x * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    h = h * 1664525u + 1013904223u;
    int base = ((h >> 8) & 255) * 16 + (threadIdx.x & 15);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fma(xs[(base + j * 16 * 17) & 4095], 1.0001, acc[j]);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2048;
  float ms;
  const char* names[4] = {"all-true", "uniform-false", "uniform-50%", "perlane-50%"};
  auto run = [&](auto kern, const char* tag, int mode, double nfma) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0); kern<<<blocks, threads>>>(out, iters, 0.999, 12345u); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double slots = (double)blocks * threads * iters * nfma;
    printf("%s %-14s %.3f ms  %.2f T-slots/s (DFMA-slot rate; full-rate DFMA = 18.5)\n", tag, names[mode], ms, slots / ms / 1e9);
  };
  run(k_pred<0>, "pred1", 0, 64); run(k_pred<1>, "pred1", 1, 64); run(k_pred<2>, "pred1", 2, 64); run(k_pred<3>, "pred1", 3, 64);
  run(k_pred2<0>, "pred16", 0, 128); run(k_pred2<1>, "pred16", 1, 128); run(k_pred2<2>, "pred16", 2, 128); run(k_pred2<3>, "pred16", 3, 128);
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0); k_lds_dfma<<<blocks, threads>>>(out, iters * 8); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("lds+dfma (8B/FMA): %.3f ms  %.2f TFLOP/s\n", ms, 2.0 * blocks * threads * iters * 8 * 8 / ms / 1e9);
  cudaError_t e = cudaDeviceSynchronize(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
