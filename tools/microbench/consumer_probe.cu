// consumer_probe.cu -- how fast is K1's consumer loop on its own? 8 consumer
// warps per CTA run the exact K1 group loop (fp32 tile in the float4
// interleaved layout, X slab with the n-tile interleave, float4 A + double2 B
// fragment loads, F2F, DMMA m8n8k4 over 2 m-tiles x 2 n-tiles) over a static
// shared-memory tile, with no producer and no barriers, one CTA per SM. The
// DMMA count equals K1's per item; the time per "item" against the 4096
// tensor cycles per SMSP an item needs shows the consumer pipeline's
// efficiency. Variants: 8 warps (2 per SMSP, K1 today), 4 and 16 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o consumer_probe consumer_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int TD = 128, NT = 2, SA = TD + 16, SX = 8 * NT + 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// PW extra "producer-like" warps per CTA stream shared-memory stores into a
// second 73.7 KB region while the consumers run: mode 1 bulk zeroing with
// 128-bit stores (K1's per-item tile clear), 2 scattered 32-bit stores (the
// entry scatter, ~6.5k per item), 3 both; 0 = no producers.
template <int CW, int PW = 0, int MODE = 0, bool GLOBALB = false>
__global__ void __launch_bounds__(32 * (CW + PW), 1) probe(int items, double* out, const double* xg) {
  constexpr int MT = TD / 8 / CW;
  extern __shared__ __align__(16) unsigned char smem[];
  float* A0 = reinterpret_cast<float*>(smem);
  double* X0 = reinterpret_cast<double*>(smem + sizeof(float) * TD * SA);
  float* Z0 = reinterpret_cast<float*>(smem + sizeof(float) * TD * SA + sizeof(double) * TD * SX);
  for (int e = threadIdx.x; e < TD * SA; e += blockDim.x) A0[e] = (e % 7) * 0.25f;
  for (int e = threadIdx.x; e < TD * SX; e += blockDim.x) X0[e] = (e % 5) * 0.5;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  if (warp >= CW) {  // producer-like warps
    const int pt = threadIdx.x - 32 * CW, np = 32 * PW;
    unsigned h = 2166136261u ^ pt;
    for (int it = 0; it < items; ++it) {
      if (MODE & 1) {
        float4* p4 = reinterpret_cast<float4*>(Z0);
        for (int k = pt; k < TD * SA / 4; k += np) p4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (MODE & 2) {
        for (int k = pt; k < 6500; k += np) {
          h = h * 1664525u + 1013904223u;
          Z0[(h >> 8) % (TD * SA)] = 1.0f;
        }
      }
    }
    return;
  }
  const int m_base = warp * 8 * MT;
  double acc[MT][NT][2] = {};
  const float* A = A0 + (m_base + g) * SA + 4 * q;
  const double* xb = X0 + q * SX + 2 * g;
  for (int it = 0; it < items; ++it) {
    double af[2][4][MT], bf[2][4][NT];
    auto load_group = [&](int grp, double (&fa)[4][MT], double (&fb)[4][NT]) {
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const float4 v4 = *reinterpret_cast<const float4*>(A + j * 8 * SA + 16 * grp);
        fa[0][j] = v4.x;
        fa[1][j] = v4.y;
        fa[2][j] = v4.z;
        fa[3][j] = v4.w;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (GLOBALB) {  // X row-major (rows of 16): columns g and 8 + g of row 4 k + q
          const double* xr = xg + static_cast<size_t>((it & 63) * TD + 4 * (4 * grp + u) + q) * 16 + g;
          fb[u][0] = __ldg(xr);
          fb[u][1] = __ldg(xr + 8);
        } else {
          const double2 v2 = *reinterpret_cast<const double2*>(xb + 4 * (4 * grp + u) * SX);
          fb[u][0] = v2.x;
          fb[u][1] = v2.y;
        }
      }
    };
    auto mma_group = [&](const double (&fa)[4][MT], const double (&fb)[4][NT]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int j = 0; j < MT; ++j) dmma(acc[j][n][0], acc[j][n][1], fa[u][j], fb[u][n]);
    };
    constexpr int kGroups = TD / 16;
    load_group(0, af[0], bf[0]);
#pragma unroll 1
    for (int grp = 0; grp < kGroups; grp += 2) {
      load_group(grp + 1, af[1], bf[1]);
      mma_group(af[0], bf[0]);
      if (grp + 2 < kGroups) load_group(grp + 2, af[0], bf[0]);
      mma_group(af[1], bf[1]);
    }
  }
  double s = 0;
  for (int j = 0; j < MT; ++j)
    for (int n = 0; n < NT; ++n) s += acc[j][n][0] + acc[j][n][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CW, int PW = 0, int MODE = 0, bool GLOBALB = false>
void run(int sms, int items, double* out, const double* xg) {
  const size_t smem = 2 * sizeof(float) * TD * SA + sizeof(double) * TD * SX;
  cudaFuncSetAttribute(probe<CW, PW, MODE, GLOBALB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<CW, PW, MODE, GLOBALB><<<sms, 32 * (CW + PW), smem>>>(10, out, xg);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<CW, PW, MODE, GLOBALB><<<sms, 32 * (CW + PW), smem>>>(items, out, xg);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // per item: 16 m-tiles x 2 n-tiles x 32 k-steps DMMA = 1024 per CTA; 37 TF/s per GPU
  const double flops = double(sms) * items * 1024 * 512;
  printf("CW=%2d PW=%d mode=%d globalB=%d  %8.3f ms  %7.2f TF/s (%5.1f %% of 37.0)  %s\n", CW, PW, MODE, (int)GLOBALB, ms, flops / ms / 1e9, flops / ms / 1e9 / 37.0 * 100,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  const int items = 1648;  // K1's items per SM on config 2
  double* xg = nullptr;  // 64 slabs of 128 rows x 16 (the partner panels' X rows)
  cudaMalloc(&xg, sizeof(double) * 64 * TD * 16);
  cudaMemset(xg, 0, sizeof(double) * 64 * TD * 16);
  run<8>(sms, items, out, xg);
  run<8, 8, 3>(sms, items, out, xg);
  run<8, 0, 0, true>(sms, items, out, xg);
  run<8, 8, 3, true>(sms, items, out, xg);
  return 0;
}
