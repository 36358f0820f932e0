// Shared-memory store wavefronts by access size: 32 lanes storing to 32
// distinct banks with 8-, 16-, 32-bit stores (read the counts with
// ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_st.sum).
#include <cstdio>
#include <cstdint>
template <typename T>
__global__ void sts_kernel(int iters, int mode, unsigned* out) {
  __shared__ __align__(16) std::uint8_t buf[16384];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    // bank = lane, row = (i + w) & 15; mode 1: byte offset within the word varies by lane
    // mode 0: one 128-byte row, bank = lane; mode 1: + byte offset varies; mode 2: bank = lane, row
    // varies per lane (distinct banks, scattered rows); mode 3: like 2 with bank = (lane * 5) & 31
    unsigned row = mode >= 2 ? ((lane * 37 + i * 11 + w * 3) & 127) : ((i + w) & 15);
    unsigned bank = mode == 3 ? ((lane * 5) & 31) : lane;
    unsigned off = row * 128 + bank * 4 + (mode == 1 ? (lane & 3) * sizeof(T) % 4 : 0);
    off &= ~(sizeof(T) - 1);
    *reinterpret_cast<volatile T*>(buf + off) = static_cast<T>(i + lane);
  }
  __syncthreads();
  acc = buf[threadIdx.x * 4];
  if (acc == 12345) out[0] = acc;
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int mode = 0; mode < 4; ++mode) {
    float ms[3];
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      sts_kernel<std::uint8_t><<<148 * 4, 256>>>(iters, mode, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[0], a, b);
      cudaEventRecord(a);
      sts_kernel<std::uint16_t><<<148 * 4, 256>>>(iters, mode, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[1], a, b);
      cudaEventRecord(a);
      sts_kernel<std::uint32_t><<<148 * 4, 256>>>(iters, mode, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[2], a, b);
    }
    const double n = 148.0 * 4 * 8 * iters;  // warp-level store instructions
    printf("mode %d: u8 %.3f ms (%.2f cyc/warp-store/SM), u16 %.3f ms, u32 %.3f ms (%.2f)\n", mode, ms[0],
           ms[0] * 1e-3 * 1.9e9 * 148 / n, ms[1], ms[2], ms[2] * 1e-3 * 1.9e9 * 148 / n);
  }
  return 0;
}
