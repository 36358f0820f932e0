// device_common.cuh -- small device helpers shared by the libcieg kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cieg {

// D(8x8) += A(8x4) * B(4x8), fp64 tensor core (SASS DMMA.8x8x4).
// Fragment ownership for lane l (g = l>>2, q = l&3):
//   a = A[g][q], b = B[q][g], {c0, c1} = C[g][2q], C[g][2q+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace cieg
