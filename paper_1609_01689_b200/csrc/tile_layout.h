// tile_layout.h -- where a tile entry sits in the SpMM kernel's shared-memory
// tile (spmm.cu), shared by the host tiler (tiling.cpp), the device
// generator (gpugen.cu) and the tile-diagonal extraction so that all of them
// agree on the packed 16-bit offsets.
//
// A tile row has stride tl_stride(te, v) elements. Columns are permuted so
// that one 128-bit shared load yields the DMMA A fragments (column 4*ks + q
// of k-step ks) of several consecutive k-steps:
//   fp32: within every 16 columns, column 16b + 4u + q is stored at
//         16b + 4q + u  -> one float4 = 4 k-steps; stride te + 16 (16 mod 32
//         banks) keeps the quarter-warp's 8 float4 loads conflict-free.
//   fp64: within every 8 columns, column 8b + 4h + q is stored at 8b + 2q + h
//         -> one double2 = 2 k-steps; stride te + 8 doubles.
// Both permutations are involutions of two bit fields; tl_unperm inverts.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define CIEG_TL __host__ __device__ __forceinline__
#else
#define CIEG_TL inline
#endif

namespace cieg_tl {

CIEG_TL std::uint32_t stride(std::uint32_t te, int precision) { return precision == 0 ? te + 16 : te + 8; }

CIEG_TL std::uint32_t perm(std::uint32_t k, int precision) {
  return precision == 0 ? ((k & ~15u) | ((k & 3u) << 2) | ((k >> 2) & 3u))
                        : ((k & ~7u) | ((k & 3u) << 1) | ((k >> 2) & 1u));
}

CIEG_TL std::uint32_t unperm(std::uint32_t p, int precision) {
  return precision == 0 ? ((p & ~15u) | ((p & 3u) << 2) | ((p >> 2) & 3u))
                        : ((p & ~7u) | ((p & 1u) << 2) | ((p >> 1) & 3u));
}

// Packed entry index: own-row placement (row r, column c) in the low half,
// the mirrored placement (row c, column r) in the high half.
CIEG_TL std::uint32_t pack(std::uint32_t r, std::uint32_t c, std::uint32_t sa, int precision) {
  return (r * sa + perm(c, precision)) | ((c * sa + perm(r, precision)) << 16);
}

}  // namespace cieg_tl
