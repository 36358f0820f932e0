// blockvec.hpp -- host wrappers of the tall-skinny block kernels (K2-K4).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "context.hpp"

namespace cieg {

// A column-concatenation of up to 3 row-major device blocks ([X W P] without
// the hcat copies of block_vectors.cpp:20-34).
struct Seg {
  const double* p;
  std::uint32_t ld;
  std::uint32_t w;
};
struct View3 {
  Seg s[3];
  int nseg;
  std::uint32_t width;
};
inline View3 view(std::initializer_list<Seg> segs) {
  View3 v{};
  v.nseg = 0;
  v.width = 0;
  for (const Seg& s : segs) {
    if (s.w == 0) continue;
    v.s[v.nseg++] = s;
    v.width += s.w;
  }
  return v;
}
inline Seg seg(const double* p, std::uint32_t w) { return Seg{p, w, w}; }

// Output split over up to two row-major blocks (columns [0, w0) -> o0,
// [w0, w0 + w1) -> o1).
struct Out2 {
  double* o0;
  std::uint32_t ld0, w0;
  double* o1;
  std::uint32_t ld1, w1;
};
inline Out2 out1(double* p, std::uint32_t w) { return Out2{p, w, w, nullptr, 0, 0}; }
inline Out2 out2(double* p0, std::uint32_t w0, double* p1, std::uint32_t w1) {
  return Out2{p0, w0, w0, p1, w1, w1};
}

// L^T R (L.width x R.width), column major on the host; deterministic
// fixed-order reduction. Synchronizes the stream.
std::vector<double> gram(cieg_ctx* ctx, std::uint32_t n, const View3& L, const View3& R);
// two independent Grams, one D2H + one synchronisation (same values as two gram() calls)
std::pair<std::vector<double>, std::vector<double>> gram_pair(cieg_ctx* ctx, std::uint32_t n, const View3& L1,
                                                              const View3& R1, const View3& L2, const View3& R2);

// out = [accumulate ? out : 0] + in * G, G (in.width x kout) column major on
// the host. Row-local: out may alias in when the widths match.
void combine(cieg_ctx* ctx, std::uint32_t n, const View3& in, const double* g_host,
             std::uint32_t kout, const Out2& out, bool accumulate);

// combine followed by a Gram of its output in the same pass: returns
// L^T out (L.width x kout) or, for L == nullptr, out^T out (kout x kout),
// column major on the host. Same values as combine + gram up to the Gram's
// summation order; falls back to the two separate passes outside the fused
// instantiations (out and L up to 32 columns).
std::vector<double> combine_gram(cieg_ctx* ctx, std::uint32_t n, const View3& in, const double* g_host,
                                 std::uint32_t kout, const Out2& out, bool accumulate, const View3* L);

// R = HX - X diag(theta) (n x k, contiguous).
void residual(cieg_ctx* ctx, std::uint32_t n, std::uint32_t k, const double* hx, const double* x,
              const double* theta_host, double* r);

// dst (n x cols.size()) = src[:, cols] (src n x ksrc).
void gather_columns(cieg_ctx* ctx, std::uint32_t n, const double* src, std::uint32_t ksrc,
                    const std::vector<std::uint32_t>& cols, double* dst);

}  // namespace cieg
