// Host memcpy throughput on the GPU box: 256 MB pageable -> 8 MB slots and back,
// OpenMP pieces of 256 KB, by thread count; regular vs non-temporal stores.
#include <emmintrin.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
static void stream_piece(char* d, const char* s, size_t n) {
  for (size_t o = 0; o + 64 <= n; o += 64) {
    __m128i a = _mm_loadu_si128((const __m128i*)(s + o)), b = _mm_loadu_si128((const __m128i*)(s + o + 16));
    __m128i c = _mm_loadu_si128((const __m128i*)(s + o + 32)), e = _mm_loadu_si128((const __m128i*)(s + o + 48));
    _mm_stream_si128((__m128i*)(d + o), a); _mm_stream_si128((__m128i*)(d + o + 16), b);
    _mm_stream_si128((__m128i*)(d + o + 32), c); _mm_stream_si128((__m128i*)(d + o + 48), e);
  }
  _mm_sfence();
}
static void copy(char* d, const char* s, size_t n, int th, int nt) {
  const size_t P = 256u << 10; long pieces = (long)((n + P - 1) / P);
#pragma omp parallel for schedule(static) num_threads(th)
  for (long i = 0; i < pieces; ++i) { size_t o = (size_t)i * P, l = n - o < P ? n - o : P; if (nt) stream_piece(d + o, s + o, l); else memcpy(d + o, s + o, l); }
}
int main(void) {
  const size_t N = 256u << 20, S = 8u << 20;
  char* big = (char*)aligned_alloc(4096, N); char* ring = (char*)aligned_alloc(4096, 4 * S);
  memset(big, 1, N); memset(ring, 2, 4 * S);
  int ths[] = {1, 2, 4, 8, 16};
  for (int t = 0; t < 5; ++t) for (int mode = 0; mode < 3; ++mode) {
    double best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      double t0 = now();
      for (size_t o = 0, c = 0; o < N; o += S, ++c) {
        if (mode == 0) copy(ring + (c % 4) * S, big + o, S, ths[t], 0);        // in: pageable -> ring
        else copy(big + o, ring + (c % 4) * S, S, ths[t], mode == 2);           // out: ring -> pageable (memcpy / NT)
      }
      double dt = now() - t0; if (dt < best) best = dt;
    }
    printf("threads %2d %s: %.2f ms, %.1f GB/s\n", ths[t], mode == 0 ? "in (memcpy)" : mode == 1 ? "out (memcpy)" : "out (stream)", best * 1e3, N / best / 1e9);
  }
  return 0;
}
