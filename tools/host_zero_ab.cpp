// host_zero_ab.cpp — memset vs non-temporal (_mm_stream_si128) zero-fill of the 80 MB dense host output of
// sttsv_apply_host on `large` (n = 1e7), 64 Ki-double chunks over the OpenMP threads.  On the B200 host (16
// threads): memset 0.373 ms, streaming stores 0.514 ms -> memset kept (plan.cpp).
//   g++ -O2 -fopenmp -o /tmp/zt tools/host_zero_ab.cpp && /tmp/zt
#include <emmintrin.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
static inline void zero_stream(double* p, int64_t cnt) {
  int64_t i = 0;
  while (i < cnt && (reinterpret_cast<uintptr_t>(p + i) & 63)) p[i++] = 0.0;
  const __m128i z = _mm_setzero_si128();
  for (; i + 8 <= cnt; i += 8) {
    __m128i* q = reinterpret_cast<__m128i*>(p + i);
    _mm_stream_si128(q, z); _mm_stream_si128(q + 1, z); _mm_stream_si128(q + 2, z); _mm_stream_si128(q + 3, z);
  }
  for (; i < cnt; ++i) p[i] = 0.0;
  _mm_sfence();
}
int main() {
  const int64_t n = 10000000;
  double* y = (double*)aligned_alloc(64, (n + 8) * 8) + 1;
  for (int mode = 0; mode < 2; ++mode) {
    double best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
      for (int64_t i = 0; i < n; i += 4096) y[i] = 1.0;
      auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
      for (int64_t c = 0; c < (n + 65535) / 65536; ++c) {
        const int64_t a = c * 65536, b = std::min<int64_t>(n, a + 65536);
        if (mode == 0) memset(y + a, 0, (size_t)(b - a) * 8); else zero_stream(y + a, b - a);
      }
      double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, dt);
    }
    double s = 0; for (int64_t i = 0; i < n; ++i) s += y[i];
    printf("mode %d best %.3f ms sum %g threads %d\n", mode, best * 1e3, s, omp_get_max_threads());
  }
}
