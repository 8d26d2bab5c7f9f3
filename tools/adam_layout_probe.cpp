// Host Adam bandwidth: separate w / m / v arrays (the store's layout) vs one
// interleaved [w16 m16 v16] array (fewer concurrent DRAM streams per thread).
// g read + bf16 shadow written in both. 16 threads, 30 B/param accounting.
#include <immintrin.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <sys/mman.h>

static void* huge(size_t b) {
  void* p = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(p, b, MADV_HUGEPAGE);
  return p;
}
static inline __m256i bf16x16(__m512 v) { return _mm512_cvtepi32_epi16(_mm512_srli_epi32(_mm512_castps_si512(v), 16)); }
#define ADAM_BODY                                                                                      \
  mm = _mm512_add_ps(_mm512_mul_ps(b1, mm), _mm512_mul_ps(o1, gg));                                    \
  vv = _mm512_add_ps(_mm512_mul_ps(b2, vv), _mm512_mul_ps(_mm512_mul_ps(o2, gg), gg));                 \
  th = _mm512_sub_ps(th, _mm512_mul_ps(lr, _mm512_div_ps(_mm512_div_ps(mm, c1),                        \
                                                         _mm512_add_ps(_mm512_sqrt_ps(_mm512_div_ps(vv, c2)), ep))));

int main() {
  const long N = 512l << 20;   // 512 Mi params
  float* g = (float*)huge(N * 4);
  float *w = (float*)huge(N * 4), *m = (float*)huge(N * 4), *v = (float*)huge(N * 4);
  float* wmv = (float*)huge(N * 12);
  uint16_t* sh = (uint16_t*)huge(N * 2);
#pragma omp parallel for
  for (long i = 0; i < N; ++i) { g[i] = 1e-3f; w[i] = 1; m[i] = 0; v[i] = 0; sh[i] = 0; }
#pragma omp parallel for
  for (long i = 0; i < 3 * N; ++i) wmv[i] = (i / 16) % 3 == 0 ? 1.f : 0.f;
  const __m512 b1 = _mm512_set1_ps(0.9f), b2 = _mm512_set1_ps(0.999f), o1 = _mm512_set1_ps(0.1f),
               o2 = _mm512_set1_ps(0.001f), c1 = _mm512_set1_ps(0.1f), c2 = _mm512_set1_ps(0.001f),
               ep = _mm512_set1_ps(1e-8f), lr = _mm512_set1_ps(1e-4f);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
    for (long c = 0; c < N / 32768; ++c)
      for (long i = c * 32768; i < (c + 1) * 32768; i += 16) {
        __m512 gg = _mm512_loadu_ps(g + i), mm = _mm512_loadu_ps(m + i), vv = _mm512_loadu_ps(v + i),
               th = _mm512_loadu_ps(w + i);
        ADAM_BODY
        _mm512_storeu_ps(m + i, mm); _mm512_storeu_ps(v + i, vv); _mm512_storeu_ps(w + i, th);
        _mm256_stream_si256((__m256i*)(sh + i), bf16x16(th));
      }
    double ta = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
    for (long c = 0; c < N / 32768; ++c)
      for (long i = c * 32768; i < (c + 1) * 32768; i += 16) {
        float* q = wmv + 3 * i;
        __m512 gg = _mm512_loadu_ps(g + i), th = _mm512_loadu_ps(q), mm = _mm512_loadu_ps(q + 16),
               vv = _mm512_loadu_ps(q + 32);
        ADAM_BODY
        _mm512_storeu_ps(q, th); _mm512_storeu_ps(q + 16, mm); _mm512_storeu_ps(q + 32, vv);
        _mm256_stream_si256((__m256i*)(sh + i), bf16x16(th));
      }
    double tb = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
    for (long c = 0; c < N / 32768; ++c)
      for (long i = c * 32768; i < (c + 1) * 32768; i += 16) {
        if ((i & 63) == 0) {   // one line per stream, 2 KiB ahead
          _mm_prefetch((const char*)(g + i + 512), _MM_HINT_T0);
          _mm_prefetch((const char*)(m + i + 512), _MM_HINT_T0);
          _mm_prefetch((const char*)(v + i + 512), _MM_HINT_T0);
          _mm_prefetch((const char*)(w + i + 512), _MM_HINT_T0);
        }
        __m512 gg = _mm512_loadu_ps(g + i), mm = _mm512_loadu_ps(m + i), vv = _mm512_loadu_ps(v + i),
               th = _mm512_loadu_ps(w + i);
        ADAM_BODY
        _mm512_storeu_ps(m + i, mm); _mm512_storeu_ps(v + i, vv); _mm512_storeu_ps(w + i, th);
        _mm256_stream_si256((__m256i*)(sh + i), bf16x16(th));
      }
    double tc = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %d: separate w/m/v %.3f s = %.0f GB/s ; interleaved %.3f s = %.0f GB/s ; separate+prefetch %.3f s = %.0f GB/s (30 B/param)\n",
           omp_get_max_threads(), ta, 30.0 * N / ta / 1e9, tb, 30.0 * N / tb / 1e9, tc, 30.0 * N / tc / 1e9);
  }
  return 0;
}
