// Does a small LLC-resident D2H ring help the host Adam? Three sources for the
// gradient: (a) 1 GiB pinned buffer (DRAM), (b) a 4 MiB pinned ring reused
// (upper bound: gradient in cache), (c) the GPU writing 4 MiB chunks into an
// 8-slot pinned ring by DMA, the CPU consuming each chunk right after its event.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static void adam_chunk(float* w, float* m, float* v, uint16_t* sh, const float* g, long n) {
  const float b1 = 0.9f, b2 = 0.999f, lr = 1e-4f, eps = 1e-8f, bc1 = 0.1f, bc2 = 0.001f;
#pragma omp parallel for schedule(static)
  for (long c = 0; c < n / 4096; ++c) {
    for (long i = c * 4096; i < (c + 1) * 4096; i += 16) {
      __m512 gg = _mm512_loadu_ps(g + i), mm = _mm512_loadu_ps(m + i), vv = _mm512_loadu_ps(v + i), th = _mm512_loadu_ps(w + i);
      mm = _mm512_add_ps(_mm512_mul_ps(_mm512_set1_ps(b1), mm), _mm512_mul_ps(_mm512_set1_ps(1 - b1), gg));
      vv = _mm512_add_ps(_mm512_mul_ps(_mm512_set1_ps(b2), vv), _mm512_mul_ps(_mm512_mul_ps(_mm512_set1_ps(1 - b2), gg), gg));
      __m512 u = _mm512_div_ps(_mm512_div_ps(mm, _mm512_set1_ps(bc1)), _mm512_add_ps(_mm512_sqrt_ps(_mm512_div_ps(vv, _mm512_set1_ps(bc2))), _mm512_set1_ps(eps)));
      th = _mm512_sub_ps(th, _mm512_mul_ps(_mm512_set1_ps(lr), u));
      _mm512_storeu_ps(m + i, mm); _mm512_storeu_ps(v + i, vv); _mm512_storeu_ps(w + i, th);
      _mm256_stream_si256((__m256i*)(sh + i), _mm512_cvtepi32_epi16(_mm512_srli_epi32(_mm512_castps_si512(th), 16)));
    }
  }
}

int main() {
  const long N = 256l << 20;          // 256 Mi params = 1 GiB per fp32 array
  const long CH = 1l << 20;           // 4 MiB chunks
  float *w = (float*)aligned_alloc(64, N * 4), *m = (float*)aligned_alloc(64, N * 4), *v = (float*)aligned_alloc(64, N * 4);
  uint16_t* sh; cudaHostAlloc((void**)&sh, N * 2, 0);
  float *gbig, *ring; cudaHostAlloc((void**)&gbig, N * 4, 0); cudaHostAlloc((void**)&ring, 8 * CH * 4, 0);
#pragma omp parallel for
  for (long i = 0; i < N; ++i) { w[i] = 1; m[i] = 0; v[i] = 0; gbig[i] = 1e-3f; }
  for (long i = 0; i < 8 * CH; ++i) ring[i] = 1e-3f;
  float* dgrad; cudaMalloc(&dgrad, N * 4); cudaMemset(dgrad, 0, N * 4);
  cudaStream_t s; cudaStreamCreate(&s);
  std::vector<cudaEvent_t> ev(8); for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  auto now = [] { return std::chrono::steady_clock::now(); };
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = now();
    for (long c = 0; c < N; c += CH) adam_chunk(w + c, m + c, v + c, sh + c, gbig + c, CH);
    double ta = std::chrono::duration<double>(now() - t0).count();
    t0 = now();
    for (long c = 0; c < N; c += CH) adam_chunk(w + c, m + c, v + c, sh + c, ring + (c / CH % 1) * CH, CH);
    double tb = std::chrono::duration<double>(now() - t0).count();
    t0 = now();
    const long nch = N / CH;
    for (long k = 0; k < 8 && k < nch; ++k) { cudaMemcpyAsync(ring + k * CH, dgrad + k * CH, CH * 4, cudaMemcpyDeviceToHost, s); cudaEventRecord(ev[k], s); }
    for (long k = 0; k < nch; ++k) {
      cudaEventSynchronize(ev[k % 8]);
      adam_chunk(w + k * CH, m + k * CH, v + k * CH, sh + k * CH, ring + (k % 8) * CH, CH);
      if (k + 8 < nch) { cudaMemcpyAsync(ring + (k % 8) * CH, dgrad + (k + 8) * CH, CH * 4, cudaMemcpyDeviceToHost, s); cudaEventRecord(ev[k % 8], s); }
    }
    double tc = std::chrono::duration<double>(now() - t0).count();
    printf("threads %d  (a) DRAM grads %.3f s = %.0f GB/s(30B)   (b) cached grads %.3f s = %.0f GB/s   (c) DMA ring %.3f s = %.0f GB/s\n",
           omp_get_max_threads(), ta, 30.0 * N / ta / 1e9, tb, 30.0 * N / tb / 1e9, tc, 30.0 * N / tc / 1e9);
  }
  return 0;
}
