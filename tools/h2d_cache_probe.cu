// Does an H2D DMA of host data that the CPU just wrote (cache-resident) take DRAM
// bandwidth away from the host Adam? 15 threads run an Adam-like stream (30 B/param)
// while the GPU pulls H2D (a) from a 2 GiB pinned buffer in DRAM, (b) from an 8 MiB
// pinned ring that one thread keeps rewriting (regular stores, cache-resident), (c) no
// H2D. If (b)'s Adam bandwidth matches (c) and beats (a), DMA reads of freshly written
// lines are served from the caches and a BF16 shadow written just before its H2D costs
// no DRAM traffic.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

static double adam_pass(float* w, float* m, float* v, float* g, long n, int threads) {
  auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(threads) schedule(static)
  for (long c = 0; c < n / 4096; ++c)
    for (long i = c * 4096; i < (c + 1) * 4096; i += 16) {
      __m512 gg = _mm512_loadu_ps(g + i), mm = _mm512_loadu_ps(m + i), vv = _mm512_loadu_ps(v + i),
             th = _mm512_loadu_ps(w + i);
      mm = _mm512_fmadd_ps(_mm512_set1_ps(0.9f), mm, _mm512_mul_ps(_mm512_set1_ps(0.1f), gg));
      vv = _mm512_fmadd_ps(_mm512_set1_ps(0.999f), vv, _mm512_mul_ps(_mm512_set1_ps(0.001f), _mm512_mul_ps(gg, gg)));
      th = _mm512_sub_ps(th, _mm512_mul_ps(_mm512_set1_ps(1e-4f), _mm512_div_ps(mm, _mm512_add_ps(_mm512_sqrt_ps(vv), _mm512_set1_ps(1e-8f)))));
      _mm512_storeu_ps(m + i, mm); _mm512_storeu_ps(v + i, vv); _mm512_storeu_ps(w + i, th);
    }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  const long N = 256l << 20;                     // 1 GiB per fp32 array
  float *w = (float*)aligned_alloc(64, N * 4), *m = (float*)aligned_alloc(64, N * 4),
        *v = (float*)aligned_alloc(64, N * 4), *g = (float*)aligned_alloc(64, N * 4);
#pragma omp parallel for
  for (long i = 0; i < N; ++i) { w[i] = 1; m[i] = 0; v[i] = 0; g[i] = 1e-3f; }
  const size_t BIG = 2ul << 30, RING = 8ul << 20, CH = 1ul << 20;
  char *big, *ring;
  cudaHostAlloc((void**)&big, BIG, 0);
  cudaHostAlloc((void**)&ring, RING, 0);
  memset(big, 1, BIG); memset(ring, 1, RING);
  char* dev; cudaMalloc(&dev, BIG);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      std::atomic<bool> stop{false};
      std::atomic<long> bytes{0};
      double dev_gbs = 0;
      std::thread dma([&] {
        if (mode == 2) return;
        cudaEvent_t t_a, t_b;
        cudaEventCreate(&t_a); cudaEventCreate(&t_b);
        cudaEventRecord(t_a, s);
        cudaEvent_t ev[8];
        for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        long k = 0;
        while (!stop.load()) {
          const int slot = k % 8;
          if (k >= 8) cudaEventSynchronize(ev[slot]);
          char* src;
          if (mode == 0) {
            src = big + (k * CH) % BIG;
          } else if (mode == 3) {   // ring reused without rewriting: DMA reads of LLC-resident lines
            src = ring + slot * CH;
          } else {   // rewrite this ring chunk (the CPU producing a fresh BF16 piece), then DMA it
            src = ring + slot * CH;
            for (size_t i = 0; i < CH; i += 64) _mm512_storeu_si512((void*)(src + i), _mm512_set1_epi32((int)k));
          }
          cudaMemcpyAsync(dev + (k * CH) % BIG, src, CH, cudaMemcpyHostToDevice, s);
          cudaEventRecord(ev[slot], s);
          bytes += CH;
          ++k;
        }
        cudaEventRecord(t_b, s);
        cudaStreamSynchronize(s);
        float ms = 0; cudaEventElapsedTime(&ms, t_a, t_b);
        dev_gbs = bytes.load() / (ms / 1e3) / 1e9;
      });
      std::this_thread::sleep_for(std::chrono::milliseconds(100));
      const auto t0 = std::chrono::steady_clock::now();
      const double ta = adam_pass(w, m, v, g, N, 15);
      const double tw = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      stop = true;
      dma.join();
      printf("mode %s: adam %.3f s = %.0f GB/s (28 B/param)  h2d %.1f GB/s\n",
             mode == 0 ? "DRAM-src H2D " : mode == 1 ? "fresh-ring H2D" : mode == 3 ? "LLC-ring H2D " : "no H2D       ", ta,
             28.0 * N / ta / 1e9, dev_gbs);
      (void)tw;
    }
  }
  return 0;
}
