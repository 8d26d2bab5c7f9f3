"""Host memory bandwidth on the GPU box vs the fused host Adam.
STREAM-like kernels via numpy (multi-threaded through numexpr-free chunking
in threads) are unreliable, so the copy/triad probe is a tiny C++ OpenMP
program compiled here; the Adam probe calls the product's host Adam."""
import ctypes, os, subprocess, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

src = r'''
#include <omp.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
int main() {
  const size_t n = 1ull << 30;  // 4 GiB per array
  float *a = (float*)aligned_alloc(64, n*4), *b = (float*)aligned_alloc(64, n*4), *c = (float*)aligned_alloc(64, n*4);
  #pragma omp parallel for
  for (size_t i = 0; i < n; ++i) { a[i] = 1.f; b[i] = 2.f; c[i] = 0.f; }
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    double s = 0;
    #pragma omp parallel for reduction(+:s)
    for (size_t i = 0; i < n; ++i) s += a[i];
    double t1 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
    #pragma omp parallel for
    for (size_t i = 0; i < n; ++i) c[i] = a[i];
    double t2 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
    #pragma omp parallel for
    for (size_t i = 0; i < n; ++i) a[i] = b[i] + 0.5f * c[i];
    double t3 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %d read %.1f GB/s copy %.1f GB/s triad %.1f GB/s (s=%g)\n", omp_get_max_threads(),
           n*4/t1/1e9, 2*n*4/t2/1e9, 3*n*4/t3/1e9, s);
  }
}
'''
d = tempfile.mkdtemp()
open(os.path.join(d, "bw.cpp"), "w").write(src)
subprocess.run(["g++", "-O3", "-march=native", "-fopenmp", "-o", os.path.join(d, "bw"), os.path.join(d, "bw.cpp")], check=True)
for th in ("16", "8"):
    subprocess.run([os.path.join(d, "bw")], env=dict(os.environ, OMP_NUM_THREADS=th, OMP_PROC_BIND="close"))

from paper_2602_04816_b200 import engine as E
c = E.ModelConfig(4, 3584, 18944, 1024, 8, 1)
s = E.Store(c, 1, "fp32", init="parallel", pin=True)
g = np.random.default_rng(0).standard_normal(s.total_params).astype(np.float32) * 1e-3
for t in (1, 2, 3):
    t0 = time.time(); s.adam_step(g, E.HyperParams(), t); dt = time.time() - t0
    print(f"adam {s.total_params/1e9:.2f} Gparam: {dt:.3f} s -> {30*s.total_params/dt/1e9:.1f} GB/s (30 B/param)")
