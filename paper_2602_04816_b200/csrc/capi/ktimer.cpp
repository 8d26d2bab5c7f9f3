// Per-launch device timing of the hot kernels inside a timed region
// (bench.py's roofline.achieved): an event pair on the launching stream around
// every GEMM / attention launch, the kernel's algorithmic flops alongside. Off
// unless hlm_ktimer_enable(1); events come from a reused pool.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "capi_util.h"
#include "hlm_cuda.h"

namespace {

struct Rec {
  int a, b;   // event pool indices
  int kind;
  double work;
};

std::mutex mu;
bool enabled = false;
std::vector<cudaEvent_t> pool;
size_t used = 0;
std::vector<Rec> recs;

int take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    pool.push_back(e);
  }
  return static_cast<int>(used++);
}

}  // namespace

namespace hlm_capi {

int ktimer_begin(void* stream) {
  std::lock_guard<std::mutex> lk(mu);
  if (!enabled) return -1;
  const int a = take();
  if (a < 0 || cudaEventRecord(pool[static_cast<size_t>(a)], static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return -1;
  return a;
}

void ktimer_end(int a, void* stream, int kind, double work) {
  if (a < 0) return;
  std::lock_guard<std::mutex> lk(mu);
  if (!enabled) return;
  const int b = take();
  if (b < 0 || cudaEventRecord(pool[static_cast<size_t>(b)], static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return;
  recs.push_back({a, b, kind, work});
}

}  // namespace hlm_capi

extern "C" int hlm_ktimer_enable(int on) {
  std::lock_guard<std::mutex> lk(mu);
  enabled = on != 0;
  return HLM_OK;
}

extern "C" int hlm_ktimer_collect(int kind, double* ms, double* work, int64_t* launches) {
  std::lock_guard<std::mutex> lk(mu);
  double t = 0.0, w = 0.0;
  int64_t n = 0;
  for (const Rec& r : recs) {
    if (r.kind != kind) continue;
    float e = 0.f;
    if (cudaEventSynchronize(pool[static_cast<size_t>(r.b)]) != cudaSuccess ||
        cudaEventElapsedTime(&e, pool[static_cast<size_t>(r.a)], pool[static_cast<size_t>(r.b)]) != cudaSuccess) {
      hlm_capi::set_error("ktimer: event query failed");
      return HLM_ERR_CUDA;
    }
    t += e;
    w += r.work;
    ++n;
  }
  if (ms) *ms = t;
  if (work) *work = w;
  if (launches) *launches = n;
  return HLM_OK;
}

extern "C" int hlm_ktimer_reset(void) {
  std::lock_guard<std::mutex> lk(mu);
  recs.clear();
  used = 0;
  return HLM_OK;
}
