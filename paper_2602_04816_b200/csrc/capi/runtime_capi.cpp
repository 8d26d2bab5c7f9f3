// The device-runtime half of the C ABI (SURVEY.md §8b "what a C-ABI replacement must
// export"): device init + capabilities, a raw device arena, typed streams and events,
// pinned H2D / D2H copies, and the fused head + cross-entropy call in the argument order
// the survey fixes. A host caller that keeps its own scheduler (the reference's
// Engine::stream_tile / evacuate, proj/src/engine.cpp:55-71, 186-203) drives the kernels
// with these and never includes a CUDA header: streams, events and the arena are opaque.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_util.h"
#include "hlm_cuda.h"

namespace {

int cuda_fail(const char* what, cudaError_t e) {
  hlm_capi::set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return HLM_ERR_CUDA;
}

#define HLM_RT_CHECK(call, what)                \
  do {                                          \
    const cudaError_t e_ = (call);              \
    if (e_ != cudaSuccess) return cuda_fail(what, e_); \
  } while (0)

int args_fail(const char* what) {
  hlm_capi::set_error(what);
  return HLM_ERR_ARGS;
}

}  // namespace

extern "C" {

int hlm_cuda_init(int device, HlmCaps* caps) {
  HLM_RT_CHECK(cudaSetDevice(device), "hlm_cuda_init: cudaSetDevice");
  cudaDeviceProp p{};
  HLM_RT_CHECK(cudaGetDeviceProperties(&p, device), "hlm_cuda_init: cudaGetDeviceProperties");
  if (caps) {
    std::memset(caps, 0, sizeof *caps);
    caps->device = device;
    caps->sm_count = p.multiProcessorCount;
    caps->cc_major = p.major;
    caps->cc_minor = p.minor;
    caps->hbm_bytes = static_cast<int64_t>(p.totalGlobalMem);
    caps->l2_bytes = p.l2CacheSize;
    caps->smem_per_block_optin = static_cast<int64_t>(p.sharedMemPerBlockOptin);
    std::snprintf(caps->name, sizeof caps->name, "%.63s", p.name);
  }
  // the library is built for sm_100a only (tcgen05 / TMEM / TMA): refuse anything else
  // up front instead of failing at the first launch
  if (p.major != 10 || p.minor != 0) {
    hlm_capi::set_error("hlm_cuda_init: this build targets sm_100a (B200); device " + std::string(p.name) +
                        " is sm_" + std::to_string(p.major) + std::to_string(p.minor));
    return HLM_ERR_CONFIG;
  }
  return HLM_OK;
}

int hlm_cuda_arena_create(size_t bytes, void** base) {
  if (!base) return args_fail("hlm_cuda_arena_create: null out pointer");
  *base = nullptr;
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes ? bytes : 1);
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    hlm_capi::set_error("hlm_cuda_arena_create: device out of memory for " + std::to_string(bytes) + " bytes");
    return HLM_ERR_OOM;
  }
  if (e != cudaSuccess) return cuda_fail("hlm_cuda_arena_create", e);
  *base = p;
  return HLM_OK;
}

int hlm_cuda_arena_destroy(void* base) {
  if (base) HLM_RT_CHECK(cudaFree(base), "hlm_cuda_arena_destroy");
  return HLM_OK;
}

int hlm_cuda_stream_create(int kind, void** stream) {
  if (!stream) return args_fail("hlm_cuda_stream_create: null out pointer");
  if (kind < HLM_STREAM_COMPUTE || kind > HLM_STREAM_OPT) return args_fail("hlm_cuda_stream_create: unknown kind");
  int least = 0, greatest = 0;
  HLM_RT_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest), "hlm_cuda_stream_create: priority range");
  // as the engine: compute at the greatest priority (side work fills the SMs it leaves)
  cudaStream_t s = nullptr;
  HLM_RT_CHECK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking,
                                            kind == HLM_STREAM_COMPUTE ? greatest : least),
               "hlm_cuda_stream_create");
  *stream = s;
  return HLM_OK;
}

int hlm_cuda_stream_destroy(void* stream) {
  if (stream) HLM_RT_CHECK(cudaStreamDestroy(static_cast<cudaStream_t>(stream)), "hlm_cuda_stream_destroy");
  return HLM_OK;
}

int hlm_cuda_stream_sync(void* stream) {
  HLM_RT_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "hlm_cuda_stream_sync");
  return HLM_OK;
}

int hlm_cuda_event_create(void** event) {
  if (!event) return args_fail("hlm_cuda_event_create: null out pointer");
  cudaEvent_t e = nullptr;
  HLM_RT_CHECK(cudaEventCreate(&e), "hlm_cuda_event_create");
  *event = e;
  return HLM_OK;
}

int hlm_cuda_event_destroy(void* event) {
  if (event) HLM_RT_CHECK(cudaEventDestroy(static_cast<cudaEvent_t>(event)), "hlm_cuda_event_destroy");
  return HLM_OK;
}

int hlm_cuda_event_record(void* event, void* stream) {
  HLM_RT_CHECK(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)),
               "hlm_cuda_event_record");
  return HLM_OK;
}

int hlm_cuda_event_wait(void* stream, void* event) {
  HLM_RT_CHECK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0),
               "hlm_cuda_event_wait");
  return HLM_OK;
}

int hlm_cuda_event_sync(void* event) {
  HLM_RT_CHECK(cudaEventSynchronize(static_cast<cudaEvent_t>(event)), "hlm_cuda_event_sync");
  return HLM_OK;
}

int hlm_cuda_event_query(void* event) {
  const cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaSuccess) return HLM_OK;
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();
    return HLM_NOT_READY;
  }
  return cuda_fail("hlm_cuda_event_query", e);
}

int hlm_cuda_event_elapsed_ms(void* start, void* end, float* ms) {
  if (!ms) return args_fail("hlm_cuda_event_elapsed_ms: null out pointer");
  HLM_RT_CHECK(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)),
               "hlm_cuda_event_elapsed_ms");
  return HLM_OK;
}

int hlm_cuda_h2d_async(void* dst, const void* pinned_src, size_t bytes, void* stream) {
  if (bytes && (!dst || !pinned_src)) return args_fail("hlm_cuda_h2d_async: null pointer");
  HLM_RT_CHECK(cudaMemcpyAsync(dst, pinned_src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
               "hlm_cuda_h2d_async");
  return HLM_OK;
}

int hlm_cuda_d2h_async(void* pinned_dst, const void* src, size_t bytes, void* stream) {
  if (bytes && (!pinned_dst || !src)) return args_fail("hlm_cuda_d2h_async: null pointer");
  HLM_RT_CHECK(cudaMemcpyAsync(pinned_dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
               "hlm_cuda_d2h_async");
  return HLM_OK;
}

// head_fwd + ce_loss_and_grad + head_bwd (proj/include/hlm/kernels.hpp:410-446) in the
// survey's argument order: the per-row losses land in loss_rows (device, `rows` floats);
// with loss_sum_out non-null the call waits for the stream and returns their sum on the
// host, accumulated in double in row order as Engine::anchor_loss does.
int hlm_cuda_head_fwd_ce_bwd(const HlmHeadDims* dims, const void* head_bf16, const float* h,
                             const int32_t* targets, float inv_global_rows, float* d_h, float* d_head_fp32,
                             float* loss_rows, double* loss_sum_out, void* ws, void* stream) {
  if (!dims) return args_fail("hlm_cuda_head_fwd_ce_bwd: null dims");
  const int rc = hlm_cuda_head_loss(dims->rows, dims->hidden, dims->vocab, head_bf16, h, targets, inv_global_rows,
                                    d_h, d_head_fp32, 0, loss_rows, ws, stream);
  if (rc != HLM_OK || !loss_sum_out) return rc;
  std::vector<float> lr(static_cast<size_t>(dims->rows));
  HLM_RT_CHECK(cudaMemcpyAsync(lr.data(), loss_rows, lr.size() * 4, cudaMemcpyDeviceToHost,
                               static_cast<cudaStream_t>(stream)),
               "hlm_cuda_head_fwd_ce_bwd: loss rows");
  HLM_RT_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "hlm_cuda_head_fwd_ce_bwd: sync");
  double s = 0.0;
  for (float v : lr) s += static_cast<double>(v);
  *loss_sum_out = s;
  return HLM_OK;
}

}  // extern "C"
