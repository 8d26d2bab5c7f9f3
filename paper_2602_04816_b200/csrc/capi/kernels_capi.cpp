// extern "C" kernel entry points: validate, launch, translate status codes.
#include <cuda_runtime.h>

#include <string>

#include "capi_util.h"
#include "hlm_cuda.h"
#include "../kernels/gemm.h"
#include "../kernels/block_ops.h"

extern "C" int hlm_cuda_gemm(const HlmGemmDesc* desc, void* stream) {
  const int rc = hlm_gemm_launch(desc, static_cast<cudaStream_t>(stream));
  if (rc != 0) {
    static const char* names[] = {"args", "align", "tensor map", "launch", "driver entry point"};
    const int i = rc - HLM_GEMM_ERR_ARGS;
    hlm_capi::set_error(std::string("hlm_cuda_gemm: ") +
                        (i >= 0 && i < 5 ? names[i] : "unknown") + " error");
  }
  return rc;
}

extern "C" long long hlm_cuda_launch_count(void) { return hlm_launches_total(); }

extern "C" int hlm_cuda_set_device(int device) {
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    hlm_capi::set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return HLM_ERR_CUDA;
  }
  return HLM_OK;
}
