// Internal launcher for the tcgen05 GEMM (gemm_sm100.cu). The public C ABI in
// include/hlm_cuda.h re-exports it as hlm_cuda_gemm.
#pragma once

#include <cuda_runtime.h>

#include "hlm_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

int hlm_gemm_launch(const HlmGemmDesc* d, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
