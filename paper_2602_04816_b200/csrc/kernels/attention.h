// Tensor-core causal flash attention (attention_flash.cu): q/k/v/o bf16 rows of
// stride ld (heads interleaved, head h at column h*hd), lse fp32 [B][H][S].
#pragma once

#include <cuda_runtime.h>

bool hlm_flash_supported(int head_dim, int seq);
int hlm_flash_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int hd,
                  int ld, cudaStream_t s);
int hlm_flash_bwd(const void* q, const void* k, const void* v, const void* o, const void* d_o, const float* lse,
                  float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int hd, int ld, cudaStream_t s);

// tcgen05 forward (attention_tc.cu): head_dim 128, seq % 128 == 0.
bool hlm_flash_tc_supported(int head_dim, int seq, int ld);
int hlm_flash_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int ld,
                     cudaStream_t s);
int hlm_flash_bwd_tc(const void* q, const void* k, const void* v, const void* d_o, const float* lse,
                     const float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int ld, cudaStream_t s);
