/* hlm_cuda.h — the C ABI between the C++ host engine (include/hlm/ headers) and
 * the sm_100a kernels. Flat extern "C" functions over POD structs, plain
 * pointers and sizes; no CUDA or torch types (streams are opaque void*).
 * Every call returns an int status (HLM_OK == 0); hlm_cuda_last_error()
 * returns the message of the last failure on the calling thread.
 *
 * Reference interfaces these entry points replace (paths under the read-only
 * reference tree /root/reference/proj):
 *   hlm_cuda_gemm            matmul_nn / matmul_nt / matmul_grad_acc  include/hlm/kernels.hpp:164-205
 *   hlm_cuda_rmsnorm_fwd/bwd rmsnorm_fwd / rmsnorm_bwd               include/hlm/kernels.hpp:129-162
 *   hlm_cuda_attention_fwd/bwd attention_fwd / attention_bwd         include/hlm/kernels.hpp:207-299
 *   hlm_cuda_block_fwd/bwd   block_forward / block_backward          include/hlm/kernels.hpp:313-383
 *   hlm_cuda_embed_fwd/bwd   embed_fwd / embed_bwd_acc               include/hlm/kernels.hpp:385-408
 *   hlm_cuda_head_loss       head_fwd + ce_loss_and_grad + head_bwd  include/hlm/kernels.hpp:410-446
 *   hlm_cuda_bf16_pack       bf16_bits_from_f32                      include/hlm/bf16.hpp:15-25
 *   hlm_engine_*             Engine / run_training                   include/hlm/engine.hpp:46-116,
 *                                                                    include/hlm/trainer.hpp:38
 */
#ifndef HLM_CUDA_H_
#define HLM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum HlmStatus {
  HLM_OK = 0,
  HLM_ERR_CONFIG = 2,   /* ConfigError / std::invalid_argument (CLI exit 2) */
  HLM_ERR_OOM = 3,      /* ArenaOomError (CLI exit 3)                       */
  HLM_ERR_PROTOCOL = 4, /* ProtocolError                                    */
  HLM_ERR_NUMERICS = 5, /* NumericsError: non-finite gradient               */
  HLM_ERR_RANGE = 6,    /* std::out_of_range: token / target id             */
  HLM_ERR_CUDA = 7,     /* CUDA runtime / driver failure                    */
  HLM_ERR_ARGS = 8      /* malformed call (null pointer, bad layout)        */
};

/* GEMM-internal codes (also surfaced through hlm_cuda_gemm) */
enum HlmGemmErr {
  HLM_GEMM_ERR_ARGS = 8,
  HLM_GEMM_ERR_ALIGN = 9,
  HLM_GEMM_ERR_TMAP = 10,
  HLM_GEMM_ERR_LAUNCH = 11,
  HLM_GEMM_ERR_DRIVER = 12
};

const char* hlm_cuda_last_error(void);

/* ------------------------------------------------------------------ GEMM
 * C[g] = A[g] . B[g]  (bf16 operands, fp32 accumulation in TMEM)
 *   A element (m,k): a_mn ? A[k*lda + m] : A[m*lda + k]
 *   B element (k,n): b_mn ? B[k*ldb + n] : B[n*ldb + k]
 *   C element (m,n): C[m*ldc + n]
 * Groups (G >= 1): operand g lives at base + g*gstride when *_grouped.
 *   kgroup == 0: one output per group at C + g*c_gstride
 *   kgroup == 1: single output, C = sum_g A[g] . B[g]
 * Epilogues: BF16 store, FP32 store, FP32 store of R + acc (R may alias C). */
enum HlmEpilogue { HLM_EPI_BF16 = 0, HLM_EPI_F32 = 1, HLM_EPI_F32_ADD = 2 };

typedef struct HlmGemmDesc {
  int M, N, K, G;
  int kgroup;
  int a_mn, b_mn;
  int a_grouped, b_grouped;
  int epi;
  const void* A;
  long long lda, a_gstride;
  const void* B;
  long long ldb, b_gstride;
  void* C;
  long long ldc, c_gstride;
  const float* R;
  long long ldr, r_gstride;
} HlmGemmDesc;

int hlm_cuda_gemm(const HlmGemmDesc* desc, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HLM_CUDA_H_ */
