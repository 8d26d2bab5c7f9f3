// Internal launchers of block_ops.cu (return 0 on a clean launch).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#define HLM_NORM_ROWS_PER_CHUNK 8

int hlm_ops_rmsnorm_fwd(const float* x, const void* scale, void* out, long long rows, int h, cudaStream_t s);
int hlm_ops_rmsnorm_bwd(const float* x, const void* scale, const float* g, const float* resid, float* out,
                        void* out_bf, float* inv_buf, float* partial, float* dscale, long long rows, int h,
                        cudaStream_t s);
int hlm_ops_cast_bf16(const float* in, void* out, long long n, cudaStream_t s);
int hlm_ops_swiglu_fwd(const void* ug, void* act, long long n, cudaStream_t s);
int hlm_ops_swiglu_bwd(const void* dact, const void* ug, void* dug, long long n, cudaStream_t s);
int hlm_ops_rope(void* x, const float* cs, const float* sn, long long rows, int h, int hd, int S, int inverse,
                 int nmats, long long mat_stride, cudaStream_t s);
int hlm_ops_embed_fwd(const int32_t* tok, const void* table, float* out, long long rows, int h, int vocab,
                      int* err, cudaStream_t s);
int hlm_ops_embed_bwd(const int32_t* row_ptr, const int32_t* pos, const float* g, float* d_table, int vocab,
                      int h, int accumulate, cudaStream_t s);
int hlm_ops_embed_bwd_compact(const int32_t* row_ptr, const int32_t* pos, const int32_t* rows, int n_rows,
                              const float* g, float* out, int h, cudaStream_t s);
int hlm_ops_ce(const float* logits, long long ld_in, const int32_t* tgt, void* dl, long long ld_out,
               float* loss_row, long long rows, int vocab, float inv_rows, int* err, cudaStream_t s);
// Vocab-chunked head (hlm_cuda_head_stats / hlm_cuda_head_grad_chunk): pass-1 row
// statistics (float2 max, 1/z per row), pass-2 d_logits of one vocab chunk, and
// the up-front finiteness certificate of d_head (word: ~0 or HLM_HEAD_UNCERTIFIED).
int hlm_ops_ce_stats(const float* logits, long long ld_in, const int32_t* tgt, void* stats, float* loss_row,
                     long long rows, int vocab, float inv_rows, int* err, cudaStream_t s);
int hlm_ops_ce_grad_chunk(const float* logits, long long ld_in, const int32_t* tgt, const void* stats, void* dl,
                          long long ld_out, long long rows, int v0, int vc, float inv_rows, cudaStream_t s);
int hlm_ops_head_certify(const void* x_bf, long long n, const void* stats, long long rows, float limit,
                         unsigned long long* word, cudaStream_t s);
int hlm_ops_attention_fwd_generic(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S,
                                  int H, int hd, int ld, cudaStream_t s);
int hlm_ops_attention_bwd_generic(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                  const float* lse, float* dsum, void* dq, void* dk, void* dv, int B, int S, int H,
                                  int hd, int ld, cudaStream_t s);

// Kernel launches issued by this library since load (all launchers add to it).
void hlm_count_launches(long long n);
long long hlm_launches_total();
// Deterministic pseudo-random bf16 fill (bench / probe inputs), |x| < 1.
int hlm_ops_fill_random_bf16(void* p, long long n, unsigned seed, cudaStream_t s);
// first[0] := smallest index of a non-finite element of g[0..n), ~0ull when none.
int hlm_ops_nonfinite(const float* g, long long n, unsigned long long* first, const unsigned long long* only_if,
                      cudaStream_t s);
// Adam on HBM-resident optimizer state (bit-identical to the host kernel); no-op when *bad != ~0.
int hlm_ops_adam_device(float* w, float* m, float* v, void* w16, const float* g, long long n,
                        const unsigned long long* bad, float lr, float b1, float b2, float eps, float wd, float bc1,
                        float bc2, cudaStream_t s);
