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

/* Select this process's GPU (call before creating stores, communicators or arenas). */
int hlm_cuda_set_device(int device);

/* ------------------------------------------------------------------ device runtime
 * SURVEY.md §8b's runtime entry points, for a host caller that keeps its own
 * scheduler (the reference's Engine::stream_tile / evacuate, proj/src/engine.cpp:55-71,
 * 186-203, and its DeviceArena, proj/src/device_arena.cpp): streams, events and the
 * arena are opaque pointers, so the caller never includes a CUDA header.
 * hlm_cuda_init selects the device and fills caps; HLM_ERR_CONFIG when the device is
 * not sm_100 (this build carries sm_100a code only). */
typedef struct HlmCaps {
  int device, sm_count, cc_major, cc_minor;
  int64_t hbm_bytes, l2_bytes, smem_per_block_optin;
  char name[64];
} HlmCaps;
enum HlmStreamKind { HLM_STREAM_COMPUTE = 0, HLM_STREAM_H2D = 1, HLM_STREAM_D2H = 2, HLM_STREAM_COMM = 3,
                     HLM_STREAM_OPT = 4 };
#define HLM_NOT_READY 1   /* hlm_cuda_event_query: recorded work still pending */
int hlm_cuda_init(int device, HlmCaps* caps);
int hlm_cuda_arena_create(size_t bytes, void** base);   /* one device allocation; HLM_ERR_OOM */
int hlm_cuda_arena_destroy(void* base);
int hlm_cuda_stream_create(int kind, void** stream);    /* non-blocking; compute at top priority */
int hlm_cuda_stream_destroy(void* stream);
int hlm_cuda_stream_sync(void* stream);
int hlm_cuda_event_create(void** event);
int hlm_cuda_event_destroy(void* event);
int hlm_cuda_event_record(void* event, void* stream);
int hlm_cuda_event_wait(void* stream, void* event);     /* stream waits for event (no host block) */
int hlm_cuda_event_sync(void* event);
int hlm_cuda_event_query(void* event);                  /* HLM_OK done, HLM_NOT_READY pending */
int hlm_cuda_event_elapsed_ms(void* start, void* end, float* ms);
int hlm_cuda_h2d_async(void* dst, const void* pinned_src, size_t bytes, void* stream);
int hlm_cuda_d2h_async(void* pinned_dst, const void* src, size_t bytes, void* stream);

/* Number of CUDA kernels this library has launched since it was loaded. */
long long hlm_cuda_launch_count(void);

/* ------------------------------------------------------------------ GEMM
 * C[g] = A[g] . B[g]  (bf16 operands, fp32 accumulation in TMEM)
 *   A element (m,k): a_mn ? A[k*lda + m] : A[m*lda + k]
 *   B element (k,n): b_mn ? B[k*ldb + n] : B[n*ldb + k]
 *   C element (m,n): C[m*ldc + n]
 * Groups (G >= 1): operand g lives at base + g*gstride when *_grouped.
 *   kgroup == 0: one output per group at C + g*c_gstride
 *   kgroup == 1: single output, C = sum_g A[g] . B[g]
 * Epilogues: BF16 store, FP32 store, FP32 store of R + acc (R may alias C).
 * Fused epilogues (the block's elementwise steps done on the accumulator, never
 * re-reading an intermediate from HBM; bit-identical to the separate kernels):
 *   HLM_EPI_BF16_ROPE  N-grouped q|k|v projection: BF16 store, with groups 0 and 1
 *                      (q, k) rotated by RoPE (rotate-half, tables rope_cos / rope_sin
 *                      [rope_seq][head_dim/2], position = row % rope_seq); head_dim
 *                      64 / 128 / 256. Replaces the GEMM + hlm rope pass.
 *   HLM_EPI_SWIGLU     up|gate projection with G = 2 (B groups w_up, w_gate; B MN-major):
 *                      each tile computes the same output columns of up and gate, stores
 *                      both BF16 (C, C + c_gstride) and act = up * silu(gate) BF16 to C2
 *                      (ldc2). Replaces the GEMM + swiglu_fwd.
 *   HLM_EPI_SWIGLU_BWD d_act = dY . W_down^T rounded to BF16, then with up / gate read
 *                      from aux (aux_ld, gate at aux + aux_gstride): d_up -> C,
 *                      d_gate -> C + c_gstride (BF16). Replaces the BF16 d_act store +
 *                      swiglu_bwd. */
enum HlmEpilogue {
  HLM_EPI_BF16 = 0,
  HLM_EPI_F32 = 1,
  HLM_EPI_F32_ADD = 2,
  HLM_EPI_BF16_ROPE = 3,
  HLM_EPI_SWIGLU = 4,
  HLM_EPI_SWIGLU_BWD = 5
};

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
  /* fused epilogues (appended; zero for the plain ones) */
  const float* rope_cos;
  const float* rope_sin;
  int rope_seq, rope_head_dim;
  const void* aux;
  long long aux_ld, aux_gstride;
  void* C2;
  long long ldc2;
} HlmGemmDesc;

int hlm_cuda_gemm(const HlmGemmDesc* desc, void* stream);

/* ------------------------------------------------------------------ block
 * One transformer block (reference kernels.hpp:313-383, plus the multi-head /
 * RoPE extension): pre-RMSNorm causal attention + residual, pre-RMSNorm
 * SwiGLU MLP + residual. Weights: the block's bf16 tile in the reference
 * offset-table order (w_q w_k w_v w_o (h,h), w_up w_gate (h,f), w_down (f,h),
 * norm1, norm2 (h); host_store.cpp:70-92). Residual stream and gradients are
 * fp32; GEMM operands bf16 with fp32 accumulation.
 *   acts: device buffer of hlm_cuda_block_acts_bytes() holding what backward
 *         consumes (n1, q|k|v after RoPE, o, lse, y, n2, up|gate, act).
 *   ws:   device scratch of hlm_cuda_block_ws_bytes().
 *   rope_cos / rope_sin: device tables [seq][head_dim/2] from
 *         hlm_cuda_rope_table(), or NULL when rope_theta == 0.
 * Backward overwrites grad_tile (fp32, tile order, block_params elements);
 * h_out must not alias h_in and g_in must not alias g_out (kernels.hpp:313,334). */
typedef struct HlmBlockDims {
  int64_t batch, seq, hidden, ffn;
  int32_t n_heads;   /* 1 = reference semantics */
  int32_t flags;     /* HLM_BLOCK_* */
} HlmBlockDims;

enum HlmBlockFlags {
  HLM_BLOCK_GENERIC_ATTENTION = 1, /* force the any-head_dim CUDA-core attention */
  HLM_BLOCK_UNFUSED = 2            /* separate RoPE / SwiGLU kernels instead of the fused GEMM
                                      epilogues (bit-identical; A/B and tests) */
};

size_t hlm_cuda_block_acts_bytes(const HlmBlockDims* d);
size_t hlm_cuda_block_ws_bytes(const HlmBlockDims* d);
int hlm_cuda_block_fwd(const HlmBlockDims* d, const void* w_tile, const float* h_in, float* h_out,
                       void* acts, void* ws, const float* rope_cos, const float* rope_sin,
                       void* stream);
int hlm_cuda_block_bwd(const HlmBlockDims* d, const void* w_tile, const float* h_in,
                       const void* acts, const float* g_out, float* g_in, float* grad_tile,
                       void* ws, const float* rope_cos, const float* rope_sin, void* stream);

/* RoPE tables [seq][head_dim/2]: angle = pos * theta^(-2i/head_dim) evaluated
 * in double on the host, rounded to fp32, copied to the device. */
int hlm_cuda_rope_table(float* dev_cos, float* dev_sin, int64_t seq, int64_t head_dim,
                        double theta);

/* ------------------------------------------------------------------ head + loss
 * logits = x . head^T (head (V,h) bf16), mean cross entropy with d_logits =
 * (softmax - onehot) * inv_rows, d_x = d_logits . head, d_head (+)= d_logits^T . x
 * (reference head_fwd / ce_loss_and_grad / head_bwd, kernels.hpp:410-446).
 * loss_rows[r] = (logz_r - logit_r[target_r]) * inv_rows; the caller sums.
 * inv_rows is 1/global_rows under data parallelism. */
size_t hlm_cuda_head_ws_bytes(int64_t rows, int64_t hidden, int64_t vocab);
/* Vocab-chunked head, the same numbers in pieces (engine's piecewise head gradient):
 * hlm_cuda_head_stats: logits row chunk by row chunk -> per-row max and 1/z kept in
 * ws, loss_rows as hlm_cuda_head_loss; then *cert = ~0 when every element of the
 * head weight gradient is provably finite before it is computed (finite row
 * statistics and rows * inv_rows * max|x| far below FLT_MAX), else
 * HLM_HEAD_UNCERTIFIED (the caller scans the gradient instead).
 * hlm_cuda_head_grad_chunk: vocab rows [v0, v0 + vc): logits chunk, d_logits,
 * d_head rows [v0, v0 + vc) of the (vocab, hidden) fp32 gradient (stored, or added
 * when accumulate_d_head), d_x (+)= d_logits_c . head_c (stored when
 * accumulate_d_x == 0). Same ws as hlm_cuda_head_loss, after hlm_cuda_head_stats.
 * hlm_cuda_head_chunk_vocab: the largest vc (multiple of 128) the ws holds. */
#define HLM_HEAD_UNCERTIFIED 0xFFFFFFFFFFFFFFFEull

/* Row-compact embedding gradient (reference embed_bwd_acc, kernels.hpp:396-408, for
 * the touched rows only): out[c] = sum of g rows at the positions of token rows[c]
 * (CSR from hlm_embed_csr; rows ascending) — equal to hlm_cuda_embed_bwd's row
 * rows[c] bit for bit; the (vocab - n_rows) untouched rows are exactly zero there. */
int hlm_cuda_embed_bwd_compact(const int32_t* row_ptr, const int32_t* pos, const int32_t* rows, int64_t n_rows,
                               const float* g, float* out, int64_t hidden, void* stream);

/* ------------------------------------------------------------------ kernel timer
 * Per-launch CUDA-event timing of the hot kernels inside a timed region (the
 * bench's roofline.achieved): when enabled, every GEMM / attention launch is
 * bracketed by an event pair on its own stream and its algorithmic flops kept.
 * collect() sums one kind (synchronises on its events); reset() recycles them. */
enum { HLM_KTIMER_GEMM = 0, HLM_KTIMER_ATTN_FWD = 1, HLM_KTIMER_ATTN_BWD = 2,
       /* HBM-bound kernels: work = algorithmic bytes (each tensor read / written once) */
       HLM_KTIMER_RMSNORM_FWD = 3, HLM_KTIMER_RMSNORM_BWD = 4, HLM_KTIMER_SWIGLU_FWD = 5,
       HLM_KTIMER_SWIGLU_BWD = 6, HLM_KTIMER_ROPE = 7, HLM_KTIMER_CAST = 8 };
int hlm_ktimer_enable(int on);
int hlm_ktimer_collect(int kind, double* ms, double* work, int64_t* launches);
int hlm_ktimer_reset(void);
int hlm_cuda_head_stats(int64_t rows, int64_t hidden, int64_t vocab, const void* head, const float* x,
                        const int32_t* targets, float inv_rows, float* loss_rows, unsigned long long* cert,
                        void* ws, void* stream);
int hlm_cuda_head_grad_chunk(int64_t rows, int64_t hidden, int64_t vocab, const void* head,
                             const int32_t* targets, float inv_rows, int64_t v0, int64_t vc, float* d_x,
                             int accumulate_d_x, float* d_head, int accumulate_d_head, void* ws, void* stream);
int64_t hlm_cuda_head_chunk_vocab(int64_t rows, int64_t vocab);
int hlm_cuda_head_loss(int64_t rows, int64_t hidden, int64_t vocab, const void* head,
                       const float* x, const int32_t* targets, float inv_rows, float* d_x,
                       float* d_head, int accumulate_d_head, float* loss_rows, void* ws,
                       void* stream);
/* The same head + cross-entropy in SURVEY.md §8b's argument order (head_fwd +
 * ce_loss_and_grad + head_bwd, proj/include/hlm/kernels.hpp:410-446; d_head overwritten):
 * per-row losses in loss_rows (device); loss_sum_out (host, optional) = their sum in row
 * order in double after the stream drains, as Engine::anchor_loss computes it. ws as
 * hlm_cuda_head_loss (hlm_cuda_head_ws_bytes). */
typedef struct HlmHeadDims {
  int64_t rows, hidden, vocab;
} HlmHeadDims;
int hlm_cuda_head_fwd_ce_bwd(const HlmHeadDims* dims, const void* head_bf16, const float* h,
                             const int32_t* targets, float inv_global_rows, float* d_h, float* d_head_fp32,
                             float* loss_rows, double* loss_sum_out, void* ws, void* stream);

/* ------------------------------------------------------------------ embedding
 * embed_fwd: out[t] = table[tokens[t]] widened to fp32 (kernels.hpp:385-394);
 *   an out-of-range id sets *err_flag |= 1 (device int) and yields zeros.
 * embed_bwd: d_table[v] (+)= sum of g[t] over the positions t of token v in
 *   ascending order (kernels.hpp:396-408 order, no atomics): row_ptr[V+1] and
 *   pos[] are the CSR of the batch tokens (hlm_embed_csr builds it on the host). */
int hlm_cuda_embed_fwd(const int32_t* tokens, const void* table, float* out, int64_t rows,
                       int64_t hidden, int64_t vocab, int* err_flag, void* stream);
int hlm_cuda_embed_bwd(const int32_t* row_ptr, const int32_t* pos, const float* g,
                       float* d_table, int64_t vocab, int64_t hidden, int accumulate,
                       void* stream);
int hlm_embed_csr(const int32_t* tokens, int64_t rows, int64_t vocab, int32_t* row_ptr,
                  int32_t* pos);

/* ------------------------------------------------------------------ small ops */
int hlm_cuda_cast_bf16(const float* in, void* out, int64_t n, void* stream);
/* Adam on HBM-resident optimizer state (w, m, v fp32, w16 bf16 out) — bit-identical
 * to the host Adam; skipped when *bad (device, from hlm_cuda_nonfinite) != ~0. */
struct HlmHyper;
int hlm_cuda_adam(float* w, float* m, float* v, void* w16, const float* g, int64_t n,
                  const unsigned long long* bad, const struct HlmHyper* hp, int64_t t, void* stream);
/* *first (device u64) := smallest index of a non-finite element of g, ~0 when all finite */
int hlm_cuda_nonfinite(const float* g, int64_t n, unsigned long long* first, void* stream);
/* the same scan only when *certificate (device, from hlm_cuda_head_stats) is
 * HLM_HEAD_UNCERTIFIED; otherwise *first := ~0 and g is not read */
int hlm_cuda_nonfinite_if_uncertified(const float* g, int64_t n, unsigned long long* first,
                                      const unsigned long long* certificate, void* stream);

/* Device-event timer for harnesses: record(slot) synchronises the device and
 * records an event on the legacy stream; elapsed_ms(a, b) between two slots. */
int hlm_timer_record(int slot);
double hlm_timer_elapsed_ms(int a, int b);

/* Live roofline probe of the dominant kernel: the 12 tcgen05 GEMM launches of
 * one block (4 forward, 8 backward: dgrad + wgrad) at the given dims, timed
 * with CUDA events over `iters` repetitions on one stream. Outputs the
 * algorithmic flops of the set, the mean ms per set and the per-launch mean. */
int hlm_cuda_bench_block_gemms(const HlmBlockDims* d, int iters, double* flops, double* ms_per_set,
                               double* ms_per_launch);
/* Achieved HBM GB/s (algorithmic bytes / CUDA-event time) of the block's
 * elementwise and norm kernels at the workload shape; gbs[6], ms[6] (ms may be
 * NULL) in the order rmsnorm_fwd, rmsnorm_bwd, swiglu_fwd, swiglu_bwd, rope, cast. */
int hlm_cuda_bench_block_ops(const HlmBlockDims* d, int iters, double* gbs, double* ms);
int hlm_cuda_attention_fwd(const HlmBlockDims* d, const void* q, const void* k, const void* v,
                           void* o, float* lse, int64_t ld, void* stream);
int hlm_cuda_attention_bwd(const HlmBlockDims* d, const void* q, const void* k, const void* v,
                           const void* o, const void* d_o, const float* lse, float* dsum,
                           void* dq, void* dk, void* dv, int64_t ld, void* stream);


/* ------------------------------------------------------------------ host engine
 * Opaque handles over the C++ engine (include/hlm/ headers): the entry points a
 * binding of the reference's Python / CLI surface (proj/python/bindings.cpp:79-96,
 * tools/hlm_main.cpp:191-236) would call. Layout of HlmModelConfig matches
 * oracle/oracle_abi.h OrcCfg. */
typedef struct HlmModelConfig {
  int64_t layers, hidden, ffn, vocab, seq, batch, k_ckpt;
  int32_t tie_embeddings;
  int32_t n_heads;     /* 1 = reference semantics */
  double rope_theta;   /* 0 = no RoPE */
} HlmModelConfig;

typedef struct HlmHyper {
  double lr, beta1, beta2, eps, weight_decay;
} HlmHyper;

typedef struct HlmEngineOptions {
  int32_t eager_optim;
  int32_t threaded_accum;
  int64_t n_slab;
  int64_t accum_delay_us;
  int32_t skip_optimizer;
  int32_t fused_recompute;
  int32_t record_trace;
  int32_t block_flags;
  int32_t overlap_optimizer_tail; /* head + top tail_blocks optimised while the next step starts */
  int32_t tail_blocks;
  /* data parallel: this process is `rank` of `world`; per-layer fp32 gradient
   * reduce-scatter on comm_grad; sharded weight H2D + all-gather on comm_weights
   * (may be NULL: full H2D per rank). Communicators from hlm_nccl_comm_create. */
  int32_t rank;
  int32_t world;
  void* comm_grad;
  void* comm_weights;
  int32_t host_threads;  /* OpenMP threads of the optimizer worker (0 = default) */
  /* HBM-resident optimizer tiles: embedding + blocks 1..resident_blocks keep FP32
   * master / m / v and BF16 weights on the GPU (device Adam, no streaming) */
  int32_t resident_embed;
  int64_t resident_blocks;
  /* vocab rows per piece of the head weight gradient (vocab-chunked head, each
   * piece's D2H and host Adam start while the next piece is computed):
   * 0 = auto (~64 Mi elements per piece when the head spans two or more), -1 = off */
  int64_t head_piece_vocab;
  /* elements per gradient D2H / host Adam / forward weight H2D piece (0 = 64 Mi) */
  int64_t piece_elems;
  /* outbound fp32 gradient buffers on the device (<= 2: the arena's two) */
  int64_t grad_buffers;
  /* row-sparse embedding gradient (only the batch's token rows computed, copied and
   * read by the host Adam; bit-identical results) */
  int32_t sparse_embed_grad;
  /* forward embedding rows gathered zero-copy from the pinned host shadow (no table H2D) */
  int32_t embed_gather_host;
  /* 1: leave the host optimizer's OpenMP team unpinned (default: pinned to cores) */
  int32_t no_pin_threads;
  /* was transit_blocks (the transit-tile mode, removed in round 2): kept so the fields after
   * it keep their offsets; must be 0 (a non-zero value is rejected with HLM_ERR_CONFIG) */
  int64_t reserved_transit_blocks;
  /* blocks L - saved_act_layers + 1 .. L keep their forward activations in HBM until
   * their backward (no recompute; bit-identical: the recompute would reproduce them) */
  int64_t saved_act_layers;
} HlmEngineOptions;

typedef struct HlmStepResult {
  double loss;
  int64_t h2d_bytes, d2h_bytes, recompute_forwards;
  double gpu_ms;
  int64_t arena_committed, arena_peak, host_total, slab_max_in_use;
} HlmStepResult;

typedef struct HlmStore HlmStore;
typedef struct HlmArena HlmArena;
typedef struct HlmEngine HlmEngine;

enum HlmStoreField { HLM_FIELD_MASTER = 0, HLM_FIELD_M = 1, HLM_FIELD_V = 2, HLM_FIELD_GRADS = 3,
                     HLM_FIELD_SHADOW = 4 };

/* dtype: 0 = bf16 init (reference bf16-store values), 1 = fp32 init.
 * init_mode: 0 = bit-identical to reference build_store, 1 = parallel. */
int hlm_store_create(const HlmModelConfig* cfg, uint64_t seed, int dtype, int init_mode, int pin_shadow,
                     HlmStore** out);
void hlm_store_destroy(HlmStore* s);
int64_t hlm_store_total_params(const HlmStore* s);
int64_t hlm_store_adam_steps(const HlmStore* s);
/* all physical tiles in store order, fp32 (shadow widened from bf16) */
int hlm_store_export(const HlmStore* s, int field, float* out);
int hlm_store_import_master(HlmStore* s, const float* w);   /* master := w, shadow re-packed */
int hlm_store_bitwise_equal(const HlmStore* a, const HlmStore* b);
/* Shared host store for one-process-per-GPU data parallelism: rank 0 creates
 * /dev/shm/<name> and initialises it, the other ranks attach. `nonce` is a per-run
 * token all ranks share (e.g. a hash of the NCCL unique id): an attaching rank only
 * accepts the segment rank 0 stamped with it, never a stale one of a crashed run;
 * it also checks the segment's model dims / world size (HLM_ERR_CONFIG otherwise). */
int hlm_store_create_shared(const HlmModelConfig* cfg, uint64_t seed, int dtype, int init_mode, int pin_shadow,
                            const char* name, int rank, int world, uint64_t nonce, HlmStore** out);
/* Data-parallel host Adam: this rank updates its 1/world shard of every tile
 * from full-size gradients (store layout) and bumps its version counters. */
int hlm_store_adam_shard(HlmStore* s, const float* grads, const HlmHyper* hp, int64_t t, int rank, int world);
/* min over ranks of the completed-update counter of physical tile p */
int64_t hlm_store_tile_version(const HlmStore* s, int64_t p);
/* Host Adam on every physical tile from caller gradients (store layout),
 * step index t (reference adam_update_tile, host_store.cpp:334-362). */
int hlm_store_adam_step(HlmStore* s, const float* grads, const HlmHyper* hp, int64_t t);
/* Host Adam on the embedding tile from a row-compact gradient: rows[c] (ascending,
 * n_rows of them) carry compact[c * hidden ...], every other row a zero gradient that
 * is not read (the engine's sparse_embed_grad path); bit-identical to hlm_store_adam_step
 * on the dense gradient for that tile. */
int hlm_store_adam_embed_rows(HlmStore* s, const int32_t* rows, int64_t n_rows, const float* compact,
                              const HlmHyper* hp, int64_t t);

/* CPUs a data-parallel rank's optimizer team is pinned to (the engine's own
 * placement rule, exposed for testing): rank's share of the CPUs of its GPU's NUMA
 * node, split among the ranks on that node. gpu_nodes[world] = node of each rank's
 * GPU (-1 unknown); allowed[n_allowed] = the process affinity (ascending); online =
 * host CPU count; node_of_cpu[n_cpus] = node of each CPU id. Writes up to out_cap
 * CPU ids to out and returns how many (negative on error). */
int hlm_rank_cpu_slice(int rank, const int* gpu_nodes, int world, const int* allowed, int n_allowed, int online,
                       const int* node_of_cpu, int n_cpus, int* out, int out_cap);

int hlm_arena_create(const HlmModelConfig* cfg, int64_t budget_cap, int device, HlmArena** out);
/* + an HBM weight cache of weight_cache_bytes (block tiles resident between the
 * forward and the backward of a step: one H2D pass for every cached layer) */
int hlm_arena_create_ex(const HlmModelConfig* cfg, int64_t budget_cap, int device, int64_t weight_cache_bytes,
                        HlmArena** out);
void hlm_arena_destroy(HlmArena* a);
/* out[5] = stream_buf, anchor_slot, anchor_slots, stack, workspace (bytes) */
int hlm_arena_footprint(const HlmModelConfig* cfg, int64_t* out);

int hlm_engine_create(HlmStore* s, HlmArena* a, const HlmHyper* hp, const HlmEngineOptions* o,
                      HlmEngine** out);
void hlm_engine_destroy(HlmEngine* e);
int hlm_engine_train_step(HlmEngine* e, const int32_t* tokens, const int32_t* targets, HlmStepResult* out);
/* wait for every pending host optimizer update and copy HBM-resident optimizer
 * tiles back (store consistent afterwards) */
int hlm_engine_sync(HlmEngine* e);
/* wait for the host optimizer only (end of the training work; no write-back) */
int hlm_engine_wait_optimizer(HlmEngine* e);
/* phase API (reference engine.hpp:62-66); out-of-order calls -> HLM_ERR_PROTOCOL */
int hlm_engine_begin_step(HlmEngine* e, const int32_t* tokens, const int32_t* targets);
int hlm_engine_forward(HlmEngine* e);
int hlm_engine_anchor_loss(HlmEngine* e, double* loss);
int hlm_engine_backward(HlmEngine* e);
int hlm_engine_finish_step(HlmEngine* e, HlmStepResult* out);
int hlm_engine_debug_hidden(HlmEngine* e, float* out);
/* JSONL of the last step's measured trace; *needed = bytes incl. NUL */
int hlm_engine_last_trace(HlmEngine* e, char* buf, size_t cap, size_t* needed);

/* Host DRAM bandwidth probe (all OpenMP threads): STREAM triad a = b + s*c over
 * three arrays of `bytes_per_array`, best of `reps`; GB/s counting 3 arrays. */
double hlm_host_triad_gbs(int64_t bytes_per_array, int reps);
/* "avx512" | "generic": host Adam / BF16-pack / finiteness loop bodies selected at load
 * time from the CPU (x86-64-v3 baseline; HLM_HOST_ISA=generic forces the portable ones).
 * Both are bit-identical to the reference's scalar arithmetic. */
const char* hlm_host_isa(void);

/* HLM2 checkpoint of the host store (master, m, v, Adam step count); load
 * re-derives the BF16 shadow and rejects mismatched geometry (HLM_ERR_CONFIG).
 * hlm_store_load also reads the reference's HLM1 files (replaces hlm::load_checkpoint,
 * /root/reference/proj/src/checkpoint.cpp:71-120: same checks and messages);
 * hlm_store_save_hlm1 writes HLM1 for the reference's loader (replaces
 * hlm::save_checkpoint, checkpoint.cpp:38-69). */
int hlm_store_save(const HlmStore* s, const char* path);
int hlm_store_load(HlmStore* s, const char* path);
int hlm_store_save_hlm1(const HlmStore* s, const char* path);

/* NCCL (loaded at run time): 128-byte unique id, communicator create / destroy */
int hlm_nccl_unique_id(uint8_t* out128);
int hlm_nccl_comm_create(const uint8_t* id128, int world, int rank, void** comm);
void hlm_nccl_comm_destroy(void* comm);
/* The data-parallel exchange steps for callers that keep their own engine:
 * per-layer fp32 gradient reduce-scatter (sum; `count` elements land on each rank, send
 * holds world x count), bf16 weight all-gather (each rank contributes `count`), and the
 * loss all-reduce (sum, in place allowed). Stream-ordered on `stream`; status codes as
 * everywhere else (HLM_ERR_CUDA on an NCCL failure). */
int hlm_nccl_reduce_scatter_f32(void* comm, const float* send, float* recv, int64_t count, void* stream);
int hlm_nccl_all_gather_bf16(void* comm, const void* send, void* recv, int64_t count, void* stream);
int hlm_nccl_allreduce_f32(void* comm, const float* send, float* recv, int64_t count, void* stream);

int hlm_make_copy_task_batch(const HlmModelConfig* cfg, uint64_t data_seed, int64_t skip, int32_t* tokens);
/* run_training (trainer.hpp): store from seed, data seed+1, `steps` steps;
 * hlm_run_training_store continues an existing store (resume: the data stream
 * is replayed past store->adam_steps batches). */
int hlm_run_training_store(HlmStore* s, const HlmHyper* hp, uint64_t seed, int64_t steps,
                           const HlmEngineOptions* o, double* losses);
int hlm_run_training(const HlmModelConfig* cfg, const HlmHyper* hp, uint64_t seed, int dtype, int64_t steps,
                     const HlmEngineOptions* o, double* losses, HlmStepResult* last);

#ifdef __cplusplus
}
#endif

#endif /* HLM_CUDA_H_ */
