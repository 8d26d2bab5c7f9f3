/* oracle_abi.h — C ABI shared by the two CPU checkers under oracle/:
 *   liboracle.so        our restatement (hlm_oracle.cpp), with the multi-head
 *                       + RoPE extension the B200 perf configs need;
 *   _ref/libhlm_ref.so  the reference itself, compiled from the read-only
 *                       sources under /root/reference/proj/src plus ref_shim.cpp.
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py. Never linked into the
 * product library.
 *
 * Parameter layout everywhere: physical tiles in store order — embed (V,h),
 * blocks 1..L in the offset-table order w_q w_k w_v w_o (h,h) w_up w_gate (h,f)
 * w_down (f,h) norm1 norm2 (h), then head (V,h) unless tied
 * (reference host_store.cpp:70-92, 94-114). */
#ifndef HLM_ORACLE_ABI_H_
#define HLM_ORACLE_ABI_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct OrcCfg {
  int64_t layers, hidden, ffn, vocab, seq, batch, k_ckpt;
  int32_t tie;        /* tied embedding / head */
  int32_t n_heads;    /* 1 = reference semantics (single head)             */
  double rope_theta;  /* 0 = no RoPE (reference semantics); Qwen2.5: 1e6   */
} OrcCfg;

typedef struct OrcHyper {
  double lr, beta1, beta2, eps, weight_decay;
} OrcHyper;

#ifdef __cplusplus
}
#endif
#endif
