// Elementwise math shared by the standalone SwiGLU / RoPE kernels (block_ops.cu) and the
// GEMM epilogues that fuse them (gemm_sm100.cu). Every product and sum is an explicit
// IEEE-rounded intrinsic, so the compiler can never contract them into FMAs differently
// in the two places: the fused and unfused paths agree bit for bit (tested).
//
// Reference semantics: SwiGLU of block_forward / block_backward
// (proj/include/hlm/kernels.hpp:301-311, 342-347); RoPE is the rotate-half extension
// (oracle/hlm_oracle.cpp rope_apply).
#pragma once

#include <cuda_bf16.h>

namespace hlm_fused {

__device__ __forceinline__ float round_bf16(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ float sigmoid(float z) { return __frcp_rn(__fadd_rn(1.0f, __expf(-z))); }

// act = up * silu(gate) = up * (gate * sigmoid(gate))
__device__ __forceinline__ float swiglu(float up, float gate) {
  return __fmul_rn(up, __fmul_rn(gate, sigmoid(gate)));
}

// d_up = d_act * gate * s ; d_gate = d_act * up * (s * (1 + gate * (1 - s))), s = sigmoid(gate)
__device__ __forceinline__ void swiglu_bwd(float d_act, float up, float gate, float& d_up, float& d_gate) {
  const float s = sigmoid(gate);
  d_up = __fmul_rn(__fmul_rn(d_act, gate), s);
  const float ds = __fmul_rn(s, __fadd_rn(1.0f, __fmul_rn(gate, __fsub_rn(1.0f, s))));
  d_gate = __fmul_rn(__fmul_rn(d_act, up), ds);
}

// rotate-half RoPE of the pair (a, b) = (x[i], x[i + half]); inverse = transpose rotation.
__device__ __forceinline__ void rope_rotate(float a, float b, float c, float s, bool inverse, float& oa, float& ob) {
  if (!inverse) {
    oa = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
    ob = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
  } else {
    oa = __fadd_rn(__fmul_rn(a, c), __fmul_rn(b, s));
    ob = __fsub_rn(__fmul_rn(b, c), __fmul_rn(a, s));
  }
}

}  // namespace hlm_fused
