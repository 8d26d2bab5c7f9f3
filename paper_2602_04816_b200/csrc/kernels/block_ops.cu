// Row-wise / elementwise kernels of the transformer block, head and embedding
// (everything in reference proj/include/hlm/kernels.hpp that is not a GEMM):
//   rmsnorm_fwd / rmsnorm_bwd        kernels.hpp:129-162
//   SwiGLU fwd / bwd                 kernels.hpp:301-311, 329, 342-347
//   embed gather / scatter-add       kernels.hpp:385-408
//   cross entropy + d_logits         kernels.hpp:423-446
//   RoPE (extension, Qwen2 rotate-half)
// All HBM-bound: 16-byte vector accesses; RMSNorm keeps a chunk's rows in
// registers between the row reduction and the output pass (one HBM read of each
// input); fixed-order (deterministic) reductions everywhere. Achieved GB/s at
// the workload shape: hlm_cuda_bench_block_ops (bench.py elementwise_roofline).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "block_ops.h"
#include "fused_math.cuh"
#include "hlm_cuda.h"

namespace {

constexpr float kEps = 1e-6f;   // kernels.hpp:127

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float bf(const __nv_bfloat16 x) { return __bfloat162float(x); }

int grid_for(long long n, int per_block) {
  long long g = (n + per_block - 1) / per_block;
  if (g > 148LL * 64) g = 148LL * 64;
  return static_cast<int>(g < 1 ? 1 : g);
}

// ------------------------------------------------------------------ RMSNorm
// out_bf16[r] = x[r] * inv_rms(x[r]) * scale ; one warp per row.
__global__ void rmsnorm_fwd_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ scale,
                                   __nv_bfloat16* __restrict__ out, long long rows, int h) {
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* xr = x + r * h;
    float ss = 0.f;
    if ((h & 3) == 0) {
      for (int j = lane * 4; j < h; j += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + j);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    } else {
      for (int j = lane; j < h; j += 32) ss += xr[j] * xr[j];
    }
    ss = warp_sum(ss);
    const float inv = 1.0f / sqrtf(ss / (float)h + kEps);
    __nv_bfloat16* o = out + r * h;
    if ((h & 3) == 0) {
      for (int j = lane * 4; j < h; j += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + j);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * bf(scale[j]), v.y * inv * bf(scale[j + 1]));
        __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * bf(scale[j + 2]), v.w * inv * bf(scale[j + 3]));
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&a);
        pk.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(o + j) = pk;
      }
    } else {
      for (int j = lane; j < h; j += 32) o[j] = __float2bfloat16_rn(xr[j] * inv * bf(scale[j]));
    }
  }
}

// Register-resident forward: one block per chunk of rows, thread owns float4
// columns q = tid + k*THREADS; x read once, scale loaded once per block.
template <int THREADS, int V>
__global__ void __launch_bounds__(THREADS)
    rmsnorm_fwd_reg_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ scale,
                           __nv_bfloat16* __restrict__ out, long long rows, int h, int rows_per_block) {
  constexpr int NW = THREADS / 32;
  __shared__ float red[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nv = h >> 2;
  float4 sc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int q = tid + k * THREADS;
    sc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q < nv) {
      const uint2 spk = *reinterpret_cast<const uint2*>(scale + 4 * q);
      const float2 s01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.x));
      const float2 s23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.y));
      sc[k] = make_float4(s01.x, s01.y, s23.x, s23.y);
    }
  }
  const long long r0 = (long long)blockIdx.x * rows_per_block;
  const long long r1 = r0 + rows_per_block < rows ? r0 + rows_per_block : rows;
  int par = 0;
  for (long long r = r0; r < r1; ++r, par ^= 1) {
    float4 xv[V];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        xv[k] = reinterpret_cast<const float4*>(x + r * h)[q];
        ss += xv[k].x * xv[k].x + xv[k].y * xv[k].y + xv[k].z * xv[k].z + xv[k].w * xv[k].w;
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) red[par][warp] = ss;
    __syncthreads();
    ss = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) ss += red[par][w];
    const float inv = 1.0f / sqrtf(ss / (float)h + kEps);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(xv[k].x * inv * sc[k].x, xv[k].y * inv * sc[k].y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(xv[k].z * inv * sc[k].z, xv[k].w * inv * sc[k].w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(out + r * h)[q] = pk;
      }
    }
  }
}

// g_x = g*s*inv - inv^3 * (sum g*s*x)/h * x ;  out = g_x + resid ; also the
// per-row inv (consumed by the deterministic scale-gradient reduction).
__global__ void rmsnorm_bwd_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ scale,
                                   const float* __restrict__ g, const float* __restrict__ resid,
                                   float* __restrict__ out, __nv_bfloat16* __restrict__ out_bf,
                                   float* __restrict__ inv_out, long long rows, int h) {
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* xr = x + r * h;
    const float* gr = g + r * h;
    float ss = 0.f, dot = 0.f;
    if ((h & 3) == 0) {
      for (int j = lane * 4; j < h; j += 128) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + j);
        const float4 gv = *reinterpret_cast<const float4*>(gr + j);
        const uint2 sp = *reinterpret_cast<const uint2*>(scale + j);
        const float2 s01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sp.x));
        const float2 s23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sp.y));
        ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        dot += gv.x * s01.x * xv.x + gv.y * s01.y * xv.y + gv.z * s23.x * xv.z + gv.w * s23.y * xv.w;
      }
    } else {
      for (int j = lane; j < h; j += 32) {
        const float xv = xr[j];
        ss += xv * xv;
        dot += gr[j] * bf(scale[j]) * xv;
      }
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    const float inv = 1.0f / sqrtf(ss / (float)h + kEps);
    const float c = inv * inv * inv * dot / (float)h;
    if (lane == 0) inv_out[r] = inv;
    const float* rr = resid ? resid + r * h : nullptr;
    if ((h & 3) == 0) {
      for (int j = lane * 4; j < h; j += 128) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + j);
        const float4 gv = *reinterpret_cast<const float4*>(gr + j);
        const uint2 sp = *reinterpret_cast<const uint2*>(scale + j);
        const float2 s01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sp.x));
        const float2 s23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sp.y));
        float4 v = make_float4(gv.x * s01.x * inv - c * xv.x, gv.y * s01.y * inv - c * xv.y,
                               gv.z * s23.x * inv - c * xv.z, gv.w * s23.y * inv - c * xv.w);
        if (rr) {
          const float4 q = *reinterpret_cast<const float4*>(rr + j);
          v.x += q.x;
          v.y += q.y;
          v.z += q.z;
          v.w += q.w;
        }
        *reinterpret_cast<float4*>(out + r * h + j) = v;
        if (out_bf) {
          __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&a);
          pk.y = *reinterpret_cast<uint32_t*>(&b);
          *reinterpret_cast<uint2*>(out_bf + r * h + j) = pk;
        }
      }
    } else {
      for (int j = lane; j < h; j += 32) {
        float v = gr[j] * bf(scale[j]) * inv - c * xr[j];
        if (rr) v += rr[j];
        out[r * h + j] = v;
        if (out_bf) out_bf[r * h + j] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Register-resident variant: one block per chunk of rows_per_chunk rows; each
// thread owns float4 columns q = tid + k*THREADS (k < V) and keeps the row's x,
// g and its scale in registers between the reduction and the output pass, so x
// and g are read from HBM once. The scale-gradient partial of the chunk
// (sum over its rows of g*x*inv, row order) accumulates in registers too.
// Deterministic: fixed-order warp and block reductions.
template <int THREADS, int V, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    rmsnorm_bwd_reg_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ scale,
                           const float* __restrict__ g, const float* __restrict__ resid, float* __restrict__ out,
                           __nv_bfloat16* __restrict__ out_bf, float* __restrict__ inv_out,
                           float* __restrict__ partial, long long rows, int h, int rows_per_chunk) {
  constexpr int NW = THREADS / 32;
  __shared__ float red[2][2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nv = h >> 2;
  float4 sc[V], acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int q = tid + k * THREADS;
    acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    sc[k] = acc[k];
    if (q < nv) {
      const uint2 spk = *reinterpret_cast<const uint2*>(scale + 4 * q);
      const float2 s01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.x));
      const float2 s23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.y));
      sc[k] = make_float4(s01.x, s01.y, s23.x, s23.y);
    }
  }
  const long long r0 = (long long)blockIdx.x * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  int par = 0;
  for (long long r = r0; r < r1; ++r, par ^= 1) {
    // x and g stay in registers between the row reduction and the output pass; the
    // residual is read in the output pass only (keeping it live spilled at 3 CTAs / SM)
    float4 xv[V], gv[V];
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        xv[k] = __ldcs(reinterpret_cast<const float4*>(x + r * h) + q);
        gv[k] = __ldcs(reinterpret_cast<const float4*>(g + r * h) + q);
        ss += xv[k].x * xv[k].x + xv[k].y * xv[k].y + xv[k].z * xv[k].z + xv[k].w * xv[k].w;
        dot += gv[k].x * sc[k].x * xv[k].x + gv[k].y * sc[k].y * xv[k].y + gv[k].z * sc[k].z * xv[k].z +
               gv[k].w * sc[k].w * xv[k].w;
      }
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    if (lane == 0) {
      red[par][0][warp] = ss;
      red[par][1][warp] = dot;
    }
    __syncthreads();   // red[par] complete; red[par ^ 1] (last row) no longer read
    ss = 0.f;
    dot = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ss += red[par][0][w];
      dot += red[par][1][w];
    }
    const float inv = 1.0f / sqrtf(ss / (float)h + kEps);
    const float c = inv * inv * inv * dot / (float)h;
    if (tid == 0) inv_out[r] = inv;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        const float4 rv = resid ? __ldcs(reinterpret_cast<const float4*>(resid + r * h) + q)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 v = make_float4(gv[k].x * sc[k].x * inv - c * xv[k].x + rv.x,
                                     gv[k].y * sc[k].y * inv - c * xv[k].y + rv.y,
                                     gv[k].z * sc[k].z * inv - c * xv[k].z + rv.z,
                                     gv[k].w * sc[k].w * inv - c * xv[k].w + rv.w);
        __stcs(reinterpret_cast<float4*>(out + r * h) + q, v);
        if (out_bf) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          reinterpret_cast<uint2*>(out_bf + r * h)[q] = pk;
        }
        acc[k].x += gv[k].x * xv[k].x * inv;
        acc[k].y += gv[k].y * xv[k].y * inv;
        acc[k].z += gv[k].z * xv[k].z * inv;
        acc[k].w += gv[k].w * xv[k].w * inv;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int q = tid + k * THREADS;
    if (q < nv) reinterpret_cast<float4*>(partial + (long long)blockIdx.x * h)[q] = acc[k];
  }
}

// The same computation with the row's scale and the chunk's scale-gradient partial in
// shared memory instead of registers (32 registers fewer per thread): 3 CTAs per SM, so
// three rows' HBM traffic is in flight per SM instead of two. Each thread owns the same
// float4 columns in both, so the per-column sums run in the same row order: bit-identical
// to rmsnorm_bwd_reg_kernel.
template <int THREADS, int V, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    rmsnorm_bwd_smem_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ scale,
                            const float* __restrict__ g, const float* __restrict__ resid, float* __restrict__ out,
                            __nv_bfloat16* __restrict__ out_bf, float* __restrict__ inv_out,
                            float* __restrict__ partial, long long rows, int h, int rows_per_chunk) {
  constexpr int NW = THREADS / 32;
  __shared__ float red[2][2][NW];
  extern __shared__ float4 dyn4[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nv = h >> 2;
  float4* ssc = dyn4;          // [nv] row scale
  float4* sacc = dyn4 + nv;    // [nv] scale-gradient partial of the chunk
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int q = tid + k * THREADS;
    if (q < nv) {
      const uint2 spk = *reinterpret_cast<const uint2*>(scale + 4 * q);
      const float2 s01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.x));
      const float2 s23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&spk.y));
      ssc[q] = make_float4(s01.x, s01.y, s23.x, s23.y);
      sacc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const long long r0 = (long long)blockIdx.x * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  int par = 0;
  for (long long r = r0; r < r1; ++r, par ^= 1) {
    float4 xv[V], gv[V];
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        xv[k] = __ldcs(reinterpret_cast<const float4*>(x + r * h) + q);
        gv[k] = __ldcs(reinterpret_cast<const float4*>(g + r * h) + q);
        const float4 sc = ssc[q];
        ss += xv[k].x * xv[k].x + xv[k].y * xv[k].y + xv[k].z * xv[k].z + xv[k].w * xv[k].w;
        dot += gv[k].x * sc.x * xv[k].x + gv[k].y * sc.y * xv[k].y + gv[k].z * sc.z * xv[k].z +
               gv[k].w * sc.w * xv[k].w;
      }
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    if (lane == 0) {
      red[par][0][warp] = ss;
      red[par][1][warp] = dot;
    }
    __syncthreads();   // red[par] complete; red[par ^ 1] (last row) no longer read
    ss = 0.f;
    dot = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ss += red[par][0][w];
      dot += red[par][1][w];
    }
    const float inv = 1.0f / sqrtf(ss / (float)h + kEps);
    const float c = inv * inv * inv * dot / (float)h;
    if (tid == 0) inv_out[r] = inv;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int q = tid + k * THREADS;
      if (q < nv) {
        const float4 sc = ssc[q];
        const float4 rv = resid ? __ldcs(reinterpret_cast<const float4*>(resid + r * h) + q)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 v = make_float4(gv[k].x * sc.x * inv - c * xv[k].x + rv.x,
                                     gv[k].y * sc.y * inv - c * xv[k].y + rv.y,
                                     gv[k].z * sc.z * inv - c * xv[k].z + rv.z,
                                     gv[k].w * sc.w * inv - c * xv[k].w + rv.w);
        __stcs(reinterpret_cast<float4*>(out + r * h) + q, v);
        if (out_bf) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          reinterpret_cast<uint2*>(out_bf + r * h)[q] = pk;
        }
        float4 a = sacc[q];
        a.x += gv[k].x * xv[k].x * inv;
        a.y += gv[k].y * xv[k].y * inv;
        a.z += gv[k].z * xv[k].z * inv;
        a.w += gv[k].w * xv[k].w * inv;
        sacc[q] = a;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int q = tid + k * THREADS;
    if (q < nv) reinterpret_cast<float4*>(partial + (long long)blockIdx.x * h)[q] = sacc[q];
  }
}

// partial[c][j] = sum_{r in chunk c} g[r][j] * x[r][j] * inv[r]   (columns across threads)
__global__ void norm_scale_partial_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                          const float* __restrict__ inv, float* __restrict__ partial,
                                          long long rows, int h, int rows_per_chunk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (j >= h) return;
  const long long r0 = (long long)c * rows_per_chunk;
  const long long r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float acc = 0.f;
  for (long long r = r0; r < r1; ++r) acc += g[r * h + j] * x[r * h + j] * inv[r];
  partial[(long long)c * h + j] = acc;
}

// out[j] = sum_c partial[c][j]: 32 columns x 8 chunk groups per block; group k
// sums chunks k, k+8, ... in order, then the 8 group sums are added in group
// order (fixed, deterministic), coalesced 128-byte rows of partial.
__global__ void __launch_bounds__(256) norm_scale_reduce_kernel(const float* __restrict__ partial,
                                                                float* __restrict__ out, int chunks, int h) {
  __shared__ float red[8][33];
  const int col = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + col;
  float acc = 0.f;
  if (j < h) {
    // eight loads in flight per thread, added in the same chunk order (bit-identical sums)
    int c = grp;
    for (; c + 7 * 8 < chunks; c += 8 * 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = partial[(long long)(c + u * 8) * h + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; c < chunks; c += 8) acc += partial[(long long)c * h + j];
  }
  red[grp][col] = acc;
  __syncthreads();
  if (grp == 0 && j < h) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][col];
    out[j] = t;
  }
}

// ------------------------------------------------------------------ casts
__global__ void cast_f32_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&a);
    pk.y = *reinterpret_cast<uint32_t*>(&b);
    reinterpret_cast<uint2*>(out)[i] = pk;
  }
  for (long long i = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __float2bfloat16_rn(in[i]);
}

// ------------------------------------------------------------------ SwiGLU

// act = up * silu(gate) ; ug = [2][rows][f] (up then gate)
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ ug, __nv_bfloat16* __restrict__ act,
                                  long long n) {
  const __nv_bfloat16* up = ug;
  const __nv_bfloat16* gate = ug + n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += stride * 8) {
    if (i + 8 <= n) {
      const uint4 u = *reinterpret_cast<const uint4*>(up + i);
      const uint4 gg = *reinterpret_cast<const uint4*>(gate + i);
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gg);
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 uf = __bfloat1622float2(u2[k]), gf = __bfloat1622float2(g2[k]);
        o2[k] = __floats2bfloat162_rn(hlm_fused::swiglu(uf.x, gf.x), hlm_fused::swiglu(uf.y, gf.y));
      }
      *reinterpret_cast<uint4*>(act + i) = o;
    } else {
      for (long long k = i; k < n; ++k) act[k] = __float2bfloat16_rn(hlm_fused::swiglu(bf(up[k]), bf(gate[k])));
    }
  }
}

// d_up = d_act * silu(gate) ; d_gate = d_act * up * silu'(gate)  -> dug [2][rows][f]
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ dact, const __nv_bfloat16* __restrict__ ug,
                                  __nv_bfloat16* __restrict__ dug, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += stride * 8) {
    if (i + 8 <= n) {
      const uint4 dv = *reinterpret_cast<const uint4*>(dact + i);
      const uint4 uv = *reinterpret_cast<const uint4*>(ug + i);
      const uint4 zv = *reinterpret_cast<const uint4*>(ug + n + i);
      const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
      const __nv_bfloat162* z2 = reinterpret_cast<const __nv_bfloat162*>(&zv);
      uint4 ou, og;
      __nv_bfloat162* ou2 = reinterpret_cast<__nv_bfloat162*>(&ou);
      __nv_bfloat162* og2 = reinterpret_cast<__nv_bfloat162*>(&og);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 da = __bfloat1622float2(d2[k]), u = __bfloat1622float2(u2[k]), z = __bfloat1622float2(z2[k]);
        float dux, duy, dgx, dgy;
        hlm_fused::swiglu_bwd(da.x, u.x, z.x, dux, dgx);
        hlm_fused::swiglu_bwd(da.y, u.y, z.y, duy, dgy);
        ou2[k] = __floats2bfloat162_rn(dux, duy);
        og2[k] = __floats2bfloat162_rn(dgx, dgy);
      }
      *reinterpret_cast<uint4*>(dug + i) = ou;
      *reinterpret_cast<uint4*>(dug + n + i) = og;
    } else {
      for (long long k = i; k < n; ++k) {
        float du, dg;
        hlm_fused::swiglu_bwd(bf(dact[k]), bf(ug[k]), bf(ug[n + k]), du, dg);
        dug[k] = __float2bfloat16_rn(du);
        dug[n + k] = __float2bfloat16_rn(dg);
      }
    }
  }
}

// ------------------------------------------------------------------ RoPE
// rotate-half per head on x (rows, h) bf16, in place; inverse for backward.
__global__ void rope_kernel(__nv_bfloat16* __restrict__ x, const float* __restrict__ cs,
                            const float* __restrict__ sn, long long rows, int h, int hd, int S,
                            int inverse, int nmats, long long mat_stride) {
  const int half = hd / 2;
  const long long pairs = rows * (h / 2);
  const long long total = pairs * nmats;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int m = (int)(t / pairs);
    const long long p = t - (long long)m * pairs;
    const long long r = p / (h / 2);
    const int k = (int)(p - r * (h / 2));
    const int head = k / half, i = k - head * half;
    const int pos = (int)(r % S);
    __nv_bfloat16* v = x + m * mat_stride + r * h + head * hd;
    const float c = cs[pos * half + i], s = sn[pos * half + i];
    float oa, ob;
    hlm_fused::rope_rotate(bf(v[i]), bf(v[i + half]), c, s, inverse != 0, oa, ob);
    v[i] = __float2bfloat16_rn(oa);
    v[i + half] = __float2bfloat16_rn(ob);
  }
}

// 8 rotation pairs per thread: 16-byte loads of x[i..i+8) and x[i+half..), two
// float4 loads of cos / sin each (hd % 16 == 0, h % 8 == 0).
__global__ void rope8_kernel(__nv_bfloat16* __restrict__ x, const float* __restrict__ cs,
                             const float* __restrict__ sn, int rows, int h, int hd, int S, int inverse,
                             int nmats, long long mat_stride) {
  const int half = hd >> 1, cph = half >> 3;
  const int per_row = (h / hd) * cph;
  const long long per_mat = (long long)rows * per_row;
  const long long total = per_mat * nmats;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int m = (int)(t / per_mat);
    const long long p = t - (long long)m * per_mat;
    const int r = (int)(p / per_row);
    const int k = (int)(p - (long long)r * per_row);
    const int head = k / cph, i = (k - head * cph) * 8;
    const int pos = r % S;
    __nv_bfloat16* v = x + m * mat_stride + (long long)r * h + head * hd + i;
    uint4 ua = *reinterpret_cast<const uint4*>(v);
    uint4 ub = *reinterpret_cast<const uint4*>(v + half);
    const float4* cp = reinterpret_cast<const float4*>(cs + (long long)pos * half + i);
    const float4* sp = reinterpret_cast<const float4*>(sn + (long long)pos * half + i);
    const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
    const float c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    __nv_bfloat162* a2 = reinterpret_cast<__nv_bfloat162*>(&ua);
    __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&ub);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 a = __bfloat1622float2(a2[q]), b = __bfloat1622float2(b2[q]);
      float oax, obx, oay, oby;
      hlm_fused::rope_rotate(a.x, b.x, c[2 * q], sv[2 * q], inverse != 0, oax, obx);
      hlm_fused::rope_rotate(a.y, b.y, c[2 * q + 1], sv[2 * q + 1], inverse != 0, oay, oby);
      a2[q] = __floats2bfloat162_rn(oax, oay);
      b2[q] = __floats2bfloat162_rn(obx, oby);
    }
    *reinterpret_cast<uint4*>(v) = ua;
    *reinterpret_cast<uint4*>(v + half) = ub;
  }
}

// ------------------------------------------------------------------ embedding
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                                 float* __restrict__ out, long long rows, int h, int vocab,
                                 int* __restrict__ err) {
  const long long n = rows * h;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long r = i / h;
    const int j = (int)(i - r * h);
    const int id = tok[r];
    if (id < 0 || id >= vocab) {
      if (j == 0) atomicOr(err, 1);
      out[i] = 0.f;
      continue;
    }
    out[i] = bf(table[(long long)id * h + j]);
  }
}

// h % 8 == 0: 16-byte reads of the table (a zero-copy table in pinned host memory is
// read over PCIe in full 16-byte pieces), two float4 writes.
__global__ void embed_fwd_vec8_kernel(const int32_t* __restrict__ tok, const uint4* __restrict__ table,
                                      float4* __restrict__ out, long long rows, int h8, int vocab,
                                      int* __restrict__ err) {
  const long long n = rows * h8;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long r = i / h8;
    const int j = (int)(i - r * h8);
    const int id = tok[r];
    if (id < 0 || id >= vocab) {
      if (j == 0) atomicOr(err, 1);
      out[2 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
      out[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const uint4 v = table[(long long)id * h8 + j];
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
    const float2 a = __bfloat1622float2(p[0]), b = __bfloat1622float2(p[1]), c = __bfloat1622float2(p[2]),
                 d = __bfloat1622float2(p[3]);
    out[2 * i] = make_float4(a.x, a.y, b.x, b.y);
    out[2 * i + 1] = make_float4(c.x, c.y, d.x, d.y);
  }
}

// d_table[v][j] = sum over positions p of token v (ascending) of g[p][j]:
// the reference's in-order scatter-add (kernels.hpp:396-408) without atomics,
// driven by a host-built CSR (row_ptr[V+1], pos[]) of the batch tokens.
__global__ void embed_bwd_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ pos,
                                 const float* __restrict__ g, float* __restrict__ d_table, int vocab, int h,
                                 int accumulate) {
  const long long n = (long long)vocab * h;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = (int)(i / h);
    const int j = (int)(i - (long long)v * h);
    float acc = accumulate ? d_table[i] : 0.f;
    for (int k = row_ptr[v]; k < row_ptr[v + 1]; ++k) acc += g[(long long)pos[k] * h + j];
    d_table[i] = acc;
  }
}

// Row-compact embedding gradient: out[c][j] = sum over the positions of token
// rows[c] (ascending, the CSR order of embed_bwd_kernel, so each touched row equals
// embed_bwd_kernel's bit for bit) of g[p][j]. Untouched rows are not materialised.
__global__ void embed_bwd_compact_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ pos,
                                         const int32_t* __restrict__ rows, int n_rows, const float* __restrict__ g,
                                         float* __restrict__ out, int h) {
  const long long n = (long long)n_rows * h;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int c = (int)(i / h);
    const int j = (int)(i - (long long)c * h);
    const int v = rows[c];
    float acc = 0.f;
    for (int k = row_ptr[v]; k < row_ptr[v + 1]; ++k) acc += g[(long long)pos[k] * h + j];
    out[i] = acc;
  }
}

// ------------------------------------------------------------------ cross entropy
// One CTA per row. loss_row[r] = (logz - l[tgt]) * inv_rows ;
// d_logits = (softmax - onehot) * inv_rows (bf16, row stride ld).
template <int THREADS>
__global__ void __launch_bounds__(THREADS) ce_kernel(const float* __restrict__ logits, long long ld_in,
                                                     const int32_t* __restrict__ tgt,
                                                     __nv_bfloat16* __restrict__ dl, long long ld_out,
                                                     float* __restrict__ loss_row, int vocab, float inv_rows,
                                                     int* __restrict__ err) {
  __shared__ float red[THREADS / 32];
  __shared__ float bcast;
  const long long r = blockIdx.x;
  const float* l = logits + r * ld_in;
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  float mx = -INFINITY;
  for (int v = threadIdx.x; v < vocab; v += THREADS) mx = fmaxf(mx, l[v]);
  mx = warp_max(mx);
  if (lane == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int i = 1; i < THREADS / 32; ++i) m = fmaxf(m, red[i]);
    bcast = m;
  }
  __syncthreads();
  mx = bcast;
  float z = 0.f;
  for (int v = threadIdx.x; v < vocab; v += THREADS) z += __expf(l[v] - mx);
  z = warp_sum(z);
  __syncthreads();
  if (lane == 0) red[w] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < THREADS / 32; ++i) s += red[i];
    bcast = s;
  }
  __syncthreads();
  z = bcast;
  const int t = tgt[r];
  const bool ok = t >= 0 && t < vocab;
  const float invz = 1.0f / z;
  __nv_bfloat16* d = dl + r * ld_out;
  for (int v = threadIdx.x; v < vocab; v += THREADS) {
    float p = __expf(l[v] - mx) * invz * inv_rows;
    if (v == t) p -= inv_rows;
    d[v] = __float2bfloat16_rn(p);
  }
  for (int v = vocab + threadIdx.x; v < ld_out; v += THREADS) d[v] = __float2bfloat16_rn(0.f);
  if (threadIdx.x == 0) {
    if (!ok) {
      atomicOr(err, 2);
      loss_row[r] = 0.f;
    } else {
      loss_row[r] = (logf(z) + mx - l[t]) * inv_rows;
    }
  }
}

// Vocab-chunked head, pass 1: the row statistics of ce_kernel (same max / sum
// order, so d_logits below equal ce_kernel's bit for bit) -> stats[r] = (max,
// 1/z), loss_row[r]; the d_logits are produced later per vocab chunk.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) ce_stats_kernel(const float* __restrict__ logits, long long ld_in,
                                                           const int32_t* __restrict__ tgt,
                                                           float2* __restrict__ stats, float* __restrict__ loss_row,
                                                           int vocab, float inv_rows, int* __restrict__ err) {
  __shared__ float red[THREADS / 32];
  __shared__ float bcast;
  const long long r = blockIdx.x;
  const float* l = logits + r * ld_in;
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  float mx = -INFINITY;
  for (int v = threadIdx.x; v < vocab; v += THREADS) mx = fmaxf(mx, l[v]);
  mx = warp_max(mx);
  if (lane == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int i = 1; i < THREADS / 32; ++i) m = fmaxf(m, red[i]);
    bcast = m;
  }
  __syncthreads();
  mx = bcast;
  float z = 0.f;
  for (int v = threadIdx.x; v < vocab; v += THREADS) z += __expf(l[v] - mx);
  z = warp_sum(z);
  __syncthreads();
  if (lane == 0) red[w] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sz = 0.f;
    for (int i = 0; i < THREADS / 32; ++i) sz += red[i];
    const int t = tgt[r];
    stats[r] = make_float2(mx, 1.0f / sz);
    if (t < 0 || t >= vocab) {
      atomicOr(err, 2);
      loss_row[r] = 0.f;
    } else {
      loss_row[r] = (logf(sz) + mx - l[t]) * inv_rows;
    }
  }
}

// Pass 2 for vocab columns [v0, v0 + vc): d_logits (bf16, row stride ld_out,
// zero in the padding columns vc..ld_out) from the chunk's logits (stride
// ld_in) and the pass-1 statistics: the formula of ce_kernel.
__global__ void ce_grad_chunk_kernel(const float* __restrict__ logits, long long ld_in,
                                     const int32_t* __restrict__ tgt, const float2* __restrict__ stats,
                                     __nv_bfloat16* __restrict__ dl, long long ld_out, long long rows, int v0,
                                     int vc, float inv_rows) {
  const long long per_row = ld_out / 2;   // bf16 pairs
  const long long n = rows * per_row;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long r = i / per_row;
    const int c = (int)(i - r * per_row) * 2;
    const float2 st = stats[r];
    const int t = tgt[r] - v0;
    float p0 = 0.f, p1 = 0.f;
    if (c < vc) {
      p0 = __expf(logits[r * ld_in + c] - st.x) * st.y * inv_rows;
      if (c == t) p0 -= inv_rows;
    }
    if (c + 1 < vc) {
      p1 = __expf(logits[r * ld_in + c + 1] - st.x) * st.y * inv_rows;
      if (c + 1 == t) p1 -= inv_rows;
    }
    reinterpret_cast<__nv_bfloat162*>(dl + r * ld_out)[c / 2] = __floats2bfloat162_rn(p0, p1);
  }
}

// Finiteness certificate of the head weight gradient, issued before any of it
// exists: with every d_logits element in [-inv_rows, inv_rows] (up to bf16
// rounding; finite when every row's statistics are), |d_head[v][j]| =
// |sum_t d_logits[t][v] x[t][j]| <= rows * inv_rows * 1.01 * max|x|. So when the
// row statistics are finite and rows * inv_rows * max|x| stays far below FLT_MAX,
// no element of d_head can be non-finite and *word keeps ~0 ("none"); otherwise
// it becomes HLM_HEAD_UNCERTIFIED and the caller falls back to scanning d_head.
__global__ void head_certify_kernel(const __nv_bfloat16* __restrict__ x, long long n,
                                    const float2* __restrict__ stats, long long rows, float limit,
                                    unsigned long long* word) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += stride) {
    const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(x)[i];
    const float a = __low2float(v), b = __high2float(v);
    bad |= !(fabsf(a) <= limit) || !(fabsf(b) <= limit);   // NaN and Inf fail the comparison
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) bad |= !(fabsf(__bfloat162float(x[n - 1])) <= limit);
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const float2 st = stats[r];
    bad |= !isfinite(st.x) || !isfinite(st.y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(word, HLM_HEAD_UNCERTIFIED);
}

// ------------------------------------------------------------------ finiteness
// first[0] = min index of a non-finite element (INT64 max when none): the
// reference's "validate before any mutation" check (host_store.cpp:340-345),
// run at HBM speed before the gradient leaves the GPU.
// Any alignment of g (a data-parallel shard starts at rank * n / world elements): the
// first `head` elements up to the next 16-byte boundary are scanned scalar, the rest
// as float4.
// `only_if` (may be null): scan only when *only_if == HLM_HEAD_UNCERTIFIED (the vocab-chunked
// head's fallback; a certified head gradient costs one read per CTA).
__global__ void nonfinite_kernel(const float* __restrict__ g, long long n, unsigned long long* first,
                                 const unsigned long long* __restrict__ only_if) {
  if (only_if != nullptr && *only_if != HLM_HEAD_UNCERTIFIED) return;
  const long long head = min(n, (long long)(((16u - ((uintptr_t)g & 15u)) & 15u) / 4u));
  if (blockIdx.x == 0 && threadIdx.x < head)
    if (!isfinite(g[threadIdx.x])) atomicMin(first, (unsigned long long)threadIdx.x);
  const float* body = g + head;
  const long long nb = n - head;
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < nb; i += stride) {
    if (i + 4 <= nb) {
      const float4 v = *reinterpret_cast<const float4*>(body + i);
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (!isfinite(e[k])) atomicMin(first, (unsigned long long)(head + i + k));
    } else {
      for (long long k = i; k < nb; ++k)
        if (!isfinite(body[k])) atomicMin(first, (unsigned long long)(head + k));
    }
  }
}

// ------------------------------------------------------------------ device Adam
// Reference adam_update_tile (host_store.cpp:334-362) for HBM-resident optimizer
// tiles: every operation an IEEE-rounded intrinsic in the host kernel's order (no
// FMA contraction), so results equal the host Adam bit for bit. Skipped entirely
// when the gradient scan flagged a non-finite element (no mutation, as the host).
__global__ void adam_device_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                                   __nv_bfloat16* __restrict__ w16, const float* __restrict__ g, long long n,
                                   const unsigned long long* __restrict__ bad, float lr, float b1, float b2,
                                   float omb1, float omb2, float eps, float wd, float bc1, float bc2) {
  if (*bad != ~0ull) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float gv = g[i];
    const float mm = __fadd_rn(__fmul_rn(b1, m[i]), __fmul_rn(omb1, gv));
    const float vv = __fadd_rn(__fmul_rn(b2, v[i]), __fmul_rn(__fmul_rn(omb2, gv), gv));
    const float mhat = __fdiv_rn(mm, bc1);
    const float vhat = __fdiv_rn(vv, bc2);
    float th = w[i];
    const float upd = __fadd_rn(__fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), eps)), __fmul_rn(wd, th));
    th = __fsub_rn(th, __fmul_rn(lr, upd));
    m[i] = mm;
    v[i] = vv;
    w[i] = th;
    w16[i] = __float2bfloat16_rn(th);
  }
}

// ------------------------------------------------------------------ generic attention
// Causal softmax attention for any head_dim <= 32*VPL: one warp per
// (batch, head, query row), online softmax over keys j <= i in fp32.
// Reference-semantics path (single head, head_dim = h) and small shapes;
// the tensor-core flash kernel (attention_sm100.cu) serves head_dim 64/128.
template <int VPL>
__global__ void attn_fwd_generic(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                                 const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ o,
                                 float* __restrict__ lse, int B, int S, int H, int hd, int ld, float scale) {
  const long long total = (long long)B * H * S;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= total) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(gw % S);
  const int hh = (int)((gw / S) % H);
  const int b = (int)(gw / ((long long)S * H));
  const long long base = (long long)b * S * ld + (long long)hh * hd;
  float qv[VPL], acc[VPL];
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    qv[e] = d < hd ? bf(q[base + (long long)i * ld + d]) : 0.f;
    acc[e] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j <= i; ++j) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      const int d = lane + 32 * e;
      if (d < hd) s += qv[e] * bf(k[base + (long long)j * ld + d]);
    }
    s = warp_sum(s) * scale;
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn);
    const float p = __expf(s - mn);
    l = l * corr + p;
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      const int d = lane + 32 * e;
      acc[e] = acc[e] * corr + (d < hd ? p * bf(v[base + (long long)j * ld + d]) : 0.f);
    }
    m = mn;
  }
  const float il = 1.0f / l;
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    if (d < hd) o[base + (long long)i * ld + d] = __float2bfloat16_rn(acc[e] * il);
  }
  if (lane == 0) lse[((long long)b * H + hh) * S + i] = m + logf(l);
}

// Dsum[b,h,i] = sum_d dO[i,d] * O[i,d]
__global__ void attn_bwd_dsum(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                              float* __restrict__ dsum, int B, int S, int H, int hd, int ld) {
  const long long total = (long long)B * H * S;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= total) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(gw % S);
  const int hh = (int)((gw / S) % H);
  const int b = (int)(gw / ((long long)S * H));
  const long long row = ((long long)b * S + i) * ld + (long long)hh * hd;
  float s = 0.f;
  for (int d = lane; d < hd; d += 32) s += bf(o[row + d]) * bf(dout[row + d]);
  s = warp_sum(s);
  if (lane == 0) dsum[((long long)b * H + hh) * S + i] = s;
}

// dQ_i = scale * sum_{j<=i} P_ij (dP_ij - D_i) K_j  (one warp per query row)
template <int VPL>
__global__ void attn_bwd_dq_generic(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                                    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
                                    const float* __restrict__ lse, const float* __restrict__ dsum,
                                    __nv_bfloat16* __restrict__ dq, int B, int S, int H, int hd, int ld,
                                    float scale) {
  const long long total = (long long)B * H * S;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= total) return;
  const int lane = threadIdx.x & 31;
  const int i = (int)(gw % S);
  const int hh = (int)((gw / S) % H);
  const int b = (int)(gw / ((long long)S * H));
  const long long base = (long long)b * S * ld + (long long)hh * hd;
  const long long st = ((long long)b * H + hh) * S;
  float qv[VPL], dov[VPL], acc[VPL];
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    qv[e] = d < hd ? bf(q[base + (long long)i * ld + d]) : 0.f;
    dov[e] = d < hd ? bf(dout[base + (long long)i * ld + d]) : 0.f;
    acc[e] = 0.f;
  }
  const float L = lse[st + i], D = dsum[st + i];
  for (int j = 0; j <= i; ++j) {
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      const int d = lane + 32 * e;
      if (d < hd) {
        s += qv[e] * bf(k[base + (long long)j * ld + d]);
        dp += dov[e] * bf(v[base + (long long)j * ld + d]);
      }
    }
    s = warp_sum(s) * scale;
    dp = warp_sum(dp);
    const float p = __expf(s - L);
    const float ds = p * (dp - D) * scale;
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      const int d = lane + 32 * e;
      if (d < hd) acc[e] += ds * bf(k[base + (long long)j * ld + d]);
    }
  }
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    if (d < hd) dq[base + (long long)i * ld + d] = __float2bfloat16_rn(acc[e]);
  }
}

// dV_j = sum_{i>=j} P_ij dO_i ; dK_j = scale * sum_{i>=j} P_ij (dP_ij - D_i) Q_i  (warp per key row)
template <int VPL>
__global__ void attn_bwd_dkv_generic(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                                     const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
                                     const float* __restrict__ lse, const float* __restrict__ dsum,
                                     __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, int B,
                                     int S, int H, int hd, int ld, float scale) {
  const long long total = (long long)B * H * S;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= total) return;
  const int lane = threadIdx.x & 31;
  const int j = (int)(gw % S);
  const int hh = (int)((gw / S) % H);
  const int b = (int)(gw / ((long long)S * H));
  const long long base = (long long)b * S * ld + (long long)hh * hd;
  const long long st = ((long long)b * H + hh) * S;
  float kv[VPL], vv[VPL], adk[VPL], adv[VPL];
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    kv[e] = d < hd ? bf(k[base + (long long)j * ld + d]) : 0.f;
    vv[e] = d < hd ? bf(v[base + (long long)j * ld + d]) : 0.f;
    adk[e] = 0.f;
    adv[e] = 0.f;
  }
  for (int i = j; i < S; ++i) {
    float s = 0.f, dp = 0.f;
    float qi[VPL], doi[VPL];
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      const int d = lane + 32 * e;
      qi[e] = d < hd ? bf(q[base + (long long)i * ld + d]) : 0.f;
      doi[e] = d < hd ? bf(dout[base + (long long)i * ld + d]) : 0.f;
      s += qi[e] * kv[e];
      dp += doi[e] * vv[e];
    }
    s = warp_sum(s) * scale;
    dp = warp_sum(dp);
    const float p = __expf(s - lse[st + i]);
    const float ds = p * (dp - dsum[st + i]) * scale;
#pragma unroll
    for (int e = 0; e < VPL; ++e) {
      adv[e] += p * doi[e];
      adk[e] += ds * qi[e];
    }
  }
#pragma unroll
  for (int e = 0; e < VPL; ++e) {
    const int d = lane + 32 * e;
    if (d < hd) {
      dk[base + (long long)j * ld + d] = __float2bfloat16_rn(adk[e]);
      dv[base + (long long)j * ld + d] = __float2bfloat16_rn(adv[e]);
    }
  }
}

__global__ void fill_random_bf16_kernel(__nv_bfloat16* p, long long n, unsigned seed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    p[i] = __float2bfloat16_rn(((float)(x >> 8) / 16777216.0f) * 2.0f - 1.0f);
  }
}

}  // namespace

// ====================================================================== launchers
#include <atomic>
static std::atomic<long long> g_launches{0};
void hlm_count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long hlm_launches_total() { return g_launches.load(std::memory_order_relaxed); }

#define HLM_CHECK_LAUNCH() return cudaGetLastError() == cudaSuccess ? 0 : 1

int hlm_ops_fill_random_bf16(void* p, long long n, unsigned seed, cudaStream_t s) {
  fill_random_bf16_kernel<<<grid_for(n, 256), 256, 0, s>>>((__nv_bfloat16*)p, n, seed);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_nonfinite(const float* g, long long n, unsigned long long* first, const unsigned long long* only_if,
                      cudaStream_t s) {
  cudaMemsetAsync(first, 0xFF, sizeof(unsigned long long), s);
  nonfinite_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, s>>>(g, n, first, only_if);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_adam_device(float* w, float* m, float* v, void* w16, const float* g, long long n,
                        const unsigned long long* bad, float lr, float b1, float b2, float eps, float wd, float bc1,
                        float bc2, cudaStream_t s) {
  adam_device_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, m, v, (__nv_bfloat16*)w16, g, n, bad, lr, b1, b2, 1.0f - b1,
                                                       1.0f - b2, eps, wd, bc1, bc2);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_rmsnorm_fwd(const float* x, const void* scale, void* out, long long rows, int h, cudaStream_t s) {
  constexpr int rpb = 8;
  const unsigned blocks = (unsigned)((rows + rpb - 1) / rpb);
  if (h % 4 == 0 && h <= 4 * 256 * 4)
    rmsnorm_fwd_reg_kernel<256, 4><<<blocks, 256, 0, s>>>(x, (const __nv_bfloat16*)scale, (__nv_bfloat16*)out, rows,
                                                          h, rpb);
  else if (h % 4 == 0 && h <= 4 * 512 * 6)
    rmsnorm_fwd_reg_kernel<512, 6><<<blocks, 512, 0, s>>>(x, (const __nv_bfloat16*)scale, (__nv_bfloat16*)out, rows,
                                                          h, rpb);
  else
    rmsnorm_fwd_kernel<<<grid_for(rows, 8), 256, 0, s>>>(x, (const __nv_bfloat16*)scale, (__nv_bfloat16*)out, rows,
                                                         h);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_rmsnorm_bwd(const float* x, const void* scale, const float* g, const float* resid, float* out,
                        void* out_bf, float* inv_buf, float* partial, float* dscale, long long rows, int h,
                        cudaStream_t s) {
  const int rpc = HLM_NORM_ROWS_PER_CHUNK;
  const int chunks = (int)((rows + rpc - 1) / rpc);
  // Default: scale / partial in shared memory, 3 CTAs / SM (78 registers): 230 us at C2 vs
  // 267 (registers, 2 CTAs / SM, 117 registers) and 287 (registers, 3 CTAs / SM, 16 B spilled),
  // alternating on one box; bit-identical (tested). HLM_RMSNORM_BWD_MINB=2 / 3 selects the
  // register variants. (A next-row x / g prefetch at 2 CTAs / SM measured 317 us.)
  static int minb = -1;
  if (minb < 0) {
    const char* e = std::getenv("HLM_RMSNORM_BWD_MINB");
    minb = (e && *e == '3') ? 3 : (e && *e == '2') ? 2 : 5;
  }
  if (h % 4 == 0 && h <= 4 * 256 * 4 && minb == 5) {   // scale / partial in shared memory, 3 CTAs / SM
    rmsnorm_bwd_smem_kernel<256, 4, 3><<<chunks, 256, 2 * h * sizeof(float), s>>>(
        x, (const __nv_bfloat16*)scale, g, resid, out, (__nv_bfloat16*)out_bf, inv_buf, partial, rows, h, rpc);
  } else if (h % 4 == 0 && h <= 4 * 256 * 4 && minb == 2) {
    rmsnorm_bwd_reg_kernel<256, 4, 2><<<chunks, 256, 0, s>>>(x, (const __nv_bfloat16*)scale, g, resid, out,
                                                             (__nv_bfloat16*)out_bf, inv_buf, partial, rows, h, rpc);
  } else if (h % 4 == 0 && h <= 4 * 256 * 4) {
    rmsnorm_bwd_reg_kernel<256, 4, 3><<<chunks, 256, 0, s>>>(x, (const __nv_bfloat16*)scale, g, resid, out,
                                                             (__nv_bfloat16*)out_bf, inv_buf, partial, rows, h, rpc);
  } else if (h % 4 == 0 && h <= 4 * 512 * 6) {
    rmsnorm_bwd_reg_kernel<512, 6, 1><<<chunks, 512, 0, s>>>(x, (const __nv_bfloat16*)scale, g, resid, out,
                                                             (__nv_bfloat16*)out_bf, inv_buf, partial, rows, h, rpc);
  } else {
    rmsnorm_bwd_kernel<<<grid_for(rows, 8), 256, 0, s>>>(x, (const __nv_bfloat16*)scale, g, resid, out,
                                                         (__nv_bfloat16*)out_bf, inv_buf, rows, h);
    dim3 grid((h + 255) / 256, chunks);
    norm_scale_partial_kernel<<<grid, 256, 0, s>>>(x, g, inv_buf, partial, rows, h, rpc);
    hlm_count_launches(1);
  }
  norm_scale_reduce_kernel<<<(h + 31) / 32, 256, 0, s>>>(partial, dscale, chunks, h);
  hlm_count_launches(2);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_cast_bf16(const float* in, void* out, long long n, cudaStream_t s) {
  cast_f32_bf16_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, s>>>(in, (__nv_bfloat16*)out, n);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_swiglu_fwd(const void* ug, void* act, long long n, cudaStream_t s) {
  swiglu_fwd_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)ug, (__nv_bfloat16*)act, n);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_swiglu_bwd(const void* dact, const void* ug, void* dug, long long n, cudaStream_t s) {
  swiglu_bwd_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)dact, (const __nv_bfloat16*)ug,
                                                    (__nv_bfloat16*)dug, n);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_rope(void* x, const float* cs, const float* sn, long long rows, int h, int hd, int S, int inverse,
                 int nmats, long long mat_stride, cudaStream_t s) {
  if (hd % 16 == 0 && h % 8 == 0 && rows < (1LL << 31))
    rope8_kernel<<<grid_for(rows * (h / 16) * nmats, 256), 256, 0, s>>>((__nv_bfloat16*)x, cs, sn, (int)rows, h, hd,
                                                                         S, inverse, nmats, mat_stride);
  else
    rope_kernel<<<grid_for(rows * (h / 2) * nmats, 256), 256, 0, s>>>((__nv_bfloat16*)x, cs, sn, rows, h, hd, S,
                                                                       inverse, nmats, mat_stride);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_embed_fwd(const int32_t* tok, const void* table, float* out, long long rows, int h, int vocab,
                      int* err, cudaStream_t s) {
  if (h % 8 == 0 && (reinterpret_cast<uintptr_t>(table) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0)
    embed_fwd_vec8_kernel<<<grid_for(rows * (h / 8), 256), 256, 0, s>>>(tok, (const uint4*)table, (float4*)out, rows,
                                                                        h / 8, vocab, err);
  else
    embed_fwd_kernel<<<grid_for(rows * h, 256), 256, 0, s>>>(tok, (const __nv_bfloat16*)table, out, rows, h, vocab,
                                                             err);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_embed_bwd_compact(const int32_t* row_ptr, const int32_t* pos, const int32_t* rows, int n_rows,
                              const float* g, float* out, int h, cudaStream_t s) {
  if (n_rows <= 0) return 0;
  embed_bwd_compact_kernel<<<grid_for((long long)n_rows * h, 256), 256, 0, s>>>(row_ptr, pos, rows, n_rows, g, out,
                                                                                 h);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_embed_bwd(const int32_t* row_ptr, const int32_t* pos, const float* g, float* d_table, int vocab,
                      int h, int accumulate, cudaStream_t s) {
  embed_bwd_kernel<<<grid_for((long long)vocab * h, 256), 256, 0, s>>>(row_ptr, pos, g, d_table, vocab, h, accumulate);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_ce(const float* logits, long long ld_in, const int32_t* tgt, void* dl, long long ld_out,
               float* loss_row, long long rows, int vocab, float inv_rows, int* err, cudaStream_t s) {
  ce_kernel<512><<<(unsigned)rows, 512, 0, s>>>(logits, ld_in, tgt, (__nv_bfloat16*)dl, ld_out, loss_row, vocab,
                                                inv_rows, err);
  hlm_count_launches(5);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_ce_stats(const float* logits, long long ld_in, const int32_t* tgt, void* stats, float* loss_row,
                     long long rows, int vocab, float inv_rows, int* err, cudaStream_t s) {
  ce_stats_kernel<512><<<(unsigned)rows, 512, 0, s>>>(logits, ld_in, tgt, (float2*)stats, loss_row, vocab,
                                                      inv_rows, err);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_ce_grad_chunk(const float* logits, long long ld_in, const int32_t* tgt, const void* stats, void* dl,
                          long long ld_out, long long rows, int v0, int vc, float inv_rows, cudaStream_t s) {
  if (ld_out % 2) return 2;
  ce_grad_chunk_kernel<<<grid_for(rows * (ld_out / 2), 256), 256, 0, s>>>(
      logits, ld_in, tgt, (const float2*)stats, (__nv_bfloat16*)dl, ld_out, rows, v0, vc, inv_rows);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

int hlm_ops_head_certify(const void* x_bf, long long n, const void* stats, long long rows, float limit,
                         unsigned long long* word, cudaStream_t s) {
  if (cudaMemsetAsync(word, 0xFF, 8, s) != cudaSuccess) return 1;
  head_certify_kernel<<<grid_for(n / 2 + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)x_bf, n,
                                                               (const float2*)stats, rows, limit, word);
  hlm_count_launches(1);
  HLM_CHECK_LAUNCH();
}

namespace {
template <int VPL>
int attn_generic(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int hd,
                 int ld, cudaStream_t s) {
  const long long warps = (long long)B * H * S;
  hlm_count_launches(1);
  attn_fwd_generic<VPL><<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(
      (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, (__nv_bfloat16*)o, lse, B, S, H,
      hd, ld, 1.0f / sqrtf((float)hd));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
template <int VPL>
int attn_bwd_generic(const void* q, const void* k, const void* v, const void* o, const void* dout,
                     const float* lse, float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int hd,
                     int ld, cudaStream_t s) {
  const long long warps = (long long)B * H * S;
  const unsigned grid = (unsigned)((warps + 7) / 8);
  const float scale = 1.0f / sqrtf((float)hd);
  hlm_count_launches(3);
  attn_bwd_dsum<<<grid, 256, 0, s>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dsum, B, S, H, hd, ld);
  attn_bwd_dq_generic<VPL><<<grid, 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                (const __nv_bfloat16*)v, (const __nv_bfloat16*)dout, lse, dsum,
                                                (__nv_bfloat16*)dq, B, S, H, hd, ld, scale);
  attn_bwd_dkv_generic<VPL><<<grid, 256, 0, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                 (const __nv_bfloat16*)v, (const __nv_bfloat16*)dout, lse, dsum,
                                                 (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, B, S, H, hd, ld, scale);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
}  // namespace

int hlm_ops_attention_fwd_generic(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S,
                                  int H, int hd, int ld, cudaStream_t s) {
  if (hd <= 32) return attn_generic<1>(q, k, v, o, lse, B, S, H, hd, ld, s);
  if (hd <= 64) return attn_generic<2>(q, k, v, o, lse, B, S, H, hd, ld, s);
  if (hd <= 128) return attn_generic<4>(q, k, v, o, lse, B, S, H, hd, ld, s);
  if (hd <= 256) return attn_generic<8>(q, k, v, o, lse, B, S, H, hd, ld, s);
  if (hd <= 512) return attn_generic<16>(q, k, v, o, lse, B, S, H, hd, ld, s);
  if (hd <= 1024) return attn_generic<32>(q, k, v, o, lse, B, S, H, hd, ld, s);
  return 2;
}

int hlm_ops_attention_bwd_generic(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                  const float* lse, float* dsum, void* dq, void* dk, void* dv, int B, int S, int H,
                                  int hd, int ld, cudaStream_t s) {
  if (hd <= 32) return attn_bwd_generic<1>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  if (hd <= 64) return attn_bwd_generic<2>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  if (hd <= 128) return attn_bwd_generic<4>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  if (hd <= 256) return attn_bwd_generic<8>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  if (hd <= 512) return attn_bwd_generic<16>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  if (hd <= 1024) return attn_bwd_generic<32>(q, k, v, o, dout, lse, dsum, dq, dk, dv, B, S, H, hd, ld, s);
  return 2;
}
