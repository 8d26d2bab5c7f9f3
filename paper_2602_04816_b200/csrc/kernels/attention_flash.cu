// Causal flash attention on tensor cores (bf16 mma.sync m16n8k16, fp32
// accumulation), head_dim 64 / 128, seq a multiple of 64.
//
// Replaces reference attention_fwd / attention_bwd (proj/include/hlm/
// kernels.hpp:207-299), which materialise P (B,S,S): here only O and the row
// log-sum-exp are kept, P is recomputed in backward. Multi-head layout: q, k,
// v, o are (B*S, ld) bf16 rows with head hh at columns [hh*hd, (hh+1)*hd).
//
// Kernels
//   flash_fwd   : grid (S/64, B*H), 4 warps x 16 query rows, K/V tiles of 64
//                 keys double-buffered through cp.async, online softmax (exp2).
//   flash_bwd_dq: grid (S/64, B*H), per query tile: recompute S, dP over the
//                 key tiles j <= i, dQ = scale * sum dS K.
//   flash_bwd_dkv: grid (S/64, B*H), per key tile: loop over query tiles
//                 i >= j, dV = sum P^T dO, dK = scale * sum dS^T Q.
// dQ and dK/dV are produced by separate kernels so every output element is
// written by exactly one thread in a fixed order: deterministic, no atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "attention.h"
#include "block_ops.h"

namespace {

constexpr int BR = 64;   // query rows per CTA
constexpr int BC = 64;   // keys per tile
constexpr int NW = 4;    // warps per CTA
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled [rows][HD] bf16 tile: 16-byte chunk c of row r lives at chunk c ^ (r & 7).
template <int HD>
struct Tile {
  static constexpr int CHUNKS = HD / 8;
  __device__ static __forceinline__ int off(int r, int c) { return r * HD + ((c ^ (r & 7)) << 3); }
};

// Async copy of a 64 x HD tile (rows row0.. of a (rows, ld) bf16 matrix, column col0).
template <int HD>
__device__ __forceinline__ void load_tile(__nv_bfloat16* s, const __nv_bfloat16* g, long long row0, int ld,
                                          int col0) {
  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < 64 * CH; i += NW * 32) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + Tile<HD>::off(r, c), g + (row0 + r) * (long long)ld + col0 + c * 8);
  }
}

// A fragment (16x16) at (r0, k0) of a swizzled tile.
template <int HD>
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const __nv_bfloat16* s, int r0, int k0) {
  const int lane = threadIdx.x & 31;
  const int r = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = (k0 >> 3) + (lane >> 4);
  ldsm_x4(a, smem_addr(s + Tile<HD>::off(r, c)));
}
// B fragments for two n-blocks (n0..n0+15) x k16 (k0) from a tile stored [n][k] (k contiguous).
template <int HD>
__device__ __forceinline__ void frag_b_nk(uint32_t (&b)[4], const __nv_bfloat16* s, int n0, int k0) {
  const int lane = threadIdx.x & 31;
  const int r = n0 + (lane & 7) + (lane >> 4) * 8;
  const int c = (k0 >> 3) + ((lane >> 3) & 1);
  ldsm_x4(b, smem_addr(s + Tile<HD>::off(r, c)));
}
// B fragments for two n-blocks (n0..n0+15) x k16 (k0) from a tile stored [k][n] (n contiguous), via .trans.
template <int HD>
__device__ __forceinline__ void frag_b_kn(uint32_t (&b)[4], const __nv_bfloat16* s, int k0, int n0) {
  const int lane = threadIdx.x & 31;
  const int r = k0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = (n0 >> 3) + (lane >> 4);
  ldsm_x4_t(b, smem_addr(s + Tile<HD>::off(r, c)));
}

// ------------------------------------------------------------------ forward
template <int HD>
__global__ void __launch_bounds__(NW * 32) flash_fwd(const __nv_bfloat16* __restrict__ q,
                                                     const __nv_bfloat16* __restrict__ k,
                                                     const __nv_bfloat16* __restrict__ v,
                                                     __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                                                     int S, int H, int ld, float scale_log2) {
  extern __shared__ __align__(128) __nv_bfloat16 smem[];
  __nv_bfloat16* sQ = smem;
  __nv_bfloat16* sK = sQ + BR * HD;   // [2][BC][HD]
  __nv_bfloat16* sV = sK + 2 * BC * HD;
  const int qt = (int)(gridDim.x - 1 - blockIdx.x);   // heavy (long) tiles first
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const long long row_base = (long long)b * S;
  const int col0 = hh * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  load_tile<HD>(sQ, q, row_base + qt * BR, ld, col0);
  load_tile<HD>(sK, k, row_base, ld, col0);
  load_tile<HD>(sV, v, row_base, ld, col0);
  cp_commit();

  float oacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[HD / 16][4];
  const int n_tiles = qt + 1;
  const int qrow0 = qt * BR + warp * 16 + g;   // query positions of this thread's two rows
  const int qrow1 = qrow0 + 8;

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      load_tile<HD>(sK + (buf ^ 1) * BC * HD, k, row_base + (j + 1) * BC, ld, col0);
      load_tile<HD>(sV + (buf ^ 1) * BC * HD, v, row_base + (j + 1) * BC, ld, col0);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) frag_a<HD>(qf[kk], sQ, warp * 16, kk * 16);
    }
    const __nv_bfloat16* cK = sK + buf * BC * HD;
    const __nv_bfloat16* cV = sV + buf * BC * HD;
    float s[BC / 8][4];
#pragma unroll
    for (int i = 0; i < BC / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < BC / 16; ++np) {
        uint32_t bb[4];
        frag_b_nk<HD>(bb, cK, np * 16, kk * 16);
        mma16816(s[2 * np], qf[kk], bb[0], bb[1]);
        mma16816(s[2 * np + 1], qf[kk], bb[2], bb[3]);
      }
    }
    // scale (log2 domain), causal mask on the diagonal tile, online softmax
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nb = 0; nb < BC / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float val = s[nb][e] * scale_log2;
        if (j == qt) {
          const int key = j * BC + nb * 8 + 2 * t + (e & 1);
          const int qr = (e < 2) ? qrow0 : qrow1;
          if (key > qr) val = -INFINITY;
        }
        s[nb][e] = val;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nb][0], s[nb][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nb][2], s[nb][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float a0 = exp2f(m0 - mx0), a1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    l0 *= a0;
    l1 *= a1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      oacc[i][0] *= a0;
      oacc[i][1] *= a0;
      oacc[i][2] *= a1;
      oacc[i][3] *= a1;
    }
#pragma unroll
    for (int nb = 0; nb < BC / 8; ++nb) {
      s[nb][0] = exp2f(s[nb][0] - m0);
      s[nb][1] = exp2f(s[nb][1] - m0);
      s[nb][2] = exp2f(s[nb][2] - m1);
      s[nb][3] = exp2f(s[nb][3] - m1);
      l0 += s[nb][0] + s[nb][1];
      l1 += s[nb][2] + s[nb][3];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BC / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t bb[4];
        frag_b_kn<HD>(bb, cV, kk * 16, np * 16);
        mma16816(oacc[2 * np], pa, bb[0], bb[1]);
        mma16816(oacc[2 * np + 1], pa, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float il0 = 1.f / l0, il1 = 1.f / l1;
  __nv_bfloat16* o0 = o + (row_base + qrow0) * (long long)ld + col0;
  __nv_bfloat16* o1 = o + (row_base + qrow1) * (long long)ld + col0;
#pragma unroll
  for (int nb = 0; nb < HD / 8; ++nb) {
    const int c = nb * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(o0 + c) = pack2(oacc[nb][0] * il0, oacc[nb][1] * il0);
    *reinterpret_cast<uint32_t*>(o1 + c) = pack2(oacc[nb][2] * il1, oacc[nb][3] * il1);
  }
  if (t == 0) {
    float* L = lse + (long long)bh * S;
    L[qrow0] = (m0 + log2f(l0)) / kLog2e;
    L[qrow1] = (m1 + log2f(l1)) / kLog2e;
  }
}

// ------------------------------------------------------------------ backward: dQ
template <int HD>
__global__ void __launch_bounds__(NW * 32) flash_bwd_dq(const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k,
                                                        const __nv_bfloat16* __restrict__ v,
                                                        const __nv_bfloat16* __restrict__ dout,
                                                        const float* __restrict__ lse,
                                                        const float* __restrict__ dsum,
                                                        __nv_bfloat16* __restrict__ dq, int S, int H, int ld,
                                                        float scale, float scale_log2) {
  extern __shared__ __align__(128) __nv_bfloat16 smem[];
  __nv_bfloat16* sQ = smem;
  __nv_bfloat16* sdO = sQ + BR * HD;
  __nv_bfloat16* sK = sdO + BR * HD;   // [2][BC][HD]
  __nv_bfloat16* sV = sK + 2 * BC * HD;
  const int qt = (int)(gridDim.x - 1 - blockIdx.x);
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const long long row_base = (long long)b * S;
  const int col0 = hh * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  load_tile<HD>(sQ, q, row_base + qt * BR, ld, col0);
  load_tile<HD>(sdO, dout, row_base + qt * BR, ld, col0);
  load_tile<HD>(sK, k, row_base, ld, col0);
  load_tile<HD>(sV, v, row_base, ld, col0);
  cp_commit();

  const int qrow0 = qt * BR + warp * 16 + g, qrow1 = qrow0 + 8;
  const float* Lr = lse + (long long)bh * S;
  const float* Dr = dsum + (long long)bh * S;
  const float lse0 = Lr[qrow0] * kLog2e, lse1 = Lr[qrow1] * kLog2e;
  const float D0 = Dr[qrow0], D1 = Dr[qrow1];
  float acc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const int n_tiles = qt + 1;
  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      load_tile<HD>(sK + (buf ^ 1) * BC * HD, k, row_base + (j + 1) * BC, ld, col0);
      load_tile<HD>(sV + (buf ^ 1) * BC * HD, v, row_base + (j + 1) * BC, ld, col0);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* cK = sK + buf * BC * HD;
    const __nv_bfloat16* cV = sV + buf * BC * HD;
    float s[BC / 8][4], dp[BC / 8][4];
#pragma unroll
    for (int i = 0; i < BC / 8; ++i) {
      s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
    }
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t qa[4], da[4];
      frag_a<HD>(qa, sQ, warp * 16, kk * 16);
      frag_a<HD>(da, sdO, warp * 16, kk * 16);
#pragma unroll
      for (int np = 0; np < BC / 16; ++np) {
        uint32_t bk[4], bv[4];
        frag_b_nk<HD>(bk, cK, np * 16, kk * 16);
        frag_b_nk<HD>(bv, cV, np * 16, kk * 16);
        mma16816(s[2 * np], qa, bk[0], bk[1]);
        mma16816(s[2 * np + 1], qa, bk[2], bk[3]);
        mma16816(dp[2 * np], da, bv[0], bv[1]);
        mma16816(dp[2 * np + 1], da, bv[2], bv[3]);
      }
    }
#pragma unroll
    for (int nb = 0; nb < BC / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool hi = e >= 2;
        float p = exp2f(s[nb][e] * scale_log2 - (hi ? lse1 : lse0));
        if (j == qt) {
          const int key = j * BC + nb * 8 + 2 * t + (e & 1);
          if (key > (hi ? qrow1 : qrow0)) p = 0.f;
        }
        s[nb][e] = p * (dp[nb][e] - (hi ? D1 : D0));   // dS
      }
    }
#pragma unroll
    for (int kk = 0; kk < BC / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t bb[4];
        frag_b_kn<HD>(bb, cK, kk * 16, np * 16);
        mma16816(acc[2 * np], pa, bb[0], bb[1]);
        mma16816(acc[2 * np + 1], pa, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
  __nv_bfloat16* o0 = dq + (row_base + qrow0) * (long long)ld + col0;
  __nv_bfloat16* o1 = dq + (row_base + qrow1) * (long long)ld + col0;
#pragma unroll
  for (int nb = 0; nb < HD / 8; ++nb) {
    const int c = nb * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(o0 + c) = pack2(acc[nb][0] * scale, acc[nb][1] * scale);
    *reinterpret_cast<uint32_t*>(o1 + c) = pack2(acc[nb][2] * scale, acc[nb][3] * scale);
  }
}

// ------------------------------------------------------------------ backward: dK, dV
template <int HD>
__global__ void __launch_bounds__(NW * 32) flash_bwd_dkv(const __nv_bfloat16* __restrict__ q,
                                                         const __nv_bfloat16* __restrict__ k,
                                                         const __nv_bfloat16* __restrict__ v,
                                                         const __nv_bfloat16* __restrict__ dout,
                                                         const float* __restrict__ lse,
                                                         const float* __restrict__ dsum,
                                                         __nv_bfloat16* __restrict__ dk,
                                                         __nv_bfloat16* __restrict__ dv, int S, int H, int ld,
                                                         float scale, float scale_log2) {
  extern __shared__ __align__(128) __nv_bfloat16 smem[];
  __nv_bfloat16* sK = smem;
  __nv_bfloat16* sV = sK + BC * HD;
  __nv_bfloat16* sQ = sV + BC * HD;    // [2][BR][HD]
  __nv_bfloat16* sdO = sQ + 2 * BR * HD;
  float* sL = reinterpret_cast<float*>(sdO + 2 * BR * HD);   // [2][BR]
  float* sD = sL + 2 * BR;
  const int nq = (int)gridDim.x;
  const int kt = (int)blockIdx.x;   // key tile; short loops for late tiles
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const long long row_base = (long long)b * S;
  const int col0 = hh * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float* Lr = lse + (long long)bh * S;
  const float* Dr = dsum + (long long)bh * S;

  load_tile<HD>(sK, k, row_base + kt * BC, ld, col0);
  load_tile<HD>(sV, v, row_base + kt * BC, ld, col0);
  load_tile<HD>(sQ, q, row_base + kt * BR, ld, col0);
  load_tile<HD>(sdO, dout, row_base + kt * BR, ld, col0);
  if (threadIdx.x < BR) {
    sL[threadIdx.x] = Lr[kt * BR + threadIdx.x] * kLog2e;
    sD[threadIdx.x] = Dr[kt * BR + threadIdx.x];
  }
  cp_commit();

  float dka[HD / 8][4], dva[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    dka[i][0] = dka[i][1] = dka[i][2] = dka[i][3] = 0.f;
    dva[i][0] = dva[i][1] = dva[i][2] = dva[i][3] = 0.f;
  }
  const int key0 = kt * BC + warp * 16 + g, key1 = key0 + 8;
  for (int it = kt; it < nq; ++it) {
    const int buf = (it - kt) & 1;
    if (it + 1 < nq) {
      load_tile<HD>(sQ + (buf ^ 1) * BR * HD, q, row_base + (it + 1) * BR, ld, col0);
      load_tile<HD>(sdO + (buf ^ 1) * BR * HD, dout, row_base + (it + 1) * BR, ld, col0);
      if (threadIdx.x < BR) {
        sL[(buf ^ 1) * BR + threadIdx.x] = Lr[(it + 1) * BR + threadIdx.x] * kLog2e;
        sD[(buf ^ 1) * BR + threadIdx.x] = Dr[(it + 1) * BR + threadIdx.x];
      }
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* cQ = sQ + buf * BR * HD;
    const __nv_bfloat16* cdO = sdO + buf * BR * HD;
    const float* cL = sL + buf * BR;
    const float* cD = sD + buf * BR;
    // S^T = K Q^T and dP^T = V dO^T  (16 keys x 64 queries per warp)
    float st[BR / 8][4], dpt[BR / 8][4];
#pragma unroll
    for (int i = 0; i < BR / 8; ++i) {
      st[i][0] = st[i][1] = st[i][2] = st[i][3] = 0.f;
      dpt[i][0] = dpt[i][1] = dpt[i][2] = dpt[i][3] = 0.f;
    }
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ka[4], va[4];
      frag_a<HD>(ka, sK, warp * 16, kk * 16);
      frag_a<HD>(va, sV, warp * 16, kk * 16);
#pragma unroll
      for (int np = 0; np < BR / 16; ++np) {
        uint32_t bq[4], bd[4];
        frag_b_nk<HD>(bq, cQ, np * 16, kk * 16);
        frag_b_nk<HD>(bd, cdO, np * 16, kk * 16);
        mma16816(st[2 * np], ka, bq[0], bq[1]);
        mma16816(st[2 * np + 1], ka, bq[2], bq[3]);
        mma16816(dpt[2 * np], va, bd[0], bd[1]);
        mma16816(dpt[2 * np + 1], va, bd[2], bd[3]);
      }
    }
    // P^T and dS^T
#pragma unroll
    for (int nb = 0; nb < BR / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = nb * 8 + 2 * t + (e & 1);   // query column within the tile
        const int qpos = it * BR + qc;
        const int key = (e < 2) ? key0 : key1;
        float p = exp2f(st[nb][e] * scale_log2 - cL[qc]);
        if (key > qpos) p = 0.f;
        st[nb][e] = p;
        dpt[nb][e] = p * (dpt[nb][e] - cD[qc]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q
#pragma unroll
    for (int kk = 0; kk < BR / 16; ++kk) {
      uint32_t pa[4], sa[4];
      pa[0] = pack2(st[2 * kk][0], st[2 * kk][1]);
      pa[1] = pack2(st[2 * kk][2], st[2 * kk][3]);
      pa[2] = pack2(st[2 * kk + 1][0], st[2 * kk + 1][1]);
      pa[3] = pack2(st[2 * kk + 1][2], st[2 * kk + 1][3]);
      sa[0] = pack2(dpt[2 * kk][0], dpt[2 * kk][1]);
      sa[1] = pack2(dpt[2 * kk][2], dpt[2 * kk][3]);
      sa[2] = pack2(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
      sa[3] = pack2(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t bd[4], bq[4];
        frag_b_kn<HD>(bd, cdO, kk * 16, np * 16);
        frag_b_kn<HD>(bq, cQ, kk * 16, np * 16);
        mma16816(dva[2 * np], pa, bd[0], bd[1]);
        mma16816(dva[2 * np + 1], pa, bd[2], bd[3]);
        mma16816(dka[2 * np], sa, bq[0], bq[1]);
        mma16816(dka[2 * np + 1], sa, bq[2], bq[3]);
      }
    }
    __syncthreads();
  }
  __nv_bfloat16* k0p = dk + (row_base + key0) * (long long)ld + col0;
  __nv_bfloat16* k1p = dk + (row_base + key1) * (long long)ld + col0;
  __nv_bfloat16* v0p = dv + (row_base + key0) * (long long)ld + col0;
  __nv_bfloat16* v1p = dv + (row_base + key1) * (long long)ld + col0;
#pragma unroll
  for (int nb = 0; nb < HD / 8; ++nb) {
    const int c = nb * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(k0p + c) = pack2(dka[nb][0] * scale, dka[nb][1] * scale);
    *reinterpret_cast<uint32_t*>(k1p + c) = pack2(dka[nb][2] * scale, dka[nb][3] * scale);
    *reinterpret_cast<uint32_t*>(v0p + c) = pack2(dva[nb][0], dva[nb][1]);
    *reinterpret_cast<uint32_t*>(v1p + c) = pack2(dva[nb][2], dva[nb][3]);
  }
}

template <int HD>
__global__ void dsum_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                            float* __restrict__ dsum, int B, int S, int H, int ld) {
  // D[b][h][i] = rowsum(dO * O) per head. One warp per token row (b, i), walking its
  // H heads contiguously: 16-byte loads, each half-warp covers one head of hd = 128
  // (hd = 64: a quarter-warp), segmented shuffle reduction. Fully coalesced. The loads of
  // kBatch head groups are issued before any math (more bytes in flight per warp).
  constexpr int kLanesPerHead = HD / 8, kHeadsPerIter = 32 / kLanesPerHead, kBatch = 4;
  const long long rows = (long long)B * S;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= rows) return;
  const int lane = threadIdx.x & 31;
  const int b = (int)(gw / S), i = (int)(gw % S);
  const __nv_bfloat16* orow = o + gw * ld;
  const __nv_bfloat16* drow = dout + gw * ld;
  const int d = (lane % kLanesPerHead) * 8;
  for (int h0 = 0; h0 < H; h0 += kBatch * kHeadsPerIter) {
    uint4 a[kBatch], c[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const int hh = h0 + k * kHeadsPerIter + lane / kLanesPerHead;
      if (hh < H) {
        a[k] = *reinterpret_cast<const uint4*>(orow + (long long)hh * HD + d);
        c[k] = *reinterpret_cast<const uint4*>(drow + (long long)hh * HD + d);
      } else {
        a[k] = make_uint4(0, 0, 0, 0);
        c[k] = a[k];
      }
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[k]);
      const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c[k]);
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(a2[e]), y = __bfloat1622float2(c2[e]);
        s += x.x * y.x + x.y * y.y;
      }
#pragma unroll
      for (int off = kLanesPerHead / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const int hh = h0 + k * kHeadsPerIter + lane / kLanesPerHead;
      if (hh < H && lane % kLanesPerHead == 0) dsum[((long long)b * H + hh) * S + i] = s;
    }
  }
}

// tcgen05 kernels (attention_tc.cu) unless HLM_ATTN_MMA_SYNC=1 (A/B comparisons)
bool use_tc() {
  static int mma_sync = -1;
  if (mma_sync < 0) {
    const char* e = getenv("HLM_ATTN_MMA_SYNC");
    mma_sync = (e && *e == '1') ? 1 : 0;
  }
  return !mma_sync;
}

template <int HD>
int fwd_impl(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int ld,
             cudaStream_t s) {
  const int smem = (BR + 4 * BC) * HD * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_fwd<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(S / BR, B * H);
  flash_fwd<HD><<<grid, NW * 32, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                            (const __nv_bfloat16*)v, (__nv_bfloat16*)o, lse, S, H, ld,
                                            (1.0f / sqrtf((float)HD)) * kLog2e);
  hlm_count_launches(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <int HD>
int bwd_impl(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
             float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int ld, cudaStream_t s) {
  const int smem_dq = (2 * BR + 4 * BC) * HD * 2;
  const int smem_dkv = (2 * BC + 4 * BR) * HD * 2 + 4 * BR * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_bwd_dq<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dq);
    cudaFuncSetAttribute(flash_bwd_dkv<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dkv);
    attr = true;
  }
  const float scale = 1.0f / sqrtf((float)HD);
  dsum_kernel<HD><<<(unsigned)(((long long)B * S + 7) / 8), 256, 0, s>>>((const __nv_bfloat16*)o,
                                                                           (const __nv_bfloat16*)dout, dsum, B, S,
                                                                           H, ld);
  if (use_tc() && hlm_flash_tc_supported(HD, S, ld)) {
    hlm_count_launches(1);
    return hlm_flash_bwd_tc(q, k, v, dout, lse, dsum, dq, dk, dv, B, S, H, ld, s);
  }
  dim3 grid(S / BR, B * H);
  flash_bwd_dq<HD><<<grid, NW * 32, smem_dq, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                  (const __nv_bfloat16*)v, (const __nv_bfloat16*)dout, lse, dsum,
                                                  (__nv_bfloat16*)dq, S, H, ld, scale, scale * kLog2e);
  flash_bwd_dkv<HD><<<grid, NW * 32, smem_dkv, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                    (const __nv_bfloat16*)v, (const __nv_bfloat16*)dout, lse, dsum,
                                                    (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, S, H, ld, scale,
                                                    scale * kLog2e);
  hlm_count_launches(3);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

bool hlm_flash_supported(int head_dim, int seq) { return (head_dim == 64 || head_dim == 128) && seq % 64 == 0; }

int hlm_flash_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int hd,
                  int ld, cudaStream_t s) {
  if (use_tc() && hlm_flash_tc_supported(hd, S, ld)) return hlm_flash_fwd_tc(q, k, v, o, lse, B, S, H, ld, s);
  if (hd == 128) return fwd_impl<128>(q, k, v, o, lse, B, S, H, ld, s);
  if (hd == 64) return fwd_impl<64>(q, k, v, o, lse, B, S, H, ld, s);
  return 2;
}

int hlm_flash_bwd(const void* q, const void* k, const void* v, const void* o, const void* d_o, const float* lse,
                  float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int hd, int ld, cudaStream_t s) {
  if (hd == 128) return bwd_impl<128>(q, k, v, o, d_o, lse, dsum, dq, dk, dv, B, S, H, ld, s);
  if (hd == 64) return bwd_impl<64>(q, k, v, o, d_o, lse, dsum, dq, dk, dv, B, S, H, ld, s);
  return 2;
}
