// Causal flash attention on tcgen05 / TMEM / TMA (head_dim 128, seq % 128 == 0), forward
// and backward. Same contract as the mma.sync kernels (attention_flash.cu) and the reference
// attention_fwd / attention_bwd (proj/include/hlm/kernels.hpp:207-299): per head, scale
// 1/sqrt(hd), O and the row log-sum-exp forward; dQ, dK, dV from O, dO, lse and D = rowsum(dO.O).
//
// Production kernels (defaults; the others stay selectable for A/B):
//   flash_fwd_pp3      persistent forward: one CTA per SM walks query-tile PAIRS (two 128-query
//                      tiles ping-ponging on the tensor core, 64-key steps, S double-buffered
//                      per tile in TMEM, P written over S, O accumulated in TMEM, lazy 2^8
//                      rescale), O stored through a shared-memory stage
//   flash_bwd_dkv_tc3  persistent dK/dV: 128-key tiles, 64-query steps, S^T / dP^T
//                      double-buffered in TMEM, P^T / dS^T written back over them as A operands
//                      from TMEM, dK / dV accumulated in TMEM, TMA-stored through a stage
//   flash_bwd_dq_tc3   persistent dQ: 128-query tiles, 64-key steps, Q / dO TMEM-resident as A
//                      operands (TMA-loaded for the next tile while this one runs), dS over dP
// Persistent kernels claim tiles from a per-launch counter (tile_counter) in grouped
// longest-first order (tile_decode). Earlier versions kept for comparison: flash_fwd_tc (one
// query tile per CTA, round 1), flash_fwd_pp (128-key steps), flash_fwd_pp2 (one CTA per pair),
// flash_bwd_dkv_tc / flash_bwd_dq_tc (128-wide steps), flash_bwd_dkv_tc2 / flash_bwd_dq_tc2 (one
// CTA per tile). DESIGN.md "Attention" has the measurements behind each step.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "attention.h"
#include "block_ops.h"
#include "sm100_ptx.cuh"

using namespace hlm_sm100;

namespace {

constexpr int TQ = 128, TK = 128, HD = 128;
constexpr int TILE_BYTES = TQ * HD * 2;            // 32 KiB
constexpr int ATOM_BYTES = 128 * 64 * 2;           // 16 KiB: 128 rows x 64 cols
constexpr int FWD_THREADS = 384;
constexpr int SMEM_BYTES = TILE_BYTES * 7 + 1024 + 256 + 1024;   // Q, K0 V0 K1 V1, P0 P1, barriers, row exchange
constexpr float kLog2e = 1.4426950408889634f;

struct Bars {
  uint64_t q_full, k_full[2], k_empty[2], s_full[2], s_free[2], p_full[2], o_full[2], o_free[2];
  uint64_t v_full[2], v_empty[2];
  uint32_t tmem;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA store of one box (shared -> global, bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Blackwell packed fp32 (two lanes per instruction, each rounded like FFMA / FADD)
// and the three-input max: fewer issue slots per score in the softmax loop.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n.reg .b64 ra, rb, rc, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %4};\nmov.b64 rc, {%5, %5};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1) {
  asm("{\n.reg .b64 ra, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rd, {%0, %1};\n"
      "add.rn.f32x2 rd, rd, ra;\nmov.b64 {%0, %1}, rd;\n}"
      : "+f"(d0), "+f"(d1) : "f"(a0), "f"(a1));
}
// general two-lane forms (per-lane operands), each lane rounded like the scalar op
__device__ __forceinline__ void fma2v(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n.reg .b64 ra, rb, rc, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// (a - b) * p per lane: the dS = P (dP - D) of the attention backward
__device__ __forceinline__ void submul2(float& d0, float& d1, float a0, float a1, float b0, float b1, float p0,
                                        float p1) {
  asm("{\n.reg .b64 ra, rb, rp, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rp, {%6, %7};\n"
      "sub.rn.f32x2 rd, ra, rb;\nmul.rn.f32x2 rd, rp, rd;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(p0), "f"(p1));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe for two lanes (the MUFU ex2 is the forward softmax's bottleneck):
// x = j + f, j = rint(x) via the 1.5 * 2^23 shift, 2^f on [-1/2, 1/2] by a degree-3
// polynomial (max relative error 1.0e-4, far below the bf16 rounding of P), 2^j added to
// the exponent field. x is clamped at -127, where the result is exactly +0 (masked scores).
__device__ __forceinline__ void ex2_poly2(float& y0, float& y1, float x0, float x1) {
  x0 = fmaxf(x0, -127.f);
  x1 = fmaxf(x1, -127.f);
  float t0, t1, f0, f1, p0, p1;
  asm("{\n.reg .b64 x, t, m, f;\n"
      "mov.b64 x, {%4, %5};\nmov.b64 m, {%6, %6};\n"
      "add.rn.f32x2 t, x, m;\nsub.rn.f32x2 f, t, m;\nsub.rn.f32x2 f, x, f;\n"
      "mov.b64 {%0, %1}, t;\nmov.b64 {%2, %3}, f;\n}"
      : "=f"(t0), "=f"(t1), "=f"(f0), "=f"(f1) : "f"(x0), "f"(x1), "f"(12582912.f));
  fma2v(p0, p1, f0, f1, 0.05499936f, 0.05499936f, 0.24221137f, 0.24221137f);
  fma2v(p0, p1, p0, p1, f0, f1, 0.69328505f, 0.69328505f);
  fma2v(p0, p1, p0, p1, f0, f1, 1.0f, 1.0f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}
// the two softmax warps sharing TMEM lanes 32q..32q+31 (named barrier 1 + q, 64 threads)
__device__ __forceinline__ void pair_sync(int q) { asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory"); }

// K-major SW128 descriptor for K step kk (16 elements) of a 128 x 128 tile stored as two atoms.
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int kk) {
  return make_sw128_desc(base + (kk >> 2) * ATOM_BYTES + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor (V): K step kk = 16 key rows; MN atoms (64 d) 16 KiB apart.
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t base, int kk) {
  return make_sw128_desc(base + kk * 2048, ATOM_BYTES, 1024);
}
// 64-row tiles (64-wide steps): two 64 x 64 boxes
constexpr int HALF_TILE = 64 * HD * 2;   // 16 KiB: 64 rows x 128 columns (two 64x64 SW128 boxes)
constexpr int HALF_ATOM = 64 * 64 * 2;   // 8 KiB: one 64-row x 64-column swizzle box
// K-major descriptor for K step kk of a 64-row x 128-column tile (two 8 KiB boxes)
__device__ __forceinline__ uint64_t kmajor_desc64(uint32_t base, int kk) {
  return make_sw128_desc(base + (kk >> 2) * HALF_ATOM + (kk & 3) * 32, 16, 1024);
}
// MN-major descriptor of the same 64-row tile used as B with N = its 128 columns, K = its rows
__device__ __forceinline__ uint64_t mnmajor_desc64(uint32_t base, int kk) {
  return make_sw128_desc(base + kk * 2048, HALF_ATOM, 1024);
}

// Round-1 forward (HLM_ATTN_FWD_V1=1): one CTA per (128-query tile, batch*head). Warp 0 TMA
// (Q once, K/V into a 2-stage ring), warp 1 MMA (S_j = Q K_j^T into TMEM S[j%2], O_j = P_j V_j
// into O[j%2] with P from shared memory; S_{j+1} issued before PV_j), warp 2 TMEM allocator,
// warps 4-11 softmax (thread = query row, column halves exchanged through shared memory).
__global__ void __launch_bounds__(FWD_THREADS, 1)
    flash_fwd_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                 const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                 int S, int H, int ld, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK[2] = {smem + TILE_BYTES, smem + 3 * TILE_BYTES};
  uint8_t* sV[2] = {smem + 2 * TILE_BYTES, smem + 4 * TILE_BYTES};
  uint8_t* sP[2] = {smem + 5 * TILE_BYTES, smem + 6 * TILE_BYTES};
  Bars* bars = reinterpret_cast<Bars*>(smem + 7 * TILE_BYTES);
  float* xch = reinterpret_cast<float*>(smem + 7 * TILE_BYTES + 256);   // [2 halves][128 rows]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = (int)(gridDim.x - 1 - blockIdx.x);   // long (late) query tiles first
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const int row0 = b * S;
  const int col0 = hh * HD;
  const int n_tiles = qt + 1;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], 8);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], 8);
      mbar_init(&bars->p_full[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->q_full, TILE_BYTES);
      tma_load_2d(sQ, &map_q, &bars->q_full, col0, row0 + qt * TQ);
      tma_load_2d(sQ + ATOM_BYTES, &map_q, &bars->q_full, col0 + 64, row0 + qt * TQ);
      // K_j is released by S_j, V_j by PV_j: the next K streams in while the softmax runs
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const int r = row0 + j * TK;
        mbar_wait(&bars->k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->k_full[st], TILE_BYTES);
        tma_load_2d(sK[st], &map_k, &bars->k_full[st], col0, r);
        tma_load_2d(sK[st] + ATOM_BYTES, &map_k, &bars->k_full[st], col0 + 64, r);
        mbar_wait(&bars->v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->v_full[st], TILE_BYTES);
        tma_load_2d(sV[st], &map_v, &bars->v_full[st], col0, r);
        tma_load_2d(sV[st] + ATOM_BYTES, &map_v, &bars->v_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    const uint32_t q_base = smem_u32(sQ);
    mbar_wait(&bars->q_full, 0);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&bars->k_full[st], (j >> 1) & 1);
      mbar_wait(&bars->s_free[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_base = smem_u32(sK[st]);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem + st * 128, kmajor_desc(q_base, kk), kmajor_desc(k_base, kk), idesc_s, kk ? 1u : 0u);
        umma_commit(&bars->s_full[st]);
        umma_commit(&bars->k_empty[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      if (j + 1 < n_tiles) issue_s(j + 1);
      mbar_wait(&bars->p_full[st], (j >> 1) & 1);
      mbar_wait(&bars->o_free[st], ((j >> 1) & 1) ^ 1);
      mbar_wait(&bars->v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t v_base = smem_u32(sV[st]);
        const uint32_t p_base = smem_u32(sP[st]);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)
          umma_bf16(tmem + 256 + st * 128, kmajor_desc(p_base, kk), mnmajor_desc(v_base, kk), idesc_o, kk ? 1u : 0u);
        umma_commit(&bars->o_full[st]);
        umma_commit(&bars->v_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2;             // S / O columns [64*half, 64*half + 64)
    const int quarter = warp & 3;                 // TMEM lanes 32*quarter .. +31
    const int r = quarter * 32 + lane;            // query row within the tile
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int cb = half * 64;
    float oacc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) oacc[i] = 0.f;
    float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
    // O_acc <- alpha * O_acc + O_j (this half's 64 columns of TMEM O[jj % 2]), then release it
    auto fold = [&](int jj, float alpha) {
      const int so = jj & 1;
      mbar_wait(&bars->o_full[so], (jj >> 1) & 1);
      tc_fence_after();
      uint32_t v0[32], v1[32];
      tmem_ld_32x32(tmem + 256 + so * 128 + cb + lane_off, v0);
      tmem_ld_32x32(tmem + 256 + so * 128 + cb + 32 + lane_off, v1);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        oacc[e] = oacc[e] * alpha + __uint_as_float(v0[e]);
        oacc[32 + e] = oacc[32 + e] * alpha + __uint_as_float(v1[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->o_free[so]);
    };
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      const bool diag = j == qt;
      mbar_wait(&bars->s_full[st], (j >> 1) & 1);
      tc_fence_after();
      uint32_t s0[32], s1[32];
      tmem_ld_32x32(tmem + st * 128 + cb + lane_off, s0);
      tmem_ld_32x32(tmem + st * 128 + cb + 32 + lane_off, s1);
      tmem_ld_wait();
      float sv[64];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        sv[e] = __uint_as_float(s0[e]) * scale_log2;
        sv[32 + e] = __uint_as_float(s1[e]) * scale_log2;
      }
      if (diag) {
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (cb + e > r) sv[e] = -INFINITY;
      }
      float mx = m;
#pragma unroll
      for (int e = 0; e < 64; ++e) mx = fmaxf(mx, sv[e]);
      // row max across the two column halves
      xch[half * 128 + r] = mx;
      pair_sync(quarter);
      mx = fmaxf(xch[r], xch[128 + r]);
      pair_sync(quarter);                         // both read before the next tile's write
      const float alpha = ex2(m - mx);
      m = mx;
      // P[st] was last read by PV_{j-2}
      if (j >= 2) mbar_wait(&bars->o_full[st], ((j - 2) >> 1) & 1);
      uint8_t* prow = sP[st] + half * ATOM_BYTES + r * 128;   // keys 64*half.. = swizzle atom `half`
      float rs = 0.f;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {               // 16-byte chunk = 8 keys
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const float p0 = ex2(sv[cc * 8 + e] - m);
          const float p1 = ex2(sv[cc * 8 + e + 1] - m);
          rs += p0 + p1;
          pk[e / 2] = pack_bf16x2(p0, p1);
        }
        *reinterpret_cast<uint4*>(prow + ((cc ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l = l * alpha + rs;
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars->s_free[st]);
        mbar_arrive(&bars->p_full[st]);
      }
      // fold the previous tile while PV_j runs on the tensor core
      if (j >= 1) fold(j - 1, alpha_prev);
      alpha_prev = alpha;
    }
    fold(n_tiles - 1, alpha_prev);
    xch[half * 128 + r] = l;
    pair_sync(quarter);
    const float lt = xch[r] + xch[128 + r];
    const float il = 1.f / lt;
    __nv_bfloat16* orow = o + (long long)(row0 + qpos) * ld + col0 + cb;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 val = make_uint4(pack_bf16x2(oacc[8 * c] * il, oacc[8 * c + 1] * il),
                             pack_bf16x2(oacc[8 * c + 2] * il, oacc[8 * c + 3] * il),
                             pack_bf16x2(oacc[8 * c + 4] * il, oacc[8 * c + 5] * il),
                             pack_bf16x2(oacc[8 * c + 6] * il, oacc[8 * c + 7] * il));
      reinterpret_cast<uint4*>(orow)[c] = val;
    }
    if (half == 0) lse[(long long)bh * S + qpos] = (m + log2f(lt)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


// ------------------------------------------------------------------ forward, ping-pong
// Two 128-query tiles per CTA (A = 2p, B = 2p + 1) share every K / V tile, and the
// softmax of one tile runs while the tensor core works on the other.
//   TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512).
//   P (bf16) overwrites the first 64 columns of its S region (tcgen05.st) and the PV
//   MMA reads it straight from TMEM (A operand in TMEM); O accumulates in TMEM.
//   The running row max is raised only when a tile's max exceeds it by more than
//   2^8 (then the owning warp rescales its O rows and l in place); otherwise P <= 256,
//   exact in the fp32 accumulators. No O traffic through registers per tile.
//   warp 0 TMA producer (Q_A, Q_B once; K / V 2-slot rings released separately),
//   warp 1 MMA issuer + TMEM allocator, warps 2-9 softmax: tile (w-2)/4, TMEM lane
//   quarter w%4, thread = query row, all 128 key columns in registers. (A 16-warp
//   variant with 64 columns per thread and a smem row-max exchange measured slower:
//   0.49 vs 0.38 ms at C2 — spills at 96 registers and the extra barriers.)
struct PPBars {
  uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2], o_final[2];
  uint32_t tmem;
};
constexpr int PP_THREADS = 320;
constexpr int PP_SMEM = TILE_BYTES * 6 + 1024 + 256;
constexpr float kRescaleLog2 = 8.0f;

__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// 32 lanes x 16 columns of 32-bit
__device__ __forceinline__ void tmem_ld_32x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_32x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
__device__ __forceinline__ void tmem_st_32x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void tmem_st_32x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// kEmu of every 4 exponentials per thread run on the FMA pipe (ex2_poly2), the rest on MUFU
template <int kEmu>
__global__ void __launch_bounds__(PP_THREADS, 1)
    flash_fwd_pp(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                 const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                 int S, int H, int ld, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // tile t / ring slot st as arithmetic, not runtime-indexed arrays (those live on the stack)
  auto sQ = [&](int t) { return smem + t * TILE_BYTES; };
  auto sK = [&](int st) { return smem + (2 + st) * TILE_BYTES; };
  auto sV = [&](int st) { return smem + (4 + st) * TILE_BYTES; };
  PPBars* bars = reinterpret_cast<PPBars*>(smem + 6 * TILE_BYTES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int pair = (int)(gridDim.x - 1 - blockIdx.x);   // long (late) query tiles first
  const int ntile_b = 2 * pair + 2;                     // key tiles of query tile B (A: one fewer)
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const int row0 = b * S;
  const int col0 = hh * HD;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 4);
      mbar_init(&bars->o_final[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->q_full, 2 * TILE_BYTES);
      for (int t = 0; t < 2; ++t) {
        tma_load_2d(sQ(t), &map_q, &bars->q_full, col0, row0 + (2 * pair + t) * TQ);
        tma_load_2d(sQ(t) + ATOM_BYTES, &map_q, &bars->q_full, col0 + 64, row0 + (2 * pair + t) * TQ);
      }
      for (int j = 0; j < ntile_b; ++j) {
        const int st = j & 1;
        const int r = row0 + j * TK;
        mbar_wait(&bars->k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->k_full[st], TILE_BYTES);
        tma_load_2d(sK(st), &map_k, &bars->k_full[st], col0, r);
        tma_load_2d(sK(st) + ATOM_BYTES, &map_k, &bars->k_full[st], col0 + 64, r);
        mbar_wait(&bars->v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->v_full[st], TILE_BYTES);
        tma_load_2d(sV(st), &map_v, &bars->v_full[st], col0, r);
        tma_load_2d(sV(st) + ATOM_BYTES, &map_v, &bars->v_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    mbar_wait(&bars->q_full, 0);
    // S_t = Q_t K_j^T; K_j is released by tile B's S (B uses every K tile, after A)
    auto issue_s = [&](int t, int j) {
      const int st = j & 1;
      mbar_wait(&bars->k_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t q_base = smem_u32(sQ(t)), k_base = smem_u32(sK(st));
      umma_chain_w<8, ATOM_BYTES / 16, 2, ATOM_BYTES / 16, 2>(tmem + t * 128, kmajor_desc(q_base, 0),
                                                             kmajor_desc(k_base, 0), idesc_s, 0u);
      umma_commit_w(&bars->s_full[t]);
      if (t == 1) umma_commit_w(&bars->k_empty[st]);
    };
    // O_t += P_t V_j with P_t in TMEM (the first 64 columns of S_t); V_j released by tile B's PV
    auto issue_pv = [&](int t, int j) {
      const int st = j & 1;
      mbar_wait(&bars->p_full[t], j & 1);
      mbar_wait(&bars->v_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_base = smem_u32(sV(st));
#pragma unroll
      for (int kk = 0; kk < TK / 16; ++kk)
        umma_bf16_ts_w(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmajor_desc(v_base, kk), idesc_o,
                       (j > 0 || kk > 0) ? 1u : 0u);
      if (t == 1) umma_commit_w(&bars->v_empty[st]);
    };
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < ntile_b; ++j) {
      if (j < ntile_b - 1) {
        issue_pv(0, j);
        if (j + 1 < ntile_b - 1) {
          issue_s(0, j + 1);
        } else {
          umma_commit_w(&bars->o_final[0]);
        }
      }
      issue_pv(1, j);
      if (j + 1 < ntile_b) {
        issue_s(1, j + 1);
      } else {
        umma_commit_w(&bars->o_final[1]);
      }
    }
  } else {
    const int t = (warp - 2) >> 2;                 // query tile A (0) or B (1)
    const int quarter = warp & 3;                  // TMEM lanes 32*quarter ..
    const int r = quarter * 32 + lane;             // query row within the tile
    const int qt = 2 * pair + t, n = qt + 1;
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_addr = tmem + t * 128 + lane_off, o_addr = tmem + 256 + t * 128 + lane_off;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      mbar_wait(&bars->s_full[t], j & 1);
      tc_fence_after();
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32(s_addr + c * 32, sv[c]);
      tmem_ld_wait();
      if (j == qt) {   // diagonal tile (warp-uniform): mask keys above the row
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (c * 32 + e > r) sv[c][e] = __float_as_uint(-INFINITY);
      }
      // max of the raw scores (scale_log2 > 0 commutes with max); 8 independent chains
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(__uint_as_float(sv[0][u]), __uint_as_float(sv[0][u + 8]));
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = (c == 0 ? 16 : 0); e < 32; e += 2)
          mx8[e & 7] = fmax3(mx8[e & 7], __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
      const float mx = scale_log2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                          fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      if (j == 0) {
        m = mx;
      } else if (__any_sync(0xffffffffu, mx > m + kRescaleLog2)) {
        // O_t holds P V of tiles < j: S_t(j) was issued after PV_t(j-1), so its
        // completion implies theirs. Rescale this warp's 32 rows in TMEM.
        const float mn = fmaxf(m, mx);
        const float alpha = ex2(m - mn);
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {   // 16 columns at a time: the 128 scores stay in registers
          uint32_t ov[16];
          tmem_ld_32x16(o_addr + c * 16, ov);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st_32x16(o_addr + c * 16, ov);
        }
        l *= alpha;
        m = mn;
      }
      // P = 2^(s * scale_log2 - m) <= 2^8 as bf16 pairs into S_t columns [0, 64)
      const float negm = -m;
      float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float a0, a1;
          ffma2(a0, a1, __uint_as_float(sv[c][2 * e]), __uint_as_float(sv[c][2 * e + 1]), scale_log2, negm);
          float p0, p1;
          if ((e & 3) < kEmu) {
            ex2_poly2(p0, p1, a0, a1);
          } else {
            p0 = ex2(a0);
            p1 = ex2(a1);
          }
          fadd2(l8[2 * (e & 3)], l8[2 * (e & 3) + 1], p0, p1);
          pk[e] = pack_bf16x2(p0, p1);
        }
        tmem_st_32x16(s_addr + c * 16, pk);
      }
      l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full[t]);
    }
    mbar_wait(&bars->o_final[t], 0);
    tc_fence_after();
    const float il = 1.f / l;
    __nv_bfloat16* orow = o + (long long)(row0 + qpos) * ld + col0;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32(o_addr + c * 32, ov);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<uint4*>(orow + c * 32)[q] =
            make_uint4(pack_bf16x2(__uint_as_float(ov[8 * q]) * il, __uint_as_float(ov[8 * q + 1]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 2]) * il, __uint_as_float(ov[8 * q + 3]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 4]) * il, __uint_as_float(ov[8 * q + 5]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 6]) * il, __uint_as_float(ov[8 * q + 7]) * il));
    }
    lse[(long long)bh * S + qpos] = (m + log2f(l)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ forward, 64-key steps
// Same two-query-tile ping-pong, but over 64-key steps with S double-buffered per tile:
//   TMEM: S_A[2] [0,128) (64 each), S_B[2] [128,256), O_A [256,384), O_B [384,512).
// S_t(j+2) goes into the buffer P_t(j) came from, right behind PV_t(j) (in-order tensor
// pipe), so S_t(j+1) is already computed when tile t's softmax of step j ends: the
// softmax of a tile no longer waits a PV + S round trip per step, only the tensor pipe.
// K / V: KF_STAGES-deep ring of 64-row stages, released by tile B's PV (B uses every key).
// A rare lazy rescale of O_t (row max up by more than 2^8) first waits for PV_t(j-1).
#ifdef HLM_ATTN_TIMELINE   // tools/attn_timeline.cu only: per-CTA global-timer stamps
__device__ unsigned long long* g_attn_tl;
__device__ __forceinline__ void tl_put_at(int rec, int slot, unsigned long long v) { g_attn_tl[rec * 16 + slot] = v; }
__device__ __forceinline__ void tl_put(int slot, unsigned long long v) {
  tl_put_at((int)(blockIdx.x + gridDim.x * blockIdx.y), slot, v);
}
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HLM_TL(slot) tl_put(slot, tl_now())
#define HLM_TL_VAL(slot, v) tl_put(slot, (unsigned long long)(v))
#define HLM_TL_AT(rec, slot) tl_put_at(rec, slot, tl_now())
#define HLM_TL_AT_VAL(rec, slot, v) tl_put_at(rec, slot, (unsigned long long)(v))
#else
#define HLM_TL_AT(rec, slot) ((void)0)
#define HLM_TL_AT_VAL(rec, slot, v) ((void)0)
#define HLM_TL(slot) ((void)0)
#define HLM_TL_VAL(slot, v) ((void)0)
#endif

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
constexpr int KF_STAGES = 4;
struct PP2Bars {
  uint64_t q_full, kv_full[KF_STAGES], kv_empty[KF_STAGES], s_full[2][2], p_full[2][2], pv_done[2], o_final[2];
  uint32_t tmem;
};
constexpr int PP2_SMEM = TILE_BYTES * 2 + KF_STAGES * 2 * HALF_TILE + 1024 + 256;

// Grid order of the production kernels. grid = (tiles per head, B * H); `rank` 0 is the
// longest tile (most causal steps). group == 0: head by head, longest tile of each head first.
// group > 0: the linear grid walks groups of `group` heads and, inside a group, all its heads'
// longest tiles first — the grid's tail then holds only short tiles, while the ~148 CTAs in
// flight still span few enough heads for their K / V (1 MB per head at S 2048) to stay in L2.
__device__ __forceinline__ void tile_decode(int lin, int nt, int nbh, int group, int& rank, int& bh) {
  if (group <= 0) {
    rank = lin % nt;
    bh = lin / nt;
    return;
  }
  const int g = lin / (nt * group), r = lin - g * nt * group;
  const int heads = min(group, nbh - g * group);
  rank = r / heads;
  bh = g * group + r % heads;
}
__device__ __forceinline__ void tile_order(int group, int& rank, int& bh) {
  tile_decode((int)blockIdx.x + (int)gridDim.x * (int)blockIdx.y, (int)gridDim.x, (int)gridDim.y, group, rank, bh);
}

template <int kEmu>
__global__ void __launch_bounds__(PP_THREADS, 1)
    flash_fwd_pp2(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k64,
                  const __grid_constant__ CUtensorMap map_v64, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                  int S, int H, int ld, float scale_log2, int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto sQ = [&](int t) { return smem + t * TILE_BYTES; };
  auto sK = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE; };
  auto sV = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE + HALF_TILE; };
  PP2Bars* bars = reinterpret_cast<PP2Bars*>(smem + 2 * TILE_BYTES + KF_STAGES * 2 * HALF_TILE);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int rank, bh;
  tile_order(order, rank, bh);
  const int pair = (int)gridDim.x - 1 - rank;           // long (late) query tiles first
  const int nb = 4 * pair + 4;                          // 64-key steps of query tile B (A: two fewer)
  const int b = bh / H, hh = bh % H;
  const int row0 = b * S;
  const int col0 = hh * HD;

  if (threadIdx.x == 0) {
    HLM_TL(0);
    {
      unsigned smid_v;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_v));
      (void)smid_v;
      HLM_TL_VAL(6, smid_v);
      HLM_TL_VAL(7, nb);
    }
    tma_prefetch(&map_q);
    tma_prefetch(&map_k64);
    tma_prefetch(&map_v64);
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < KF_STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars->s_full[t][0], 1);
      mbar_init(&bars->s_full[t][1], 1);
      mbar_init(&bars->p_full[t][0], 4);   // per buffer: a softmax can run a step ahead of its PV
      mbar_init(&bars->p_full[t][1], 4);
      mbar_init(&bars->pv_done[t], 1);
      mbar_init(&bars->o_final[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->q_full, 2 * TILE_BYTES);
      for (int t = 0; t < 2; ++t) {
        tma_load_2d(sQ(t), &map_q, &bars->q_full, col0, row0 + (2 * pair + t) * TQ);
        tma_load_2d(sQ(t) + ATOM_BYTES, &map_q, &bars->q_full, col0 + 64, row0 + (2 * pair + t) * TQ);
      }
      for (int j = 0; j < nb; ++j) {
        const int st = j % KF_STAGES;
        const int r = row0 + j * 64;
        mbar_wait(&bars->kv_empty[st], ((j / KF_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[st], 2 * HALF_TILE);
        tma_load_2d(sK(st), &map_k64, &bars->kv_full[st], col0, r);
        tma_load_2d(sK(st) + HALF_ATOM, &map_k64, &bars->kv_full[st], col0 + 64, r);
        tma_load_2d(sV(st), &map_v64, &bars->kv_full[st], col0, r);
        tma_load_2d(sV(st) + HALF_ATOM, &map_v64, &bars->kv_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    const int n_t[2] = {nb - 2, nb};
    mbar_wait(&bars->q_full, 0);
    if (lane == 0) HLM_TL(1);
    auto issue_s = [&](int t, int j) {
      const int st = j % KF_STAGES;
      mbar_wait(&bars->kv_full[st], (j / KF_STAGES) & 1);
      tc_fence_after();
      umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + t * 128 + (j & 1) * 64,
                                                            kmajor_desc(smem_u32(sQ(t)), 0),
                                                            kmajor_desc64(smem_u32(sK(st)), 0), idesc_s, 0u);
      umma_commit_w(&bars->s_full[t][j & 1]);
    };
    // O_t += P_t(j) V_j, P_t(j) (bf16) in the first 32 columns of S_t[j % 2]
    auto issue_pv = [&](int t, int j) {
      const int st = j % KF_STAGES;
      mbar_wait(&bars->p_full[t][j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_base = smem_u32(sV(st));
      const uint32_t p_tmem = tmem + t * 128 + (j & 1) * 64;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_ts_w(tmem + 256 + t * 128, p_tmem + kk * 8, mnmajor_desc64(v_base, kk), idesc_o,
                       (j > 0 || kk > 0) ? 1u : 0u);
      if (j + 2 == n_t[t]) umma_commit_w(&bars->pv_done[t]);   // PV_t(n-2): for a rescale at the last step
      if (t == 1) umma_commit_w(&bars->kv_empty[st]);
      if (j + 1 == n_t[t]) umma_commit_w(&bars->o_final[t]);
    };
    issue_s(0, 0);
    issue_s(1, 0);
    issue_s(0, 1);
    issue_s(1, 1);
    for (int j = 0; j < nb; ++j) {
      for (int t = 0; t < 2; ++t) {
        if (j >= n_t[t]) continue;
        issue_pv(t, j);
        if (j + 2 < n_t[t]) issue_s(t, j + 2);
      }
    }
  } else {
    const int t = (warp - 2) >> 2;                 // query tile A (0) or B (1)
    const int quarter = warp & 3;                  // TMEM lanes 32*quarter ..
    const int r = quarter * 32 + lane;             // query row within the tile
    const int qt = 2 * pair + t, n = 2 * qt + 2;
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_base = tmem + t * 128 + lane_off, o_addr = tmem + 256 + t * 128 + lane_off;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      const uint32_t s_addr = s_base + (j & 1) * 64;
      mbar_wait(&bars->s_full[t][j & 1], (j >> 1) & 1);
      if (j == 0 && warp == 6 && lane == 0) HLM_TL(2);
      tc_fence_after();
      uint32_t sv[2][32];
      tmem_ld_32x32(s_addr, sv[0]);
      tmem_ld_32x32(s_addr + 32, sv[1]);
      tmem_ld_wait();
      if (j >= 2 * qt) {   // the two diagonal steps (warp-uniform): mask keys above the row
        const int k0 = j * 64;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (k0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
      }
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(__uint_as_float(sv[0][u]), __uint_as_float(sv[0][u + 8]));
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = (c == 0 ? 16 : 0); e < 32; e += 2)
          mx8[e & 7] = fmax3(mx8[e & 7], __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
      const float mx = scale_log2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                          fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      if (j == 0) {
        m = mx;
      } else if (__any_sync(0xffffffffu, mx > m + kRescaleLog2)) {
        // O_t holds P V of steps < j; PV_t(j-1) may still run: wait for it, then rescale.
        // S_t(j+1) was issued right behind PV_t(j-1) (in-order tensor pipe), so its s_full
        // covers it; the last step has no S_t(j+1) and waits pv_done (PV_t(n-2) only)
        if (j + 1 < n)
          mbar_wait(&bars->s_full[t][(j + 1) & 1], ((j + 1) >> 1) & 1);
        else
          mbar_wait(&bars->pv_done[t], 0);
        tc_fence_after();
        const float mn = fmaxf(m, mx);
        const float alpha = ex2(m - mn);
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t ov[16];
          tmem_ld_32x16(o_addr + c * 16, ov);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st_32x16(o_addr + c * 16, ov);
        }
        tmem_st_wait();
        l *= alpha;
        m = mn;
      }
      // P = 2^(s * scale_log2 - m) <= 2^8 as bf16 pairs into the first 32 columns of S_t[j % 2]
      const float negm = -m;
      float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float a0, a1;
          ffma2(a0, a1, __uint_as_float(sv[c][2 * e]), __uint_as_float(sv[c][2 * e + 1]), scale_log2, negm);
          float p0, p1;
          if ((e & 3) < kEmu) {
            ex2_poly2(p0, p1, a0, a1);
          } else {
            p0 = ex2(a0);
            p1 = ex2(a1);
          }
          fadd2(l8[2 * (e & 3)], l8[2 * (e & 3) + 1], p0, p1);
          pk[e] = pack_bf16x2(p0, p1);
        }
        tmem_st_32x16(s_addr + c * 16, pk);
      }
      l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full[t][j & 1]);
    }
    mbar_wait(&bars->o_final[t], 0);
    mbar_wait(&bars->pv_done[t], 0);   // its one phase (complete with o_final)
    if (warp == 6 && lane == 0) HLM_TL(3);
    tc_fence_after();
    const float il = 1.f / l;
    // O through shared memory (this tile's Q buffer: every S_t MMA has completed with o_final)
    // so the global stores are row-contiguous: a warp store straight from the TMEM layout
    // (thread = row) touches 32 rows (XOR swizzle by row: conflict-free both ways)
    const uint32_t stage = smem_u32(sQ(t));
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32(o_addr + c * 32, ov);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ch = c * 4 + q;
        st_shared_v4(stage + r * 256 + ((ch ^ (r & 7)) << 4),
                     pack_bf16x2(__uint_as_float(ov[8 * q]) * il, __uint_as_float(ov[8 * q + 1]) * il),
                     pack_bf16x2(__uint_as_float(ov[8 * q + 2]) * il, __uint_as_float(ov[8 * q + 3]) * il),
                     pack_bf16x2(__uint_as_float(ov[8 * q + 4]) * il, __uint_as_float(ov[8 * q + 5]) * il),
                     pack_bf16x2(__uint_as_float(ov[8 * q + 6]) * il, __uint_as_float(ov[8 * q + 7]) * il));
      }
    }
    lse[(long long)bh * S + qpos] = (m + log2f(l)) / kLog2e;
    asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");   // this tile's 4 warps
    __nv_bfloat16* otile = o + (long long)(row0 + qt * TQ) * ld + col0;
    const int et = quarter * 32 + lane;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int idx = i * 128 + et, row = idx >> 4, ch = idx & 15;
      uint4 w;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                   : "r"(stage + row * 256 + ((ch ^ (row & 7)) << 4)));
      *reinterpret_cast<uint4*>(otile + (long long)row * ld + ch * 8) = w;
    }
    if (warp == 6 && lane == 0) HLM_TL(4);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) HLM_TL(5);
}

// Persistent forward: one CTA per SM walks the query-tile pairs (claimed from a per-launch
// counter by the producer, as the persistent backward kernels), everything else as
// flash_fwd_pp2 per pair. The tile boundary (the timeline's forward mode: ~5 us per CTA of Q
// load, first S, O store and CTA-to-CTA gap on a 0.94 us step):
//   * O goes out through a dedicated 32 KB stage (used by A and B in turn, stage_done), so a
//     tile's Q buffer frees as soon as its last S MMA completes (q_free, committed by the MMA
//     warp) and the producer loads the next pair's Q there while the tile finishes;
//   * the next pair's first S MMAs follow this pair's last PV on the tensor pipe, under the
//     O stores;
//   * per-tile S / P buffers and their barrier parities continue across pairs (global step
//     counts); pv_done / o_final / q_full / q_free complete once per pair.
struct PP3Bars {
  uint64_t q_full[2], q_free[2], kv_full[KF_STAGES], kv_empty[KF_STAGES], s_full[2][2], p_full[2][2], pv_done[2],
      o_final[2], stage_done, tile_full[2], tile_empty[2];
  int tile_id[2];
  uint32_t tmem;
};
static_assert(sizeof(PP3Bars) <= 256, "barrier block");
constexpr int PP3_SMEM = TILE_BYTES * 2 + KF_STAGES * 2 * HALF_TILE + TILE_BYTES + 256;
static_assert(PP3_SMEM <= 227 * 1024, "shared memory");
constexpr int PP3_TILE_READERS = 9;   // the MMA warp + 8 softmax warps

template <int kEmu>
__global__ void __launch_bounds__(PP_THREADS, 1)
    flash_fwd_pp3(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k64,
                  const __grid_constant__ CUtensorMap map_v64, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                  int S, int H, int ld, float scale_log2, int order, int nbh, int* __restrict__ tile_ctr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // 1024-aligned window, no slack in PP3_SMEM; checked
  if (smem_u32(smem) & 1023) __trap();
  auto sQ = [&](int t) { return smem + t * TILE_BYTES; };
  auto sK = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE; };
  auto sV = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE + HALF_TILE; };
  const uint32_t s_out = smem_u32(smem + 2 * TILE_BYTES + KF_STAGES * 2 * HALF_TILE);
  PP3Bars* bars = reinterpret_cast<PP3Bars*>(smem + 3 * TILE_BYTES + KF_STAGES * 2 * HALF_TILE);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int npairs = S / (2 * TQ), total = npairs * nbh;
  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k64);
    tma_prefetch(&map_v64);
    for (int i = 0; i < KF_STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars->q_full[t], 1);
      mbar_init(&bars->q_free[t], 1);
      mbar_init(&bars->s_full[t][0], 1);
      mbar_init(&bars->s_full[t][1], 1);
      mbar_init(&bars->p_full[t][0], 4);
      mbar_init(&bars->p_full[t][1], 4);
      mbar_init(&bars->pv_done[t], 1);
      mbar_init(&bars->o_final[t], 1);
      mbar_init(&bars->tile_full[t], 1);
      mbar_init(&bars->tile_empty[t], PP3_TILE_READERS);
    }
    mbar_init(&bars->stage_done, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;
  auto next_tile = [&](int j) {
    const int slot = j & 1;
    mbar_wait(&bars->tile_full[slot], (j >> 1) & 1);
    const int id = *reinterpret_cast<volatile int*>(&bars->tile_id[slot]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->tile_empty[slot]);
    return id;
  };
  auto decode = [&](int id, int& pair, int& bh) {
    int rank;
    tile_decode(id, npairs, nbh, order, rank, bh);
    pair = npairs - 1 - rank;   // long (late) query tiles first
  };

  if (warp == 0) {
    // claim pair p, publish it, load its Q (each tile's buffer once that tile's last S of
    // the previous pair has completed), then stream its K / V steps through the ring
    auto claim = [&](int p) {
      int t = 0;
      if (lane == 0) {
        const int slot = p & 1;
        mbar_wait(&bars->tile_empty[slot], ((p >> 1) & 1) ^ 1);
        t = atomicAdd(tile_ctr, 1);
        if (t >= total) t = -1;
        bars->tile_id[slot] = t;
        mbar_arrive(&bars->tile_full[slot]);
      }
      return __shfl_sync(0xffffffffu, t, 0);
    };
    int g = 0;
    int id = claim(0);
    for (int p = 0; id >= 0; ++p) {
      int pair, bh;
      decode(id, pair, bh);
      const int nb = 4 * pair + 4, row0 = (bh / H) * S, col0 = (bh % H) * HD;
      if (lane == 0) {
        for (int t = 0; t < 2; ++t) {
          if (p > 0) mbar_wait(&bars->q_free[t], (p - 1) & 1);
          mbar_arrive_expect_tx(&bars->q_full[t], TILE_BYTES);
          tma_load_2d(sQ(t), &map_q, &bars->q_full[t], col0, row0 + (2 * pair + t) * TQ);
          tma_load_2d(sQ(t) + ATOM_BYTES, &map_q, &bars->q_full[t], col0 + 64, row0 + (2 * pair + t) * TQ);
        }
        for (int j = 0; j < nb; ++j) {
          const int gg = g + j, st = gg % KF_STAGES;
          const int r = row0 + j * 64;
          mbar_wait(&bars->kv_empty[st], ((gg / KF_STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars->kv_full[st], 2 * HALF_TILE);
          tma_load_2d(sK(st), &map_k64, &bars->kv_full[st], col0, r);
          tma_load_2d(sK(st) + HALF_ATOM, &map_k64, &bars->kv_full[st], col0 + 64, r);
          tma_load_2d(sV(st), &map_v64, &bars->kv_full[st], col0, r);
          tma_load_2d(sV(st) + HALF_ATOM, &map_v64, &bars->kv_full[st], col0 + 64, r);
        }
      }
      __syncwarp();
      g += nb;
      id = claim(p + 1);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    int g0 = 0, base[2] = {0, 0};
    for (int p = 0;; ++p) {
      const int id = next_tile(p);
      if (id < 0) break;
      int pair, bh;
      decode(id, pair, bh);
      const int nb = 4 * pair + 4;
      const int n_t[2] = {nb - 2, nb};
      auto issue_s = [&](int t, int j) {
        const int gg = g0 + j, st = gg % KF_STAGES, gs = base[t] + j;
        mbar_wait(&bars->kv_full[st], (gg / KF_STAGES) & 1);
        tc_fence_after();
        umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + t * 128 + (gs & 1) * 64,
                                                              kmajor_desc(smem_u32(sQ(t)), 0),
                                                              kmajor_desc64(smem_u32(sK(st)), 0), idesc_s, 0u);
        umma_commit_w(&bars->s_full[t][gs & 1]);
        if (j + 1 == n_t[t]) umma_commit_w(&bars->q_free[t]);   // Q_t read for the last time
      };
      // O_t += P_t(j) V_j, P_t(j) (bf16) in the first 32 columns of S_t[gs % 2]
      auto issue_pv = [&](int t, int j) {
        const int gg = g0 + j, st = gg % KF_STAGES, gs = base[t] + j;
        mbar_wait(&bars->p_full[t][gs & 1], (gs >> 1) & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sV(st));
        const uint32_t p_tmem = tmem + t * 128 + (gs & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ts_w(tmem + 256 + t * 128, p_tmem + kk * 8, mnmajor_desc64(v_base, kk), idesc_o,
                         (j > 0 || kk > 0) ? 1u : 0u);
        if (j + 2 == n_t[t]) umma_commit_w(&bars->pv_done[t]);   // PV_t(n-2): for a rescale at the last step
        if (t == 1) umma_commit_w(&bars->kv_empty[st]);
        if (j + 1 == n_t[t]) umma_commit_w(&bars->o_final[t]);
      };
      mbar_wait(&bars->q_full[0], p & 1);
      issue_s(0, 0);
      issue_s(0, 1);
      mbar_wait(&bars->q_full[1], p & 1);
      issue_s(1, 0);
      issue_s(1, 1);
      for (int j = 0; j < nb; ++j) {
        for (int t = 0; t < 2; ++t) {
          if (j >= n_t[t]) continue;
          issue_pv(t, j);
          if (j + 2 < n_t[t]) issue_s(t, j + 2);
        }
      }
      g0 += nb;
      base[0] += n_t[0];
      base[1] += n_t[1];
    }
  } else {
    const int t = (warp - 2) >> 2;                 // query tile A (0) or B (1)
    const int quarter = warp & 3;                  // TMEM lanes 32*quarter ..
    const int r = quarter * 32 + lane;             // query row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_base = tmem + t * 128 + lane_off, o_addr = tmem + 256 + t * 128 + lane_off;
    int base = 0;
    for (int p = 0;; ++p) {
      const int id = next_tile(p);
      if (id < 0) break;
      int pair, bh;
      decode(id, pair, bh);
      const int row0 = (bh / H) * S, col0 = (bh % H) * HD;
      const int qt = 2 * pair + t, n = 2 * qt + 2;
      const int qpos = qt * TQ + r;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        const int gs = base + j;
        const uint32_t s_addr = s_base + (gs & 1) * 64;
        mbar_wait(&bars->s_full[t][gs & 1], (gs >> 1) & 1);
        tc_fence_after();
        uint32_t sv[2][32];
        tmem_ld_32x32(s_addr, sv[0]);
        tmem_ld_32x32(s_addr + 32, sv[1]);
        tmem_ld_wait();
        if (j >= 2 * qt) {   // the two diagonal steps (warp-uniform): mask keys above the row
          const int k0 = j * 64;
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (k0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(__uint_as_float(sv[0][u]), __uint_as_float(sv[0][u + 8]));
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = (c == 0 ? 16 : 0); e < 32; e += 2)
            mx8[e & 7] = fmax3(mx8[e & 7], __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
        const float mx = scale_log2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                            fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if (j == 0) {
          m = mx;
        } else if (__any_sync(0xffffffffu, mx > m + kRescaleLog2)) {
          // O_t holds P V of steps < j; PV_t(j-1) may still run: wait for it (S_t(j+1), issued
          // behind it, or at the last step the pair's pv_done), then rescale
          if (j + 1 < n)
            mbar_wait(&bars->s_full[t][(gs + 1) & 1], ((gs + 1) >> 1) & 1);
          else
            mbar_wait(&bars->pv_done[t], p & 1);
          tc_fence_after();
          const float mn = fmaxf(m, mx);
          const float alpha = ex2(m - mn);
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t ov[16];
            tmem_ld_32x16(o_addr + c * 16, ov);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st_32x16(o_addr + c * 16, ov);
          }
          tmem_st_wait();
          l *= alpha;
          m = mn;
        }
        const float negm = -m;
        float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a0, a1;
            ffma2(a0, a1, __uint_as_float(sv[c][2 * e]), __uint_as_float(sv[c][2 * e + 1]), scale_log2, negm);
            float p0, p1;
            if ((e & 3) < kEmu) {
              ex2_poly2(p0, p1, a0, a1);
            } else {
              p0 = ex2(a0);
              p1 = ex2(a1);
            }
            fadd2(l8[2 * (e & 3)], l8[2 * (e & 3) + 1], p0, p1);
            pk[e] = pack_bf16x2(p0, p1);
          }
          tmem_st_32x16(s_addr + c * 16, pk);
        }
        l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->p_full[t][gs & 1]);
      }
      base += n;
      mbar_wait(&bars->o_final[t], p & 1);
      mbar_wait(&bars->pv_done[t], p & 1);   // this pair's phase (complete with o_final)
      tc_fence_after();
      const float il = 1.f / l;
      // the O stage goes A(0), B(0), A(1), B(1), ...: epilogue k = 2p + t waits for k - 1
      const int k = 2 * p + t;
      if (k > 0) mbar_wait(&bars->stage_done, (k - 1) & 1);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32(o_addr + c * 32, ov);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ch = c * 4 + q;
          st_shared_v4(s_out + r * 256 + ((ch ^ (r & 7)) << 4),
                       pack_bf16x2(__uint_as_float(ov[8 * q]) * il, __uint_as_float(ov[8 * q + 1]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 2]) * il, __uint_as_float(ov[8 * q + 3]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 4]) * il, __uint_as_float(ov[8 * q + 5]) * il),
                       pack_bf16x2(__uint_as_float(ov[8 * q + 6]) * il, __uint_as_float(ov[8 * q + 7]) * il));
        }
      }
      // O_t is read out: the next pair's first PV_t may overwrite it once this tile's next
      // P arrives (tc_fence_before there orders the loads above)
      lse[(long long)bh * S + qpos] = (m + log2f(l)) / kLog2e;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");   // this tile's 4 warps
      __nv_bfloat16* otile = o + (long long)(row0 + qt * TQ) * ld + col0;
      const int et = quarter * 32 + lane;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int idx = i * 128 + et, row = idx >> 4, ch = idx & 15;
        uint4 w;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(s_out + row * 256 + ((ch ^ (row & 7)) << 4)));
        *reinterpret_cast<uint4*>(otile + (long long)row * ld + ch * 8) = w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->stage_done);   // this warp's stage reads are done
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ backward
// Shared pieces: a 128-row bf16 tile written by 128 threads (thread = row) into
// the K-major SW128 layout the MMA A operand expects (two 64-column atoms).
__device__ __forceinline__ void store_row_kmajor(uint8_t* tile, int r, int c, const uint32_t (&pk)[16]) {
  // columns c*32 .. c*32+31 of row r: atom c/2, 16-byte chunks (c%2)*4 .. +3
  uint8_t* row = tile + (c >> 1) * ATOM_BYTES + r * 128;
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    const int chunk = (c & 1) * 4 + q4;
    *reinterpret_cast<uint4*>(row + ((chunk ^ (r & 7)) << 4)) =
        make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
  }
}

// 64 accumulator columns (one half) of a row: TMEM -> scaled bf16 in global memory
__device__ __forceinline__ void store_acc_half(__nv_bfloat16* dst, uint32_t taddr, float scale) {
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld_32x32(taddr + c * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 4; ++q)
      reinterpret_cast<uint4*>(dst + c * 32)[q] =
          make_uint4(pack_bf16x2(__uint_as_float(v[8 * q]) * scale, __uint_as_float(v[8 * q + 1]) * scale),
                     pack_bf16x2(__uint_as_float(v[8 * q + 2]) * scale, __uint_as_float(v[8 * q + 3]) * scale),
                     pack_bf16x2(__uint_as_float(v[8 * q + 4]) * scale, __uint_as_float(v[8 * q + 5]) * scale),
                     pack_bf16x2(__uint_as_float(v[8 * q + 6]) * scale, __uint_as_float(v[8 * q + 7]) * scale));
  }
}

// 16 columns (c16-th group of 16 along the 128) of row r of a K-major SW128 bf16 tile
__device__ __forceinline__ void store_row16_kmajor(uint8_t* tile, int r, int c16, const uint32_t (&pk)[8]) {
  uint8_t* row = tile + (c16 >> 2) * ATOM_BYTES + r * 128;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int chunk = (c16 & 3) * 2 + q;
    *reinterpret_cast<uint4*>(row + ((chunk ^ (r & 7)) << 4)) =
        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}
// 32 accumulator columns of a row: TMEM -> scaled bf16 in global memory
__device__ __forceinline__ void store_acc_32(__nv_bfloat16* dst, uint32_t taddr, float scale) {
  uint32_t v[32];
  tmem_ld_32x32(taddr, v);
  tmem_ld_wait();
#pragma unroll
  for (int q = 0; q < 4; ++q)
    reinterpret_cast<uint4*>(dst)[q] =
        make_uint4(pack_bf16x2(__uint_as_float(v[8 * q]) * scale, __uint_as_float(v[8 * q + 1]) * scale),
                   pack_bf16x2(__uint_as_float(v[8 * q + 2]) * scale, __uint_as_float(v[8 * q + 3]) * scale),
                   pack_bf16x2(__uint_as_float(v[8 * q + 4]) * scale, __uint_as_float(v[8 * q + 5]) * scale),
                   pack_bf16x2(__uint_as_float(v[8 * q + 6]) * scale, __uint_as_float(v[8 * q + 7]) * scale));
}
// dK, dV for one 128-key tile: loop over query tiles i >= kt.
//   TMEM: S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512)
//   smem: K, V (fixed), Q_i, dO_i, P^T, dS^T (bf16, K-major), lse2/D of tile i
//   Q is double-buffered (released by the dK MMA), dO single (released by the dV
//   MMA, issued first): the next Q / dO stream in under this tile's MMAs.
struct BwdKVBars {
  uint64_t kv_full, q_full[2], q_empty[2], do_full, do_empty, s_full, p_full, acc_full;
  uint32_t tmem;
};
constexpr int BWD_KV_SMEM = TILE_BYTES * 7 + 1024 + 1024 + 256;
constexpr int BWD_KV_THREADS = 640;   // 4 control warps + 16 elementwise warps (4 column quarters)

__global__ void __launch_bounds__(BWD_KV_THREADS, 1)
    flash_bwd_dkv_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                     const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dk,
                     __nv_bfloat16* __restrict__ dv, int S, int H, int ld, float scale, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sK = smem, *sV = smem + TILE_BYTES, *sdO = smem + 3 * TILE_BYTES, *sPT = smem + 4 * TILE_BYTES,
          *sdST = smem + 5 * TILE_BYTES;
  uint8_t* sQ[2] = {smem + 2 * TILE_BYTES, smem + 6 * TILE_BYTES};
  float* sL = reinterpret_cast<float*>(smem + 7 * TILE_BYTES);
  float* sD = sL + 128;
  BwdKVBars* bars = reinterpret_cast<BwdKVBars*>(smem + 7 * TILE_BYTES + 1024);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kt = (int)blockIdx.x;        // key tile (early tiles have the longest loops: launched first)
  const int nq = S / TQ;
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const int row0 = b * S, col0 = hh * HD;
  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do);
    mbar_init(&bars->kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
    }
    mbar_init(&bars->do_full, 1);
    mbar_init(&bars->do_empty, 1);
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_full, 16);
    mbar_init(&bars->acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &map_k, &bars->kv_full, col0, row0 + kt * TK);
      tma_load_2d(sK + ATOM_BYTES, &map_k, &bars->kv_full, col0 + 64, row0 + kt * TK);
      tma_load_2d(sV, &map_v, &bars->kv_full, col0, row0 + kt * TK);
      tma_load_2d(sV + ATOM_BYTES, &map_v, &bars->kv_full, col0 + 64, row0 + kt * TK);
      for (int i = kt; i < nq; ++i) {
        const int it = i - kt;
        const int qs = it & 1;
        const int r = row0 + i * TQ;
        mbar_wait(&bars->q_empty[qs], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->q_full[qs], TILE_BYTES);
        tma_load_2d(sQ[qs], &map_q, &bars->q_full[qs], col0, r);
        tma_load_2d(sQ[qs] + ATOM_BYTES, &map_q, &bars->q_full[qs], col0 + 64, r);
        mbar_wait(&bars->do_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->do_full, TILE_BYTES);
        tma_load_2d(sdO, &map_do, &bars->do_full, col0, r);
        tma_load_2d(sdO + ATOM_BYTES, &map_do, &bars->do_full, col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_kk = make_idesc_bf16(128, 128, false, false);   // A K-major, B K-major
    constexpr uint32_t idesc_kmn = make_idesc_bf16(128, 128, false, true);   // A K-major, B MN-major
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV), do_base = smem_u32(sdO),
                   pt_base = smem_u32(sPT), dst_base = smem_u32(sdST);
    mbar_wait(&bars->kv_full, 0);
    for (int i = kt; i < nq; ++i) {
      const int it = i - kt;
      const int qs = it & 1;
      const uint32_t q_base = smem_u32(sQ[qs]);
      mbar_wait(&bars->q_full[qs], (it >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem, kmajor_desc(k_base, kk), kmajor_desc(q_base, kk), idesc_kk, kk ? 1u : 0u);
      }
      __syncwarp();
      mbar_wait(&bars->do_full, it & 1);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem + 128, kmajor_desc(v_base, kk), kmajor_desc(do_base, kk), idesc_kk, kk ? 1u : 0u);
        umma_commit(&bars->s_full);
      }
      __syncwarp();
      mbar_wait(&bars->p_full, it & 1);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < TQ / 16; ++kk)
          umma_bf16(tmem + 256, kmajor_desc(pt_base, kk), mnmajor_desc(do_base, kk), idesc_kmn,
                    (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&bars->do_empty);
#pragma unroll
        for (int kk = 0; kk < TQ / 16; ++kk)
          umma_bf16(tmem + 384, kmajor_desc(dst_base, kk), mnmajor_desc(q_base, kk), idesc_kmn,
                    (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&bars->q_empty[qs]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(&bars->acc_full);
    __syncwarp();
  } else if (warp >= 4) {
    // warp w: key rows 32*(w%4).. (its TMEM lanes), query columns [32*cq, +32), cq = (w-4)/4:
    // sixteen elementwise warps, four per scheduler, two 16-column rounds each
    const int cq = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // key row within the tile
    const int key = kt * TK + r;
    const int tid = (warp - 4) * 32 + lane;        // 0..511
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float* L = lse + (long long)bh * S;
    const float* Dr = dsum + (long long)bh * S;
    for (int i = kt; i < nq; ++i) {
      const int it = i - kt;
      // lse (log2 units) and D of this query tile; the previous tile's readers are done
      asm volatile("bar.sync 1, 512;" ::: "memory");
      if (tid < 128)
        sL[tid] = -L[i * TQ + tid] * kLog2e;   // negated: exp argument is one FFMA
      else if (tid < 256)
        sD[tid - 128] = Dr[i * TQ + tid - 128];
      asm volatile("bar.sync 1, 512;" ::: "memory");
      mbar_wait(&bars->s_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        const int c16 = cq * 2 + h2;               // 16-column group of the 128 query columns
        uint32_t sv[16], dpv[16];
        tmem_ld_32x16(tmem + c16 * 16 + lane_off, sv);
        tmem_ld_32x16(tmem + 128 + c16 * 16 + lane_off, dpv);
        tmem_ld_wait();
        uint32_t pk[8], dk8[8];
        const float4* L4 = reinterpret_cast<const float4*>(sL + c16 * 16);
        const float4* D4 = reinterpret_cast<const float4*>(sD + c16 * 16);
        auto body = [&](auto diag_tag) {
          constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const float4 lv = L4[e4], dv4 = D4[e4];
            const float ln[4] = {lv.x, lv.y, lv.z, lv.w}, dn[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
            float p[4], ds[4];
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              const int e = e4 * 4 + u;
              float x0, x1;
              fma2v(x0, x1, __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]), scale_log2, scale_log2, ln[u],
                    ln[u + 1]);
              float p0 = ex2(x0), p1 = ex2(x1);
              if (kDiag && r > c16 * 16 + e) p0 = 0.f;
              if (kDiag && r > c16 * 16 + e + 1) p1 = 0.f;
              p[u] = p0;
              p[u + 1] = p1;
              submul2(ds[u], ds[u + 1], __uint_as_float(dpv[e]), __uint_as_float(dpv[e + 1]), dn[u], dn[u + 1], p0,
                      p1);
            }
            pk[e4 * 2] = pack_bf16x2(p[0], p[1]);
            pk[e4 * 2 + 1] = pack_bf16x2(p[2], p[3]);
            dk8[e4 * 2] = pack_bf16x2(ds[0], ds[1]);
            dk8[e4 * 2 + 1] = pack_bf16x2(ds[2], ds[3]);
          }
        };
        if (i == kt)
          body(std::true_type{});
        else
          body(std::false_type{});
        store_row16_kmajor(sPT, r, c16, pk);
        store_row16_kmajor(sdST, r, c16, dk8);
      }
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full);
    }
    mbar_wait(&bars->acc_full, 0);
    tc_fence_after();
    store_acc_32(dv + (long long)(row0 + key) * ld + col0 + cq * 32, tmem + 256 + cq * 32 + lane_off, 1.0f);
    store_acc_32(dk + (long long)(row0 + key) * ld + col0 + cq * 32, tmem + 384 + cq * 32 + lane_off, scale);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// dQ for one 128-query tile: loop over key tiles j <= qt (K/V double-buffered).
//   TMEM: S [0,128) dP [128,256) dQ [256,384)
struct BwdQBars {
  uint64_t q_full, kv_full[2], kv_empty[2], s_full, ds_full, ds_free, acc_full;
  uint32_t tmem;
};
constexpr int BWD_Q_SMEM = TILE_BYTES * 7 + 1024 + 256;

__global__ void __launch_bounds__(FWD_THREADS, 1)
    flash_bwd_dq_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                    const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dq,
                    int S, int H, int ld, float scale, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem, *sdO = smem + TILE_BYTES, *sdS = smem + 6 * TILE_BYTES;
  // stage st: K at (2 + 2 st) tiles, V at (3 + 2 st) tiles
  auto sK = [&](int st) { return smem + (2 + 2 * st) * TILE_BYTES; };
  auto sV = [&](int st) { return smem + (3 + 2 * st) * TILE_BYTES; };
  BwdQBars* bars = reinterpret_cast<BwdQBars*>(smem + 7 * TILE_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = (int)(gridDim.x - 1 - blockIdx.x);
  const int bh = blockIdx.y, b = bh / H, hh = bh % H;
  const int row0 = b * S, col0 = hh * HD;
  const int n_tiles = qt + 1;
  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do);
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->ds_full, 8);
    mbar_init(&bars->ds_free, 1);
    mbar_init(&bars->acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->q_full, 2 * TILE_BYTES);
      tma_load_2d(sQ, &map_q, &bars->q_full, col0, row0 + qt * TQ);
      tma_load_2d(sQ + ATOM_BYTES, &map_q, &bars->q_full, col0 + 64, row0 + qt * TQ);
      tma_load_2d(sdO, &map_do, &bars->q_full, col0, row0 + qt * TQ);
      tma_load_2d(sdO + ATOM_BYTES, &map_do, &bars->q_full, col0 + 64, row0 + qt * TQ);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        mbar_wait(&bars->kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[st], 2 * TILE_BYTES);
        const int r = row0 + j * TK;
        tma_load_2d(sK(st), &map_k, &bars->kv_full[st], col0, r);
        tma_load_2d(sK(st) + ATOM_BYTES, &map_k, &bars->kv_full[st], col0 + 64, r);
        tma_load_2d(sV(st), &map_v, &bars->kv_full[st], col0, r);
        tma_load_2d(sV(st) + ATOM_BYTES, &map_v, &bars->kv_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_kk = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_kmn = make_idesc_bf16(128, 128, false, true);
    const uint32_t q_base = smem_u32(sQ), do_base = smem_u32(sdO), ds_base = smem_u32(sdS);
    // S_j, dP_j into TMEM [0,256)
    auto issue_sdp = [&](int j) {
      const int st = j & 1;
      mbar_wait(&bars->kv_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_base = smem_u32(sK(st)), v_base = smem_u32(sV(st));
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem, kmajor_desc(q_base, kk), kmajor_desc(k_base, kk), idesc_kk, kk ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem + 128, kmajor_desc(do_base, kk), kmajor_desc(v_base, kk), idesc_kk, kk ? 1u : 0u);
        umma_commit(&bars->s_full);
      }
      __syncwarp();
    };
    mbar_wait(&bars->q_full, 0);
    issue_sdp(0);
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      mbar_wait(&bars->ds_full, j & 1);
      // S / dP of the next key tile first (the elementwise warps are done reading TMEM),
      // so they compute under this tile's dQ MMA; dS_j's smem is released by ds_free
      if (j + 1 < n_tiles) issue_sdp(j + 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_base = smem_u32(sK(st));
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)
          umma_bf16(tmem + 256, kmajor_desc(ds_base, kk), mnmajor_desc(k_base, kk), idesc_kmn,
                    (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&bars->kv_empty[st]);
        umma_commit(&bars->ds_free);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(&bars->acc_full);
    __syncwarp();
  } else if (warp >= 4) {
    // warp w: query rows 32*(w%4).. (its TMEM lanes), key columns [64*half, +64)
    const int half = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // query row within the tile
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float neg_l2 = -lse[(long long)bh * S + qpos] * kLog2e;
    const float D = dsum[(long long)bh * S + qpos];
    for (int j = 0; j < n_tiles; ++j) {
      const bool diag = j == qt;
      mbar_wait(&bars->s_full, j & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        const int c = half * 2 + h2;
        uint32_t sv[32], dpv[32];
        tmem_ld_32x32(tmem + c * 32 + lane_off, sv);
        tmem_ld_32x32(tmem + 128 + c * 32 + lane_off, dpv);
        tmem_ld_wait();
        uint32_t pk[16];
        auto body = [&](auto diag_tag) {
          constexpr bool kDiag = decltype(diag_tag)::value;
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float ds[2], x0, x1;
            fma2v(x0, x1, __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]), scale_log2, scale_log2, neg_l2, neg_l2);
            float p0 = ex2(x0), p1 = ex2(x1);
            if (kDiag && c * 32 + e > r) p0 = 0.f;
            if (kDiag && c * 32 + e + 1 > r) p1 = 0.f;
            submul2(ds[0], ds[1], __uint_as_float(dpv[e]), __uint_as_float(dpv[e + 1]), D, D, p0, p1);
            pk[e / 2] = pack_bf16x2(ds[0], ds[1]);
          }
        };
        if (diag)   // warp-uniform: only the diagonal tile masks
          body(std::true_type{});
        else
          body(std::false_type{});
        if (h2 == 0 && j > 0) mbar_wait(&bars->ds_free, (j - 1) & 1);   // dQ_{j-1} has read dS
        store_row_kmajor(sdS, r, c, pk);
      }
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->ds_full);
    }
    mbar_wait(&bars->acc_full, 0);
    tc_fence_after();
    store_acc_half(dq + (long long)(row0 + qpos) * ld + col0 + half * 64, tmem + 256 + half * 64 + lane_off, scale);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ backward, 64-wide steps
// The two kernels above hold one S / dP pair in TMEM, so the tensor core idles while the
// elementwise warps turn S, dP into P, dS. These step over the inner sequence dimension 64
// at a time: S and dP of a step take 64 TMEM columns each and are double-buffered, so the
// MMAs of step i+1 (and the accumulating MMAs of step i-1) run under the elementwise work
// of step i. The elementwise warps copy S / dP into registers and release the TMEM buffer
// before computing. Same per-element arithmetic as the 128-wide kernels.
// K-major descriptor of a 128-row x 64-column bf16 tile (one swizzle atom column), K step kk < 4
__device__ __forceinline__ uint64_t kmajor_desc_narrow(uint32_t base, int kk) {
  return make_sw128_desc(base + kk * 32, 16, 1024);
}
// 16 bf16 columns (group c16 < 4) of row r of a 128 x 64 K-major SW128 tile
__device__ __forceinline__ void store_row16_narrow(uint8_t* tile, int r, int c16, const uint32_t (&pk)[8]) {
  uint8_t* row = tile + r * 128;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int chunk = c16 * 2 + q;
    *reinterpret_cast<uint4*>(row + ((chunk ^ (r & 7)) << 4)) =
        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}


// P, dS of 16 (row, column) scores held by one thread, the reference backward's
// dS = P (dP - D) (kernels.hpp:269-299), P from the forward's log-sum-exp.
//   nl[e] = -lse * log2(e) of column e; dn[e] = D of column e (row sums for dQ, column
//   values for dK/dV); masked entries (kDiag, e >= keep) get P = 0.
template <bool kDiag>
__device__ __forceinline__ void p_ds_16(const uint32_t (&sv)[16], const uint32_t (&dpv)[16], const float (&nl)[16],
                                        const float (&dn)[16], float scale_log2, int keep_from, bool mask_below,
                                        uint32_t (&pk)[8], uint32_t (&dk8)[8]) {
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float x0, x1, d0, d1;
    fma2v(x0, x1, __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]), scale_log2, scale_log2, nl[e], nl[e + 1]);
    float p0 = ex2(x0), p1 = ex2(x1);
    if (kDiag) {
      // dK/dV (mask_below): column e is masked when e < keep_from; dQ: when e > keep_from
      if (mask_below ? (e < keep_from) : (e > keep_from)) p0 = 0.f;
      if (mask_below ? (e + 1 < keep_from) : (e + 1 > keep_from)) p1 = 0.f;
    }
    submul2(d0, d1, __uint_as_float(dpv[e]), __uint_as_float(dpv[e + 1]), dn[e], dn[e + 1], p0, p1);
    pk[e / 2] = pack_bf16x2(p0, p1);
    dk8[e / 2] = pack_bf16x2(d0, d1);
  }
}

// dK, dV for one 128-key tile, 64 queries per step.
//   TMEM: S^T[2] [0,128) (64 each), dP^T[2] [128,256), dV [256,384), dK [384,512)
//   P^T and dS^T (bf16) are written back over S^T[b] / dP^T[b] and feed dV / dK as
//   A operands from TMEM: the tensor core reads only Q and dO from shared memory (the
//   shared-memory operand traffic of the 64-wide steps bounded the previous version).
//   Warp cq turns its 16 query columns of S^T / dP^T into 8 packed columns at the same
//   offset (16 cq), so the dV / dK MMA of K step kk reads its A at column 16 kk.
//   smem: K, V (fixed); a ring of KV2_STAGES stages, each Q|dO (64 rows) plus that step's
//   log-sum-exp and D (bulk-copied beside them, read as broadcasts).
//   MMA order: S0 dP0 S1 dP1 | dV0 dK0 S2 dP2 | dV1 dK1 S3 dP3 | ...; S(i+2) reuses the
//   buffers of step i behind dV(i) / dK(i) (in-order tensor pipe).
constexpr int KV2_STAGES = 4;
struct BwdKV2Bars {
  uint64_t kv_full, q_full[KV2_STAGES], q_empty[KV2_STAGES], s_full[2], p_full[2], acc_full;
  uint32_t tmem;
};
constexpr int KV2_LD_BYTES = 2 * 64 * 4;   // per stage: lse[64], D[64]
constexpr int BWD_KV2_SMEM = TILE_BYTES * 2 + KV2_STAGES * 2 * HALF_TILE + KV2_STAGES * KV2_LD_BYTES + 1024 + 256;
constexpr int BWD_KV2_THREADS = 640;   // 4 control warps + 16 elementwise warps

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// 16 bf16 columns (group c16 < 4) of row r of a 128 x 64 K-major SW128 tile at shared address `tile`
__device__ __forceinline__ void st_row16_narrow(uint32_t tile, int r, int c16, const uint32_t (&pk)[8]) {
  const uint32_t row = tile + r * 128;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int chunk = c16 * 2 + q;
    st_shared_v4(row + ((chunk ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}

// kExp (timing experiments only, results invalid when != 0): 1 skips the elementwise math,
// 2 also skips the S / dP TMEM loads (HLM_ATTN_BWD_EXPERIMENT)
template <int kExp>
__global__ void __launch_bounds__(BWD_KV2_THREADS, 1)
    flash_bwd_dkv_tc2(const __grid_constant__ CUtensorMap map_q64, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do64,
                      const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dk,
                      __nv_bfloat16* __restrict__ dv, int S, int H, int ld, float scale, float scale_log2,
                      int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sK = smem, *sV = smem + TILE_BYTES;
  auto sQ = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE; };
  auto sdO = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE + HALF_TILE; };
  float* sLD = reinterpret_cast<float*>(smem + 2 * TILE_BYTES + KV2_STAGES * 2 * HALF_TILE);   // [stage][lse|D]
  BwdKV2Bars* bars = reinterpret_cast<BwdKV2Bars*>(reinterpret_cast<uint8_t*>(sLD) + KV2_STAGES * KV2_LD_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int kt, bh;
  tile_order(order, kt, bh);             // key tile (early tiles have the longest loops: launched first)
  const int i0 = 2 * kt, n = S / 64 - i0;   // query steps i0 .. S/64 - 1
  const int b = bh / H, hh = bh % H;
  const int row0 = b * S, col0 = hh * HD;
  if (threadIdx.x == 0) {
    HLM_TL(0);
    {
      unsigned smid_v;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_v));
      (void)smid_v;
      HLM_TL_VAL(6, smid_v);
      HLM_TL_VAL(7, n);
    }
    tma_prefetch(&map_q64);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do64);
    mbar_init(&bars->kv_full, 1);
    for (int i = 0; i < KV2_STAGES; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 16);
    }
    mbar_init(&bars->acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &map_k, &bars->kv_full, col0, row0 + kt * TK);
      tma_load_2d(sK + ATOM_BYTES, &map_k, &bars->kv_full, col0 + 64, row0 + kt * TK);
      tma_load_2d(sV, &map_v, &bars->kv_full, col0, row0 + kt * TK);
      tma_load_2d(sV + ATOM_BYTES, &map_v, &bars->kv_full, col0 + 64, row0 + kt * TK);
      const float* L = lse + (long long)bh * S;
      const float* Dr = dsum + (long long)bh * S;
      for (int it = 0; it < n; ++it) {
        const int st = it % KV2_STAGES, ph = (it / KV2_STAGES) & 1;
        const int q0 = (i0 + it) * 64;
        mbar_wait(&bars->q_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&bars->q_full[st], 2 * HALF_TILE + KV2_LD_BYTES);
        tma_load_2d(sQ(st), &map_q64, &bars->q_full[st], col0, row0 + q0);
        tma_load_2d(sQ(st) + HALF_ATOM, &map_q64, &bars->q_full[st], col0 + 64, row0 + q0);
        tma_load_2d(sdO(st), &map_do64, &bars->q_full[st], col0, row0 + q0);
        tma_load_2d(sdO(st) + HALF_ATOM, &map_do64, &bars->q_full[st], col0 + 64, row0 + q0);
        bulk_load(sLD + st * 128, L + q0, 256, &bars->q_full[st]);
        bulk_load(sLD + st * 128 + 64, Dr + q0, 256, &bars->q_full[st]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);    // S^T, dP^T: N = 64 queries
    constexpr uint32_t idesc_acc = make_idesc_bf16(128, 128, false, true);  // dV, dK: B MN-major
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
    mbar_wait(&bars->kv_full, 0);
    if (lane == 0) HLM_TL(1);
    auto issue_sdp = [&](int it) {
      const int st = it % KV2_STAGES, bb = it & 1;
      mbar_wait(&bars->q_full[st], (it / KV2_STAGES) & 1);
      tc_fence_after();
      const uint32_t q_base = smem_u32(sQ(st)), do_base = smem_u32(sdO(st));
      umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + bb * 64, kmajor_desc(k_base, 0),
                                                            kmajor_desc64(q_base, 0), idesc_s, 0u);
      umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + 128 + bb * 64, kmajor_desc(v_base, 0),
                                                            kmajor_desc64(do_base, 0), idesc_s, 0u);
      umma_commit_w(&bars->s_full[bb]);
    };
    issue_sdp(0);
    if (n > 1) issue_sdp(1);
    for (int it = 0; it < n; ++it) {
      const int st = it % KV2_STAGES, bb = it & 1;
      mbar_wait(&bars->p_full[bb], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t q_base = smem_u32(sQ(st)), do_base = smem_u32(sdO(st));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_ts_w(tmem + 256, tmem + bb * 64 + 16 * kk, mnmajor_desc64(do_base, kk), idesc_acc,
                       (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_ts_w(tmem + 384, tmem + 128 + bb * 64 + 16 * kk, mnmajor_desc64(q_base, kk), idesc_acc,
                       (it > 0 || kk > 0) ? 1u : 0u);
      umma_commit_w(&bars->q_empty[st]);
      if (it + 2 < n) issue_sdp(it + 2);
    }
    umma_commit_w(&bars->acc_full);
  } else if (warp >= 4) {
    // warp w: key rows 32*(w%4).. (its TMEM lanes), query columns [16*cq, +16) of each step
    const int cq = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // key row within the tile
    const int key = kt * TK + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t ld_base = smem_u32(sLD) + cq * 64;   // this warp's 16 columns of lse / D
    for (int it = 0; it < n; ++it) {
      const int bb = it & 1, st = it % KV2_STAGES;
      const int q0 = (i0 + it) * 64 + cq * 16;     // first query column of this thread's 16
      mbar_wait(&bars->s_full[bb], (it >> 1) & 1);
      if (it == 0 && warp == 4 && lane == 0) HLM_TL(2);
      tc_fence_after();
      uint32_t sv[16], dpv[16];
      if (kExp < 2) {
        tmem_ld_32x16(tmem + bb * 64 + cq * 16 + lane_off, sv);
        tmem_ld_32x16(tmem + 128 + bb * 64 + cq * 16 + lane_off, dpv);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) sv[e] = dpv[e] = (uint32_t)e;
      }
      mbar_wait(&bars->q_full[st], (it / KV2_STAGES) & 1);   // lse / D landed with this step's Q
      float nl[16], dn[16];
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        const float4 lv = ld_shared_f4(ld_base + st * KV2_LD_BYTES + e4 * 16);
        const float4 dv4 = ld_shared_f4(ld_base + st * KV2_LD_BYTES + 256 + e4 * 16);
        nl[4 * e4] = -lv.x * kLog2e;
        nl[4 * e4 + 1] = -lv.y * kLog2e;
        nl[4 * e4 + 2] = -lv.z * kLog2e;
        nl[4 * e4 + 3] = -lv.w * kLog2e;
        dn[4 * e4] = dv4.x;
        dn[4 * e4 + 1] = dv4.y;
        dn[4 * e4 + 2] = dv4.z;
        dn[4 * e4 + 3] = dv4.w;
      }
      tmem_ld_wait();
      uint32_t pk[8], dk8[8];
      // causal: P = 0 where key > query, i.e. column e < key - q0
      if (kExp >= 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) pk[e] = dk8[e] = sv[e] ^ dpv[e + 8] ^ __float_as_uint(nl[e] + dn[e]);
      } else if (q0 < kt * TK + TK)   // warp-uniform: only the two diagonal steps mask
        p_ds_16<true>(sv, dpv, nl, dn, scale_log2, key - q0, true, pk, dk8);
      else
        p_ds_16<false>(sv, dpv, nl, dn, scale_log2, 0, true, pk, dk8);
      // P^T / dS^T over the columns this warp just read (A operands of dV / dK)
      tmem_st_32x8(tmem + bb * 64 + cq * 16 + lane_off, pk);
      tmem_st_32x8(tmem + 128 + bb * 64 + cq * 16 + lane_off, dk8);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full[bb]);
      if (it == n - 1 && warp == 4 && lane == 0) HLM_TL(3);
    }
    mbar_wait(&bars->acc_full, 0);
    if (warp == 4 && lane == 0) HLM_TL(4);
    tc_fence_after();
    store_acc_32(dv + (long long)(row0 + key) * ld + col0 + cq * 32, tmem + 256 + cq * 32 + lane_off, 1.0f);
    store_acc_32(dk + (long long)(row0 + key) * ld + col0 + cq * 32, tmem + 384 + cq * 32 + lane_off, scale);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) HLM_TL(5);
}

// One 128 x 128 fp32 accumulator (TMEM) -> bf16 rows of a global tile, through a 32 KB
// shared-memory stage so the global stores are row-contiguous (each warp instruction writes two
// full 256-byte rows; storing straight from the TMEM layout, thread = row, made every warp
// instruction touch 32 rows: 4.45 us per tile for dK + dV at C2). Called by all 16 elementwise
// warps (named barrier 1): thread (quarter, cq, lane) owns row 32 quarter + lane, columns
// 32 cq .. +32 at `taddr`; `et` = 0..511 is its index among the 512 threads. The stage is
// XOR-swizzled by row (16-byte chunk c of row r at c ^ (r & 7)): conflict-free both ways.
__device__ __forceinline__ void store_acc_staged(__nv_bfloat16* tile, int ld, uint32_t taddr, float scale,
                                                 uint32_t stage, int r, int cq, int et) {
  uint32_t v[32];
  tmem_ld_32x32(taddr, v);
  tmem_ld_wait();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = cq * 4 + q;
    st_shared_v4(stage + r * 256 + ((c ^ (r & 7)) << 4),
                 pack_bf16x2(__uint_as_float(v[8 * q]) * scale, __uint_as_float(v[8 * q + 1]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 2]) * scale, __uint_as_float(v[8 * q + 3]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 4]) * scale, __uint_as_float(v[8 * q + 5]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 6]) * scale, __uint_as_float(v[8 * q + 7]) * scale));
  }
  asm volatile("bar.sync 1, 512;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = i * 512 + et, row = idx >> 4, c = idx & 15;
    uint4 w;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(stage + row * 256 + ((c ^ (row & 7)) << 4)));
    *reinterpret_cast<uint4*>(tile + (long long)row * ld + c * 8) = w;
  }
  asm volatile("bar.sync 1, 512;" ::: "memory");   // the stage is free again
}

// The same 128 x 128 accumulator -> bf16 tile, written by TMA from the 32 KB stage laid out as
// the store map's two 128 x 64 SW128 boxes: the warps only move TMEM -> shared memory, the
// copy engine writes global memory while they go on. The stage is reused after the previous
// store has read it (the issuing thread, et == 0, waits for that before the first barrier);
// the caller waits for all stores (bulk_wait0 by et == 0) before the CTA exits.
__device__ __forceinline__ void store_acc_tma(const CUtensorMap* map, int c0, int r0, uint32_t taddr, float scale,
                                              uint32_t stage, int r, int cq, int et) {
  uint32_t v[32];
  tmem_ld_32x32(taddr, v);
  if (et == 0) bulk_wait_read0();
  asm volatile("bar.sync 1, 512;" ::: "memory");
  tmem_ld_wait();
  const uint32_t row = stage + (cq >> 1) * ATOM_BYTES + r * 128;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int chunk = (cq & 1) * 4 + q;
    st_shared_v4(row + ((chunk ^ (r & 7)) << 4),
                 pack_bf16x2(__uint_as_float(v[8 * q]) * scale, __uint_as_float(v[8 * q + 1]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 2]) * scale, __uint_as_float(v[8 * q + 3]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 4]) * scale, __uint_as_float(v[8 * q + 5]) * scale),
                 pack_bf16x2(__uint_as_float(v[8 * q + 6]) * scale, __uint_as_float(v[8 * q + 7]) * scale));
  }
  fence_proxy_async();
  asm volatile("bar.sync 1, 512;" ::: "memory");
  if (et == 0) {
    tma_store_2d(map, stage, c0, r0);
    tma_store_2d(map, stage + ATOM_BYTES, c0 + 64, r0);
    bulk_commit();
  }
}

// Persistent dK / dV: one CTA per SM walks the 128-key tiles (fetched from a global counter,
// so the causal lengths balance dynamically) with the TMEM allocation, barriers and the Q|dO
// ring kept across tiles. Per tile the work is flash_bwd_dkv_tc2's; what changes is the tile
// boundary (tools/attn_timeline.cu measured ~7.8 us per CTA of prologue, epilogue and
// CTA-to-CTA gap at C2 on a 0.8 us step, a third of the kernel):
//   * the next tile's K / V load as soon as the MMA warp has issued this tile's last S / dP
//     (kv_empty), i.e. under its last two dV / dK steps;
//   * the next tile's first S / dP run on the tensor core while the elementwise warps store
//     this tile's dK / dV (their P / dS hand-off for the next tile doubles as the signal that
//     the accumulators are free);
//   * no CTA launch / teardown between tiles.
// Tile ids go through a 2-slot ring in shared memory written by the producer warp (which
// claims them) and read by the MMA warp and the 16 elementwise warps (tile_empty counts 17).
struct BwdKV3Bars {
  uint64_t kv_full, kv_empty, q_full[KV2_STAGES], q_empty[KV2_STAGES], s_full[2], p_full[2], acc_full;
  uint64_t tile_full[2], tile_empty[2];
  int tile_id[2];
  uint32_t tmem;
};
constexpr int KV3_TILE_READERS = 17;   // the MMA warp + 16 elementwise warps
static_assert(sizeof(BwdKV3Bars) <= 256, "barrier block");
constexpr int BWD_KV3_SMEM = TILE_BYTES * 2 + KV2_STAGES * 2 * HALF_TILE + TILE_BYTES + KV2_STAGES * KV2_LD_BYTES + 256;
static_assert(BWD_KV3_SMEM <= 227 * 1024, "shared memory");

__global__ void __launch_bounds__(BWD_KV2_THREADS, 1)
    flash_bwd_dkv_tc3(const __grid_constant__ CUtensorMap map_q64, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do64,
                      const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dk,
                      __nv_bfloat16* __restrict__ dv, int S, int H, int ld, float scale, float scale_log2,
                      int order, int nbh, int* __restrict__ tile_ctr, const __grid_constant__ CUtensorMap map_dk,
                      const __grid_constant__ CUtensorMap map_dv, int tma_out) {
  // no alignment slack in BWD_KV3_SMEM (the 32 KB store stage needs it): the dynamic
  // shared-memory window starts 1024-aligned (no static shared memory here); checked
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem) & 1023) __trap();
  uint8_t *sK = smem, *sV = smem + TILE_BYTES;
  auto sQ = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE; };
  auto sdO = [&](int st) { return smem + 2 * TILE_BYTES + st * 2 * HALF_TILE + HALF_TILE; };
  const uint32_t s_out = smem_u32(smem + 2 * TILE_BYTES + KV2_STAGES * 2 * HALF_TILE);   // 32 KB store stage
  float* sLD = reinterpret_cast<float*>(smem + 2 * TILE_BYTES + KV2_STAGES * 2 * HALF_TILE + TILE_BYTES);
  BwdKV3Bars* bars = reinterpret_cast<BwdKV3Bars*>(reinterpret_cast<uint8_t*>(sLD) + KV2_STAGES * KV2_LD_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = S / TK, total = nt * nbh;
  if (threadIdx.x == 0) {
    tma_prefetch(&map_q64);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do64);
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < KV2_STAGES; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 16);
      mbar_init(&bars->tile_full[i], 1);
      mbar_init(&bars->tile_empty[i], KV3_TILE_READERS);
    }
    mbar_init(&bars->acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;
  // j-th tile of this CTA (-1: none left); the caller's lane 0 releases the slot
  auto next_tile = [&](int j) {
    const int slot = j & 1;
    mbar_wait(&bars->tile_full[slot], (j >> 1) & 1);
    const int id = *reinterpret_cast<volatile int*>(&bars->tile_id[slot]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->tile_empty[slot]);
    return id;
  };

  // the producer claims tile j (global counter) and publishes it to the readers; it claims
  // the next tile only once this one's loads are issued, so a CTA holds at most the ring's
  // depth of work in reserve (a whole claimed tile in reserve left long tiles waiting behind
  // long tiles at the end of the grid)
  auto claim = [&](int j) {
    int t = 0;
    if (lane == 0) {
      const int slot = j & 1;
      mbar_wait(&bars->tile_empty[slot], ((j >> 1) & 1) ^ 1);
      t = atomicAdd(tile_ctr, 1);
      if (t >= total) t = -1;
      bars->tile_id[slot] = t;
      mbar_arrive(&bars->tile_full[slot]);
    }
    return __shfl_sync(0xffffffffu, t, 0);
  };

  if (warp == 0) {
    int g = 0;
    int id = claim(0);
    for (int j = 0; id >= 0; ++j) {
      int kt, bh;
      tile_decode(id, nt, nbh, order, kt, bh);
      const int i0 = 2 * kt, n = S / 64 - i0;
      const int b = bh / H, hh = bh % H, row0 = b * S, col0 = hh * HD;
      if (lane == 0) {
        if (j > 0) mbar_wait(&bars->kv_empty, (j - 1) & 1);   // the last tile's S / dP are done with K / V
        mbar_arrive_expect_tx(&bars->kv_full, 2 * TILE_BYTES);
        tma_load_2d(sK, &map_k, &bars->kv_full, col0, row0 + kt * TK);
        tma_load_2d(sK + ATOM_BYTES, &map_k, &bars->kv_full, col0 + 64, row0 + kt * TK);
        tma_load_2d(sV, &map_v, &bars->kv_full, col0, row0 + kt * TK);
        tma_load_2d(sV + ATOM_BYTES, &map_v, &bars->kv_full, col0 + 64, row0 + kt * TK);
        const float* L = lse + (long long)bh * S;
        const float* Dr = dsum + (long long)bh * S;
        for (int it = 0; it < n; ++it) {
          const int gg = g + it, st = gg % KV2_STAGES, ph = (gg / KV2_STAGES) & 1;
          const int q0 = (i0 + it) * 64;
          mbar_wait(&bars->q_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&bars->q_full[st], 2 * HALF_TILE + KV2_LD_BYTES);
          tma_load_2d(sQ(st), &map_q64, &bars->q_full[st], col0, row0 + q0);
          tma_load_2d(sQ(st) + HALF_ATOM, &map_q64, &bars->q_full[st], col0 + 64, row0 + q0);
          tma_load_2d(sdO(st), &map_do64, &bars->q_full[st], col0, row0 + q0);
          tma_load_2d(sdO(st) + HALF_ATOM, &map_do64, &bars->q_full[st], col0 + 64, row0 + q0);
          bulk_load(sLD + st * 128, L + q0, 256, &bars->q_full[st]);
          bulk_load(sLD + st * 128 + 64, Dr + q0, 256, &bars->q_full[st]);
        }
      }
      __syncwarp();
      g += n;
      id = claim(j + 1);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);    // S^T, dP^T: N = 64 queries
    constexpr uint32_t idesc_acc = make_idesc_bf16(128, 128, false, true);  // dV, dK: B MN-major
    const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
    int g0 = 0;
    for (int j = 0;; ++j) {
      const int id = next_tile(j);
      if (id < 0) break;
      int kt, bh;
      tile_decode(id, nt, nbh, order, kt, bh);
      const int n = S / 64 - 2 * kt;
      mbar_wait(&bars->kv_full, j & 1);
      tc_fence_after();
      auto issue_sdp = [&](int it) {
        const int gg = g0 + it, st = gg % KV2_STAGES, bb = gg & 1;
        mbar_wait(&bars->q_full[st], (gg / KV2_STAGES) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ(st)), do_base = smem_u32(sdO(st));
        umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + bb * 64, kmajor_desc(k_base, 0),
                                                              kmajor_desc64(q_base, 0), idesc_s, 0u);
        umma_chain_w<8, ATOM_BYTES / 16, 2, HALF_ATOM / 16, 2>(tmem + 128 + bb * 64, kmajor_desc(v_base, 0),
                                                              kmajor_desc64(do_base, 0), idesc_s, 0u);
        umma_commit_w(&bars->s_full[bb]);
        if (it == n - 1) umma_commit_w(&bars->kv_empty);   // K / V free for the next tile
      };
      issue_sdp(0);
      issue_sdp(1);   // n >= 2
      for (int it = 0; it < n; ++it) {
        const int gg = g0 + it, st = gg % KV2_STAGES, bb = gg & 1;
        mbar_wait(&bars->p_full[bb], (gg >> 1) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ(st)), do_base = smem_u32(sdO(st));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ts_w(tmem + 256, tmem + bb * 64 + 16 * kk, mnmajor_desc64(do_base, kk), idesc_acc,
                         (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ts_w(tmem + 384, tmem + 128 + bb * 64 + 16 * kk, mnmajor_desc64(q_base, kk), idesc_acc,
                         (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit_w(&bars->q_empty[st]);
        if (it + 2 < n) issue_sdp(it + 2);
      }
      umma_commit_w(&bars->acc_full);
      g0 += n;
    }
  } else if (warp >= 4) {
    // warp w: key rows 32*(w%4).. (its TMEM lanes), query columns [16*cq, +16) of each step
    const int cq = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // key row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t ld_base = smem_u32(sLD) + cq * 64;   // this warp's 16 columns of lse / D
    int g0 = 0;
    for (int j = 0;; ++j) {
      const int id = next_tile(j);
      if (id < 0) break;
      int kt, bh;
      tile_decode(id, nt, nbh, order, kt, bh);
      const int i0 = 2 * kt, n = S / 64 - i0;
      const int b = bh / H, hh = bh % H, row0 = b * S, col0 = hh * HD;
      const int key = kt * TK + r;
      const bool stamp = warp == 4 && lane == 0;
      if (stamp) {
        HLM_TL_AT(id, 0);
        unsigned smid_v;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_v));
        (void)smid_v;
        HLM_TL_AT_VAL(id, 6, smid_v);
        HLM_TL_AT_VAL(id, 7, n);
      }
      for (int it = 0; it < n; ++it) {
        const int gg = g0 + it, bb = gg & 1, st = gg % KV2_STAGES;
        const int q0 = (i0 + it) * 64 + cq * 16;     // first query column of this thread's 16
        mbar_wait(&bars->s_full[bb], (gg >> 1) & 1);
        if (stamp && it == 0) HLM_TL_AT(id, 1);
        tc_fence_after();
        uint32_t sv[16], dpv[16];
        tmem_ld_32x16(tmem + bb * 64 + cq * 16 + lane_off, sv);
        tmem_ld_32x16(tmem + 128 + bb * 64 + cq * 16 + lane_off, dpv);
        mbar_wait(&bars->q_full[st], (gg / KV2_STAGES) & 1);   // lse / D landed with this step's Q
        float nl[16], dn[16];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const float4 lv = ld_shared_f4(ld_base + st * KV2_LD_BYTES + e4 * 16);
          const float4 dv4 = ld_shared_f4(ld_base + st * KV2_LD_BYTES + 256 + e4 * 16);
          nl[4 * e4] = -lv.x * kLog2e;
          nl[4 * e4 + 1] = -lv.y * kLog2e;
          nl[4 * e4 + 2] = -lv.z * kLog2e;
          nl[4 * e4 + 3] = -lv.w * kLog2e;
          dn[4 * e4] = dv4.x;
          dn[4 * e4 + 1] = dv4.y;
          dn[4 * e4 + 2] = dv4.z;
          dn[4 * e4 + 3] = dv4.w;
        }
        tmem_ld_wait();
        uint32_t pk[8], dk8[8];
        // causal: P = 0 where key > query, i.e. column e < key - q0
        if (q0 < kt * TK + TK)   // warp-uniform: only the two diagonal steps mask
          p_ds_16<true>(sv, dpv, nl, dn, scale_log2, key - q0, true, pk, dk8);
        else
          p_ds_16<false>(sv, dpv, nl, dn, scale_log2, 0, true, pk, dk8);
        tmem_st_32x8(tmem + bb * 64 + cq * 16 + lane_off, pk);
        tmem_st_32x8(tmem + 128 + bb * 64 + cq * 16 + lane_off, dk8);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->p_full[bb]);
        if (stamp && it == n - 1) HLM_TL_AT(id, 2);
      }
      mbar_wait(&bars->acc_full, j & 1);
      if (stamp) HLM_TL_AT(id, 3);
      tc_fence_after();
      const int et = (warp - 4) * 32 + lane;
      const long long tile_off = (long long)(row0 + kt * TK) * ld + col0;
      if (tma_out) {
        store_acc_tma(&map_dv, col0, row0 + kt * TK, tmem + 256 + cq * 32 + lane_off, 1.0f, s_out, r, cq, et);
        store_acc_tma(&map_dk, col0, row0 + kt * TK, tmem + 384 + cq * 32 + lane_off, scale, s_out, r, cq, et);
      } else {
        store_acc_staged(dv + tile_off, ld, tmem + 256 + cq * 32 + lane_off, 1.0f, s_out, r, cq, et);
        store_acc_staged(dk + tile_off, ld, tmem + 384 + cq * 32 + lane_off, scale, s_out, r, cq, et);
      }
      if (stamp) HLM_TL_AT(id, 4);
      // the tcgen05.ld above completed (store_acc_32 waits); the next tile's first P / dS
      // arrive (after tc_fence_before) is what lets the MMA warp overwrite dV / dK
      g0 += n;
    }
  }
  if (tma_out && warp == 4 && lane == 0) bulk_wait0();   // et == 0: every dK / dV store has landed
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// dQ for one 128-query tile, 64 keys per step.
//   TMEM: S[2] [0,128), dP[2] [128,256), dQ [256,384), Q [384,448), dO [448,512) (bf16 pairs)
//   Q and dO are written into TMEM once by the elementwise warps (thread = row) and feed S
//   and dP as A operands; dS (bf16) goes back over the dP columns it came from (warp ck:
//   columns 16 ck .. +8) and feeds dQ as the A operand at column 16 kk. The tensor core
//   reads only K and V from shared memory: 48 KB per step instead of 144 KB.
//   smem: K|V ring of Q2_STAGES 64-row stages.
//   MMA order: S0 dP0 S1 dP1 | dQ0 S2 dP2 | dQ1 S3 dP3 | ...; S / dP (j+2) reuse the
//   buffers of step j behind dQ(j) (in-order tensor pipe).
constexpr int Q2_STAGES = 6;
struct BwdQ2Bars {
  uint64_t q_ready, kv_full[Q2_STAGES], kv_empty[Q2_STAGES], s_full[2], ds_full[2], acc_full;
  uint32_t tmem;
};
constexpr int BWD_Q2_SMEM = Q2_STAGES * 2 * HALF_TILE + 1024 + 256;
constexpr int BWD_Q2_THREADS = 640;

// 32 bf16 of a global row into 16 TMEM columns (one tcgen05.st per warp: thread = lane = row)
__device__ __forceinline__ void row32_to_tmem(uint32_t taddr, const __nv_bfloat16* src) {
  uint32_t w[16];
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = __ldg(s4 + q);
    w[4 * q] = v.x;
    w[4 * q + 1] = v.y;
    w[4 * q + 2] = v.z;
    w[4 * q + 3] = v.w;
  }
  tmem_st_32x16(taddr, w);
}

__global__ void __launch_bounds__(BWD_Q2_THREADS, 1)
    flash_bwd_dq_tc2(const __nv_bfloat16* __restrict__ q, const __grid_constant__ CUtensorMap map_k64,
                     const __grid_constant__ CUtensorMap map_v64, const __nv_bfloat16* __restrict__ d_o,
                     const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dq,
                     int S, int H, int ld, float scale, float scale_log2, int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto sK = [&](int st) { return smem + st * 2 * HALF_TILE; };
  auto sV = [&](int st) { return smem + st * 2 * HALF_TILE + HALF_TILE; };
  BwdQ2Bars* bars = reinterpret_cast<BwdQ2Bars*>(smem + Q2_STAGES * 2 * HALF_TILE);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int rank, bh;
  tile_order(order, rank, bh);
  const int qt = (int)gridDim.x - 1 - rank;
  const int b = bh / H, hh = bh % H;
  const int row0 = b * S, col0 = hh * HD;
  const int n = 2 * qt + 2;                        // 64-key steps 0 .. 2 qt + 1
  if (threadIdx.x == 0) {
    tma_prefetch(&map_k64);
    tma_prefetch(&map_v64);
    mbar_init(&bars->q_ready, 16);
    for (int i = 0; i < Q2_STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->ds_full[i], 16);
    }
    mbar_init(&bars->acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < n; ++j) {
        const int st = j % Q2_STAGES, ph = (j / Q2_STAGES) & 1;
        const int r = row0 + j * 64;
        mbar_wait(&bars->kv_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[st], 2 * HALF_TILE);
        tma_load_2d(sK(st), &map_k64, &bars->kv_full[st], col0, r);
        tma_load_2d(sK(st) + HALF_ATOM, &map_k64, &bars->kv_full[st], col0 + 64, r);
        tma_load_2d(sV(st), &map_v64, &bars->kv_full[st], col0, r);
        tma_load_2d(sV(st) + HALF_ATOM, &map_v64, &bars->kv_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idesc_acc = make_idesc_bf16(128, 128, false, true);
    mbar_wait(&bars->q_ready, 0);
    tc_fence_after();
    auto issue_sdp = [&](int j) {
      const int st = j % Q2_STAGES, bb = j & 1;
      mbar_wait(&bars->kv_full[st], (j / Q2_STAGES) & 1);
      tc_fence_after();
      const uint32_t k_base = smem_u32(sK(st)), v_base = smem_u32(sV(st));
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        umma_bf16_ts_w(tmem + bb * 64, tmem + 384 + kk * 8, kmajor_desc64(k_base, kk), idesc_s, kk ? 1u : 0u);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        umma_bf16_ts_w(tmem + 128 + bb * 64, tmem + 448 + kk * 8, kmajor_desc64(v_base, kk), idesc_s,
                       kk ? 1u : 0u);
      umma_commit_w(&bars->s_full[bb]);
    };
    issue_sdp(0);
    issue_sdp(1);
    for (int j = 0; j < n; ++j) {
      const int st = j % Q2_STAGES, bb = j & 1;
      mbar_wait(&bars->ds_full[bb], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t k_base = smem_u32(sK(st));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_ts_w(tmem + 256, tmem + 128 + bb * 64 + 16 * kk, mnmajor_desc64(k_base, kk), idesc_acc,
                       (j > 0 || kk > 0) ? 1u : 0u);
      umma_commit_w(&bars->kv_empty[st]);
      if (j + 2 < n) issue_sdp(j + 2);
    }
    umma_commit_w(&bars->acc_full);
  } else if (warp >= 4) {
    // warp w: query rows 32*(w%4).. (its TMEM lanes), key columns [16*ck, +16) of each step
    const int ck = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // query row within the tile
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    // this row's Q / dO, hd columns [32 ck, +32), into TMEM as bf16 pairs
    const long long grow = (long long)(row0 + qpos) * ld + col0 + ck * 32;
    row32_to_tmem(tmem + 384 + ck * 16 + lane_off, q + grow);
    row32_to_tmem(tmem + 448 + ck * 16 + lane_off, d_o + grow);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->q_ready);
    const float nl0 = -lse[(long long)bh * S + qpos] * kLog2e;
    const float D = dsum[(long long)bh * S + qpos];
    float nl[16], dn[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      nl[e] = nl0;
      dn[e] = D;
    }
    for (int j = 0; j < n; ++j) {
      const int bb = j & 1;
      const int k0 = j * 64 + ck * 16;             // first key column of this thread's 16
      mbar_wait(&bars->s_full[bb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[16], dpv[16];
      tmem_ld_32x16(tmem + bb * 64 + ck * 16 + lane_off, sv);
      tmem_ld_32x16(tmem + 128 + bb * 64 + ck * 16 + lane_off, dpv);
      tmem_ld_wait();
      uint32_t pk[8], ds8[8];
      // causal: P = 0 where key > query, i.e. column e > qpos - k0
      if (j >= 2 * qt)   // warp-uniform: the two diagonal steps
        p_ds_16<true>(sv, dpv, nl, dn, scale_log2, qpos - k0, false, pk, ds8);
      else
        p_ds_16<false>(sv, dpv, nl, dn, scale_log2, 0, false, pk, ds8);
      tmem_st_32x8(tmem + 128 + bb * 64 + ck * 16 + lane_off, ds8);   // over the dP columns just read
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->ds_full[bb]);
    }
    mbar_wait(&bars->acc_full, 0);
    tc_fence_after();
    store_acc_32(dq + (long long)(row0 + qpos) * ld + col0 + ck * 32, tmem + 256 + ck * 32 + lane_off, scale);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// Persistent dQ: one CTA per SM walks the 128-query tiles (per-launch counter, as
// flash_bwd_dkv_tc3), the K|V ring, barriers and TMEM kept across tiles.
//   smem: K|V ring of Q3_STAGES 64-row stages | the next tile's Q and dO (TMA, 64 KB) | the
//   32 KB dQ store stage.
// The producer TMA-loads the next tile's Q / dO as soon as it has claimed the tile (loading
// them row by row in the elementwise warps took ~4.9 us per tile: every warp load touched 32
// rows); at the tile boundary the elementwise warps copy them from shared memory into TMEM as
// soon as this tile's last S / dP have landed, so the tensor core starts the next tile's S / dP
// while they store dQ (through the store stage, row-contiguous).
constexpr int Q3_STAGES = 4;
struct BwdQ3Bars {
  uint64_t q_ready, kv_full[Q3_STAGES], kv_empty[Q3_STAGES], s_full[2], ds_full[2], acc_full;
  uint64_t qs_full, qs_empty, tile_full[2], tile_empty[2];
  int tile_id[2];
  uint32_t tmem;
};
static_assert(sizeof(BwdQ3Bars) <= 256, "barrier block");
constexpr int BWD_Q3_SMEM = Q3_STAGES * 2 * HALF_TILE + 3 * TILE_BYTES + 256;
static_assert(BWD_Q3_SMEM <= 227 * 1024, "shared memory");

// 32 bf16 (columns 32 c32 .. +32) of row r of a 128 x 128 tile held as two 128 x 64 SW128
// K-major atoms at shared address `tile`, into 16 TMEM columns (thread = lane = row)
__device__ __forceinline__ void smem_row32_to_tmem(uint32_t taddr, uint32_t tile, int r, int c32) {
  uint32_t w[16];
  const uint32_t row = tile + (c32 >> 1) * ATOM_BYTES + r * 128;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int chunk = (c32 & 1) * 4 + q;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[4 * q]), "=r"(w[4 * q + 1]), "=r"(w[4 * q + 2]), "=r"(w[4 * q + 3])
                 : "r"(row + ((chunk ^ (r & 7)) << 4)));
  }
  tmem_st_32x16(taddr, w);
}

__global__ void __launch_bounds__(BWD_Q2_THREADS, 1)
    flash_bwd_dq_tc3(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k64,
                     const __grid_constant__ CUtensorMap map_v64, const __grid_constant__ CUtensorMap map_do,
                     const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dq,
                     int S, int H, int ld, float scale, float scale_log2, int order, int nbh,
                     int* __restrict__ tile_ctr, const __grid_constant__ CUtensorMap map_dq, int tma_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // 1024-aligned window, no slack in BWD_Q3_SMEM; checked
  if (smem_u32(smem) & 1023) __trap();
  auto sK = [&](int st) { return smem + st * 2 * HALF_TILE; };
  auto sV = [&](int st) { return smem + st * 2 * HALF_TILE + HALF_TILE; };
  uint8_t* sQ = smem + Q3_STAGES * 2 * HALF_TILE;   // next tile's Q, then dO
  uint8_t* sdO = sQ + TILE_BYTES;
  const uint32_t s_out = smem_u32(sQ + 2 * TILE_BYTES);   // 32 KB store stage
  BwdQ3Bars* bars = reinterpret_cast<BwdQ3Bars*>(sQ + 3 * TILE_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = S / TQ, total = nt * nbh;
  if (threadIdx.x == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_do);
    tma_prefetch(&map_k64);
    tma_prefetch(&map_v64);
    mbar_init(&bars->q_ready, 16);
    for (int i = 0; i < Q3_STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->ds_full[i], 16);
      mbar_init(&bars->tile_full[i], 1);
      mbar_init(&bars->tile_empty[i], KV3_TILE_READERS);
    }
    mbar_init(&bars->acc_full, 1);
    mbar_init(&bars->qs_full, 1);
    mbar_init(&bars->qs_empty, 16);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;
  auto next_tile = [&](int j) {
    const int slot = j & 1;
    mbar_wait(&bars->tile_full[slot], (j >> 1) & 1);
    const int id = *reinterpret_cast<volatile int*>(&bars->tile_id[slot]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->tile_empty[slot]);
    return id;
  };
  // tile id -> query tile (long ones first within a head group), (batch, head)
  auto decode = [&](int id, int& qt, int& bh) {
    int rank;
    tile_decode(id, nt, nbh, order, rank, bh);
    qt = nt - 1 - rank;
  };
  // the producer claims tile j, publishes it, and TMA-loads its Q / dO (lane 0 only)
  auto claim_lane0 = [&](int j) {
    int t = 0;
    {
      const int slot = j & 1;
      mbar_wait(&bars->tile_empty[slot], ((j >> 1) & 1) ^ 1);
      t = atomicAdd(tile_ctr, 1);
      if (t >= total) t = -1;
      bars->tile_id[slot] = t;
      mbar_arrive(&bars->tile_full[slot]);
      if (t >= 0) {
        int qt, bh;
        decode(t, qt, bh);
        const int r0 = (bh / H) * S + qt * TQ, c0 = (bh % H) * HD;
        mbar_wait(&bars->qs_empty, (j & 1) ^ 1);   // the previous tile's Q / dO are in TMEM
        mbar_arrive_expect_tx(&bars->qs_full, 2 * TILE_BYTES);
        tma_load_2d(sQ, &map_q, &bars->qs_full, c0, r0);
        tma_load_2d(sQ + ATOM_BYTES, &map_q, &bars->qs_full, c0 + 64, r0);
        tma_load_2d(sdO, &map_do, &bars->qs_full, c0, r0);
        tma_load_2d(sdO + ATOM_BYTES, &map_do, &bars->qs_full, c0 + 64, r0);
      }
    }
    return t;
  };
  // the next tile is claimed kClaimAhead steps before this one's last K / V load: its Q / dO
  // (TMA, ~1.5 us) then land before the elementwise warps reach the boundary
  constexpr int kClaimAhead = 8;

  if (warp == 0) {
    int g = 0;
    int id = __shfl_sync(0xffffffffu, lane == 0 ? claim_lane0(0) : 0, 0);
    for (int j = 0; id >= 0; ++j) {
      int qt, bh;
      decode(id, qt, bh);
      const int n = 2 * qt + 2, row0 = (bh / H) * S, col0 = (bh % H) * HD;
      int nid = 0;
      if (lane == 0) {
        const int ahead = n > kClaimAhead ? n - kClaimAhead : 0;
        for (int jj = 0; jj < n; ++jj) {
          if (jj == ahead) nid = claim_lane0(j + 1);
          const int gg = g + jj, st = gg % Q3_STAGES, ph = (gg / Q3_STAGES) & 1;
          const int r = row0 + jj * 64;
          mbar_wait(&bars->kv_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&bars->kv_full[st], 2 * HALF_TILE);
          tma_load_2d(sK(st), &map_k64, &bars->kv_full[st], col0, r);
          tma_load_2d(sK(st) + HALF_ATOM, &map_k64, &bars->kv_full[st], col0 + 64, r);
          tma_load_2d(sV(st), &map_v64, &bars->kv_full[st], col0, r);
          tma_load_2d(sV(st) + HALF_ATOM, &map_v64, &bars->kv_full[st], col0 + 64, r);
        }
      }
      g += n;
      id = __shfl_sync(0xffffffffu, nid, 0);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t idesc_acc = make_idesc_bf16(128, 128, false, true);
    int g0 = 0;
    for (int j = 0;; ++j) {
      const int id = next_tile(j);
      if (id < 0) break;
      int qt, bh;
      decode(id, qt, bh);
      const int n = 2 * qt + 2;
      mbar_wait(&bars->q_ready, j & 1);
      tc_fence_after();
      auto issue_sdp = [&](int jj) {
        const int gg = g0 + jj, st = gg % Q3_STAGES, bb = gg & 1;
        mbar_wait(&bars->kv_full[st], (gg / Q3_STAGES) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sK(st)), v_base = smem_u32(sV(st));
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16_ts_w(tmem + bb * 64, tmem + 384 + kk * 8, kmajor_desc64(k_base, kk), idesc_s, kk ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16_ts_w(tmem + 128 + bb * 64, tmem + 448 + kk * 8, kmajor_desc64(v_base, kk), idesc_s,
                         kk ? 1u : 0u);
        umma_commit_w(&bars->s_full[bb]);
      };
      issue_sdp(0);
      issue_sdp(1);
      for (int jj = 0; jj < n; ++jj) {
        const int gg = g0 + jj, st = gg % Q3_STAGES, bb = gg & 1;
        mbar_wait(&bars->ds_full[bb], (gg >> 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sK(st));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ts_w(tmem + 256, tmem + 128 + bb * 64 + 16 * kk, mnmajor_desc64(k_base, kk), idesc_acc,
                         (jj > 0 || kk > 0) ? 1u : 0u);
        umma_commit_w(&bars->kv_empty[st]);
        if (jj + 2 < n) issue_sdp(jj + 2);
      }
      umma_commit_w(&bars->acc_full);
      g0 += n;
    }
  } else if (warp >= 4) {
    // warp w: query rows 32*(w%4).. (its TMEM lanes), key columns [16*ck, +16) of each step
    const int ck = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // query row within the tile
    const int et = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    // tile j's Q / dO rows (hd columns [32 ck, +32)) from shared memory into TMEM; q_ready
    auto load_q = [&](int j) {
      mbar_wait(&bars->qs_full, j & 1);
      smem_row32_to_tmem(tmem + 384 + ck * 16 + lane_off, smem_u32(sQ), r, ck);
      smem_row32_to_tmem(tmem + 448 + ck * 16 + lane_off, smem_u32(sdO), r, ck);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars->q_ready);
        mbar_arrive(&bars->qs_empty);
      }
    };
    int id = next_tile(0), qt = 0, bh = 0;
    float nl0 = 0.f, D = 0.f;
    if (id >= 0) {
      decode(id, qt, bh);
      load_q(0);
      nl0 = -lse[(long long)bh * S + qt * TQ + r] * kLog2e;
      D = dsum[(long long)bh * S + qt * TQ + r];
    }
    int g0 = 0;
    for (int j = 0; id >= 0; ++j) {
      const int n = 2 * qt + 2, row0 = (bh / H) * S, col0 = (bh % H) * HD;
      const int qpos = qt * TQ + r;
      const bool stamp = warp == 4 && lane == 0;
      if (stamp) {
        HLM_TL_AT(id + total, 0);
        unsigned smid_v;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_v));
        (void)smid_v;
        HLM_TL_AT_VAL(id + total, 6, smid_v);
        HLM_TL_AT_VAL(id + total, 7, n);
      }
      float nl[16], dn[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        nl[e] = nl0;
        dn[e] = D;
      }
      for (int jj = 0; jj < n; ++jj) {
        const int gg = g0 + jj, bb = gg & 1;
        const int k0 = jj * 64 + ck * 16;             // first key column of this thread's 16
        mbar_wait(&bars->s_full[bb], (gg >> 1) & 1);
        if (stamp && jj == 0) HLM_TL_AT(id + total, 1);
        tc_fence_after();
        uint32_t sv[16], dpv[16];
        tmem_ld_32x16(tmem + bb * 64 + ck * 16 + lane_off, sv);
        tmem_ld_32x16(tmem + 128 + bb * 64 + ck * 16 + lane_off, dpv);
        tmem_ld_wait();
        uint32_t pk[8], ds8[8];
        // causal: P = 0 where key > query, i.e. column e > qpos - k0
        if (jj >= 2 * qt)   // warp-uniform: the two diagonal steps
          p_ds_16<true>(sv, dpv, nl, dn, scale_log2, qpos - k0, false, pk, ds8);
        else
          p_ds_16<false>(sv, dpv, nl, dn, scale_log2, 0, false, pk, ds8);
        tmem_st_32x8(tmem + 128 + bb * 64 + ck * 16 + lane_off, ds8);   // over the dP columns just read
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->ds_full[bb]);
        if (stamp && jj == n - 1) HLM_TL_AT(id + total, 2);
      }
      g0 += n;
      // this tile's S / dP have all landed (s_full of its last step): Q / dO columns are free
      const int nid = next_tile(j + 1);
      int nqt = 0, nbh2 = 0;
      float nnl0 = 0.f, nD = 0.f;
      if (nid >= 0) {
        decode(nid, nqt, nbh2);
        load_q(j + 1);
        nnl0 = lse[(long long)nbh2 * S + nqt * TQ + r];   // first used after the dQ store (latency hidden)
        nD = dsum[(long long)nbh2 * S + nqt * TQ + r];
      }
      if (stamp) HLM_TL_AT(id + total, 5);
      mbar_wait(&bars->acc_full, j & 1);
      if (stamp) HLM_TL_AT(id + total, 3);
      tc_fence_after();
      if (tma_out)
        store_acc_tma(&map_dq, col0, row0 + qt * TQ, tmem + 256 + ck * 32 + lane_off, scale, s_out, r, ck, et);
      else
        store_acc_staged(dq + (long long)(row0 + qt * TQ) * ld + col0, ld, tmem + 256 + ck * 32 + lane_off, scale,
                         s_out, r, ck, et);
      if (stamp) HLM_TL_AT(id + total, 4);
      id = nid;
      qt = nqt;
      bh = nbh2;
      nl0 = -nnl0 * kLog2e;
      D = nD;
    }
  }
  if (tma_out && warp == 4 && lane == 0) bulk_wait0();   // et == 0: every dQ store has landed
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode_map_2d(CUtensorMap* map, const void* ptr, long long rows, int ld, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor maps by (pointer, rows, ld, box): a block's attention runs on the same arena
// buffers layer after layer, and encoding a map costs microseconds of host time per call
// (8 per backward) on the thread that feeds the compute stream. Direct-mapped, 128 entries;
// a map depends only on its key, so a hit is exact.
bool make_map_2d(CUtensorMap* map, const void* ptr, long long rows, int ld, int box_rows = 128) {
  struct Entry {
    const void* ptr;
    long long rows;
    int ld, box;
    bool valid;
    CUtensorMap map;
  };
  constexpr int kEntries = 128;
  static Entry cache[kEntries];
  static std::mutex mu;
  const size_t slot = ((reinterpret_cast<uintptr_t>(ptr) >> 7) ^ (size_t)rows * 131u ^ (size_t)ld * 31u ^
                       (size_t)box_rows) % kEntries;
  {
    std::lock_guard<std::mutex> lock(mu);
    const Entry& e = cache[slot];
    if (e.valid && e.ptr == ptr && e.rows == rows && e.ld == ld && e.box == box_rows) {
      *map = e.map;
      return true;
    }
  }
  if (!encode_map_2d(map, ptr, rows, ld, box_rows)) return false;
  std::lock_guard<std::mutex> lock(mu);
  cache[slot] = Entry{ptr, rows, ld, box_rows, true, *map};
  return true;
}

// Work counters of the persistent kernels: a ring of 1024 per device, one slot per launch
// (zeroed on the launch's stream first), so launches in flight on different streams never
// share a counter. Allocated on first use; the SM count comes with it.
bool tile_counter(int** ctr, int* nsm) {
  constexpr int kSlots = 1024, kDevs = 64;
  static int* ring[kDevs] = {};
  static int sms[kDevs] = {};
  static std::atomic<unsigned> next{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kDevs) return false;
  if (!ring[dev]) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!ring[dev]) {
      int* p = nullptr;
      if (cudaMalloc(&p, kSlots * sizeof(int)) != cudaSuccess) return false;
      if (cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return false;
      ring[dev] = p;
    }
  }
  *ctr = ring[dev] + next.fetch_add(1, std::memory_order_relaxed) % kSlots;
  // HLM_ATTN_PERSIST_CTAS caps the persistent grids (tests: many tiles per CTA at small shapes)
  static const int cap = [] {
    const char* e = std::getenv("HLM_ATTN_PERSIST_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  *nsm = cap > 0 ? std::min(cap, sms[dev]) : sms[dev];
  return true;
}

// Persistent backward kernels store dK / dV / dQ by TMA from their stage (default) or with
// row-contiguous st.global (HLM_ATTN_TMA_STORE=0).
int tma_out() {
  static const int v = [] {
    const char* e = std::getenv("HLM_ATTN_TMA_STORE");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// Heads per tile-order group (tile_decode). Forward: 16 (0.272 vs 0.279 ms head by head at
// C2). Backward (persistent kernels, tiles claimed in this order): 8 (dK/dV 453 vs 462 us head
// by head, dQ indifferent; with one CTA per tile, grouping lost more L2 locality than the tail
// cost). HLM_ATTN_TILE_GROUP / HLM_ATTN_BWD_TILE_GROUP override.
int tile_group(bool bwd) {
  static const int g[2] = {[] {
                             const char* e = std::getenv("HLM_ATTN_TILE_GROUP");
                             return e ? std::atoi(e) : 16;
                           }(),
                           [] {
                             const char* e = std::getenv("HLM_ATTN_BWD_TILE_GROUP");
                             return e ? std::atoi(e) : 8;
                           }()};
  return g[bwd ? 1 : 0];
}

}  // namespace

bool hlm_flash_tc_supported(int head_dim, int seq, int ld) {
  return head_dim == HD && seq % TQ == 0 && (ld * 2) % 16 == 0;
}

int hlm_flash_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse, int B, int S, int H, int ld,
                     cudaStream_t s) {
  CUtensorMap mq, mk, mv;
  const long long rows = (long long)B * S;
  if (!make_map_2d(&mq, q, rows, ld) || !make_map_2d(&mk, k, rows, ld) || !make_map_2d(&mv, v, rows, ld)) return 3;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  static const bool pp = std::getenv("HLM_ATTN_FWD_V1") == nullptr;
  if (pp && S % (2 * TQ) == 0) {   // two query tiles per CTA
    static const int emu = [] {
      const char* e = std::getenv("HLM_ATTN_EXP_EMU");
      return e ? std::atoi(e) : 1;
    }();
    static const bool v2 = std::getenv("HLM_ATTN_FWD_PP1") == nullptr;
    static const bool persist = [] {
      const char* e = std::getenv("HLM_ATTN_FWD_PERSIST");
      return e ? std::atoi(e) != 0 : true;
    }();
    if (v2 && persist) {   // persistent over query-tile pairs (default)
      CUtensorMap mk64, mv64;
      if (!make_map_2d(&mk64, k, rows, ld, 64) || !make_map_2d(&mv64, v, rows, ld, 64)) return 3;
      auto kern3 = emu >= 2 ? flash_fwd_pp3<2> : emu == 1 ? flash_fwd_pp3<1> : flash_fwd_pp3<0>;
      static bool attr_pp3 = false;
      if (!attr_pp3) {
        cudaFuncSetAttribute(flash_fwd_pp3<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP3_SMEM);
        cudaFuncSetAttribute(flash_fwd_pp3<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP3_SMEM);
        cudaFuncSetAttribute(flash_fwd_pp3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP3_SMEM);
        attr_pp3 = true;
      }
      int* ctr = nullptr;
      int nsm = 0;
      if (!tile_counter(&ctr, &nsm)) return 1;
      if (cudaMemsetAsync(ctr, 0, sizeof(int), s) != cudaSuccess) return 1;
      const int pairs = (S / (2 * TQ)) * B * H;
      kern3<<<std::min(nsm, pairs), PP_THREADS, PP3_SMEM, s>>>(mq, mk64, mv64, (__nv_bfloat16*)o, lse, S, H, ld,
                                                                (1.0f / sqrtf((float)HD)) * kLog2e,
                                                                tile_group(false), B * H, ctr);
      hlm_count_launches(1);
      return cudaGetLastError() == cudaSuccess ? 0 : 1;
    }
    if (v2) {   // 64-key steps, S double-buffered per tile, one CTA per pair
      CUtensorMap mk64, mv64;
      if (!make_map_2d(&mk64, k, rows, ld, 64) || !make_map_2d(&mv64, v, rows, ld, 64)) return 3;
      auto kern2 = emu >= 2 ? flash_fwd_pp2<2> : emu == 1 ? flash_fwd_pp2<1> : flash_fwd_pp2<0>;
      static bool attr_pp2 = false;
      if (!attr_pp2) {
        cudaFuncSetAttribute(flash_fwd_pp2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP2_SMEM);
        cudaFuncSetAttribute(flash_fwd_pp2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP2_SMEM);
        cudaFuncSetAttribute(flash_fwd_pp2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP2_SMEM);
        attr_pp2 = true;
      }
      dim3 grid(S / (2 * TQ), B * H);
      kern2<<<grid, PP_THREADS, PP2_SMEM, s>>>(mq, mk64, mv64, (__nv_bfloat16*)o, lse, S, H, ld,
                                               (1.0f / sqrtf((float)HD)) * kLog2e, tile_group(false));
      hlm_count_launches(1);
      return cudaGetLastError() == cudaSuccess ? 0 : 1;
    }
    auto kern = emu >= 2 ? flash_fwd_pp<2> : emu == 1 ? flash_fwd_pp<1> : flash_fwd_pp<0>;
    static bool attr_pp = false;
    if (!attr_pp) {
      cudaFuncSetAttribute(flash_fwd_pp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP_SMEM);
      cudaFuncSetAttribute(flash_fwd_pp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP_SMEM);
      cudaFuncSetAttribute(flash_fwd_pp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PP_SMEM);
      attr_pp = true;
    }
    dim3 grid(S / (2 * TQ), B * H);
    kern<<<grid, PP_THREADS, PP_SMEM, s>>>(mq, mk, mv, (__nv_bfloat16*)o, lse, S, H, ld,
                                           (1.0f / sqrtf((float)HD)) * kLog2e);
    hlm_count_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
  }
  dim3 grid(S / TQ, B * H);
  flash_fwd_tc<<<grid, FWD_THREADS, SMEM_BYTES, s>>>(mq, mk, mv, (__nv_bfloat16*)o, lse, S, H, ld,
                                             (1.0f / sqrtf((float)HD)) * kLog2e);
  hlm_count_launches(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// D (rowsum dO . O) comes from the caller (dsum, computed by dsum_kernel in attention_flash.cu).
int hlm_flash_bwd_tc(const void* q, const void* k, const void* v, const void* d_o, const float* lse,
                     const float* dsum, void* dq, void* dk, void* dv, int B, int S, int H, int ld, cudaStream_t s) {
  CUtensorMap mq, mk, mv, mdo;
  const long long rows = (long long)B * S;
  if (!make_map_2d(&mq, q, rows, ld) || !make_map_2d(&mk, k, rows, ld) || !make_map_2d(&mv, v, rows, ld) ||
      !make_map_2d(&mdo, d_o, rows, ld))
    return 3;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_bwd_dkv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_KV_SMEM);
    cudaFuncSetAttribute(flash_bwd_dq_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_Q_SMEM);
    attr = true;
  }
  const float scale = 1.0f / sqrtf((float)HD);
  dim3 grid(S / TQ, B * H);
  static const bool v1 = std::getenv("HLM_ATTN_BWD_V1") != nullptr;
  if (!v1) {   // 64-wide steps, double-buffered S / dP (default)
    CUtensorMap mq64, mk64, mv64, mdo64;
    if (!make_map_2d(&mq64, q, rows, ld, 64) || !make_map_2d(&mk64, k, rows, ld, 64) ||
        !make_map_2d(&mv64, v, rows, ld, 64) || !make_map_2d(&mdo64, d_o, rows, ld, 64))
      return 3;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(flash_bwd_dkv_tc2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_KV2_SMEM);
      cudaFuncSetAttribute(flash_bwd_dkv_tc2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_KV2_SMEM);
      cudaFuncSetAttribute(flash_bwd_dkv_tc2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_KV2_SMEM);
      cudaFuncSetAttribute(flash_bwd_dq_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_Q2_SMEM);
      attr2 = true;
    }
    static const int xp = [] {
      const char* e = std::getenv("HLM_ATTN_BWD_EXPERIMENT");
      return e ? std::atoi(e) : 0;
    }();
    static const bool persist = [] {
      const char* e = std::getenv("HLM_ATTN_BWD_PERSIST");
      return e ? std::atoi(e) != 0 : true;
    }();
    if (persist && xp == 0) {
      int* ctr = nullptr;
      int nsm = 0;
      if (!tile_counter(&ctr, &nsm)) return 1;
      static bool attr3 = false;
      if (!attr3) {
        cudaFuncSetAttribute(flash_bwd_dkv_tc3, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_KV3_SMEM);
        attr3 = true;
      }
      if (cudaMemsetAsync(ctr, 0, sizeof(int), s) != cudaSuccess) return 1;
      const int tiles = (S / TK) * B * H;
      CUtensorMap mdk, mdv;
      if (!make_map_2d(&mdk, dk, rows, ld) || !make_map_2d(&mdv, dv, rows, ld)) return 3;
      flash_bwd_dkv_tc3<<<std::min(nsm, tiles), BWD_KV2_THREADS, BWD_KV3_SMEM, s>>>(
          mq64, mk, mv, mdo64, lse, dsum, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, S, H, ld, scale, scale * kLog2e,
          tile_group(true), B * H, ctr, mdk, mdv, tma_out());
    } else {
    auto kv_kern = xp == 1 ? flash_bwd_dkv_tc2<1> : xp == 2 ? flash_bwd_dkv_tc2<2> : flash_bwd_dkv_tc2<0>;
    kv_kern<<<grid, BWD_KV2_THREADS, BWD_KV2_SMEM, s>>>(
        mq64, mk, mv, mdo64, lse, dsum, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, S, H, ld, scale, scale * kLog2e,
        tile_group(true));
    }
    if (persist) {
      int* ctr = nullptr;
      int nsm = 0;
      if (!tile_counter(&ctr, &nsm)) return 1;
      static bool attr_q3 = false;
      if (!attr_q3) {
        cudaFuncSetAttribute(flash_bwd_dq_tc3, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_Q3_SMEM);
        attr_q3 = true;
      }
      if (cudaMemsetAsync(ctr, 0, sizeof(int), s) != cudaSuccess) return 1;
      const int tiles = (S / TQ) * B * H;
      CUtensorMap mdq;
      if (!make_map_2d(&mdq, dq, rows, ld)) return 3;
      flash_bwd_dq_tc3<<<std::min(nsm, tiles), BWD_Q2_THREADS, BWD_Q3_SMEM, s>>>(
          mq, mk64, mv64, mdo, lse, dsum, (__nv_bfloat16*)dq, S, H, ld, scale, scale * kLog2e, tile_group(true),
          B * H, ctr, mdq, tma_out());
    } else
    flash_bwd_dq_tc2<<<grid, BWD_Q2_THREADS, BWD_Q2_SMEM, s>>>(
        (const __nv_bfloat16*)q, mk64, mv64, (const __nv_bfloat16*)d_o, lse, dsum, (__nv_bfloat16*)dq, S, H, ld, scale,
        scale * kLog2e, tile_group(true));
    hlm_count_launches(2);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
  }
  flash_bwd_dkv_tc<<<grid, BWD_KV_THREADS, BWD_KV_SMEM, s>>>(mq, mk, mv, mdo, lse, dsum, (__nv_bfloat16*)dk,
                                                   (__nv_bfloat16*)dv, S, H, ld, scale, scale * kLog2e);
  flash_bwd_dq_tc<<<grid, FWD_THREADS, BWD_Q_SMEM, s>>>(mq, mk, mv, mdo, lse, dsum, (__nv_bfloat16*)dq, S, H, ld, scale,
                                                 scale * kLog2e);
  hlm_count_launches(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
