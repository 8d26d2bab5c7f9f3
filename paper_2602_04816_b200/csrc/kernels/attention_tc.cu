// Causal flash-attention FORWARD on tcgen05 (head_dim 128, seq % 128 == 0).
//
// Same contract as flash_fwd (attention_flash.cu; reference attention_fwd,
// proj/include/hlm/kernels.hpp:207-245): O and the row log-sum-exp per head.
// One CTA per (128-query tile, batch*head), 256 threads:
//   warp 0  TMA producer: Q once, K/V tiles into a 2-stage ring (SW128, 2 boxes
//           of 64 columns per 128x128 tile = two K-major swizzle atoms)
//   warp 1  MMA issuer (one lane): S_j = Q K_j^T into TMEM S[j%2] (M=N=128,
//           K=128), then O_j = P_j V_j into TMEM O[j%2] (V as an MN-major B
//           operand, P from shared memory); S_{j+1} is issued before PV_j so the
//           tensor core overlaps the softmax of tile j
//   warp 2  TMEM allocator (512 columns: S0 S1 O0 O1)
//   warps 4-7 softmax: thread = query row; two TMEM passes over S (row max,
//           then exp2 + row sum + bf16 P written to swizzled smem), then the
//           online rescale O_acc = alpha * O_acc + O_j in registers.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attention.h"
#include "block_ops.h"
#include "sm100_ptx.cuh"

using namespace hlm_sm100;

namespace {

constexpr int TQ = 128, TK = 128, HD = 128;
constexpr int TILE_BYTES = TQ * HD * 2;            // 32 KiB
constexpr int ATOM_BYTES = 128 * 64 * 2;           // 16 KiB: 128 rows x 64 cols
constexpr int SMEM_BYTES = TILE_BYTES * 7 + 1024 + 256;   // Q, K0 V0 K1 V1, P0 P1
constexpr float kLog2e = 1.4426950408889634f;

struct Bars {
  uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], s_free[2], p_full[2], o_full[2], o_free[2];
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

// K-major SW128 descriptor for K step kk (16 elements) of a 128 x 128 tile stored as two atoms.
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int kk) {
  return make_sw128_desc(base + (kk >> 2) * ATOM_BYTES + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor (V): K step kk = 16 key rows; MN atoms (64 d) 16 KiB apart.
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t base, int kk) {
  return make_sw128_desc(base + kk * 2048, ATOM_BYTES, 1024);
}

__global__ void __launch_bounds__(256, 1)
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
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], 4);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], 4);
      mbar_init(&bars->p_full[i], 4);
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
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        mbar_wait(&bars->kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->kv_full[st], 2 * TILE_BYTES);
        const int r = row0 + j * TK;
        tma_load_2d(sK[st], &map_k, &bars->kv_full[st], col0, r);
        tma_load_2d(sK[st] + ATOM_BYTES, &map_k, &bars->kv_full[st], col0 + 64, r);
        tma_load_2d(sV[st], &map_v, &bars->kv_full[st], col0, r);
        tma_load_2d(sV[st] + ATOM_BYTES, &map_v, &bars->kv_full[st], col0 + 64, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    const uint32_t q_base = smem_u32(sQ);
    mbar_wait(&bars->q_full, 0);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&bars->kv_full[st], (j >> 1) & 1);
      mbar_wait(&bars->s_free[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_base = smem_u32(sK[st]);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem + st * 128, kmajor_desc(q_base, kk), kmajor_desc(k_base, kk), idesc_s, kk ? 1u : 0u);
        umma_commit(&bars->s_full[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      if (j + 1 < n_tiles) issue_s(j + 1);
      mbar_wait(&bars->p_full[st], (j >> 1) & 1);
      mbar_wait(&bars->o_free[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t v_base = smem_u32(sV[st]);
        const uint32_t p_base = smem_u32(sP[st]);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)
          umma_bf16(tmem + 256 + st * 128, kmajor_desc(p_base, kk), mnmajor_desc(v_base, kk), idesc_o, kk ? 1u : 0u);
        umma_commit(&bars->o_full[st]);
        umma_commit(&bars->kv_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane;                 // query row within the tile
    const int qpos = qt * TQ + r;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float oacc[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) oacc[i] = 0.f;
    float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
    // O_acc <- alpha * O_acc + O_j (TMEM O[jj % 2]), then release that O buffer
    auto fold = [&](int jj, float alpha) {
      const int so = jj & 1;
      mbar_wait(&bars->o_full[so], (jj >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32(tmem + 256 + so * 128 + c * 32 + lane_off, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) oacc[c * 32 + e] = oacc[c * 32 + e] * alpha + __uint_as_float(v[e]);
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
      // pass 1: row max
      float mx = m;
#pragma unroll 1
      for (int c = 0; c < TK / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32(tmem + st * 128 + c * 32 + lane_off, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float sv = __uint_as_float(v[e]) * scale_log2;
          if (!diag || c * 32 + e <= r) mx = fmaxf(mx, sv);
        }
      }
      const float alpha = exp2f(m - mx);
      m = mx;
      // P[st] was last read by PV_{j-2}
      if (j >= 2) mbar_wait(&bars->o_full[st], ((j - 2) >> 1) & 1);
      uint8_t* prow = sP[st] + r * 128;
      // pass 2: p = exp2(s - m), row sum, bf16 P into the swizzled K-major tile
      float rs = 0.f;
#pragma unroll 1
      for (int c = 0; c < TK / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32(tmem + st * 128 + c * 32 + lane_off, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p0 = exp2f(__uint_as_float(v[e]) * scale_log2 - m);
          float p1 = exp2f(__uint_as_float(v[e + 1]) * scale_log2 - m);
          if (diag && c * 32 + e > r) p0 = 0.f;
          if (diag && c * 32 + e + 1 > r) p1 = 0.f;
          rs += p0 + p1;
          pk[e / 2] = pack_bf16x2(p0, p1);
        }
        const int atom = c >> 1;   // keys c*32 .. c*32+31: atom (c/2), 16-byte chunks (c%2)*4 .. +3
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int chunk = (c & 1) * 4 + q4;
          uint4 val = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          *reinterpret_cast<uint4*>(prow + atom * ATOM_BYTES + ((chunk ^ (r & 7)) << 4)) = val;
        }
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
    const float il = 1.f / l;
    __nv_bfloat16* orow = o + (long long)(row0 + qpos) * ld + col0;
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      uint4 val = make_uint4(pack_bf16x2(oacc[8 * c] * il, oacc[8 * c + 1] * il),
                             pack_bf16x2(oacc[8 * c + 2] * il, oacc[8 * c + 3] * il),
                             pack_bf16x2(oacc[8 * c + 4] * il, oacc[8 * c + 5] * il),
                             pack_bf16x2(oacc[8 * c + 6] * il, oacc[8 * c + 7] * il));
      reinterpret_cast<uint4*>(orow)[c] = val;
    }
    lse[(long long)bh * S + qpos] = (m + log2f(l)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_map_2d(CUtensorMap* map, const void* ptr, long long rows, int ld) {
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
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
  dim3 grid(S / TQ, B * H);
  flash_fwd_tc<<<grid, 256, SMEM_BYTES, s>>>(mq, mk, mv, (__nv_bfloat16*)o, lse, S, H, ld,
                                             (1.0f / sqrtf((float)HD)) * kLog2e);
  hlm_count_launches(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
