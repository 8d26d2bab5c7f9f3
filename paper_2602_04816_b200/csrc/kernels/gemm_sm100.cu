// Persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
// One kernel template serves every projection of the block and the head:
//   forward      X(T,in) . W(in,out)        A K-major, B MN-major
//   dgrad        dY(T,out) . W(in,out)^T    A K-major, B K-major
//   wgrad        X(T,in)^T . dY(T,out)      A MN-major, B MN-major
// i.e. the three CPU loops matmul_nn / matmul_nt / matmul_grad_acc of
// reference proj/include/hlm/kernels.hpp:164-205, with W kept in the
// reference's (in, out) row-major tile layout (host_store.cpp:70-92) so no
// transposed weight copy is ever made: majorness is a descriptor bit.
//
// Groups: three (h,h) matrices w_q|w_k|w_v (and w_up|w_gate) sit back to back
// in the tile, so a "group" dimension lets one launch cover QKV (N-grouped:
// independent outputs [G][M][N]) or sum the three dgrads into one output
// (K-grouped: the K loop runs over groups too).
//
// Tile 128x256x64, 4-stage TMA->smem ring, 2 TMEM accumulators (512 cols) so
// the epilogue of tile i overlaps the MMAs of tile i+1.
// Warp roles: w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4..7 epilogue.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm.h"
#include "sm100_ptx.cuh"
#include "block_ops.h"
#include "fused_math.cuh"

using namespace hlm_sm100;

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;   // 16 KiB
constexpr int B_STAGE = BN * BK * 2;   // 32 KiB
constexpr int ATOM = 64 * BK * 2;      // one 64-wide MN atom of a MN-major stage: 8 KiB
constexpr int NUM_THREADS = 256;
constexpr int GROUP_M = 8;             // raster: 8 M-tiles share each B panel in L2 (default; see launch())
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + 1024 /*align*/ + 256 /*barriers*/;

struct KArgs {
  int M, N, K, G;
  int kgroup, a_grouped, b_grouped;
  int tiles_m, tiles_n, kblocks, num_tiles;
  int group_m;   // raster group (M-tiles sharing a B panel)
  void* C;
  long long ldc, c_gstride;
  const float* R;
  long long ldr, r_gstride;
  int epi;
  // fused epilogues (HLM_EPI_BF16_ROPE / SWIGLU / SWIGLU_BWD, include/hlm_cuda.h)
  int paired;            // SWIGLU: B atoms of groups 0 | 1 for the same output columns
  const float* rope_cos;
  const float* rope_sin;
  int rope_seq, rope_hd;
  const __nv_bfloat16* aux;
  long long aux_ld, aux_gstride;
  __nv_bfloat16* C2;
  long long ldc2;
  int l2_prefetch;       // SWIGLU_BWD: bulk-prefetch the next tile's up / gate into L2 (A/B)
  int l2_hint;           // 2-CTA operand loads: 0 evict_normal, 1 evict_last, 2 evict_first
  int* tile_ctr;         // 2-CTA: tiles claimed from this per-launch counter (nullptr: static stride)
};

__device__ __forceinline__ void tile_coords(const KArgs& a, int t, int& g, int& m, int& n) {
  const int per_group = a.tiles_m * a.tiles_n;
  g = a.kgroup ? 0 : t / per_group;
  const int rem = t - g * per_group;
  const int per_panel = a.group_m * a.tiles_n;
  const int panel = rem / per_panel;
  const int first_m = panel * a.group_m;
  const int gm = min(a.tiles_m - first_m, a.group_m);
  const int r = rem - panel * per_panel;
  m = first_m + r % gm;
  n = r / gm;
}

// TMEM accumulator row (32x32b loads, 8 chunks of 32 columns) -> global C.
__device__ __forceinline__ void epilogue_plain(const KArgs& args, uint32_t taddr, int row, int tg, int col_base,
                                               int epi) {
  const bool row_ok = row < args.M;
  const long long c_off = (long long)tg * args.c_gstride + (long long)row * args.ldc;
  const long long r_off = (long long)tg * args.r_gstride + (long long)row * args.ldr;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld_32x32(taddr + c * 32, r);
    tmem_ld_wait();
    const int col0 = col_base + c * 32;
      if (!row_ok || col0 >= args.N) continue;
      const bool full_chunk = col0 + 32 <= args.N;
      if (epi == HLM_EPI_BF16) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.C) + c_off + col0;
        if (full_chunk && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(r[8 * j + 0]), __uint_as_float(r[8 * j + 1]));
            v.y = pack_bf16x2(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3]));
            v.z = pack_bf16x2(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5]));
            v.w = pack_bf16x2(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7]));
            d4[j] = v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < args.N) dst[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
        }
      } else {
        float* dst = reinterpret_cast<float*>(args.C) + c_off + col0;
        const float* res = epi == HLM_EPI_F32_ADD ? args.R + r_off + col0 : nullptr;
        if (full_chunk && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) &&
            (res == nullptr || (reinterpret_cast<uintptr_t>(res) & 15) == 0)) {
          float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 v = make_float4(__uint_as_float(r[4 * j + 0]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            if (res) {
              const float4 q = reinterpret_cast<const float4*>(res)[j];
              v.x += q.x;
              v.y += q.y;
              v.z += q.z;
              v.w += q.w;
            }
            d4[j] = v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < args.N) dst[j] = __uint_as_float(r[j]) + (res ? res[j] : 0.0f);
        }
      }
    }
}

// 32 consecutive bf16 values of one row (16-byte stores when the chunk is whole and aligned).
// Streaming (evict-first) stores: the fused epilogues' outputs must not push the GEMM's
// operand panels out of L2.
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32], int valid) {
  if (valid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      __stcs(d4 + j, make_uint4(pack_bf16x2(v[8 * j + 0], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7])));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < valid) dst[j] = __float2bfloat16_rn(v[j]);
  }
}

__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* src, float (&v)[32], int valid) {
  if (valid == 32 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 q = s4[j];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[8 * j + 2 * e] = __uint_as_float(w[e] << 16);
        v[8 * j + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j < valid ? __bfloat162float(src[j]) : 0.0f;
  }
}

// q|k|v projection + RoPE: groups 0 (q) and 1 (k) are rotated in registers before the
// BF16 store (rotate-half pairs (i, i + hd/2) of a head sit in chunks c and c + hd/64 of
// the same thread's row); group 2 (v) is a plain BF16 store. Same rounding points as
// the GEMM's BF16 epilogue followed by the in-place rope pass.
__device__ __forceinline__ void epilogue_rope(const KArgs& args, uint32_t taddr, int row, int tg, int col_base) {
  if (tg >= 2) {   // v: the plain BF16 store
    epilogue_plain(args, taddr, row, tg, col_base, HLM_EPI_BF16);
    return;
  }
  const int hd = args.rope_hd, half = hd >> 1, dist = half >> 5;
  const bool row_ok = row < args.M;
  const int pos = row_ok ? row % args.rope_seq : 0;
  __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(args.C) + (long long)tg * args.c_gstride +
                        (long long)row * args.ldc;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    const int w = (c * 32) & (hd - 1);
    if (w >= half) continue;   // second half of a head: rotated together with chunk c - dist
    uint32_t ra[32], rb[32];
    tmem_ld_32x32(taddr + c * 32, ra);
    tmem_ld_32x32(taddr + (c + dist) * 32, rb);
    tmem_ld_wait();
    const int col0 = col_base + c * 32;
    if (!row_ok || col0 >= args.N) continue;
    const float4* cp = reinterpret_cast<const float4*>(args.rope_cos + (long long)pos * half + w);
    const float4* sp = reinterpret_cast<const float4*>(args.rope_sin + (long long)pos * half + w);
    float oa[32], ob[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 c4 = cp[q], s4 = sp[q];
      const float cv[4] = {c4.x, c4.y, c4.z, c4.w}, sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 4 * q + e;
        hlm_fused::rope_rotate(hlm_fused::round_bf16(__uint_as_float(ra[j])),
                               hlm_fused::round_bf16(__uint_as_float(rb[j])), cv[e], sv[e], false, oa[j], ob[j]);
      }
    }
    store_bf16x32(crow + col0, oa, 32);
    store_bf16x32(crow + col0 + half, ob, 32);
  }
}

// up|gate projection (paired tile: TMEM columns 0..127 = up, 128..255 = gate of the same
// 128 output columns): up, gate rounded to BF16 and stored for the backward, and
// act = up * silu(gate) from the rounded values — the swiglu_fwd kernel's arithmetic.
__device__ __forceinline__ void epilogue_swiglu(const KArgs& args, uint32_t taddr, int row, int col_base) {
  const bool row_ok = row < args.M;
  __nv_bfloat16* up_row = reinterpret_cast<__nv_bfloat16*>(args.C) + (long long)row * args.ldc;
  __nv_bfloat16* gate_row = up_row + args.c_gstride;
  __nv_bfloat16* act_row = args.C2 + (long long)row * args.ldc2;
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    uint32_t ru[32], rg[32];
    tmem_ld_32x32(taddr + c * 32, ru);
    tmem_ld_32x32(taddr + BN / 2 + c * 32, rg);
    tmem_ld_wait();
    const int col0 = col_base + c * 32;
    if (!row_ok || col0 >= args.N) continue;
    const int valid = min(32, args.N - col0);
    float u[32], z[32], a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      u[j] = hlm_fused::round_bf16(__uint_as_float(ru[j]));
      z[j] = hlm_fused::round_bf16(__uint_as_float(rg[j]));
      a[j] = hlm_fused::swiglu(u[j], z[j]);
    }
    store_bf16x32(up_row + col0, u, valid);
    store_bf16x32(gate_row + col0, z, valid);
    store_bf16x32(act_row + col0, a, valid);
  }
}

// 16-byte streaming load issued where it is written: volatile asm keeps the compiler from
// sinking a prefetch down to its use (it does that under register pressure).
__device__ __forceinline__ uint4 ld_cs_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// down-projection dgrad: d_act rounded to BF16 (the plain epilogue's value), then the
// swiglu_bwd kernel's arithmetic against up / gate read from aux. The up / gate loads of
// chunk c + 1 are issued before chunk c's math, so their latency hides under it and the
// epilogue keeps pace with the next tile's MMAs.
__device__ __forceinline__ void epilogue_swiglu_bwd(const KArgs& args, uint32_t taddr, int row, int col_base) {
  const bool row_ok = row < args.M;
  __nv_bfloat16* du_row = reinterpret_cast<__nv_bfloat16*>(args.C) + (long long)row * args.ldc;
  __nv_bfloat16* dg_row = du_row + args.c_gstride;
  const __nv_bfloat16* up_row = args.aux + (long long)row * args.aux_ld;
  const __nv_bfloat16* gate_row = up_row + args.aux_gstride;
  // whole 32-column chunks of 16-byte aligned rows use the prefetched vector path
  const bool vec = ((args.aux_ld & 7) == 0) && ((reinterpret_cast<uintptr_t>(args.aux) & 15) == 0) &&
                   ((args.aux_gstride & 7) == 0);
  auto whole = [&](int c) { return row_ok && vec && col_base + c * 32 + 32 <= args.N; };
  uint4 pu[4], pz[4];
  if (whole(0)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pu[j] = ld_cs_v4(reinterpret_cast<const uint4*>(up_row + col_base) + j);
      pz[j] = ld_cs_v4(reinterpret_cast<const uint4*>(gate_row + col_base) + j);
    }
  }
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t rd[32];
    tmem_ld_32x32(taddr + c * 32, rd);
    const int col0 = col_base + c * 32;
    uint4 nu[4], nz[4];
    if (c + 1 < BN / 32 && whole(c + 1)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        nu[j] = ld_cs_v4(reinterpret_cast<const uint4*>(up_row + col0 + 32) + j);
        nz[j] = ld_cs_v4(reinterpret_cast<const uint4*>(gate_row + col0 + 32) + j);
      }
    }
    tmem_ld_wait();
    if (row_ok && col0 < args.N) {
      const int valid = min(32, args.N - col0);
      float u[32], z[32], du[32], dg[32];
      if (whole(c)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t wu[4] = {pu[j].x, pu[j].y, pu[j].z, pu[j].w};
          const uint32_t wz[4] = {pz[j].x, pz[j].y, pz[j].z, pz[j].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            u[8 * j + 2 * e] = __uint_as_float(wu[e] << 16);
            u[8 * j + 2 * e + 1] = __uint_as_float(wu[e] & 0xFFFF0000u);
            z[8 * j + 2 * e] = __uint_as_float(wz[e] << 16);
            z[8 * j + 2 * e + 1] = __uint_as_float(wz[e] & 0xFFFF0000u);
          }
        }
      } else {
        load_bf16x32(up_row + col0, u, valid);
        load_bf16x32(gate_row + col0, z, valid);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j)
        hlm_fused::swiglu_bwd(hlm_fused::round_bf16(__uint_as_float(rd[j])), u[j], z[j], du[j], dg[j]);
      store_bf16x32(du_row + col0, du, valid);
      store_bf16x32(dg_row + col0, dg, valid);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pu[j] = nu[j];
      pz[j] = nz[j];
    }
  }
}

// F32 + residual (the o / down projections' h + x W): the residual of chunk c + 1 is loaded
// while chunk c's accumulator comes out of TMEM, and both streams bypass L2 retention
// (evict-first loads / stores) so they do not push the operand panels out. Same fp32 adds
// as the plain epilogue. (Loading the residual per float4 right before its store, behind
// the previous store to a possibly aliasing row, serialised eight global latencies per
// chunk and left the tensor pipe 39 % idle in this GEMM.)
__device__ __forceinline__ void epilogue_f32_add(const KArgs& args, uint32_t taddr, int row, int tg, int col_base) {
  const bool row_ok = row < args.M;
  float* crow = reinterpret_cast<float*>(args.C) + (long long)tg * args.c_gstride + (long long)row * args.ldc;
  const float* rrow = args.R + (long long)tg * args.r_gstride + (long long)row * args.ldr;
  const bool vec = row_ok && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(rrow) & 15) == 0) && ((args.ldc & 3) == 0) && ((args.ldr & 3) == 0);
  auto whole = [&](int c) { return vec && col_base + c * 32 + 32 <= args.N; };
  uint4 pr[8];
  if (whole(0)) {
#pragma unroll
    for (int j = 0; j < 8; ++j) pr[j] = ld_cs_v4(rrow + col_base + 4 * j);
  }
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    tmem_ld_32x32(taddr + c * 32, r);
    const int col0 = col_base + c * 32;
    uint4 nr[8];
    if (c + 1 < BN / 32 && whole(c + 1)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) nr[j] = ld_cs_v4(rrow + col0 + 32 + 4 * j);
    }
    tmem_ld_wait();
    if (row_ok && col0 < args.N) {
      if (whole(c)) {
        float4* d4 = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          __stcs(d4 + j, make_float4(__uint_as_float(r[4 * j + 0]) + __uint_as_float(pr[j].x),
                                     __uint_as_float(r[4 * j + 1]) + __uint_as_float(pr[j].y),
                                     __uint_as_float(r[4 * j + 2]) + __uint_as_float(pr[j].z),
                                     __uint_as_float(r[4 * j + 3]) + __uint_as_float(pr[j].w)));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < args.N) crow[col0 + j] = __uint_as_float(r[j]) + rrow[col0 + j];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) pr[j] = nr[j];
  }
}

// SWIGLU_BWD: pull the up / gate row segments a tile's epilogue will read into L2 while
// that tile's MMAs are still running (issued one tile ahead by the epilogue threads).
__device__ __forceinline__ void epilogue_prefetch(const KArgs& args, int row, int tn) {
  if (!args.l2_prefetch || args.epi != HLM_EPI_SWIGLU_BWD || row >= args.M) return;
  const int col0 = tn * BN;
  if (col0 >= args.N || (args.aux_ld & 7) || (args.aux_gstride & 7) || (reinterpret_cast<uintptr_t>(args.aux) & 15))
    return;
  const uint32_t bytes = (uint32_t)((min(BN, args.N - col0) * 2 + 15) & ~15);
  const __nv_bfloat16* up = args.aux + (long long)row * args.aux_ld + col0;
  l2_prefetch_bulk(up, bytes);
  l2_prefetch_bulk(up + args.aux_gstride, bytes);
}

__device__ __forceinline__ void epilogue_store(const KArgs& args, uint32_t taddr, int row, int tg, int tn) {
  switch (args.epi) {
    case HLM_EPI_BF16_ROPE: epilogue_rope(args, taddr, row, tg, tn * BN); break;
    case HLM_EPI_SWIGLU: epilogue_swiglu(args, taddr, row, tn * (BN / 2)); break;
    case HLM_EPI_SWIGLU_BWD: epilogue_swiglu_bwd(args, taddr, row, tn * BN); break;
    case HLM_EPI_F32_ADD: epilogue_f32_add(args, taddr, row, tg, tn * BN); break;
    default: epilogue_plain(args, taddr, row, tg, tn * BN, args.epi);
  }
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const KArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int g_iters = args.kgroup ? args.G : 1;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        int tg, tm, tn;
        tile_coords(args, t, tg, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int gi = 0; gi < g_iters; ++gi) {
          const int g = args.kgroup ? gi : tg;
          const int ag = args.a_grouped ? g : 0;
          const int bg = args.b_grouped ? g : 0;
          for (int kb = 0; kb < args.kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], A_STAGE + B_STAGE);
            const int k0 = kb * BK;
            uint8_t* a_dst = sA + stage * A_STAGE;
            uint8_t* b_dst = sB + stage * B_STAGE;
            if (A_MN) {
              tma_load_3d(a_dst, &map_a, &full[stage], m0, k0, ag);
              tma_load_3d(a_dst + ATOM, &map_a, &full[stage], m0 + 64, k0, ag);
            } else {
              tma_load_3d(a_dst, &map_a, &full[stage], k0, m0, ag);
            }
            if (B_MN) {
              if (args.paired) {   // atoms 0,1: group 0 (up); atoms 2,3: group 1 (gate), same columns
                const int np = tn * (BN / 2);
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  tma_load_3d(b_dst + j * ATOM, &map_b, &full[stage], np + 64 * (j & 1), k0, j >> 1);
              } else {
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  tma_load_3d(b_dst + j * ATOM, &map_b, &full[stage], n0 + 64 * j, k0, bg);
              }
            } else {
              tma_load_3d(b_dst, &map_b, &full[stage], k0, n0, bg);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      bool first = true;
      for (int gi = 0; gi < g_iters; ++gi) {
        for (int kb = 0; kb < args.kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          {
            const uint32_t a_base = smem_u32(sA + stage * A_STAGE);
            const uint32_t b_base = smem_u32(sB + stage * B_STAGE);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              // K-major: advance 16 elements = 32 B inside the 128 B swizzle row.
              // MN-major: advance 16 K-rows = 2 KiB (two 8-row swizzle atoms).
              const uint64_t ad = A_MN ? make_sw128_desc(a_base + kk * 2048, ATOM, 1024)
                                       : make_sw128_desc(a_base + kk * 32, 16, 1024);
              const uint64_t bd = B_MN ? make_sw128_desc(b_base + kk * 2048, ATOM, 1024)
                                       : make_sw128_desc(b_base + kk * 32, 16, 1024);
              umma_bf16_w(d_tmem, ad, bd, idesc, (first && kk == 0) ? 0u : 1u);
            }
            umma_commit_w(&empty[stage]);
          }
          first = false;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      umma_commit_w(&tmem_full[acc]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue: TMEM -> regs -> global
    const int ew = warp - 4;   // TMEM lanes 32*ew .. 32*ew+31
    int local = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++local) {
      int tg, tm, tn;
      tile_coords(args, t, tg, tm, tn);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      if (local == 0) epilogue_prefetch(args, tm * BM + ew * 32 + lane, tn);
      if (t + (int)gridDim.x < args.num_tiles) {   // the next tile's epilogue inputs
        int ng, nm, nn;
        tile_coords(args, t + gridDim.x, ng, nm, nn);
        epilogue_prefetch(args, nm * BM + ew * 32 + lane, nn);
      }
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row = tm * BM + ew * 32 + lane;
      epilogue_store(args, tmem_base + acc * BN + ((uint32_t)(ew * 32) << 16), row, tg, tn);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
  }

  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem_base);
}


// ------------------------------------------------------------------ 2-CTA variant
// CTA pair (cluster of 2) computes a 256x256 tile with tcgen05.mma.cta_group::2
// (M=256): each CTA stages its 128 rows of A and its 128 columns of B, so the
// pair reads B once for 256 rows (a third less L2->SMEM traffic per MMA than
// the 1-CTA 128x256 tile) and each CTA holds only 32 KiB per stage (6 stages).
// The leader (rank 0) issues the MMAs; both CTAs' TMA bytes complete on the
// leader's full barrier; MMA commits multicast to both CTAs' barriers; both
// epilogues read their own TMEM rows and release the leader's accumulator.
constexpr int STAGES2 = 6;
constexpr int HALF_STAGE = 128 * BK * 2;   // 16 KiB: 128 rows (A) or 128 cols (B) x 64 K
constexpr int SMEM2_BYTES = STAGES2 * 2 * HALF_STAGE + 1024 + 256;

__device__ __forceinline__ void tile_coords_2sm(const KArgs& a, int t, int& g, int& m, int& n) {
  tile_coords(a, t, g, m, n);   // KArgs.tiles_m already counts 256-row tiles
}

template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel_2sm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const KArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * HALF_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES2 * HALF_STAGE);
  uint64_t* empty = full + STAGES2;
  uint64_t* tmem_full = empty + STAGES2;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  // dynamic schedule: a 4-slot ring of claimed tile ids, written by the leader's producer
  // into both CTAs; tile_empty (leader) collects the 10 readers (leader MMA + 4 epilogue
  // warps, peer producer + 4 epilogue warps)
  uint64_t* tile_full = tmem_empty + 3;
  uint64_t* tile_empty = tile_full + 4;
  int* tile_ids = reinterpret_cast<int*>(tile_empty + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = cluster_ctarank();
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const bool dyn = args.tile_ctr != nullptr;
  // the i-th tile of this pair (static: pair + i * npairs), or -1 when none is left; readers
  // release their slot as soon as they hold the id
  auto read_tile = [&](int i, bool release_lane) -> int {
    if (!dyn) {
      const int t = pair + i * npairs;
      return t < args.num_tiles ? t : -1;
    }
    const int slot = i & 3;
    const uint32_t ph = (i >> 2) & 1;
    if (crank == 0) mbar_wait(&tile_full[slot], ph);
    else mbar_wait_cluster(&tile_full[slot], ph);
    const int t = *reinterpret_cast<volatile int*>(&tile_ids[slot]);
    __syncwarp(__activemask());
    if (release_lane) {
      if (crank == 0) mbar_arrive(&tile_empty[slot]);
      else mbar_arrive_cluster(mapa(&tile_empty[slot], 0));
    }
    return t;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 8);   // 4 epilogue warps x 2 CTAs
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&tile_full[s], 1);
      mbar_init(&tile_empty[s], 10);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int g_iters = args.kgroup ? args.G : 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // operand panels are read by every tile of the wave that shares them: L2 evict_last
      // (HLM_GEMM_L2_HINT=0 leaves the default policy, 2 = evict_first)
      // l2_hint < 10: both operands; otherwise tens digit = A's policy, units digit = B's
      auto policy = [](int h) {
        return h == 2 ? l2_policy_evict_first() : h == 1 ? l2_policy_evict_last() : l2_policy_evict_normal();
      };
      const uint64_t pol_a = policy(args.l2_hint < 10 ? args.l2_hint : args.l2_hint / 10 % 10);
      const uint64_t pol_b = policy(args.l2_hint < 10 ? args.l2_hint : args.l2_hint % 10);
      for (int i = 0;; ++i) {
        int t;
        if (dyn && crank == 0) {   // claim the next tile and publish it to both CTAs
          const int slot = i & 3;
          mbar_wait(&tile_empty[slot], ((i >> 2) & 1) ^ 1);
          t = atomicAdd(args.tile_ctr, 1);
          if (t >= args.num_tiles) t = -1;
          tile_ids[slot] = t;
          st_shared_cluster_u32(mapa(&tile_ids[slot], 1), (uint32_t)t);
          mbar_arrive(&tile_full[slot]);
          mbar_arrive_cluster(mapa(&tile_full[slot], 1));
        } else {
          t = read_tile(i, true);
        }
        if (t < 0) break;
        int tg, tm, tn;
        tile_coords_2sm(args, t, tg, tm, tn);
        // paired (SWIGLU): both CTAs load the same 128 output columns, CTA 0 of w_up and
        // CTA 1 of w_gate, so TMEM columns 0..127 / 128..255 are up / gate
        const int m0 = tm * 256 + (int)crank * 128;
        const int n0 = args.paired ? tn * 128 : tn * 256 + (int)crank * 128;
        for (int gi = 0; gi < g_iters; ++gi) {
          const int g = args.kgroup ? gi : tg;
          const int ag = args.a_grouped ? g : 0;
          const int bg = args.paired ? (int)crank : (args.b_grouped ? g : 0);
          for (int kb = 0; kb < args.kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], 4 * HALF_STAGE);
            const int k0 = kb * BK;
            uint8_t* a_dst = sA + stage * HALF_STAGE;
            uint8_t* b_dst = sB + stage * HALF_STAGE;
            if (A_MN) {
              tma_load_3d_2sm_hint(a_dst, &map_a, &full[stage], m0, k0, ag, pol_a);
              tma_load_3d_2sm_hint(a_dst + ATOM, &map_a, &full[stage], m0 + 64, k0, ag, pol_a);
            } else {
              tma_load_3d_2sm_hint(a_dst, &map_a, &full[stage], k0, m0, ag, pol_a);
            }
            if (B_MN) {
              tma_load_3d_2sm_hint(b_dst, &map_b, &full[stage], n0, k0, bg, pol_b);
              tma_load_3d_2sm_hint(b_dst + ATOM, &map_b, &full[stage], n0 + 64, k0, bg, pol_b);
            } else {
              tma_load_3d_2sm_hint(b_dst, &map_b, &full[stage], k0, n0, bg, pol_b);
            }
            if (++stage == STAGES2) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (crank == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      for (int local = 0;; ++local) {
        if (read_tile(local, lane == 0) < 0) break;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        bool first = true;
        for (int gi = 0; gi < g_iters; ++gi) {
          for (int kb = 0; kb < args.kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            {
              const uint32_t a_base = smem_u32(sA + stage * HALF_STAGE);
              const uint32_t b_base = smem_u32(sB + stage * HALF_STAGE);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint64_t ad = A_MN ? make_sw128_desc(a_base + kk * 2048, ATOM, 1024)
                                         : make_sw128_desc(a_base + kk * 32, 16, 1024);
                const uint64_t bd = B_MN ? make_sw128_desc(b_base + kk * 2048, ATOM, 1024)
                                         : make_sw128_desc(b_base + kk * 32, 16, 1024);
                umma_bf16_2sm_w(d_tmem, ad, bd, idesc, (first && kk == 0) ? 0u : 1u);
              }
              umma_commit_2sm_mc_w(&empty[stage]);
            }
            first = false;
            if (++stage == STAGES2) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        umma_commit_2sm_mc_w(&tmem_full[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const uint32_t leader_empty0 = mapa(&tmem_empty[0], 0);
    const uint32_t leader_empty1 = mapa(&tmem_empty[1], 0);
    for (int local = 0;; ++local) {
      const int t = read_tile(local, lane == 0);
      if (t < 0) break;
      int tg, tm, tn;
      tile_coords_2sm(args, t, tg, tm, tn);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      // epilogue inputs: static schedule one tile ahead; dynamic: the next id is not known yet
      if (local == 0 || dyn) epilogue_prefetch(args, tm * 256 + (int)crank * 128 + ew * 32 + lane, tn);
      if (!dyn && t + npairs < args.num_tiles) {   // the next tile's epilogue inputs
        int ng, nm, nn;
        tile_coords_2sm(args, t + npairs, ng, nm, nn);
        epilogue_prefetch(args, nm * 256 + (int)crank * 128 + ew * 32 + lane, nn);
      }
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row = tm * 256 + (int)crank * 128 + ew * 32 + lane;
      epilogue_store(args, tmem_base + acc * 256 + ((uint32_t)(ew * 32) << 16), row, tg, tn);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? leader_empty1 : leader_empty0);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc_2sm<512>(tmem_base);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D bf16 map: dims {inner, outer, groups}; box {64, box_outer, 1}; 128 B swizzle.
int make_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long groups,
             long long ld, long long gstride, int box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return HLM_GEMM_ERR_DRIVER;
  if (groups <= 1) gstride = ld * outer;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(groups < 1 ? 1 : groups)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(gstride * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : HLM_GEMM_ERR_TMAP;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Default: CTA pairs claim tiles from a per-launch counter in raster order, so the tiles in
// flight stay a contiguous window of the raster however far individual pairs drift (the
// static stride lets a slow pair fall whole tiles behind its wave). Measured at C2: -2 %
// serialized block-GEMM time under ncu, the GPU-bound HBM-resident bench variant +2 %
// (908 vs 924-930 ms per step, two A/B pairs), the host-bound headline unchanged (five A/B
// pairs); bitwise equal to the static stride. HLM_GEMM_DYNAMIC=0 restores the static stride.
bool dynamic_schedule() {
  static const int v = [] {
    const char* e = std::getenv("HLM_GEMM_DYNAMIC");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// Per-launch tile counters: a ring of 1024 per device, one slot per launch (zeroed on the
// launch's stream first), so launches in flight on different streams never share one.
int* tile_counter() {
  constexpr int kSlots = 1024, kDevs = 64;
  static int* ring[kDevs] = {};
  static std::atomic<unsigned> next{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kDevs) return nullptr;
  if (!ring[dev]) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!ring[dev] && cudaMalloc(&ring[dev], kSlots * sizeof(int)) != cudaSuccess) {
      ring[dev] = nullptr;
      return nullptr;
    }
  }
  return ring[dev] + next.fetch_add(1, std::memory_order_relaxed) % kSlots;
}

// HLM_GEMM_1SM=1 forces the 1-CTA kernel (A/B comparisons); otherwise the
// 2-CTA kernel serves every non-K-grouped problem with M > 128.
bool use_2sm(int M, int kgroup) {
  static int force1 = -1, kgroup2 = -1;
  if (force1 < 0) {
    const char* e = std::getenv("HLM_GEMM_1SM");
    force1 = (e && *e == '1') ? 1 : 0;
    const char* k = std::getenv("HLM_GEMM_KGROUP_2SM");
    kgroup2 = (k && *k == '0') ? 0 : 1;
  }
  // measured in isolation (late r01, C2 shapes): K-grouped dgrad qkv 1425 TFLOP/s on pair
  // tiles vs 1348 on 1-CTA tiles, dgrad up|gate within noise (1340-1405 either way);
  // HLM_GEMM_KGROUP_2SM=0 routes K-grouped problems to 1-CTA tiles
  return !force1 && M > 128 && (!kgroup || kgroup2);
}

template <bool A_MN, bool B_MN>
int launch(const HlmGemmDesc& d, cudaStream_t stream) {
  const bool two = use_2sm(d.M, d.kgroup);
  CUtensorMap ma, mb;
  int rc;
  const long long ga = d.a_grouped ? d.G : 1, gb = d.b_grouped ? d.G : 1;
  if (A_MN)
    rc = make_map(&ma, d.A, d.M, d.K, ga, d.lda, d.a_gstride, BK);
  else
    rc = make_map(&ma, d.A, d.K, d.M, ga, d.lda, d.a_gstride, 128);
  if (rc) return rc;
  if (B_MN)
    rc = make_map(&mb, d.B, d.N, d.K, gb, d.ldb, d.b_gstride, BK);
  else
    rc = make_map(&mb, d.B, d.K, d.N, gb, d.ldb, d.b_gstride, two ? 128 : BN);
  if (rc) return rc;

  const int tile_m = two ? 256 : BM;
  KArgs a;
  a.M = d.M;
  a.N = d.N;
  a.K = d.K;
  a.G = d.G < 1 ? 1 : d.G;
  a.kgroup = d.kgroup;
  a.a_grouped = d.a_grouped;
  a.b_grouped = d.b_grouped;
  a.paired = d.epi == HLM_EPI_SWIGLU;
  const int tile_n = a.paired ? BN / 2 : BN;
  a.tiles_m = (d.M + tile_m - 1) / tile_m;
  a.tiles_n = (d.N + tile_n - 1) / tile_n;
  a.kblocks = (d.K + BK - 1) / BK;
  a.num_tiles = a.tiles_m * a.tiles_n * ((d.kgroup || a.paired) ? 1 : a.G);
  {
    static int gm_env = -1;
    if (gm_env < 0) {
      const char* e = std::getenv("HLM_GEMM_GROUP_M");
      gm_env = e ? std::atoi(e) : 0;
    }
    // 8 under the dynamic schedule: the 74 tiles in flight span 8 M x ~9 N tiles. Block fwd+bwd
    // at C2 (tools/block_bench.py, power-capped back-to-back): 22.28 vs 22.76 ms with 16; full
    // bench HBM-resident variant 896-901 vs 914-933 ms (profiles/r02/r02_gemm_group_m_ab.jsonl)
    a.group_m = gm_env > 0 ? gm_env : GROUP_M;
  }
  a.C = d.C;
  a.ldc = d.ldc;
  a.c_gstride = d.c_gstride;
  a.R = d.R;
  a.ldr = d.ldr;
  a.r_gstride = d.r_gstride;
  a.epi = d.epi;
  a.rope_cos = d.rope_cos;
  a.rope_sin = d.rope_sin;
  a.rope_seq = d.rope_seq;
  a.rope_hd = d.rope_head_dim;
  a.aux = static_cast<const __nv_bfloat16*>(d.aux);
  a.aux_ld = d.aux_ld;
  a.aux_gstride = d.aux_gstride;
  a.C2 = static_cast<__nv_bfloat16*>(d.C2);
  a.ldc2 = d.ldc2;
  {
    static int pf = -1;
    if (pf < 0) {
      const char* e = std::getenv("HLM_GEMM_L2_PREFETCH");
      pf = (e && *e == '1') ? 1 : 0;
    }
    a.l2_prefetch = pf;
  }
  {
    static int hint = -1;
    if (hint < 0) {
      const char* e = std::getenv("HLM_GEMM_L2_HINT");
      hint = e ? std::atoi(e) : 1;   // evict_last: -5 % DRAM, -2 % time (block GEMMs, ncu)
    }
    a.l2_hint = hint;
  }

  if (two) {
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(gemm_kernel_2sm<A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES);
      attr2 = true;
    }
    const int pairs = a.num_tiles < sm_count() / 2 ? a.num_tiles : sm_count() / 2;
    a.tile_ctr = nullptr;
    if (dynamic_schedule() && a.num_tiles > pairs) {
      a.tile_ctr = tile_counter();
      if (!a.tile_ctr || cudaMemsetAsync(a.tile_ctr, 0, sizeof(int), stream) != cudaSuccess)
        return HLM_GEMM_ERR_LAUNCH;
    }
    gemm_kernel_2sm<A_MN, B_MN><<<2 * pairs, NUM_THREADS, SMEM2_BYTES, stream>>>(ma, mb, a);
  } else {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(gemm_kernel<A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      attr_set = true;
    }
    const int grid = a.num_tiles < sm_count() ? a.num_tiles : sm_count();
    gemm_kernel<A_MN, B_MN><<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ma, mb, a);
  }
  hlm_count_launches(1);
  return cudaGetLastError() == cudaSuccess ? 0 : HLM_GEMM_ERR_LAUNCH;
}

}  // namespace

extern "C" int hlm_gemm_launch(const HlmGemmDesc* d, cudaStream_t stream) {
  if (!d) return HLM_GEMM_ERR_ARGS;
  if (d->M <= 0 || d->N <= 0 || d->K <= 0) return 0;
  if (d->epi == HLM_EPI_F32_ADD && d->R == nullptr) return HLM_GEMM_ERR_ARGS;
  if (d->epi < HLM_EPI_BF16 || d->epi > HLM_EPI_SWIGLU_BWD) return HLM_GEMM_ERR_ARGS;
  if (d->epi == HLM_EPI_BF16_ROPE) {   // whole heads inside a 256-column tile, q and k groups
    const int hd = d->rope_head_dim;
    if (d->kgroup || d->G < 2 || !d->rope_cos || !d->rope_sin || d->rope_seq <= 0 || d->N % 32 ||
        !(hd == 64 || hd == 128 || hd == 256) || d->N % hd || (d->ldc % 8))
      return HLM_GEMM_ERR_ARGS;
  }
  if (d->epi == HLM_EPI_SWIGLU && (d->G != 2 || d->kgroup || !d->b_mn || !d->b_grouped || !d->C2))
    return HLM_GEMM_ERR_ARGS;
  if (d->epi == HLM_EPI_SWIGLU_BWD && (d->G != 1 || d->kgroup || !d->aux)) return HLM_GEMM_ERR_ARGS;
  // TMA: global strides must be multiples of 16 bytes, base 16-byte aligned.
  if ((d->lda * 2) % 16 || (d->ldb * 2) % 16) return HLM_GEMM_ERR_ALIGN;
  if ((reinterpret_cast<uintptr_t>(d->A) & 15) || (reinterpret_cast<uintptr_t>(d->B) & 15))
    return HLM_GEMM_ERR_ALIGN;
  if ((d->a_grouped && (d->a_gstride * 2) % 16) || (d->b_grouped && (d->b_gstride * 2) % 16))
    return HLM_GEMM_ERR_ALIGN;
  if (d->a_mn) {
    if (d->b_mn) return launch<true, true>(*d, stream);
    return launch<true, false>(*d, stream);
  }
  if (d->b_mn) return launch<false, true>(*d, stream);
  return launch<false, false>(*d, stream);
}
