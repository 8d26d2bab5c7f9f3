// tcgen05.mma issue-rate probe (sm_100a): one CTA per SM issues R chains of MMAs of one
// shape back to back into TMEM (operands: whatever sits in shared memory), commit + wait
// per chain; prints cycles per MMA instruction for
//   0: SS M=128 N=64  K=16 (attention S / dP steps)     1: SS M=128 N=128 K=16
//   2: TS M=128 N=128 K=16 (A from TMEM)                3: SS M=128 N=256 K=16 (GEMM tile)
//   4: TS M=128 N=64  K=16
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_04816_b200/csrc/kernels/sm100_ptx.cuh"
using namespace hlm_sm100;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b),
               "r"(idesc), "r"(acc));
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(int chains, int per_chain, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  constexpr int N = (MODE == 0 || MODE == 4) ? 64 : (MODE == 3 ? 256 : 128);
  constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    unsigned long long t0 = clock64();
    for (int c = 0; c < chains; ++c) {
      for (int k = 0; k < per_chain; ++k) {
        const uint64_t ad = make_sw128_desc(a + (k & 3) * 32, 16, 1024);
        const uint64_t bd = make_sw128_desc(b + (k & 3) * 32, 16, 1024);
        if (MODE == 2 || MODE == 4)
          umma_ts(tmem, tmem + 256 + (k & 7) * 8, bd, idesc, 1u);
        else
          umma_bf16_w(tmem, ad, bd, idesc, 1u);
      }
      umma_commit_w(&bar);
      mbar_wait(&bar, c & 1);
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 200 * 1024;
  auto run = [&](auto kern, const char* name, int chains, int per_chain) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, 128, smem>>>(chains, per_chain, d);
    kern<<<148, 128, smem>>>(chains, per_chain, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-34s chain %3d: %7.1f cycles / MMA (%s)\n", name, per_chain, avg / (chains * per_chain),
           cudaGetErrorString(e));
  };
  for (int pc : {8, 32, 256}) {
    run(probe<0>, "SS M128 N64  (attn S/dP)", 2048 / pc * 8, pc);
    run(probe<4>, "TS M128 N64", 2048 / pc * 8, pc);
    run(probe<1>, "SS M128 N128", 2048 / pc * 8, pc);
    run(probe<2>, "TS M128 N128 (attn PV/dV/dK/dQ)", 2048 / pc * 8, pc);
    run(probe<3>, "SS M128 N256 (GEMM)", 2048 / pc * 8, pc);
  }
  return 0;
}
