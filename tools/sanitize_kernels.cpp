// Drives every hand-written kernel family once at small shapes through the C ABI, for
// compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the tcgen05 GEMMs
// (1-CTA and cta_group::2 pair tiles, N-grouped, K-grouped, all majorness variants, the
// three epilogues), the tcgen05 flash attention forward / backward (hd 128) and the
// mma.sync fallback (hd 64), a whole block forward + backward with RoPE, the row- and
// vocab-chunked head + CE, the embedding gather / scatter, the finiteness scan and the
// device Adam. No torch in the process: the sanitizer sees only this library's launches.
//
//   nvcc -std=c++17 -Iinclude tools/sanitize_kernels.cpp -Lpaper_2602_04816_b200 -lhlm_b200 \
//        -Xlinker -rpath=paper_2602_04816_b200 -o tools/sanitize_kernels
//   compute-sanitizer --tool racecheck tools/sanitize_kernels
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "hlm_cuda.h"

namespace {

int failures = 0;

void check(int rc, const char* what) {
    if (rc != 0) {
        std::printf("FAIL %s: %s\n", what, hlm_cuda_last_error());
        ++failures;
    } else {
        std::printf("ok   %s\n", what);
    }
}

std::mt19937 rng(7);

uint16_t bf16(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    return static_cast<uint16_t>((b + 0x7FFF + ((b >> 16) & 1)) >> 16);
}

void* dev_bf16(size_t n, float scale = 1.0f) {
    std::normal_distribution<float> d(0.f, scale);
    std::vector<uint16_t> h(n);
    for (auto& v : h) v = bf16(d(rng));
    void* p = nullptr;
    cudaMalloc(&p, n * 2);
    cudaMemcpy(p, h.data(), n * 2, cudaMemcpyHostToDevice);
    return p;
}

float* dev_f32(size_t n, float scale = 1.0f, float offset = 0.f) {
    std::normal_distribution<float> d(0.f, scale);
    std::vector<float> h(n);
    for (auto& v : h) v = offset + d(rng);
    float* p = nullptr;
    cudaMalloc(&p, n * 4);
    cudaMemcpy(p, h.data(), n * 4, cudaMemcpyHostToDevice);
    return p;
}

void* dev_zero(size_t bytes) {
    void* p = nullptr;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0, bytes);
    return p;
}

void gemm(int M, int N, int K, int a_mn, int b_mn, int epi, int G = 1, int kgroup = 0) {
    HlmGemmDesc d{};
    d.M = M; d.N = N; d.K = K; d.G = G; d.kgroup = kgroup;
    d.a_mn = a_mn; d.b_mn = b_mn; d.epi = epi;
    const long long lda = a_mn ? M : K, ldb = b_mn ? N : K;
    const long long a_elems = static_cast<long long>(a_mn ? K : M) * lda;
    const long long b_elems = static_cast<long long>(b_mn ? K : N) * ldb;
    d.a_grouped = G > 1 && kgroup;
    d.b_grouped = G > 1;
    d.A = dev_bf16(static_cast<size_t>(a_elems * (d.a_grouped ? G : 1)));
    d.lda = lda;
    d.a_gstride = d.a_grouped ? a_elems : 0;
    d.B = dev_bf16(static_cast<size_t>(b_elems * G));
    d.ldb = ldb;
    d.b_gstride = b_elems;
    const int outs = kgroup ? 1 : G;
    d.C = dev_zero(static_cast<size_t>(M) * N * 4 * outs);
    d.ldc = N;
    d.c_gstride = kgroup ? 0 : static_cast<long long>(M) * N;
    if (epi == HLM_EPI_F32_ADD) {
        d.R = dev_f32(static_cast<size_t>(M) * N * outs);
        d.ldr = N;
        d.r_gstride = d.c_gstride;
    }
    char what[160];
    std::snprintf(what, sizeof what, "gemm M%d N%d K%d a_mn%d b_mn%d epi%d G%d kgroup%d", M, N, K, a_mn, b_mn, epi,
                  G, kgroup);
    check(hlm_cuda_gemm(&d, nullptr), what);
    cudaDeviceSynchronize();
    cudaFree(const_cast<void*>(d.A));
    cudaFree(const_cast<void*>(d.B));
    cudaFree(d.C);
    if (d.R) cudaFree(const_cast<float*>(d.R));
}

void attention(int B, int S, int H, int hd, int generic) {
    const int h = H * hd;
    const size_t T = static_cast<size_t>(B) * S;
    HlmBlockDims d{B, S, h, 8, H, generic};
    void *q = dev_bf16(T * h), *k = dev_bf16(T * h), *v = dev_bf16(T * h), *dO = dev_bf16(T * h);
    void* o = dev_zero(T * h * 2);
    float* lse = static_cast<float*>(dev_zero(T * H * 4));
    float* dsum = static_cast<float*>(dev_zero(T * H * 4));
    void *dq = dev_zero(T * h * 2), *dk = dev_zero(T * h * 2), *dv = dev_zero(T * h * 2);
    char what[128];
    std::snprintf(what, sizeof what, "attention fwd B%d S%d H%d hd%d generic%d", B, S, H, hd, generic);
    check(hlm_cuda_attention_fwd(&d, q, k, v, o, lse, h, nullptr), what);
    std::snprintf(what, sizeof what, "attention bwd B%d S%d H%d hd%d generic%d", B, S, H, hd, generic);
    check(hlm_cuda_attention_bwd(&d, q, k, v, o, dO, lse, dsum, dq, dk, dv, h, nullptr), what);
    cudaDeviceSynchronize();
    for (void* p : {q, k, v, dO, o, static_cast<void*>(lse), static_cast<void*>(dsum), dq, dk, dv}) cudaFree(p);
}

void block(int B, int S, int h, int f, int H) {
    HlmBlockDims d{B, S, h, f, H, 0};
    const size_t T = static_cast<size_t>(B) * S;
    const size_t n = 4ull * h * h + 3ull * h * f + 2ull * h;
    void* w = dev_bf16(n, 0.02f);
    float *x = dev_f32(T * h), *y = static_cast<float*>(dev_zero(T * h * 4));
    float *g = dev_f32(T * h, 0.01f), *gi = static_cast<float*>(dev_zero(T * h * 4));
    float* grad = static_cast<float*>(dev_zero(n * 4));
    void* acts = dev_zero(hlm_cuda_block_acts_bytes(&d));
    void* ws = dev_zero(hlm_cuda_block_ws_bytes(&d));
    const int hd = h / H;
    float* cs = static_cast<float*>(dev_zero(static_cast<size_t>(S) * hd / 2 * 4));
    float* sn = static_cast<float*>(dev_zero(static_cast<size_t>(S) * hd / 2 * 4));
    check(hlm_cuda_rope_table(cs, sn, S, hd, 1e6), "rope table");
    check(hlm_cuda_block_fwd(&d, w, x, y, acts, ws, cs, sn, nullptr), "block fwd");
    check(hlm_cuda_block_bwd(&d, w, x, acts, g, gi, grad, ws, cs, sn, nullptr), "block bwd");
    cudaDeviceSynchronize();
    unsigned long long* first = static_cast<unsigned long long*>(dev_zero(8));
    check(hlm_cuda_nonfinite(grad + 1, static_cast<int64_t>(n - 1), first, nullptr), "finiteness scan (misaligned)");
    float *mm = static_cast<float*>(dev_zero(n * 4)), *vv = static_cast<float*>(dev_zero(n * 4));
    float* master = dev_f32(n, 0.02f);
    HlmHyper hp{1e-3, 0.9, 0.999, 1e-8, 0.0};
    check(hlm_cuda_adam(master, mm, vv, w, grad, static_cast<int64_t>(n), first, &hp, 1, nullptr), "device adam");
    cudaDeviceSynchronize();
    for (void* p : {w, static_cast<void*>(x), static_cast<void*>(y), static_cast<void*>(g), static_cast<void*>(gi),
                    static_cast<void*>(grad), acts, ws, static_cast<void*>(cs), static_cast<void*>(sn),
                    static_cast<void*>(first), static_cast<void*>(mm), static_cast<void*>(vv),
                    static_cast<void*>(master)})
        cudaFree(p);
}

void head(int64_t rows, int64_t hid, int64_t V) {
    void* headw = dev_bf16(static_cast<size_t>(V * hid), 0.02f);
    float* x = dev_f32(static_cast<size_t>(rows * hid));
    std::vector<int32_t> tg(static_cast<size_t>(rows));
    for (auto& t : tg) t = static_cast<int32_t>(rng() % V);
    int32_t* tgt = static_cast<int32_t*>(dev_zero(tg.size() * 4));
    cudaMemcpy(tgt, tg.data(), tg.size() * 4, cudaMemcpyHostToDevice);
    float* dx = static_cast<float*>(dev_zero(static_cast<size_t>(rows * hid) * 4));
    float* dh = static_cast<float*>(dev_zero(static_cast<size_t>(V * hid) * 4));
    float* lr = static_cast<float*>(dev_zero(static_cast<size_t>(rows) * 4));
    void* ws = dev_zero(hlm_cuda_head_ws_bytes(rows, hid, V));
    const float inv = 1.0f / static_cast<float>(rows);
    check(hlm_cuda_head_loss(rows, hid, V, headw, x, tgt, inv, dx, dh, 0, lr, ws, nullptr), "head + CE (row chunks)");
    unsigned long long* cert = static_cast<unsigned long long*>(dev_zero(8));
    check(hlm_cuda_head_stats(rows, hid, V, headw, x, tgt, inv, lr, cert, ws, nullptr), "head stats");
    const int64_t vc = hlm_cuda_head_chunk_vocab(rows, V) < V / 2 ? hlm_cuda_head_chunk_vocab(rows, V) : V / 2;
    for (int64_t v0 = 0; v0 < V; v0 += vc) {
        const int64_t n = V - v0 < vc ? V - v0 : vc;
        check(hlm_cuda_head_grad_chunk(rows, hid, V, headw, tgt, inv, v0, n, dx, v0 > 0, dh, 0, ws, nullptr),
              "head grad chunk");
    }
    cudaDeviceSynchronize();
    for (void* p : {headw, static_cast<void*>(x), static_cast<void*>(tgt), static_cast<void*>(dx),
                    static_cast<void*>(dh), static_cast<void*>(lr), ws, static_cast<void*>(cert)})
        cudaFree(p);
}

}  // namespace

int main(int argc, char** argv) {
    const bool quick = argc > 1 && std::strcmp(argv[1], "quick") == 0;
    // GEMMs: 1-CTA (M <= 128), CTA-pair tiles (M > 128), ragged edges, groups, epilogues
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) gemm(128, 256, 128, a, b, HLM_EPI_F32);
    gemm(512, 512, 256, 0, 1, HLM_EPI_BF16);
    gemm(520, 296, 200, 1, 1, HLM_EPI_F32);   // ragged M / N edges (ld multiple of 8 for TMA)
    gemm(512, 512, 256, 0, 1, HLM_EPI_F32_ADD);
    gemm(256, 384, 512, 0, 1, HLM_EPI_BF16, 3, 0);     // N-grouped (qkv)
    gemm(256, 256, 384, 0, 0, HLM_EPI_F32, 2, 1);      // K-grouped (dgrad up|gate)
    gemm(256, 512, 1024, 1, 1, HLM_EPI_F32, 2, 0);     // wgrad (MN-major A and B), grouped
    gemm(4096, 4096, 128, 0, 1, HLM_EPI_F32);          // 256 pair tiles > 74 pairs: dynamic tile claiming
    if (!quick) gemm(1024, 768, 1536, 0, 1, HLM_EPI_F32);
    // attention: tcgen05 (hd 128, S % 128) and mma.sync (hd 64) paths, plus the generic one
    attention(1, 256, 2, 128, 0);   // two-query-tile forward (64-key steps), 64-wide backward
    attention(1, 512, 1, 128, 0);   // the same over 8 steps: K / V and Q / dO rings wrap
    attention(1, 384, 1, 128, 0);   // one-tile forward (S % 256 != 0)
    attention(2, 128, 2, 64, 0);
    attention(1, 64, 2, 32, 1);
    // a whole block with RoPE (hd 128), the head + CE both ways
    block(1, 128, 256, 512, 2);
    head(256, 128, 1024);
    std::printf("sanitize driver: %d failures\n", failures);
    return failures ? 1 : 0;
}
