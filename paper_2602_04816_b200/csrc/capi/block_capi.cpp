// Block / head / embedding orchestration behind the C ABI: the device-side
// equivalents of reference block_forward / block_backward
// (proj/include/hlm/kernels.hpp:313-383), anchor_loss_impl's head + CE
// (proj/src/engine.cpp:227-269) and the embedding gather / scatter.
//
// Every GEMM reads the bf16 weight tile in place (offset-table order,
// proj/src/host_store.cpp:70-92); the three q/k/v (and up/gate) projections
// are single grouped launches. Weight gradients are written straight into the
// fp32 flat tile gradient in the same order, ready for the D2H copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "capi_util.h"
#include "hlm_cuda.h"
#include "../kernels/block_ops.h"
#include "../kernels/gemm.h"
#include "../kernels/attention.h"

namespace {

using i64 = int64_t;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Carves a device buffer into 256-byte aligned pieces in a fixed order.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += align_up(count * sizeof(T));
    return p;
  }
};

struct BlockActs {
  uint16_t *n1, *qkv, *o, *n2, *ug, *act;
  float *lse, *y;
};

BlockActs carve_acts(const HlmBlockDims& d, void* buf, size_t* total) {
  const i64 T = d.batch * d.seq, h = d.hidden, f = d.ffn, H = d.n_heads;
  Carver c(buf);
  BlockActs a;
  a.n1 = c.take<uint16_t>(T * h);
  a.qkv = c.take<uint16_t>(3 * T * h);
  a.o = c.take<uint16_t>(T * h);
  a.lse = c.take<float>(d.batch * H * d.seq);
  a.y = c.take<float>(T * h);
  a.n2 = c.take<uint16_t>(T * h);
  a.ug = c.take<uint16_t>(2 * T * f);
  a.act = c.take<uint16_t>(T * f);
  if (total) *total = c.off;
  return a;
}

struct BlockWs {
  uint16_t *g_bf, *d_act, *dug, *d_y_bf, *d_o, *dqkv;
  float *d_n, *d_y, *dsum, *inv, *partial;
};

BlockWs carve_ws(const HlmBlockDims& d, void* buf, size_t* total) {
  const i64 T = d.batch * d.seq, h = d.hidden, f = d.ffn, H = d.n_heads;
  Carver c(buf);
  BlockWs w;
  w.g_bf = c.take<uint16_t>(T * h);
  w.d_act = c.take<uint16_t>(T * f);
  w.dug = c.take<uint16_t>(2 * T * f);
  w.d_y_bf = c.take<uint16_t>(T * h);
  w.d_o = c.take<uint16_t>(T * h);
  w.dqkv = c.take<uint16_t>(3 * T * h);
  w.d_n = c.take<float>(T * h);
  w.d_y = c.take<float>(T * h);
  w.dsum = c.take<float>(d.batch * H * d.seq);
  w.inv = c.take<float>(T);
  w.partial = c.take<float>(((T + HLM_NORM_ROWS_PER_CHUNK - 1) / HLM_NORM_ROWS_PER_CHUNK) * h);
  if (total) *total = c.off;
  return w;
}

// Tile offsets (elements), host_store.cpp:70-92.
struct TileOff {
  i64 q, o, up, down, norm1, norm2;
  TileOff(i64 h, i64 f)
      : q(0), o(3 * h * h), up(4 * h * h), down(4 * h * h + 2 * h * f), norm1(4 * h * h + 3 * h * f),
        norm2(4 * h * h + 3 * h * f + h) {}
};

HlmGemmDesc gdesc(int M, int N, int K, const void* A, i64 lda, int a_mn, const void* B, i64 ldb, int b_mn,
                  void* C, i64 ldc, int epi) {
  HlmGemmDesc g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.G = 1;
  g.A = A;
  g.lda = lda;
  g.a_mn = a_mn;
  g.B = B;
  g.ldb = ldb;
  g.b_mn = b_mn;
  g.C = C;
  g.ldc = ldc;
  g.epi = epi;
  return g;
}

struct Failure {
  std::string msg;
  int code;
};

void chk_gemm(const HlmGemmDesc& g, cudaStream_t s, const char* what) {
  const int tk = hlm_capi::ktimer_begin(s);
  const int rc = hlm_gemm_launch(&g, s);
  hlm_capi::ktimer_end(tk, s, HLM_KTIMER_GEMM, 2.0 * g.M * g.N * (double)g.K * (g.G > 0 ? g.G : 1));
  if (rc) throw Failure{std::string("gemm ") + what + " failed (code " + std::to_string(rc) + ")", HLM_ERR_CUDA};
}
void chk(int rc, const char* what) {
  if (rc) {
    const cudaError_t e = cudaGetLastError();
    throw Failure{std::string(what) + " launch failed: " + cudaGetErrorString(e), HLM_ERR_CUDA};
  }
}
// An HBM-bound launch timed by the kernel timer (work = algorithmic bytes).
template <typename F>
void timed(int kind, double bytes, cudaStream_t s, F&& launch) {
  const int tk = hlm_capi::ktimer_begin(s);
  launch();
  hlm_capi::ktimer_end(tk, s, kind, bytes);
}

// Fused GEMM epilogues (RoPE, SwiGLU fwd / bwd) unless the caller asks for the separate
// kernels (HLM_BLOCK_UNFUSED) or HLM_FUSE=0 is set for an A/B run.
bool fused(const HlmBlockDims& d) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("HLM_FUSE");
    env = (e && *e == '0') ? 0 : 1;
  }
  return env && !(d.flags & HLM_BLOCK_UNFUSED);
}

// The SwiGLU backward in the down-dgrad epilogue is off by default: measured at C2 (ncu,
// tools/block_bench.py) the epilogue's up / gate reads stall the accumulator hand-off and
// the GEMM drops to 50 % tensor-pipe activity (2.24 ms vs 1.46 ms + 0.47 ms for the
// separate swiglu_bwd kernel). HLM_FUSE_SWIGLU_BWD=1 turns it on (bit-identical).
bool fuse_swiglu_bwd() {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("HLM_FUSE_SWIGLU_BWD");
    env = (e && *e == '1') ? 1 : 0;
  }
  return env != 0;
}

void validate(const HlmBlockDims* d) {
  if (!d || d->batch <= 0 || d->seq <= 0 || d->hidden <= 0 || d->ffn <= 0 || d->n_heads <= 0)
    throw Failure{"block dims must be positive", HLM_ERR_CONFIG};
  if (d->hidden % 8 || d->ffn % 8)
    throw Failure{"hidden and ffn must be multiples of 8 (16-byte TMA rows)", HLM_ERR_CONFIG};
  if (d->hidden % d->n_heads) throw Failure{"hidden must be divisible by n_heads", HLM_ERR_CONFIG};
}

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return HLM_OK;
  } catch (const Failure& f) {
    hlm_capi::set_error(f.msg);
    return f.code;
  }
}

void attention_fwd(const HlmBlockDims& d, const uint16_t* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                   float* lse, i64 ld, cudaStream_t s) {
  const int hd = static_cast<int>(d.hidden / d.n_heads);
  // causal attention flops: 2 * B * S^2 * h forward
  const double fl = 2.0 * d.batch * (double)d.seq * d.seq * d.hidden;
  const int tk = hlm_capi::ktimer_begin(s);
  struct End {
    int tk; cudaStream_t s; double fl;
    ~End() { hlm_capi::ktimer_end(tk, s, HLM_KTIMER_ATTN_FWD, fl); }
  } end{tk, s, fl};
  if (!(d.flags & HLM_BLOCK_GENERIC_ATTENTION) && hlm_flash_supported(hd, static_cast<int>(d.seq))) {
    chk(hlm_flash_fwd(q, k, v, o, lse, (int)d.batch, (int)d.seq, (int)d.n_heads, hd, (int)ld, s), "flash fwd");
  } else {
    chk(hlm_ops_attention_fwd_generic(q, k, v, o, lse, (int)d.batch, (int)d.seq, (int)d.n_heads, hd, (int)ld, s),
        "attention fwd");
  }
}

void attention_bwd(const HlmBlockDims& d, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                   const uint16_t* o, const uint16_t* d_o, const float* lse, float* dsum, uint16_t* dq,
                   uint16_t* dk, uint16_t* dv, i64 ld, cudaStream_t s) {
  const int hd = static_cast<int>(d.hidden / d.n_heads);
  // backward = 2.5 x forward flops (dV, dP, dQ, dK: 4 + 1 recomputed S per tile pair, causal)
  const double fl = 2.5 * 2.0 * d.batch * (double)d.seq * d.seq * d.hidden;
  const int tk = hlm_capi::ktimer_begin(s);
  struct End {
    int tk; cudaStream_t s; double fl;
    ~End() { hlm_capi::ktimer_end(tk, s, HLM_KTIMER_ATTN_BWD, fl); }
  } end{tk, s, fl};
  if (!(d.flags & HLM_BLOCK_GENERIC_ATTENTION) && hlm_flash_supported(hd, static_cast<int>(d.seq))) {
    chk(hlm_flash_bwd(q, k, v, o, d_o, lse, dsum, dq, dk, dv, (int)d.batch, (int)d.seq, (int)d.n_heads, hd,
                      (int)ld, s),
        "flash bwd");
  } else {
    chk(hlm_ops_attention_bwd_generic(q, k, v, o, d_o, lse, dsum, dq, dk, dv, (int)d.batch, (int)d.seq,
                                      (int)d.n_heads, hd, (int)ld, s),
        "attention bwd");
  }
}

void** hlm_timer_events() {
  static void* ev[16] = {};
  return ev;
}

}  // namespace

extern "C" {

size_t hlm_cuda_block_acts_bytes(const HlmBlockDims* d) {
  size_t t = 0;
  carve_acts(*d, nullptr, &t);
  return t;
}

size_t hlm_cuda_block_ws_bytes(const HlmBlockDims* d) {
  size_t t = 0;
  carve_ws(*d, nullptr, &t);
  return t;
}

int hlm_cuda_block_fwd(const HlmBlockDims* d, const void* w_tile, const float* h_in, float* h_out, void* acts,
                       void* ws, const float* rope_cos, const float* rope_sin, void* stream) {
  (void)ws;
  return guarded([&] {
    validate(d);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const i64 T = d->batch * d->seq, h = d->hidden, f = d->ffn;
    const int Ti = (int)T, hi = (int)h, fi = (int)f;
    const TileOff off(h, f);
    const uint16_t* W = static_cast<const uint16_t*>(w_tile);
    BlockActs a = carve_acts(*d, acts, nullptr);

    const bool fuse = fused(*d);
    const int hd = (int)(h / d->n_heads);
    const bool rope_fused = fuse && rope_cos && (hd == 64 || hd == 128 || hd == 256) && h % 32 == 0;
    timed(HLM_KTIMER_RMSNORM_FWD, 6.0 * T * h, s, [&] { chk(hlm_ops_rmsnorm_fwd(h_in, W + off.norm1, a.n1, T, hi, s), "rmsnorm1"); });
    HlmGemmDesc g = gdesc(Ti, hi, hi, a.n1, h, 0, W + off.q, h, 1, a.qkv, h, HLM_EPI_BF16);
    g.G = 3;
    g.b_grouped = 1;
    g.b_gstride = h * h;
    g.c_gstride = T * h;
    if (rope_fused) {   // RoPE of q and k in the projection's epilogue
      g.epi = HLM_EPI_BF16_ROPE;
      g.rope_cos = rope_cos;
      g.rope_sin = rope_sin;
      g.rope_seq = (int)d->seq;
      g.rope_head_dim = hd;
    }
    chk_gemm(g, s, "qkv");
    if (rope_cos && !rope_fused)
      timed(HLM_KTIMER_ROPE, 8.0 * T * h, s, [&] {
        chk(hlm_ops_rope(a.qkv, rope_cos, rope_sin, T, hi, hd, (int)d->seq, 0, 2, T * h, s), "rope");
      });
    attention_fwd(*d, a.qkv, a.qkv + T * h, a.qkv + 2 * T * h, a.o, a.lse, h, s);
    g = gdesc(Ti, hi, hi, a.o, h, 0, W + off.o, h, 1, a.y, h, HLM_EPI_F32_ADD);
    g.R = h_in;
    g.ldr = h;
    chk_gemm(g, s, "o-proj");
    timed(HLM_KTIMER_RMSNORM_FWD, 6.0 * T * h, s, [&] { chk(hlm_ops_rmsnorm_fwd(a.y, W + off.norm2, a.n2, T, hi, s), "rmsnorm2"); });
    g = gdesc(Ti, fi, hi, a.n2, h, 0, W + off.up, f, 1, a.ug, f, HLM_EPI_BF16);
    g.G = 2;
    g.b_grouped = 1;
    g.b_gstride = h * f;
    g.c_gstride = T * f;
    if (fuse) {   // act = up * silu(gate) in the epilogue of paired up|gate tiles
      g.epi = HLM_EPI_SWIGLU;
      g.C2 = a.act;
      g.ldc2 = f;
    }
    chk_gemm(g, s, "up|gate");
    if (!fuse)
      timed(HLM_KTIMER_SWIGLU_FWD, 6.0 * T * f, s, [&] { chk(hlm_ops_swiglu_fwd(a.ug, a.act, T * f, s), "swiglu"); });
    g = gdesc(Ti, hi, fi, a.act, f, 0, W + off.down, h, 1, h_out, h, HLM_EPI_F32_ADD);
    g.R = a.y;
    g.ldr = h;
    chk_gemm(g, s, "down");
  });
}

int hlm_cuda_block_bwd(const HlmBlockDims* d, const void* w_tile, const float* h_in, const void* acts,
                       const float* g_out, float* g_in, float* grad_tile, void* ws, const float* rope_cos,
                       const float* rope_sin, void* stream) {
  return guarded([&] {
    validate(d);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const i64 T = d->batch * d->seq, h = d->hidden, f = d->ffn;
    const int Ti = (int)T, hi = (int)h, fi = (int)f;
    const TileOff off(h, f);
    const uint16_t* W = static_cast<const uint16_t*>(w_tile);
    const BlockActs a = carve_acts(*d, const_cast<void*>(acts), nullptr);
    BlockWs w = carve_ws(*d, ws, nullptr);
    float* G = grad_tile;

    // MLP branch
    timed(HLM_KTIMER_CAST, 6.0 * T * h, s, [&] { chk(hlm_ops_cast_bf16(g_out, w.g_bf, T * h, s), "cast g_out"); });
    chk_gemm(gdesc(fi, hi, Ti, a.act, f, 1, w.g_bf, h, 1, G + off.down, h, HLM_EPI_F32), s, "wgrad down");
    if (fused(*d) && fuse_swiglu_bwd()) {   // d_act never stored: SwiGLU backward in the dgrad epilogue
      HlmGemmDesc gd = gdesc(Ti, fi, hi, w.g_bf, h, 0, W + off.down, h, 0, w.dug, f, HLM_EPI_SWIGLU_BWD);
      gd.c_gstride = T * f;
      gd.aux = a.ug;
      gd.aux_ld = f;
      gd.aux_gstride = T * f;
      chk_gemm(gd, s, "dgrad down + swiglu bwd");
    } else {
      chk_gemm(gdesc(Ti, fi, hi, w.g_bf, h, 0, W + off.down, h, 0, w.d_act, f, HLM_EPI_BF16), s, "dgrad down");
      timed(HLM_KTIMER_SWIGLU_BWD, 10.0 * T * f, s, [&] { chk(hlm_ops_swiglu_bwd(w.d_act, a.ug, w.dug, T * f, s), "swiglu bwd"); });
    }
    HlmGemmDesc g = gdesc(hi, fi, Ti, a.n2, h, 1, w.dug, f, 1, G + off.up, f, HLM_EPI_F32);
    g.G = 2;
    g.b_grouped = 1;
    g.b_gstride = T * f;
    g.c_gstride = h * f;
    chk_gemm(g, s, "wgrad up|gate");
    g = gdesc(Ti, hi, fi, w.dug, f, 0, W + off.up, f, 0, w.d_n, h, HLM_EPI_F32);
    g.G = 2;
    g.kgroup = 1;
    g.a_grouped = 1;
    g.a_gstride = T * f;
    g.b_grouped = 1;
    g.b_gstride = h * f;
    chk_gemm(g, s, "dgrad up|gate");
    timed(HLM_KTIMER_RMSNORM_BWD, 18.0 * T * h, s, [&] {
      chk(hlm_ops_rmsnorm_bwd(a.y, W + off.norm2, w.d_n, g_out, w.d_y, w.d_y_bf, w.inv, w.partial, G + off.norm2,
                              T, hi, s),
          "rmsnorm2 bwd");
    });
    // attention branch
    chk_gemm(gdesc(hi, hi, Ti, a.o, h, 1, w.d_y_bf, h, 1, G + off.o, h, HLM_EPI_F32), s, "wgrad o");
    chk_gemm(gdesc(Ti, hi, hi, w.d_y_bf, h, 0, W + off.o, h, 0, w.d_o, h, HLM_EPI_BF16), s, "dgrad o");
    attention_bwd(*d, a.qkv, a.qkv + T * h, a.qkv + 2 * T * h, a.o, w.d_o, a.lse, w.dsum, w.dqkv, w.dqkv + T * h,
                  w.dqkv + 2 * T * h, h, s);
    if (rope_cos)
      timed(HLM_KTIMER_ROPE, 8.0 * T * h, s, [&] {
        chk(hlm_ops_rope(w.dqkv, rope_cos, rope_sin, T, hi, hi / d->n_heads, (int)d->seq, 1, 2, T * h, s),
            "rope bwd");
      });
    g = gdesc(hi, hi, Ti, a.n1, h, 1, w.dqkv, h, 1, G + off.q, h, HLM_EPI_F32);
    g.G = 3;
    g.b_grouped = 1;
    g.b_gstride = T * h;
    g.c_gstride = h * h;
    chk_gemm(g, s, "wgrad qkv");
    g = gdesc(Ti, hi, hi, w.dqkv, h, 0, W + off.q, h, 0, w.d_n, h, HLM_EPI_F32);
    g.G = 3;
    g.kgroup = 1;
    g.a_grouped = 1;
    g.a_gstride = T * h;
    g.b_grouped = 1;
    g.b_gstride = h * h;
    chk_gemm(g, s, "dgrad qkv");
    timed(HLM_KTIMER_RMSNORM_BWD, 16.0 * T * h, s, [&] {
      chk(hlm_ops_rmsnorm_bwd(h_in, W + off.norm1, w.d_n, w.d_y, g_in, nullptr, w.inv, w.partial, G + off.norm1,
                              T, hi, s),
          "rmsnorm1 bwd");
    });
  });
}

int hlm_cuda_rope_table(float* dev_cos, float* dev_sin, int64_t seq, int64_t head_dim, double theta) {
  return guarded([&] {
    if (head_dim % 2 || theta <= 0) throw Failure{"rope table: even head_dim and theta > 0 required", HLM_ERR_CONFIG};
    const i64 half = head_dim / 2;
    std::vector<float> c(static_cast<size_t>(seq * half)), sn(c.size());
    for (i64 p = 0; p < seq; ++p)
      for (i64 i = 0; i < half; ++i) {
        // identical to oracle/hlm_oracle.cpp Rope (double math, fp32 angle)
        const double inv = std::pow(theta, -2.0 * static_cast<double>(i) / static_cast<double>(head_dim));
        const float ang = static_cast<float>(static_cast<double>(p) * inv);
        c[p * half + i] = static_cast<float>(std::cos(static_cast<double>(ang)));
        sn[p * half + i] = static_cast<float>(std::sin(static_cast<double>(ang)));
      }
    if (cudaMemcpy(dev_cos, c.data(), c.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dev_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      throw Failure{"rope table copy failed", HLM_ERR_CUDA};
  });
}

// ------------------------------------------------------------------ head + loss
static i64 padded_vocab(i64 V) { return (V + 7) / 8 * 8; }

// Rows per head chunk: logits (fp32) + d_logits (bf16) of one chunk fit in
// ~kHeadChunkBytes, so the (T, V) buffers of the reference never exist whole.
static const int64_t kHeadChunkBytes = 2ll << 30;
static i64 head_chunk_rows(i64 rows, i64 vocab) {
  i64 r = kHeadChunkBytes / (6 * padded_vocab(vocab));
  r = r / 128 * 128;
  if (r < 128) r = 128;
  return r < rows ? r : rows;
}

size_t hlm_cuda_head_ws_bytes(int64_t rows, int64_t hidden, int64_t vocab) {
  Carver c(nullptr);
  const i64 ldv = padded_vocab(vocab), cr = head_chunk_rows(rows, vocab);
  c.take<uint16_t>(rows * hidden);
  c.take<float>(cr * ldv);
  c.take<uint16_t>(cr * ldv);
  c.take<int>(4);
  c.take<float>(2 * rows);   // vocab-chunked head: per-row (max, 1/z)
  return c.off;
}

int64_t hlm_cuda_head_chunk_vocab(int64_t rows, int64_t vocab) {
  if (rows <= 0 || vocab <= 0) return 0;
  const i64 ldv = padded_vocab(vocab), cr = head_chunk_rows(rows, vocab);
  const i64 cap = cr * ldv / rows;   // padded columns per row the logits / d_logits regions hold
  if (cap >= vocab) return vocab;
  return cap >= 128 ? cap / 128 * 128 : std::max<i64>(8, cap / 8 * 8);
}

namespace {
struct HeadWs {
  uint16_t* x_bf;
  float* logits;
  uint16_t* dl;
  int* err;
  float* stats;
};
HeadWs carve_head(void* ws, i64 rows, i64 hidden, i64 vocab) {
  const i64 ldv = padded_vocab(vocab), cr = head_chunk_rows(rows, vocab);
  Carver c(ws);
  HeadWs w;
  w.x_bf = c.take<uint16_t>(rows * hidden);
  w.logits = c.take<float>(cr * ldv);
  w.dl = c.take<uint16_t>(cr * ldv);
  w.err = c.take<int>(4);
  w.stats = c.take<float>(2 * rows);
  return w;
}
}  // namespace

int hlm_cuda_head_stats(int64_t rows, int64_t hidden, int64_t vocab, const void* head, const float* x,
                        const int32_t* targets, float inv_rows, float* loss_rows, unsigned long long* cert,
                        void* ws, void* stream) {
  return guarded([&] {
    if (rows <= 0 || hidden <= 0 || vocab <= 0 || hidden % 8)
      throw Failure{"head: bad dims (hidden must be a multiple of 8)", HLM_ERR_CONFIG};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const i64 ldv = padded_vocab(vocab), cr = head_chunk_rows(rows, vocab);
    HeadWs w = carve_head(ws, rows, hidden, vocab);
    chk(hlm_ops_cast_bf16(x, w.x_bf, rows * hidden, s), "cast x");
    for (i64 r0 = 0; r0 < rows; r0 += cr) {
      const i64 n = rows - r0 < cr ? rows - r0 : cr;
      chk_gemm(gdesc((int)n, (int)vocab, (int)hidden, w.x_bf + r0 * hidden, hidden, 0, head, hidden, 0, w.logits,
                     ldv, HLM_EPI_F32),
               s, "head fwd");
      chk(hlm_ops_ce_stats(w.logits, ldv, targets + r0, w.stats + 2 * r0, loss_rows + r0, n, (int)vocab, inv_rows,
                           w.err, s),
          "ce stats");
    }
    // |d_head| <= rows * inv_rows * 1.01 * max|x|: certify far below FLT_MAX
    const double lim = 1e36 / std::max(1.0, static_cast<double>(rows) * static_cast<double>(inv_rows));
    chk(hlm_ops_head_certify(w.x_bf, rows * hidden, w.stats, rows, static_cast<float>(std::min(lim, 1e36)), cert,
                             s),
        "head certificate");
  });
}

int hlm_cuda_head_grad_chunk(int64_t rows, int64_t hidden, int64_t vocab, const void* head,
                             const int32_t* targets, float inv_rows, int64_t v0, int64_t vc, float* d_x,
                             int accumulate_d_x, float* d_head, int accumulate_d_head, void* ws, void* stream) {
  return guarded([&] {
    if (rows <= 0 || hidden <= 0 || vocab <= 0 || hidden % 8)
      throw Failure{"head: bad dims (hidden must be a multiple of 8)", HLM_ERR_CONFIG};
    if (v0 < 0 || vc <= 0 || v0 + vc > vocab || vc > hlm_cuda_head_chunk_vocab(rows, vocab))
      throw Failure{"head: bad vocab chunk", HLM_ERR_ARGS};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    HeadWs w = carve_head(ws, rows, hidden, vocab);
    const i64 ld = (vc + 7) / 8 * 8;
    const uint16_t* hc = static_cast<const uint16_t*>(head) + v0 * hidden;
    const int R = (int)rows, Hh = (int)hidden, Vc = (int)vc;
    chk_gemm(gdesc(R, Vc, Hh, w.x_bf, hidden, 0, hc, hidden, 0, w.logits, ld, HLM_EPI_F32), s, "head fwd chunk");
    chk(hlm_ops_ce_grad_chunk(w.logits, ld, targets, w.stats, w.dl, ld, rows, (int)v0, Vc, inv_rows, s),
        "ce grad chunk");
    HlmGemmDesc gw = gdesc(Vc, Hh, R, w.dl, ld, 1, w.x_bf, hidden, 1, d_head + v0 * hidden, hidden,
                           accumulate_d_head ? HLM_EPI_F32_ADD : HLM_EPI_F32);
    if (accumulate_d_head) {
      gw.R = d_head + v0 * hidden;
      gw.ldr = hidden;
    }
    chk_gemm(gw, s, "head wgrad chunk");
    HlmGemmDesc gd = gdesc(R, Hh, Vc, w.dl, ld, 0, hc, hidden, 1, d_x, hidden,
                           accumulate_d_x ? HLM_EPI_F32_ADD : HLM_EPI_F32);
    if (accumulate_d_x) {
      gd.R = d_x;
      gd.ldr = hidden;
    }
    chk_gemm(gd, s, "head dgrad chunk");
  });
}

// Chunked over rows: per chunk, logits = x_c . head^T (fp32), CE -> d_logits_c
// (bf16), d_x_c = d_logits_c . head, d_head (+)= d_logits_c^T . x_c (the first
// chunk stores or accumulates per the caller, later chunks accumulate).
int hlm_cuda_head_loss(int64_t rows, int64_t hidden, int64_t vocab, const void* head, const float* x,
                       const int32_t* targets, float inv_rows, float* d_x, float* d_head, int accumulate_d_head,
                       float* loss_rows, void* ws, void* stream) {
  return guarded([&] {
    if (rows <= 0 || hidden <= 0 || vocab <= 0 || hidden % 8)
      throw Failure{"head: bad dims (hidden must be a multiple of 8)", HLM_ERR_CONFIG};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const i64 ldv = padded_vocab(vocab), cr = head_chunk_rows(rows, vocab);
    Carver c(ws);
    uint16_t* x_bf = c.take<uint16_t>(rows * hidden);
    float* logits = c.take<float>(cr * ldv);
    uint16_t* dl = c.take<uint16_t>(cr * ldv);
    int* err = c.take<int>(4);
    const int Hh = (int)hidden, V = (int)vocab;
    chk(hlm_ops_cast_bf16(x, x_bf, rows * hidden, s), "cast x");
    for (i64 r0 = 0; r0 < rows; r0 += cr) {
      const i64 n = rows - r0 < cr ? rows - r0 : cr;
      const int R = (int)n;
      const uint16_t* xc = x_bf + r0 * hidden;
      chk_gemm(gdesc(R, V, Hh, xc, hidden, 0, head, hidden, 0, logits, ldv, HLM_EPI_F32), s, "head fwd");
      chk(hlm_ops_ce(logits, ldv, targets + r0, dl, ldv, loss_rows + r0, n, V, inv_rows, err, s), "cross entropy");
      chk_gemm(gdesc(R, Hh, V, dl, ldv, 0, head, hidden, 1, d_x + r0 * hidden, hidden, HLM_EPI_F32), s, "head dgrad");
      const bool acc = accumulate_d_head || r0 > 0;
      HlmGemmDesc g = gdesc(V, Hh, R, dl, ldv, 1, xc, hidden, 1, d_head, hidden, acc ? HLM_EPI_F32_ADD : HLM_EPI_F32);
      if (acc) {
        g.R = d_head;
        g.ldr = hidden;
      }
      chk_gemm(g, s, "head wgrad");
    }
  });
}

// ------------------------------------------------------------------ embedding
int hlm_cuda_embed_fwd(const int32_t* tokens, const void* table, float* out, int64_t rows, int64_t hidden,
                       int64_t vocab, int* err_flag, void* stream) {
  return guarded([&] {
    chk(hlm_ops_embed_fwd(tokens, table, out, rows, (int)hidden, (int)vocab, err_flag,
                          static_cast<cudaStream_t>(stream)),
        "embed fwd");
  });
}

int hlm_cuda_embed_bwd(const int32_t* row_ptr, const int32_t* pos, const float* g, float* d_table, int64_t vocab,
                       int64_t hidden, int accumulate, void* stream) {
  return guarded([&] {
    chk(hlm_ops_embed_bwd(row_ptr, pos, g, d_table, (int)vocab, (int)hidden, accumulate,
                          static_cast<cudaStream_t>(stream)),
        "embed bwd");
  });
}

int hlm_cuda_embed_bwd_compact(const int32_t* row_ptr, const int32_t* pos, const int32_t* rows, int64_t n_rows,
                               const float* g, float* out, int64_t hidden, void* stream) {
  return guarded([&] {
    chk(hlm_ops_embed_bwd_compact(row_ptr, pos, rows, (int)n_rows, g, out, (int)hidden,
                                  static_cast<cudaStream_t>(stream)),
        "embed bwd compact");
  });
}

int hlm_embed_csr(const int32_t* tokens, int64_t rows, int64_t vocab, int32_t* row_ptr, int32_t* pos) {
  for (int64_t v = 0; v <= vocab; ++v) row_ptr[v] = 0;
  for (int64_t t = 0; t < rows; ++t) {
    if (tokens[t] < 0 || tokens[t] >= vocab) {
      hlm_capi::set_error("embed_bwd: token id out of range");
      return HLM_ERR_RANGE;
    }
    ++row_ptr[tokens[t] + 1];
  }
  for (int64_t v = 0; v < vocab; ++v) row_ptr[v + 1] += row_ptr[v];
  std::vector<int32_t> fill(row_ptr, row_ptr + vocab);
  for (int64_t t = 0; t < rows; ++t) pos[fill[tokens[t]]++] = static_cast<int32_t>(t);
  return HLM_OK;
}

// ------------------------------------------------------------------ small ops
int hlm_cuda_adam(float* w, float* m, float* v, void* w16, const float* g, int64_t n, const unsigned long long* bad,
                  const HlmHyper* hp, int64_t t, void* stream) {
  return guarded([&] {
    if (t < 1) throw Failure{"adam step index must be >= 1", HLM_ERR_PROTOCOL};
    const float lr = (float)hp->lr, b1 = (float)hp->beta1, b2 = (float)hp->beta2, eps = (float)hp->eps,
                wd = (float)hp->weight_decay;
    const float bc1 = 1.0f - std::pow(b1, static_cast<float>(t));   // as the host (host_store.cpp)
    const float bc2 = 1.0f - std::pow(b2, static_cast<float>(t));
    chk(hlm_ops_adam_device(w, m, v, w16, g, n, bad, lr, b1, b2, eps, wd, bc1, bc2, static_cast<cudaStream_t>(stream)),
        "adam device");
  });
}

int hlm_cuda_nonfinite(const float* g, int64_t n, unsigned long long* first, void* stream) {
  return guarded([&] { chk(hlm_ops_nonfinite(g, n, first, nullptr, static_cast<cudaStream_t>(stream)), "nonfinite"); });
}

int hlm_cuda_nonfinite_if_uncertified(const float* g, int64_t n, unsigned long long* first,
                                      const unsigned long long* certificate, void* stream) {
  return guarded([&] {
    chk(hlm_ops_nonfinite(g, n, first, certificate, static_cast<cudaStream_t>(stream)), "nonfinite (fallback)");
  });
}

int hlm_cuda_cast_bf16(const float* in, void* out, int64_t n, void* stream) {
  return guarded([&] { chk(hlm_ops_cast_bf16(in, out, n, static_cast<cudaStream_t>(stream)), "cast"); });
}

int hlm_cuda_attention_fwd(const HlmBlockDims* d, const void* q, const void* k, const void* v, void* o, float* lse,
                           int64_t ld, void* stream) {
  return guarded([&] {
    validate(d);
    attention_fwd(*d, (const uint16_t*)q, (const uint16_t*)k, (const uint16_t*)v, (uint16_t*)o, lse, ld,
                  static_cast<cudaStream_t>(stream));
  });
}

int hlm_cuda_attention_bwd(const HlmBlockDims* d, const void* q, const void* k, const void* v, const void* o,
                           const void* d_o, const float* lse, float* dsum, void* dq, void* dk, void* dv, int64_t ld,
                           void* stream) {
  return guarded([&] {
    validate(d);
    attention_bwd(*d, (const uint16_t*)q, (const uint16_t*)k, (const uint16_t*)v, (const uint16_t*)o,
                  (const uint16_t*)d_o, lse, dsum, (uint16_t*)dq, (uint16_t*)dk, (uint16_t*)dv, ld,
                  static_cast<cudaStream_t>(stream));
  });
}

int hlm_timer_record(int slot) {
  static cudaEvent_t ev[16] = {};
  if (slot < 0 || slot >= 16) return HLM_ERR_ARGS;
  if (!ev[slot]) cudaEventCreate(&ev[slot]);
  cudaDeviceSynchronize();
  cudaEventRecord(ev[slot], 0);
  cudaEventSynchronize(ev[slot]);
  hlm_timer_events()[slot] = ev[slot];
  return HLM_OK;
}

double hlm_timer_elapsed_ms(int a, int b) {
  float ms = -1.f;
  cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(hlm_timer_events()[a]), static_cast<cudaEvent_t>(hlm_timer_events()[b]));
  return ms;
}

int hlm_cuda_bench_block_gemms(const HlmBlockDims* d, int iters, double* flops, double* ms_per_set, double* ms_per_launch) {
  return guarded([&] {
    validate(d);
    const i64 T = d->batch * d->seq, h = d->hidden, f = d->ffn;
    const int Ti = (int)T, hi = (int)h, fi = (int)f;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto alloc = [s](size_t bytes) {
      void* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess) throw Failure{"bench alloc failed", HLM_ERR_CUDA};
      // random bf16 bit patterns in [-1, 1) magnitude range: zero operands understate tensor-core power
      hlm_ops_fill_random_bf16(p, static_cast<long long>(bytes / 2), 0x1234u, s);
      return p;
    };
    const i64 n = 4 * h * h + 3 * h * f + 2 * h;
    uint16_t* W = (uint16_t*)alloc(n * 2);
    uint16_t* X = (uint16_t*)alloc(T * f * 2);      // activations (T,h) / (T,f)
    uint16_t* X3 = (uint16_t*)alloc(3 * T * h * 2);
    uint16_t* U = (uint16_t*)alloc(2 * T * f * 2);
    float* Y = (float*)alloc(T * f * 4);
    float* G = (float*)alloc(n * 4);
    const TileOff off(h, f);
    std::vector<HlmGemmDesc> set;
    HlmGemmDesc g = gdesc(Ti, hi, hi, X, h, 0, W + off.q, h, 1, X3, h, HLM_EPI_BF16);
    g.G = 3; g.b_grouped = 1; g.b_gstride = h * h; g.c_gstride = T * h; set.push_back(g);
    set.push_back(gdesc(Ti, hi, hi, X, h, 0, W + off.o, h, 1, Y, h, HLM_EPI_F32));
    g = gdesc(Ti, fi, hi, X, h, 0, W + off.up, f, 1, U, f, HLM_EPI_BF16);
    g.G = 2; g.b_grouped = 1; g.b_gstride = h * f; g.c_gstride = T * f; set.push_back(g);
    set.push_back(gdesc(Ti, hi, fi, X, f, 0, W + off.down, h, 1, Y, h, HLM_EPI_F32));
    set.push_back(gdesc(fi, hi, Ti, X, f, 1, X, h, 1, G + off.down, h, HLM_EPI_F32));
    set.push_back(gdesc(Ti, fi, hi, X, h, 0, W + off.down, h, 0, U, f, HLM_EPI_BF16));
    g = gdesc(hi, fi, Ti, X, h, 1, U, f, 1, G + off.up, f, HLM_EPI_F32);
    g.G = 2; g.b_grouped = 1; g.b_gstride = T * f; g.c_gstride = h * f; set.push_back(g);
    g = gdesc(Ti, hi, fi, U, f, 0, W + off.up, f, 0, Y, h, HLM_EPI_F32);
    g.G = 2; g.kgroup = 1; g.a_grouped = 1; g.a_gstride = T * f; g.b_grouped = 1; g.b_gstride = h * f; set.push_back(g);
    set.push_back(gdesc(hi, hi, Ti, X, h, 1, X, h, 1, G + off.o, h, HLM_EPI_F32));
    set.push_back(gdesc(Ti, hi, hi, X, h, 0, W + off.o, h, 0, X3, h, HLM_EPI_BF16));
    g = gdesc(hi, hi, Ti, X, h, 1, X3, h, 1, G + off.q, h, HLM_EPI_F32);
    g.G = 3; g.b_grouped = 1; g.b_gstride = T * h; g.c_gstride = h * h; set.push_back(g);
    g = gdesc(Ti, hi, hi, X3, h, 0, W + off.q, h, 0, Y, h, HLM_EPI_F32);
    g.G = 3; g.kgroup = 1; g.a_grouped = 1; g.a_gstride = T * h; g.b_grouped = 1; g.b_gstride = h * h; set.push_back(g);
    double fl = 0;
    for (const auto& q : set) fl += 2.0 * q.M * (double)q.N * q.K * (q.G > 1 ? q.G : 1);
    for (const auto& q : set) chk_gemm(q, s, "bench warmup");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int it = 0; it < iters; ++it)
      for (const auto& q : set) chk_gemm(q, s, "bench");
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *flops = fl;
    *ms_per_set = ms / iters;
    *ms_per_launch = ms / iters / (double)set.size();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    for (void* p : {(void*)W, (void*)X, (void*)X3, (void*)U, (void*)Y, (void*)G}) cudaFree(p);
    cudaStreamDestroy(s);
  });
}

// Achieved HBM bandwidth of the block's elementwise / norm kernels at the
// workload shape (random data, CUDA events, `iters` back-to-back launches).
// Algorithmic bytes per call (each tensor read / written once):
//   0 rmsnorm_fwd  x f32 -> bf16              6 B x T*h
//   1 rmsnorm_bwd  x, g, resid f32 -> f32 + bf16 (+ scale grad)   18 B x T*h
//   2 swiglu_fwd   up, gate bf16 -> act       6 B x T*f
//   3 swiglu_bwd   d_act, up, gate -> d_up, d_gate   10 B x T*f
//   4 rope         q, k bf16 in place         8 B x T*h
//   5 cast         f32 -> bf16                6 B x T*h
int hlm_cuda_bench_block_ops(const HlmBlockDims* d, int iters, double* gbs, double* ms_out) {
  return guarded([&] {
    validate(d);
    const i64 T = d->batch * d->seq, h = d->hidden, f = d->ffn;
    const int hd = (int)(h / d->n_heads);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    std::vector<void*> bufs;
    auto alloc = [&](size_t bytes) {
      void* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess) throw Failure{"bench alloc failed", HLM_ERR_CUDA};
      hlm_ops_fill_random_bf16(p, static_cast<long long>(bytes / 2), 0x9e37u, s);
      bufs.push_back(p);
      return p;
    };
    float* x = (float*)alloc(T * h * 4);
    float* g = (float*)alloc(T * h * 4);
    float* resid = (float*)alloc(T * h * 4);
    float* out = (float*)alloc(T * h * 4);
    void* out_bf = alloc(T * h * 2);
    void* scale = alloc(h * 2);
    float* inv = (float*)alloc(T * 4);
    float* partial = (float*)alloc(((T + HLM_NORM_ROWS_PER_CHUNK - 1) / HLM_NORM_ROWS_PER_CHUNK) * h * 4);
    float* dscale = (float*)alloc(h * 4);
    void* ug = alloc(2 * T * f * 2);
    void* act = alloc(T * f * 2);
    void* dug = alloc(2 * T * f * 2);
    void* qk = alloc(2 * T * h * 2);
    float* cs = (float*)alloc(d->seq * (hd / 2) * 4);
    float* sn = (float*)alloc(d->seq * (hd / 2) * 4);
    const double bytes[6] = {6.0 * T * h, 18.0 * T * h, 6.0 * T * f, 10.0 * T * f, 8.0 * T * h, 6.0 * T * h};
    auto run = [&](int k) {
      switch (k) {
        case 0: chk(hlm_ops_rmsnorm_fwd(x, scale, out_bf, T, (int)h, s), "rmsnorm fwd"); break;
        case 1:
          chk(hlm_ops_rmsnorm_bwd(x, scale, g, resid, out, out_bf, inv, partial, dscale, T, (int)h, s), "rmsnorm bwd");
          break;
        case 2: chk(hlm_ops_swiglu_fwd(ug, act, T * f, s), "swiglu fwd"); break;
        case 3: chk(hlm_ops_swiglu_bwd(act, ug, dug, T * f, s), "swiglu bwd"); break;
        case 4: chk(hlm_ops_rope(qk, cs, sn, T, (int)h, hd, (int)d->seq, 0, 2, T * h, s), "rope"); break;
        default: chk(hlm_ops_cast_bf16(x, out_bf, T * h, s), "cast"); break;
      }
    };
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < 6; ++k) {
      run(k);
      cudaEventRecord(a, s);
      for (int it = 0; it < iters; ++it) run(k);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double per = ms / iters;
      if (ms_out) ms_out[k] = per;
      gbs[k] = bytes[k] / (per * 1e-3) / 1e9;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    for (void* p : bufs) cudaFree(p);
    cudaStreamDestroy(s);
  });
}

}  // extern "C"
