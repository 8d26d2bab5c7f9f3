// hlm_oracle.cpp — CPU restatement of the reference's layer-streaming
// training step, used ONLY as the parity checker (tests/, smoke(), bench.py's
// cpu_baseline leg). Never linked into libhlm_b200.so.
//
// Each function restates the reference algorithm it cites (paths relative to
// /root/reference/proj). Loop orders follow the reference so that in
// reference semantics (n_heads == 1, rope_theta == 0) results are bitwise
// identical to the compiled reference (checked by tests/test_oracle.py against
// oracle/_ref/libhlm_ref.so and the committed golden fixtures).
//
// Extension beyond the reference (SURVEY.md §7 hard part 1): multi-head
// causal attention (n_heads, head_dim = h / n_heads, scale 1/sqrt(head_dim))
// and Qwen2-style rotate-half RoPE on q and k after the projection. Neither
// adds parameters, so tile layouts and every size formula are unchanged.
// This path has no reference implementation; it is validated by reduction to
// the reference at n_heads = 1 / no RoPE and by central finite differences
// (tests/test_oracle.py), as reference tests/test_kernels.cpp:114-146 does.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_abi.h"

namespace orc {

using i64 = int64_t;

// ---------------------------------------------------------------- BF16
// include/hlm/bf16.hpp:15-25: RNE via (bits + 0x7FFF + lsb) >> 16; Inf passes;
// NaN keeps sign/upper payload and sets the quiet bit 0x0040.
uint16_t bf16_bits(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  if (((b >> 23) & 0xFFu) == 0xFFu) {
    uint16_t hi = static_cast<uint16_t>(b >> 16);
    if (b & 0x7FFFFFu) hi |= 0x0040u;
    return hi;
  }
  return static_cast<uint16_t>((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}
float bf16_widen(uint16_t h) {
  const uint32_t b = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}
float bf16_round(float x) { return bf16_widen(bf16_bits(x)); }

// ---------------------------------------------------------------- RNG
// include/hlm/tensor.hpp:86-131: mt19937 seeded with the low 32 bits;
// uniform = top 24 bits / 2^24; Box-Muller with a cached spare; truncated
// normal resamples outside +-2 sigma; uniform_int(n) = gen() % n.
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(static_cast<uint32_t>(seed)) {}
  float uniform() { return static_cast<float>(gen_() >> 8) * (1.0f / 16777216.0f); }
  float normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    float u1;
    do {
      u1 = uniform();
    } while (u1 <= 1e-12f);
    const float u2 = uniform();
    const float r = std::sqrt(-2.0f * std::log(u1));
    const float a = 6.2831853071795864769f * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }
  float trunc_normal(float sd) {
    float v;
    do {
      v = normal() * sd;
    } while (v < -2.0f * sd || v > 2.0f * sd);
    return v;
  }
  int32_t uniform_int(int32_t n) { return static_cast<int32_t>(gen_() % static_cast<uint32_t>(n)); }

 private:
  std::mt19937 gen_;
  bool have_spare_ = false;
  float spare_ = 0.0f;
};

// ---------------------------------------------------------------- config
struct Cfg {
  i64 L, h, f, V, S, B, K;
  bool tie;
  i64 heads;
  double theta;
  i64 hd() const { return h / heads; }
  i64 rows() const { return B * S; }
  i64 block_params() const { return 4 * h * h + 3 * h * f + 2 * h; }   // model_config.hpp:42
  i64 table_params() const { return V * h; }
  i64 total_params() const {                                           // model_config.hpp:67-71
    return table_params() * (tie ? 1 : 2) + L * block_params();
  }
  i64 block_offset(i64 l) const { return table_params() + (l - 1) * block_params(); }
  i64 head_offset() const { return tie ? 0 : table_params() + L * block_params(); }
};

Cfg from_abi(const OrcCfg* c) {
  Cfg g{c->layers, c->hidden, c->ffn, c->vocab, c->seq, c->batch, c->k_ckpt, c->tie != 0,
        c->n_heads < 1 ? 1 : c->n_heads, c->rope_theta};
  if (g.L <= 0 || g.h <= 0 || g.f <= 0 || g.V <= 0 || g.S <= 0 || g.B <= 0)
    throw std::invalid_argument("oracle config: dimensions must be positive");
  if (g.h % g.heads) throw std::invalid_argument("oracle config: hidden % n_heads != 0");
  if (g.theta > 0 && g.hd() % 2) throw std::invalid_argument("oracle config: odd head_dim with RoPE");
  return g;
}

// Block tile views in offset-table order (host_store.cpp:70-92).
template <typename T>
struct BlockView {
  T *w_q, *w_k, *w_v, *w_o, *w_up, *w_gate, *w_down, *norm1, *norm2;
};
template <typename T>
BlockView<T> block_view(T* base, i64 h, i64 f) {
  BlockView<T> v;
  T* p = base;
  auto take = [&](i64 n) {
    T* r = p;
    p += n;
    return r;
  };
  v.w_q = take(h * h);
  v.w_k = take(h * h);
  v.w_v = take(h * h);
  v.w_o = take(h * h);
  v.w_up = take(h * f);
  v.w_gate = take(h * f);
  v.w_down = take(f * h);
  v.norm1 = take(h);
  v.norm2 = take(h);
  return v;
}

// ---------------------------------------------------------------- kernels
constexpr double kEps = 1e-6;   // kernels.hpp:127

// kernels.hpp:129-140
template <typename T>
void rmsnorm_fwd(const T* x, const T* s, T* out, i64 rows, i64 h) {
  for (i64 r = 0; r < rows; ++r) {
    const T* xr = x + r * h;
    T ms = T(0);
    for (i64 j = 0; j < h; ++j) ms += xr[j] * xr[j];
    const T inv = T(1) / std::sqrt(ms / T(h) + T(kEps));
    for (i64 j = 0; j < h; ++j) out[r * h + j] = xr[j] * inv * s[j];
  }
}

// kernels.hpp:142-162 (g_x assigned, g_s accumulated)
template <typename T>
void rmsnorm_bwd(const T* x, const T* s, const T* g, T* gx, T* gs, i64 rows, i64 h) {
  for (i64 r = 0; r < rows; ++r) {
    const T* xr = x + r * h;
    const T* gr = g + r * h;
    T ms = T(0);
    for (i64 j = 0; j < h; ++j) ms += xr[j] * xr[j];
    const T inv = T(1) / std::sqrt(ms / T(h) + T(kEps));
    T dot = T(0);
    for (i64 j = 0; j < h; ++j) {
      gs[j] += gr[j] * xr[j] * inv;
      dot += gr[j] * s[j] * xr[j];
    }
    const T c = inv * inv * inv * dot / T(h);
    for (i64 j = 0; j < h; ++j) gx[r * h + j] = gr[j] * s[j] * inv - c * xr[j];
  }
}

// kernels.hpp:164-176: out = a . W, W (K,N)
template <typename T>
void mm_nn(const T* a, const T* w, T* out, i64 rows, i64 K, i64 N) {
  for (i64 r = 0; r < rows; ++r) {
    T* o = out + r * N;
    for (i64 n = 0; n < N; ++n) o[n] = T(0);
    for (i64 k = 0; k < K; ++k) {
      const T av = a[r * K + k];
      for (i64 n = 0; n < N; ++n) o[n] += av * w[k * N + n];
    }
  }
}

// kernels.hpp:178-190: out = a . W^T, W (K,N); a is (rows,N)
template <typename T>
void mm_nt(const T* a, const T* w, T* out, i64 rows, i64 N, i64 K, bool accumulate) {
  for (i64 r = 0; r < rows; ++r)
    for (i64 k = 0; k < K; ++k) {
      T acc = T(0);
      for (i64 n = 0; n < N; ++n) acc += a[r * N + n] * w[k * N + n];
      out[r * K + k] = accumulate ? out[r * K + k] + acc : acc;
    }
}

// kernels.hpp:192-205: dw += x^T . g (zero rows of x skipped)
template <typename T>
void mm_grad_acc(const T* x, const T* g, T* dw, i64 rows, i64 K, i64 N) {
  for (i64 r = 0; r < rows; ++r)
    for (i64 k = 0; k < K; ++k) {
      const T xv = x[r * K + k];
      if (xv == T(0)) continue;
      for (i64 n = 0; n < N; ++n) dw[k * N + n] += xv * g[r * N + n];
    }
}

// RoPE table: angle(pos, i) = pos * theta^(-2i/hd), evaluated in double and
// rounded to the compute type (the GPU path uses the same table).
struct Rope {
  std::vector<double> c, s;   // [S][hd/2]
  i64 half = 0;
  Rope(i64 S, i64 hd, double theta) : half(hd / 2) {
    c.resize(static_cast<size_t>(S * half));
    s.resize(c.size());
    for (i64 p = 0; p < S; ++p)
      for (i64 i = 0; i < half; ++i) {
        const double inv = std::pow(theta, -2.0 * static_cast<double>(i) / static_cast<double>(hd));
        const float a = static_cast<float>(static_cast<double>(p) * inv);
        c[p * half + i] = static_cast<double>(static_cast<float>(std::cos(static_cast<double>(a))));
        s[p * half + i] = static_cast<double>(static_cast<float>(std::sin(static_cast<double>(a))));
      }
  }
};

// rotate-half RoPE over every head of x (rows, h); inverse = transpose rotation.
template <typename T>
void rope_apply(T* x, const Rope& R, const Cfg& g, bool inverse) {
  const i64 hd = g.hd(), half = hd / 2;
  for (i64 r = 0; r < g.rows(); ++r) {
    const i64 pos = r % g.S;
    for (i64 hh = 0; hh < g.heads; ++hh) {
      T* v = x + r * g.h + hh * hd;
      for (i64 i = 0; i < half; ++i) {
        const T c = T(R.c[pos * half + i]), s = T(R.s[pos * half + i]);
        const T a = v[i], b = v[i + half];
        if (!inverse) {
          v[i] = a * c - b * s;
          v[i + half] = b * c + a * s;
        } else {
          v[i] = a * c + b * s;
          v[i + half] = b * c - a * s;
        }
      }
    }
  }
}

// kernels.hpp:207-245, per head: p (B,H,S,S) causal softmax probabilities,
// attn = p . v. With heads == 1 this is the reference loop exactly.
template <typename T>
void attention_fwd(const T* q, const T* k, const T* v, T* p, T* attn, const Cfg& g) {
  const i64 S = g.S, h = g.h, hd = g.hd();
  const T scale = T(1) / std::sqrt(T(hd));
  for (i64 b = 0; b < g.B; ++b)
    for (i64 hh = 0; hh < g.heads; ++hh) {
      const i64 c0 = hh * hd;
      T* pb = p + (b * g.heads + hh) * S * S;
      for (i64 i = 0; i < S; ++i) {
        T* pr = pb + i * S;
        T mx = T(0);
        for (i64 j = 0; j <= i; ++j) {
          T sc = T(0);
          for (i64 d = 0; d < hd; ++d) sc += q[(b * S + i) * h + c0 + d] * k[(b * S + j) * h + c0 + d];
          sc *= scale;
          pr[j] = sc;
          if (j == 0 || sc > mx) mx = sc;
        }
        T z = T(0);
        for (i64 j = 0; j <= i; ++j) {
          pr[j] = std::exp(pr[j] - mx);
          z += pr[j];
        }
        const T inv = T(1) / z;
        for (i64 j = 0; j <= i; ++j) pr[j] *= inv;
        for (i64 j = i + 1; j < S; ++j) pr[j] = T(0);
        T* ar = attn + (b * S + i) * h + c0;
        for (i64 d = 0; d < hd; ++d) ar[d] = T(0);
        for (i64 j = 0; j <= i; ++j)
          for (i64 d = 0; d < hd; ++d) ar[d] += pr[j] * v[(b * S + j) * h + c0 + d];
      }
    }
}

// kernels.hpp:247-299, per head; d_q, d_k, d_v assigned.
template <typename T>
void attention_bwd(const T* q, const T* k, const T* v, const T* p, const T* da, T* dq, T* dk, T* dv,
                   const Cfg& g) {
  const i64 S = g.S, h = g.h, hd = g.hd();
  const T scale = T(1) / std::sqrt(T(hd));
  std::vector<T> dp(static_cast<size_t>(S * S));
  for (i64 b = 0; b < g.B; ++b)
    for (i64 hh = 0; hh < g.heads; ++hh) {
      const i64 c0 = hh * hd;
      const T* pb = p + (b * g.heads + hh) * S * S;
      auto at = [&](const T* x, i64 s, i64 d) -> T { return x[(b * S + s) * h + c0 + d]; };
      for (i64 j = 0; j < S; ++j)
        for (i64 d = 0; d < hd; ++d) dv[(b * S + j) * h + c0 + d] = T(0);
      for (i64 i = 0; i < S; ++i) {
        const T* pr = pb + i * S;
        T* dpr = dp.data() + i * S;
        for (i64 j = 0; j <= i; ++j) {
          T sc = T(0);
          for (i64 d = 0; d < hd; ++d) sc += at(da, i, d) * at(v, j, d);
          dpr[j] = sc;
          for (i64 d = 0; d < hd; ++d) dv[(b * S + j) * h + c0 + d] += pr[j] * at(da, i, d);
        }
        T dot = T(0);
        for (i64 j = 0; j <= i; ++j) dot += dpr[j] * pr[j];
        for (i64 j = 0; j <= i; ++j) dpr[j] = pr[j] * (dpr[j] - dot);
        for (i64 j = i + 1; j < S; ++j) dpr[j] = T(0);
      }
      for (i64 i = 0; i < S; ++i) {
        T* dqr = dq + (b * S + i) * h + c0;
        for (i64 d = 0; d < hd; ++d) dqr[d] = T(0);
        for (i64 j = 0; j <= i; ++j) {
          const T ds = dp[i * S + j] * scale;
          for (i64 d = 0; d < hd; ++d) dqr[d] += ds * at(k, j, d);
        }
      }
      for (i64 j = 0; j < S; ++j)
        for (i64 d = 0; d < hd; ++d) dk[(b * S + j) * h + c0 + d] = T(0);
      for (i64 i = 0; i < S; ++i)
        for (i64 j = 0; j <= i; ++j) {
          const T ds = dp[i * S + j] * scale;
          for (i64 d = 0; d < hd; ++d) dk[(b * S + j) * h + c0 + d] += ds * at(q, i, d);
        }
    }
}

// kernels.hpp:301-311
template <typename T>
T silu(T z) {
  const T s = T(1) / (T(1) + std::exp(-z));
  return z * s;
}
template <typename T>
T silu_grad(T z) {
  const T s = T(1) / (T(1) + std::exp(-z));
  return s * (T(1) + z * (T(1) - s));
}

template <typename T>
struct Acts {   // per-block saved state (q, k are post-RoPE)
  std::vector<T> h_in, n1, q, k, v, p, attn, y, n2, up, gate;
};

// kernels.hpp:313-332, plus the RoPE/multi-head extension.
template <typename T>
void block_forward(const T* h_in, const BlockView<const T>& w, const Cfg& g, const Rope* rope,
                   Acts<T>& a, T* h_out) {
  const i64 rows = g.rows(), h = g.h, f = g.f;
  auto sz = [](i64 n) { return static_cast<size_t>(n); };
  a.h_in.assign(h_in, h_in + rows * h);
  a.n1.resize(sz(rows * h));
  a.q.resize(sz(rows * h));
  a.k.resize(sz(rows * h));
  a.v.resize(sz(rows * h));
  a.p.resize(sz(g.B * g.heads * g.S * g.S));
  a.attn.resize(sz(rows * h));
  a.y.resize(sz(rows * h));
  a.n2.resize(sz(rows * h));
  a.up.resize(sz(rows * f));
  a.gate.resize(sz(rows * f));
  std::vector<T> th0(sz(rows * h)), fa(sz(rows * f)), th1(sz(rows * h));
  rmsnorm_fwd(h_in, w.norm1, a.n1.data(), rows, h);
  mm_nn(a.n1.data(), w.w_q, a.q.data(), rows, h, h);
  mm_nn(a.n1.data(), w.w_k, a.k.data(), rows, h, h);
  mm_nn(a.n1.data(), w.w_v, a.v.data(), rows, h, h);
  if (rope) {
    rope_apply(a.q.data(), *rope, g, false);
    rope_apply(a.k.data(), *rope, g, false);
  }
  attention_fwd(a.q.data(), a.k.data(), a.v.data(), a.p.data(), a.attn.data(), g);
  mm_nn(a.attn.data(), w.w_o, th0.data(), rows, h, h);
  for (i64 i = 0; i < rows * h; ++i) a.y[i] = h_in[i] + th0[i];
  rmsnorm_fwd(a.y.data(), w.norm2, a.n2.data(), rows, h);
  mm_nn(a.n2.data(), w.w_up, a.up.data(), rows, h, f);
  mm_nn(a.n2.data(), w.w_gate, a.gate.data(), rows, h, f);
  for (i64 i = 0; i < rows * f; ++i) fa[i] = a.up[i] * silu(a.gate[i]);
  mm_nn(fa.data(), w.w_down, th1.data(), rows, f, h);
  for (i64 i = 0; i < rows * h; ++i) h_out[i] = a.y[i] + th1[i];
}

// kernels.hpp:334-383 (parameter grads accumulated into gr; g_in assigned).
template <typename T>
void block_backward(const BlockView<const T>& w, const Cfg& g, const Rope* rope, const Acts<T>& a,
                    const T* g_out, T* g_in, const BlockView<T>& gr) {
  const i64 rows = g.rows(), h = g.h, f = g.f;
  auto sz = [](i64 n) { return static_cast<size_t>(n); };
  std::vector<T> fa(sz(rows * f)), fb(sz(rows * f)), fc(sz(rows * f));
  std::vector<T> th0(sz(rows * h)), th1(sz(rows * h)), th2(sz(rows * h)), th3(sz(rows * h)),
      qd(sz(rows * h)), kd(sz(rows * h)), dattn(sz(rows * h));
  for (i64 i = 0; i < rows * f; ++i) fa[i] = silu(a.gate[i]);
  for (i64 i = 0; i < rows * f; ++i) fb[i] = a.up[i] * fa[i];
  mm_grad_acc(fb.data(), g_out, gr.w_down, rows, f, h);
  mm_nt(g_out, w.w_down, fb.data(), rows, h, f, false);   // d_act
  for (i64 i = 0; i < rows * f; ++i) fc[i] = fb[i] * fa[i];                         // d_up
  for (i64 i = 0; i < rows * f; ++i) fb[i] = fb[i] * a.up[i] * silu_grad(a.gate[i]);  // d_gate
  mm_grad_acc(a.n2.data(), fc.data(), gr.w_up, rows, h, f);
  mm_grad_acc(a.n2.data(), fb.data(), gr.w_gate, rows, h, f);
  mm_nt(fc.data(), w.w_up, th0.data(), rows, f, h, false);
  mm_nt(fb.data(), w.w_gate, th0.data(), rows, f, h, true);   // d_n2
  rmsnorm_bwd(a.y.data(), w.norm2, th0.data(), th1.data(), gr.norm2, rows, h);
  for (i64 i = 0; i < rows * h; ++i) th1[i] += g_out[i];   // d_y
  mm_grad_acc(a.attn.data(), th1.data(), gr.w_o, rows, h, h);
  mm_nt(th1.data(), w.w_o, dattn.data(), rows, h, h, false);   // d_attn
  attention_bwd(a.q.data(), a.k.data(), a.v.data(), a.p.data(), dattn.data(), th0.data(),
                th2.data(), th3.data(), g);
  if (rope) {
    rope_apply(th0.data(), *rope, g, true);
    rope_apply(th2.data(), *rope, g, true);
  }
  mm_grad_acc(a.n1.data(), th0.data(), gr.w_q, rows, h, h);
  mm_grad_acc(a.n1.data(), th2.data(), gr.w_k, rows, h, h);
  mm_grad_acc(a.n1.data(), th3.data(), gr.w_v, rows, h, h);
  mm_nt(th0.data(), w.w_q, qd.data(), rows, h, h, false);
  mm_nt(th2.data(), w.w_k, qd.data(), rows, h, h, true);
  mm_nt(th3.data(), w.w_v, qd.data(), rows, h, h, true);   // d_n1
  rmsnorm_bwd(a.h_in.data(), w.norm1, qd.data(), kd.data(), gr.norm1, rows, h);
  for (i64 i = 0; i < rows * h; ++i) g_in[i] = th1[i] + kd[i];
}

// kernels.hpp:423-446: mean CE; d_logits = (softmax - onehot) / rows.
// `inv_rows_override` > 0 replaces 1/rows (data-parallel: 1/global_rows).
template <typename T>
T ce_loss_and_grad(const T* logits, const int32_t* tgt, T* dl, i64 rows, i64 V, T inv_rows) {
  T loss = T(0);
  for (i64 r = 0; r < rows; ++r) {
    if (tgt[r] < 0 || tgt[r] >= V) throw std::out_of_range("ce_loss_and_grad: target id out of range");
    const T* lr = logits + r * V;
    T* dr = dl + r * V;
    T mx = lr[0];
    for (i64 v = 1; v < V; ++v) mx = lr[v] > mx ? lr[v] : mx;
    T z = T(0);
    for (i64 v = 0; v < V; ++v) z += std::exp(lr[v] - mx);
    const T logz = std::log(z) + mx;
    loss += (logz - lr[tgt[r]]) * inv_rows;
    const T invz = T(1) / z;
    for (i64 v = 0; v < V; ++v) dr[v] = std::exp(lr[v] - mx) * invz * inv_rows;
    dr[tgt[r]] -= inv_rows;
  }
  return loss;
}

// Whole-model forward + backward: engine.cpp:176-368 semantics (the result is
// independent of the checkpoint interval K, reference test_engine.cpp:212).
// params/grads in store layout; tied tables get head then embed contributions.
template <typename T>
T forward_backward(const Cfg& g, const T* params, const int32_t* tokens, const int32_t* targets,
                   T* grads, T inv_rows) {
  const i64 rows = g.rows(), h = g.h, V = g.V;
  for (i64 i = 0; i < g.total_params(); ++i) grads[i] = T(0);
  std::unique_ptr<Rope> rope;
  if (g.theta > 0) rope.reset(new Rope(g.S, g.hd(), g.theta));
  std::vector<T> x(static_cast<size_t>(rows * h)), nx(x.size());
  // embed_fwd kernels.hpp:385-394
  for (i64 t = 0; t < rows; ++t) {
    if (tokens[t] < 0 || tokens[t] >= V) throw std::out_of_range("embed_fwd: token id out of range");
    for (i64 j = 0; j < h; ++j) x[t * h + j] = params[static_cast<i64>(tokens[t]) * h + j];
  }
  std::vector<Acts<T>> acts(static_cast<size_t>(g.L));
  for (i64 l = 1; l <= g.L; ++l) {
    const auto w = block_view<const T>(params + g.block_offset(l), h, g.f);
    block_forward(x.data(), w, g, rope.get(), acts[static_cast<size_t>(l - 1)], nx.data());
    std::swap(x, nx);
  }
  // head_fwd / ce / head_bwd kernels.hpp:410-421 (engine.cpp:227-269)
  const T* head = params + g.head_offset();
  std::vector<T> logits(static_cast<size_t>(rows * V)), dl(logits.size()), gx(x.size()), gy(x.size());
  mm_nt(x.data(), head, logits.data(), rows, h, V, false);
  const T loss = ce_loss_and_grad(logits.data(), targets, dl.data(), rows, V, inv_rows);
  std::vector<T> dhead(static_cast<size_t>(V * h), T(0));
  mm_nn(dl.data(), head, gx.data(), rows, V, h);
  mm_grad_acc(dl.data(), x.data(), dhead.data(), rows, V, h);
  for (i64 l = g.L; l >= 1; --l) {
    const auto w = block_view<const T>(params + g.block_offset(l), h, g.f);
    const auto gr = block_view<T>(grads + g.block_offset(l), h, g.f);
    block_backward(w, g, rope.get(), acts[static_cast<size_t>(l - 1)], gx.data(), gy.data(), gr);
    std::swap(gx, gy);
  }
  // embed_bwd_acc kernels.hpp:396-408, in token order
  std::vector<T> dembed(static_cast<size_t>(V * h), T(0));
  for (i64 t = 0; t < rows; ++t)
    for (i64 j = 0; j < h; ++j) dembed[static_cast<i64>(tokens[t]) * h + j] += gx[t * h + j];
  if (g.tie) {
    // SlabPool accumulation order: head slab first, then embed (engine.cpp:255-368).
    for (i64 i = 0; i < V * h; ++i) grads[i] = (T(0) + dhead[i]) + dembed[i];
  } else {
    for (i64 i = 0; i < V * h; ++i) grads[i] = dembed[i];
    for (i64 i = 0; i < V * h; ++i) grads[g.head_offset() + i] = dhead[i];
  }
  return loss;
}

// host_store.cpp:334-362: FP32 Adam with bias correction powf(beta, t).
void adam(float* w, const float* gr, float* m, float* v, i64 n, const OrcHyper& hp, i64 t,
          bool bf16_weights) {
  const float lr = static_cast<float>(hp.lr), b1 = static_cast<float>(hp.beta1),
              b2 = static_cast<float>(hp.beta2), eps = static_cast<float>(hp.eps),
              wd = static_cast<float>(hp.weight_decay);
  const float bc1 = 1.0f - std::pow(b1, static_cast<float>(t));
  const float bc2 = 1.0f - std::pow(b2, static_cast<float>(t));
  for (i64 i = 0; i < n; ++i) {
    const float g = gr[i];
    m[i] = b1 * m[i] + (1.0f - b1) * g;
    v[i] = b2 * v[i] + (1.0f - b2) * g * g;
    const float mhat = m[i] / bc1;
    const float vhat = v[i] / bc2;
    float th = w[i];
    th -= lr * (mhat / (std::sqrt(vhat) + eps) + wd * th);
    w[i] = bf16_weights ? bf16_round(th) : th;
  }
}

// host_store.cpp:141-156: one Rng over physical tiles in store order; norms
// 1.0, everything else trunc_normal(0.02); stored through the dtype.
void init_weights(const Cfg& g, uint64_t seed, bool bf16, float* out) {
  Rng rng(seed);
  auto put = [&](float v) { *out++ = bf16 ? bf16_round(v) : v; };
  for (i64 i = 0; i < g.V * g.h; ++i) put(rng.trunc_normal(0.02f));
  for (i64 l = 1; l <= g.L; ++l) {
    const i64 n_mat = 4 * g.h * g.h + 3 * g.h * g.f;
    for (i64 i = 0; i < n_mat; ++i) put(rng.trunc_normal(0.02f));
    for (i64 i = 0; i < 2 * g.h; ++i) put(1.0f);
  }
  if (!g.tie)
    for (i64 i = 0; i < g.V * g.h; ++i) put(rng.trunc_normal(0.02f));
}

// engine.cpp:434-441: tokens uniform_int(V) in (b, s) order; targets = tokens.
void copy_task(const Cfg& g, Rng& rng, int32_t* tokens) {
  for (i64 i = 0; i < g.rows(); ++i) tokens[i] = rng.uniform_int(static_cast<int32_t>(g.V));
}

}  // namespace orc

// ====================================================================== ABI
namespace {
thread_local std::string g_err;
template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
uint16_t orc_bf16_bits(float x) { return orc::bf16_bits(x); }
int64_t orc_total_params(const OrcCfg* c) { return orc::from_abi(c).total_params(); }

int orc_init_weights(const OrcCfg* c, uint64_t seed, int bf16, float* out) {
  return guarded([&] { orc::init_weights(orc::from_abi(c), seed, bf16 != 0, out); });
}

// Tokens of batch number `skip` of the stream Rng(data_seed) (trainer.cpp:16-19).
int orc_copy_task_tokens(const OrcCfg* c, uint64_t data_seed, int64_t skip, int32_t* tokens) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    orc::Rng rng(data_seed);
    std::vector<int32_t> tmp(static_cast<size_t>(g.rows()));
    for (int64_t s = 0; s < skip; ++s) orc::copy_task(g, rng, tmp.data());
    orc::copy_task(g, rng, tokens);
  });
}

// Loss and all parameter gradients (store layout) in FP32 (or FP64 when
// `f64` is set, inputs widened). inv_rows <= 0 means 1/(B*S).
int orc_forward_backward(const OrcCfg* c, const float* params, const int32_t* tokens,
                         const int32_t* targets, double inv_rows, int f64, double* loss,
                         float* grads) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    const double ir = inv_rows > 0 ? inv_rows : 1.0 / static_cast<double>(g.rows());
    const int64_t n = g.total_params();
    if (f64) {
      std::vector<double> p(params, params + n), gr(static_cast<size_t>(n));
      *loss = orc::forward_backward<double>(g, p.data(), tokens, targets, gr.data(), ir);
      for (int64_t i = 0; i < n; ++i) grads[i] = static_cast<float>(gr[i]);
    } else {
      *loss = orc::forward_backward<float>(g, params, tokens, targets, grads, static_cast<float>(ir));
    }
  });
}

// Double-precision loss only (finite-difference checks).
int orc_loss_f64(const OrcCfg* c, const double* params, const int32_t* tokens,
                 const int32_t* targets, double* loss) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    std::vector<double> gr(static_cast<size_t>(g.total_params()));
    *loss = orc::forward_backward<double>(g, params, tokens, targets, gr.data(),
                                          1.0 / static_cast<double>(g.rows()));
  });
}

int orc_adam(const OrcHyper* hp, int64_t t, float* w, const float* g, float* m, float* v,
             int64_t n, int bf16_weights) {
  return guarded([&] {
    if (t < 1) throw std::invalid_argument("adam step index must be >= 1");
    orc::adam(w, g, m, v, n, *hp, t, bf16_weights != 0);
  });
}

// Training loop (trainer.cpp:8-42 + engine semantics). mode:
//   0 = FP32 store           (reference "fp32")
//   1 = BF16 store           (reference "bf16-store": bf16 weights, grads
//                              rounded to bf16 on evacuation, engine.cpp:93-101)
//   2 = mixed / north-star   FP32 master + Adam, forward/backward on the
//                              BF16 shadow RNE(master), FP32 gradients
int orc_train(const OrcCfg* c, const OrcHyper* hp, uint64_t seed, int mode, int64_t steps,
              double* losses, float* final_weights) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    const int64_t n = g.total_params();
    std::vector<float> w(static_cast<size_t>(n)), gr(w.size()), m(w.size(), 0.f), v(w.size(), 0.f),
        shadow(w.size());
    orc::init_weights(g, seed, mode == 1, w.data());
    orc::Rng data(seed + 1);
    std::vector<int32_t> tok(static_cast<size_t>(g.rows()));
    const float ir = 1.0f / static_cast<float>(g.rows());
    for (int64_t s = 0; s < steps; ++s) {
      orc::copy_task(g, data, tok.data());
      const float* wp = w.data();
      if (mode == 2) {
        for (int64_t i = 0; i < n; ++i) shadow[i] = orc::bf16_round(w[i]);
        wp = shadow.data();
      }
      losses[s] = orc::forward_backward<float>(g, wp, tok.data(), tok.data(), gr.data(), ir);
      if (mode == 1) {
        // bf16 evacuation per tile; tied table: round(head) then round(round(head)+round(embed))
        // is what the slab accumulation produces (host_store.cpp:254-284).
        for (int64_t i = 0; i < n; ++i) gr[i] = orc::bf16_round(gr[i]);
      }
      for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(gr[i])) throw std::runtime_error("non-finite gradient");
      orc::adam(w.data(), gr.data(), m.data(), v.data(), n, *hp, s + 1, mode == 1);
    }
    if (final_weights) std::memcpy(final_weights, w.data(), sizeof(float) * static_cast<size_t>(n));
  });
}

// Single-block forward / backward on a flat tile (kernel-level parity).
// acts layout (floats): n1, q, k, v (post-RoPE), attn, y, n2 (rows*h each),
// up, gate (rows*f each), p (B*H*S*S).
int orc_block_forward(const OrcCfg* c, const float* w_tile, const float* h_in, float* h_out,
                      float* acts) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    std::unique_ptr<orc::Rope> rope;
    if (g.theta > 0) rope.reset(new orc::Rope(g.S, g.hd(), g.theta));
    orc::Acts<float> a;
    orc::block_forward(h_in, orc::block_view<const float>(w_tile, g.h, g.f), g, rope.get(), a, h_out);
    if (acts) {
      float* o = acts;
      for (auto* vec : {&a.n1, &a.q, &a.k, &a.v, &a.attn, &a.y, &a.n2, &a.up, &a.gate, &a.p}) {
        std::memcpy(o, vec->data(), vec->size() * sizeof(float));
        o += vec->size();
      }
    }
  });
}

int orc_block_backward(const OrcCfg* c, const float* w_tile, const float* h_in, const float* g_out,
                       float* g_in, float* grad_tile) {
  return guarded([&] {
    const orc::Cfg g = orc::from_abi(c);
    std::unique_ptr<orc::Rope> rope;
    if (g.theta > 0) rope.reset(new orc::Rope(g.S, g.hd(), g.theta));
    orc::Acts<float> a;
    std::vector<float> h_out(static_cast<size_t>(g.rows() * g.h));
    const auto w = orc::block_view<const float>(w_tile, g.h, g.f);
    orc::block_forward(h_in, w, g, rope.get(), a, h_out.data());
    for (int64_t i = 0; i < g.block_params(); ++i) grad_tile[i] = 0.f;
    orc::block_backward(w, g, rope.get(), a, g_out, g_in, orc::block_view<float>(grad_tile, g.h, g.f));
  });
}

// RoPE cos/sin table [S][hd/2] exactly as the oracle uses it.
int orc_rope_table(int64_t S, int64_t hd, double theta, float* cos_out, float* sin_out) {
  return guarded([&] {
    orc::Rope r(S, hd, theta);
    for (size_t i = 0; i < r.c.size(); ++i) {
      cos_out[i] = static_cast<float>(r.c[i]);
      sin_out[i] = static_cast<float>(r.s[i]);
    }
  });
}

}  // extern "C"
