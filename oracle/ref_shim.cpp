// extern "C" shim over the reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It only
// calls the reference's public API; every number it returns is computed by
// reference code:
//   build_store            proj/src/host_store.cpp:141-156
//   Engine::train_step     proj/src/engine.cpp:426-432 (skip_optimizer for grads)
//   oracle_forward_backward proj/src/oracle.cpp:592-617
//   run_training           proj/src/trainer.cpp:8-42
//   make_copy_task_batch   proj/src/engine.cpp:434-441
//   block_forward/backward proj/include/hlm/kernels.hpp:313-383
//   bf16_bits_from_f32     proj/include/hlm/bf16.hpp:15-25
//   save/load_checkpoint   proj/src/checkpoint.cpp:38-120 (HLM1)
#include <chrono>
#include <memory>
#include <cstring>
#include <exception>
#include <string>

#include "hlm/bf16.hpp"
#include "hlm/checkpoint.hpp"
#include "hlm/engine.hpp"
#include "hlm/kernels.hpp"
#include "hlm/oracle.hpp"
#include "hlm/trainer.hpp"
#include "oracle_abi.h"

using namespace hlm;

namespace {

thread_local std::string g_err;

ModelConfig to_model(const OrcCfg* c) {
  ModelConfig m;
  m.layers = c->layers;
  m.hidden = c->hidden;
  m.ffn = c->ffn;
  m.vocab = c->vocab;
  m.seq = c->seq;
  m.batch = c->batch;
  m.k_ckpt = c->k_ckpt;
  m.tie_embeddings = c->tie != 0;
  return m;
}

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

void export_weights(const MasterStore& s, float* out) {
  for (i64 p = 0; p < s.physical_tiles(); ++p) {
    const LayerTile& t = s.physical(p);
    for (i64 i = 0; i < t.n_params(); ++i) *out++ = t.load_weight(i);
  }
}

void export_grads(const MasterStore& s, float* out) {
  for (i64 p = 0; p < s.physical_tiles(); ++p) {
    const LayerTile& t = s.physical(p);
    for (i64 i = 0; i < t.n_params(); ++i) *out++ = t.load_grad(i);
  }
}

Batch make_batch(const ModelConfig& m, const int32_t* tokens, const int32_t* targets) {
  Batch b;
  const i64 n = m.batch * m.seq;
  b.tokens.assign(tokens, tokens + n);
  b.targets.assign(targets, targets + n);
  return b;
}

BlockWeights<PlainMat<float>> block_views(const float* w, i64 h, i64 f) {
  BlockWeights<PlainMat<float>> bw;
  const float* p = w;
  auto take = [&](i64 r, i64 c) {
    PlainMat<float> v{p, r, c};
    p += r * c;
    return v;
  };
  bw.w_q = take(h, h);
  bw.w_k = take(h, h);
  bw.w_v = take(h, h);
  bw.w_o = take(h, h);
  bw.w_up = take(h, f);
  bw.w_gate = take(h, f);
  bw.w_down = take(f, h);
  bw.norm1 = take(1, h);
  bw.norm2 = take(1, h);
  return bw;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint16_t ref_bf16_bits(float x) { return bf16_bits_from_f32(x); }

int64_t ref_total_params(const OrcCfg* c) { return to_model(c).total_params(); }

int ref_init_weights(const OrcCfg* c, uint64_t seed, int bf16, float* out) {
  try {
    auto store = build_store(to_model(c), seed, bf16 ? Dtype::BF16 : Dtype::FP32);
    export_weights(*store, out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_copy_task_tokens(const OrcCfg* c, uint64_t data_seed, int64_t skip, int32_t* tokens) {
  try {
    const ModelConfig m = to_model(c);
    Rng rng(data_seed);
    for (int64_t s = 0; s < skip; ++s) (void)make_copy_task_batch(m, rng);
    const Batch b = make_copy_task_batch(m, rng);
    std::memcpy(tokens, b.tokens.data(), b.tokens.size() * sizeof(int32_t));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One engine step without the optimizer on a store built from `seed`; the
// store's accumulated gradients are exported (reference test_engine.cpp:47-54).
int ref_grad_step(const OrcCfg* c, uint64_t seed, int bf16, const int32_t* tokens,
                  const int32_t* targets, double* loss, float* grads) {
  try {
    const ModelConfig m = to_model(c);
    const Dtype dt = bf16 ? Dtype::BF16 : Dtype::FP32;
    auto store = build_store(m, seed, dt);
    DeviceArena arena(m, dt);
    EngineOptions opts;
    opts.skip_optimizer = true;
    Engine engine(*store, arena, HyperParams{}, opts);
    const StepResult r = engine.train_step(make_batch(m, tokens, targets));
    *loss = r.loss;
    export_grads(*store, grads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Tape oracle on caller-provided FP32 parameters (store layout).
int ref_oracle_fb(const OrcCfg* c, const float* params, const int32_t* tokens,
                  const int32_t* targets, float* loss, float* grads) {
  try {
    const ModelConfig m = to_model(c);
    oracle::Params p;
    p.config = m;
    const i64 h = m.hidden, f = m.ffn, V = m.vocab;
    const float* q = params;
    auto take = [&](std::vector<float>& v, i64 n) {
      v.assign(q, q + n);
      q += n;
    };
    take(p.embed, V * h);
    p.blocks.resize(static_cast<std::size_t>(m.layers));
    for (auto& b : p.blocks) {
      take(b.w_q, h * h);
      take(b.w_k, h * h);
      take(b.w_v, h * h);
      take(b.w_o, h * h);
      take(b.w_up, h * f);
      take(b.w_gate, h * f);
      take(b.w_down, f * h);
      take(b.norm1, h);
      take(b.norm2, h);
    }
    if (m.tie_embeddings)
      p.head = p.embed;
    else
      take(p.head, V * h);
    const auto fb = oracle::oracle_forward_backward(p, make_batch(m, tokens, targets));
    *loss = fb.loss;
    float* o = grads;
    auto put = [&](const std::vector<float>& v) {
      std::memcpy(o, v.data(), v.size() * sizeof(float));
      o += v.size();
    };
    put(fb.grads.embed);
    for (const auto& b : fb.grads.blocks) {
      put(b.w_q);
      put(b.w_k);
      put(b.w_v);
      put(b.w_o);
      put(b.w_up);
      put(b.w_gate);
      put(b.w_down);
      put(b.norm1);
      put(b.norm2);
    }
    if (!m.tie_embeddings) put(fb.grads.head);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_training: store built from seed, data stream seeded seed+1.
int ref_train(const OrcCfg* c, const OrcHyper* hp, uint64_t seed, int bf16, int64_t steps,
              double* losses, float* final_weights) {
  try {
    RunConfig cfg;
    cfg.model = to_model(c);
    cfg.has_model = true;
    cfg.hyper.lr = hp->lr;
    cfg.hyper.beta1 = hp->beta1;
    cfg.hyper.beta2 = hp->beta2;
    cfg.hyper.eps = hp->eps;
    cfg.hyper.weight_decay = hp->weight_decay;
    cfg.run.steps = steps;
    cfg.run.seed = seed;
    cfg.run.dtype = bf16 ? Dtype::BF16 : Dtype::FP32;
    auto store = build_store(cfg.model, seed, cfg.run.dtype);
    DeviceArena arena(cfg.model, cfg.run.dtype);
    const TrainOutput out = run_training(cfg, *store, arena);
    for (std::size_t i = 0; i < out.steps.size(); ++i) losses[i] = out.steps[i].loss;
    if (final_weights) export_weights(*store, final_weights);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_training for `steps` steps, then the reference's HLM1 save_checkpoint of the store
// (golden checkpoint files; tests/golden/make_golden.py).
int ref_train_save_hlm1(const OrcCfg* c, const OrcHyper* hp, uint64_t seed, int bf16, int64_t steps,
                        const char* path) {
  try {
    RunConfig cfg;
    cfg.model = to_model(c);
    cfg.has_model = true;
    cfg.hyper.lr = hp->lr;
    cfg.hyper.beta1 = hp->beta1;
    cfg.hyper.beta2 = hp->beta2;
    cfg.hyper.eps = hp->eps;
    cfg.hyper.weight_decay = hp->weight_decay;
    cfg.run.steps = steps;
    cfg.run.seed = seed;
    cfg.run.dtype = bf16 ? Dtype::BF16 : Dtype::FP32;
    auto store = build_store(cfg.model, seed, cfg.run.dtype);
    DeviceArena arena(cfg.model, cfg.run.dtype);
    run_training(cfg, *store, arena);
    save_checkpoint(*store, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's load_checkpoint of `path` into a store of this geometry; exports the
// loaded weights (as f32), m, v (flat, physical tile order) and the Adam step count.
int ref_load_hlm1(const OrcCfg* c, int bf16, const char* path, float* weights, float* m, float* v,
                  int64_t* adam_steps) {
  try {
    auto store = build_store(to_model(c), 1, bf16 ? Dtype::BF16 : Dtype::FP32);
    load_checkpoint(*store, path);
    export_weights(*store, weights);
    for (i64 p = 0; p < store->physical_tiles(); ++p) {
      LayerTile& t = store->physical(p);
      std::memcpy(m, t.moment_m(), static_cast<size_t>(t.n_params()) * 4);
      std::memcpy(v, t.moment_v(), static_cast<size_t>(t.n_params()) * 4);
      m += t.n_params();
      v += t.n_params();
    }
    *adam_steps = store->adam_steps();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Reference block kernels (FP32 instantiation) on flat tile-ordered weights.
int ref_block_forward(int64_t B, int64_t S, int64_t h, int64_t f, const float* w_tile,
                      const float* h_in, float* h_out, float* n1, float* p, float* y, float* n2,
                      float* up, float* gate) {
  try {
    const BlockDims d{B, S, h, f};
    ScratchBuf<float> scratch(B, S, h, f);
    ActPtrs<float> acts{n1, p, y, n2, up, gate};
    block_forward(h_in, block_views(w_tile, h, f), d, acts, h_out, scratch.view());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_block_backward(int64_t B, int64_t S, int64_t h, int64_t f, const float* w_tile,
                       const float* h_in, const float* n1, const float* p, const float* y,
                       const float* n2, const float* up, const float* gate, const float* g_out,
                       float* g_in, float* grad_tile) {
  try {
    const BlockDims d{B, S, h, f};
    ScratchBuf<float> scratch(B, S, h, f);
    ActPtrs<float> acts{const_cast<float*>(n1), const_cast<float*>(p), const_cast<float*>(y),
                        const_cast<float*>(n2), const_cast<float*>(up), const_cast<float*>(gate)};
    BlockGradPtrs<float> g;
    float* q = grad_tile;
    auto take = [&](i64 n) {
      float* r = q;
      q += n;
      return r;
    };
    g.w_q = take(h * h);
    g.w_k = take(h * h);
    g.w_v = take(h * h);
    g.w_o = take(h * h);
    g.w_up = take(h * f);
    g.w_gate = take(h * f);
    g.w_down = take(f * h);
    g.norm1 = take(h);
    g.norm2 = take(h);
    block_backward(h_in, block_views(w_tile, h, f), d, acts, g_out, g_in, g, scratch.view());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Wall-clock seconds per Engine::train_step (bf16-store or fp32) after
// `warmup` untimed steps — the CPU reference arm of bench.py.
double ref_time_train_step(const OrcCfg* c, int bf16, int64_t steps, int64_t warmup) {
  try {
    const ModelConfig m = to_model(c);
    const Dtype dt = bf16 ? Dtype::BF16 : Dtype::FP32;
    auto store = build_store(m, 1234, dt);
    DeviceArena arena(m, dt);
    Engine engine(*store, arena, HyperParams{});
    Rng rng(1235);
    for (int64_t s = 0; s < warmup; ++s) engine.train_step(make_copy_task_batch(m, rng));
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t s = 0; s < steps; ++s) engine.train_step(make_copy_task_batch(m, rng));
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
           static_cast<double>(steps);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Wall-clock seconds of one block forward + recompute + backward with the
// reference kernels at width (h, f) and B x S tokens (bench C2+ estimate).
double ref_time_block(int64_t B, int64_t S, int64_t h, int64_t f, int64_t reps) {
  try {
    const i64 n = 4 * h * h + 3 * h * f + 2 * h, T = B * S;
    std::vector<float> w(static_cast<std::size_t>(n)), grads(static_cast<std::size_t>(n), 0.f);
    Rng rng(7);
    for (auto& x : w) x = rng.trunc_normal(0.02f);
    for (i64 i = 4 * h * h + 3 * h * f; i < n; ++i) w[static_cast<std::size_t>(i)] = 1.0f;
    std::vector<float> x(static_cast<std::size_t>(T * h)), hout(x.size()), g(x.size()), gin(x.size());
    for (auto& v : x) v = rng.normal();
    for (auto& v : g) v = rng.normal() * 1e-3f;
    std::vector<float> n1(x.size()), y(x.size()), n2(x.size()), p(static_cast<std::size_t>(B * S * S)),
        up(static_cast<std::size_t>(T * f)), gate(up.size());
    const BlockDims d{B, S, h, f};
    ScratchBuf<float> scratch(B, S, h, f);
    ActPtrs<float> acts{n1.data(), p.data(), y.data(), n2.data(), up.data(), gate.data()};
    const auto bw = block_views(w.data(), h, f);
    BlockGradPtrs<float> gp;
    float* q = grads.data();
    auto take = [&](i64 k) { float* r = q; q += k; return r; };
    gp.w_q = take(h * h); gp.w_k = take(h * h); gp.w_v = take(h * h); gp.w_o = take(h * h);
    gp.w_up = take(h * f); gp.w_gate = take(h * f); gp.w_down = take(f * h);
    gp.norm1 = take(h); gp.norm2 = take(h);
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t r = 0; r < reps; ++r) {
      block_forward(x.data(), bw, d, acts, hout.data(), scratch.view());   // forward
      block_forward(x.data(), bw, d, acts, hout.data(), scratch.view());   // recompute
      block_backward(x.data(), bw, d, acts, g.data(), gin.data(), gp, scratch.view());
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
           static_cast<double>(reps);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Wall-clock seconds of the head: head_fwd + ce_loss_and_grad + head_bwd
// (kernels.hpp:410-446) at (rows, h, V) — the other half of the C2+ estimate.
double ref_time_head(int64_t rows, int64_t h, int64_t V, int64_t reps) {
  try {
    std::vector<float> head(static_cast<std::size_t>(V * h)), x(static_cast<std::size_t>(rows * h)),
        logits(static_cast<std::size_t>(rows * V)), dl(logits.size()), dx(x.size()), dhead(head.size(), 0.f);
    Rng rng(11);
    for (auto& v : head) v = rng.trunc_normal(0.02f);
    for (auto& v : x) v = rng.normal();
    std::vector<std::int32_t> tgt(static_cast<std::size_t>(rows));
    for (auto& t : tgt) t = rng.uniform_int(static_cast<std::int32_t>(V));
    PlainMat<float> hm{head.data(), V, h};
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t r = 0; r < reps; ++r) {
      head_fwd(x.data(), hm, logits.data(), rows, h, V);
      (void)ce_loss_and_grad(logits.data(), tgt.data(), dl.data(), rows, V);
      head_bwd(x.data(), dl.data(), hm, dx.data(), dhead.data(), rows, h, V);
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
           static_cast<double>(reps);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Persistent context for the bench's reference arm: one block (fwd +
// recompute + bwd) and the head (fwd + CE + bwd) at full width (h, f, V) on a
// reduced token count T = B*S, run through the reference kernels. Weights are
// filled with a cheap nonzero pattern (timing does not depend on values; the
// zero-skip in matmul_grad_acc never triggers).
struct RefBench {
  int64_t B, S, h, f, V, T;
  std::vector<float> w, grads, x, hout, g, gin, n1, y, n2, p, up, gate;
  std::vector<float> head, xh, logits, dl, dx, dhead;
  std::vector<std::int32_t> tgt;
  std::unique_ptr<ScratchBuf<float>> scratch;
};

void* ref_bench_create(int64_t B, int64_t S, int64_t h, int64_t f, int64_t V) {
  try {
    auto* b = new RefBench{B, S, h, f, V, B * S, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, {}, nullptr};
    const int64_t n = 4 * h * h + 3 * h * f + 2 * h, T = b->T;
    uint32_t st = 12345u;
    auto fill = [&](std::vector<float>& v, std::size_t sz, float scale) {
      v.resize(sz);
      for (auto& e : v) {
        st = st * 1664525u + 1013904223u;
        e = scale * (static_cast<float>((st >> 9) & 0x3FFF) / 8192.0f - 1.0f + 1e-3f);
      }
    };
    fill(b->w, static_cast<std::size_t>(n), 0.02f);
    b->grads.assign(static_cast<std::size_t>(n), 0.f);
    fill(b->x, static_cast<std::size_t>(T * h), 1.0f);
    fill(b->g, static_cast<std::size_t>(T * h), 1e-3f);
    b->hout.resize(b->x.size()); b->gin.resize(b->x.size()); b->n1.resize(b->x.size());
    b->y.resize(b->x.size()); b->n2.resize(b->x.size());
    b->p.resize(static_cast<std::size_t>(B * S * S));
    b->up.resize(static_cast<std::size_t>(T * f)); b->gate.resize(b->up.size());
    fill(b->head, static_cast<std::size_t>(V * h), 0.02f);
    fill(b->xh, static_cast<std::size_t>(T * h), 1.0f);
    b->logits.resize(static_cast<std::size_t>(T * V)); b->dl.resize(b->logits.size());
    b->dx.resize(b->xh.size()); b->dhead.assign(b->head.size(), 0.f);
    b->tgt.resize(static_cast<std::size_t>(T));
    for (auto& t : b->tgt) { st = st * 1664525u + 1013904223u; t = static_cast<std::int32_t>(st % static_cast<uint32_t>(V)); }
    b->scratch = std::make_unique<ScratchBuf<float>>(B, S, h, f);
    return b;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// seconds of {block fwd, block recompute, block bwd} and of {head fwd+CE+bwd}
int ref_bench_run(void* ctx, double* block_s, double* head_s) {
  try {
    auto* b = static_cast<RefBench*>(ctx);
    const BlockDims d{b->B, b->S, b->h, b->f};
    ActPtrs<float> acts{b->n1.data(), b->p.data(), b->y.data(), b->n2.data(), b->up.data(), b->gate.data()};
    const auto bw = block_views(b->w.data(), b->h, b->f);
    BlockGradPtrs<float> gp;
    float* q = b->grads.data();
    auto take = [&](int64_t k) { float* r = q; q += k; return r; };
    const int64_t h = b->h, f = b->f;
    gp.w_q = take(h * h); gp.w_k = take(h * h); gp.w_v = take(h * h); gp.w_o = take(h * h);
    gp.w_up = take(h * f); gp.w_gate = take(h * f); gp.w_down = take(f * h);
    gp.norm1 = take(h); gp.norm2 = take(h);
    auto t0 = std::chrono::steady_clock::now();
    block_forward(b->x.data(), bw, d, acts, b->hout.data(), b->scratch->view());
    block_forward(b->x.data(), bw, d, acts, b->hout.data(), b->scratch->view());
    block_backward(b->x.data(), bw, d, acts, b->g.data(), b->gin.data(), gp, b->scratch->view());
    *block_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    PlainMat<float> hm{b->head.data(), b->V, b->h};
    t0 = std::chrono::steady_clock::now();
    head_fwd(b->xh.data(), hm, b->logits.data(), b->T, b->h, b->V);
    (void)ce_loss_and_grad(b->logits.data(), b->tgt.data(), b->dl.data(), b->T, b->V);
    head_bwd(b->xh.data(), b->dl.data(), hm, b->dx.data(), b->dhead.data(), b->T, b->h, b->V);
    *head_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_bench_destroy(void* ctx) { delete static_cast<RefBench*>(ctx); }

}  // extern "C"
