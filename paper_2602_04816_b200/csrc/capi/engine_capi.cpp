// extern "C" surface over the C++ host engine. Exceptions become HlmStatus
// codes (reference errors.hpp:13-50 / hlm_main.cpp:418-430 mapping).
#include <vector>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "capi_util.h"
#include "hlm/bf16.hpp"
#include "hlm/checkpoint.hpp"
#include "hlm/engine.hpp"
#include "hlm/numa_place.hpp"
#include "hlm/trainer.hpp"
#include "hlm_cuda.h"
#include "../host/nccl_dyn.h"

#include <algorithm>

struct HlmStore {
    std::unique_ptr<hlm::MasterStore> s;
};
struct HlmArena {
    std::unique_ptr<hlm::DeviceArena> a;
};
struct HlmEngine {
    std::unique_ptr<hlm::Engine> e;
    std::string last_trace;
};

namespace {

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return HLM_OK;
    } catch (const hlm::ArenaOomError& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_OOM;
    } catch (const hlm::ConfigError& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_CONFIG;
    } catch (const std::invalid_argument& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_CONFIG;
    } catch (const hlm::ProtocolError& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_PROTOCOL;
    } catch (const hlm::NumericsError& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_NUMERICS;
    } catch (const std::out_of_range& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_RANGE;
    } catch (const hlm::CudaError& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_CUDA;
    } catch (const std::exception& e) {
        hlm_capi::set_error(e.what());
        return HLM_ERR_ARGS;
    }
}

hlm::ModelConfig to_model(const HlmModelConfig* c) {
    if (!c) throw std::invalid_argument("null model config");
    hlm::ModelConfig m;
    m.layers = c->layers;
    m.hidden = c->hidden;
    m.ffn = c->ffn;
    m.vocab = c->vocab;
    m.seq = c->seq;
    m.batch = c->batch;
    m.k_ckpt = c->k_ckpt;
    m.tie_embeddings = c->tie_embeddings != 0;
    m.n_heads = c->n_heads > 0 ? c->n_heads : 1;
    m.rope_theta = c->rope_theta;
    m.validate();
    return m;
}

hlm::HyperParams to_hyper(const HlmHyper* h) {
    hlm::HyperParams p;
    if (h) {
        p.lr = h->lr;
        p.beta1 = h->beta1;
        p.beta2 = h->beta2;
        p.eps = h->eps;
        p.weight_decay = h->weight_decay;
    }
    return p;
}

hlm::EngineOptions to_opts(const HlmEngineOptions* o) {
    hlm::EngineOptions e;
    if (o) {
        e.eager_optim = o->eager_optim != 0;
        e.threaded_accum = o->threaded_accum != 0;
        e.n_slab = o->n_slab > 0 ? o->n_slab : 12;
        e.accum_delay_us = o->accum_delay_us;
        e.skip_optimizer = o->skip_optimizer != 0;
        e.fused_recompute = o->fused_recompute != 0;
        e.record_trace = o->record_trace != 0;
        e.block_flags = o->block_flags;
        e.overlap_optimizer_tail = o->overlap_optimizer_tail != 0;
        e.tail_blocks = o->tail_blocks;
        e.rank = o->rank;
        e.world = o->world > 0 ? o->world : 1;
        e.comm_grad = o->comm_grad;
        e.comm_weights = o->comm_weights;
        e.host_threads = o->host_threads;
        e.resident_embed = o->resident_embed != 0;
        e.resident_blocks = o->resident_blocks;
        e.head_piece_vocab = o->head_piece_vocab;
        e.piece_elems = o->piece_elems;
        e.grad_buffers = o->grad_buffers > 2 ? o->grad_buffers : 2;
        e.sparse_embed_grad = o->sparse_embed_grad != 0;
        e.embed_gather_host = o->embed_gather_host != 0;
        e.pin_threads = o->no_pin_threads == 0;
        if (o->reserved_transit_blocks != 0)
            throw hlm::ConfigError("engine options: transit tiles (transit_blocks) were removed; the field must be 0");
        e.saved_act_layers = o->saved_act_layers > 0 ? o->saved_act_layers : 0;
    }
    return e;
}

void fill_result(const hlm::StepResult& r, const hlm::Engine& eng, HlmStepResult* out) {
    if (!out) return;
    out->loss = r.loss;
    out->h2d_bytes = r.h2d_bytes;
    out->d2h_bytes = r.d2h_bytes;
    out->recompute_forwards = r.recompute_forwards;
    out->gpu_ms = r.gpu_ms;
    out->arena_committed = r.arena.committed_total;
    out->arena_peak = r.arena.step_peak_total;
    out->host_total = r.host.total;
    out->slab_max_in_use = const_cast<hlm::Engine&>(eng).pool().max_in_use();
}

hlm::Batch to_batch(const hlm::ModelConfig& m, const int32_t* tokens, const int32_t* targets) {
    if (!tokens || !targets) throw std::invalid_argument("null batch");
    hlm::Batch b;
    b.tokens.assign(tokens, tokens + m.rows());
    b.targets.assign(targets, targets + m.rows());
    return b;
}

}  // namespace

extern "C" {

int hlm_store_create(const HlmModelConfig* cfg, uint64_t seed, int dtype, int init_mode, int pin_shadow,
                     HlmStore** out) {
    return guarded([&] {
        auto st = std::make_unique<HlmStore>();
        st->s = hlm::build_store(to_model(cfg), seed, dtype == 1 ? hlm::Dtype::FP32 : hlm::Dtype::BF16,
                                 init_mode == 1 ? hlm::InitMode::Parallel : hlm::InitMode::Reference, pin_shadow != 0);
        *out = st.release();
    });
}

int hlm_store_create_shared(const HlmModelConfig* cfg, uint64_t seed, int dtype, int init_mode, int pin_shadow,
                            const char* name, int rank, int world, uint64_t nonce, HlmStore** out) {
    return guarded([&] {
        if (!name || !*name) throw std::invalid_argument("shared store needs a name");
        hlm::SharedStoreSpec spec{name, rank, world, nonce};
        auto st = std::make_unique<HlmStore>();
        st->s = hlm::build_store(to_model(cfg), seed, dtype == 1 ? hlm::Dtype::FP32 : hlm::Dtype::BF16,
                                 init_mode == 1 ? hlm::InitMode::Parallel : hlm::InitMode::Reference, pin_shadow != 0,
                                 &spec);
        *out = st.release();
    });
}

int hlm_store_adam_shard(HlmStore* s, const float* grads, const HlmHyper* hp, int64_t t, int rank, int world) {
    return guarded([&] {
        hlm::MasterStore& st = *s->s;
        const hlm::HyperParams h = to_hyper(hp);
        for (hlm::i64 p = 0; p < st.physical_tiles(); ++p) {
            hlm::LayerTile& tile = st.physical(p);
            if (tile.n_params() % world) throw std::invalid_argument("tile not divisible by world");
            const hlm::i64 cnt = tile.n_params() / world, begin = rank * cnt;
            hlm::adam_step_range(tile, grads + begin, begin, cnt, h, t);
            tile.bump_version(rank);
            grads += tile.n_params();
        }
        st.set_adam_steps(t);
    });
}

int64_t hlm_store_tile_version(const HlmStore* s, int64_t p) { return s->s->physical(p).min_version(); }

int hlm_store_save(const HlmStore* s, const char* path) {
    return guarded([&] { hlm::save_checkpoint(*s->s, path); });
}

int hlm_store_load(HlmStore* s, const char* path) {
    return guarded([&] { hlm::load_checkpoint(*s->s, path); });
}

int hlm_store_save_hlm1(const HlmStore* s, const char* path) {
    return guarded([&] { hlm::save_checkpoint_hlm1(*s->s, path); });
}

int hlm_run_training_store(HlmStore* s, const HlmHyper* hp, uint64_t seed, int64_t steps,
                           const HlmEngineOptions* o, double* losses) {
    return guarded([&] {
        hlm::RunConfig rc;
        rc.model = s->s->config();
        rc.hyper = to_hyper(hp);
        rc.run.steps = steps;
        rc.run.seed = seed;
        const hlm::EngineOptions eo = to_opts(o);
        rc.run.eager_optim = eo.eager_optim;
        rc.run.n_slab = eo.n_slab;
        rc.run.threaded_accum = eo.threaded_accum;
        hlm::DeviceArena arena(rc.model);
        const hlm::TrainOutput out = hlm::run_training(rc, *s->s, arena, {}, eo);
        for (size_t i = 0; i < out.steps.size(); ++i) losses[i] = out.steps[i].loss;
    });
}

int hlm_nccl_unique_id(uint8_t* out128) {
    return guarded([&] {
        ncclUniqueId id;
        hlm::nccl_check(hlm::nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int hlm_nccl_comm_create(const uint8_t* id128, int world, int rank, void** comm) {
    return guarded([&] {
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t c;
        hlm::nccl_check(hlm::nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
        *comm = c;
    });
}

void hlm_nccl_comm_destroy(void* comm) {
    if (comm) hlm::nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

int hlm_nccl_reduce_scatter_f32(void* comm, const float* send, float* recv, int64_t count, void* stream) {
    return guarded([&] {
        if (!comm || count < 0) throw std::invalid_argument("reduce-scatter: communicator and count >= 0 required");
        hlm::nccl_check(hlm::nccl().ReduceScatter(send, recv, static_cast<size_t>(count), ncclFloat32, ncclSum,
                                                  static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)),
                        "ncclReduceScatter");
    });
}

int hlm_nccl_all_gather_bf16(void* comm, const void* send, void* recv, int64_t count, void* stream) {
    return guarded([&] {
        if (!comm || count < 0) throw std::invalid_argument("all-gather: communicator and count >= 0 required");
        hlm::nccl_check(hlm::nccl().AllGather(send, recv, static_cast<size_t>(count), ncclBfloat16,
                                              static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)),
                        "ncclAllGather");
    });
}

int hlm_nccl_allreduce_f32(void* comm, const float* send, float* recv, int64_t count, void* stream) {
    return guarded([&] {
        if (!comm || count < 0) throw std::invalid_argument("all-reduce: communicator and count >= 0 required");
        hlm::nccl_check(hlm::nccl().AllReduce(send, recv, static_cast<size_t>(count), ncclFloat32, ncclSum,
                                              static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)),
                        "ncclAllReduce");
    });
}

void hlm_store_destroy(HlmStore* s) { delete s; }

int64_t hlm_store_total_params(const HlmStore* s) { return s ? s->s->total_params() : -1; }
int64_t hlm_store_adam_steps(const HlmStore* s) { return s ? s->s->adam_steps() : -1; }

int hlm_store_export(const HlmStore* s, int field, float* out) {
    return guarded([&] {
        const hlm::MasterStore& st = *s->s;
        st.quiesce(false);   // an attached engine's optimizer tail / resident tiles land first
        for (hlm::i64 p = 0; p < st.physical_tiles(); ++p) {
            const hlm::LayerTile& t = st.physical(p);
            const size_t n = static_cast<size_t>(t.n_params());
            switch (field) {
                case HLM_FIELD_MASTER: std::memcpy(out, t.master(), n * 4); break;
                case HLM_FIELD_M: std::memcpy(out, t.moment_m(), n * 4); break;
                case HLM_FIELD_V: std::memcpy(out, t.moment_v(), n * 4); break;
                case HLM_FIELD_GRADS:
                    if (t.grads_or_null())
                        std::memcpy(out, t.grads_or_null(), n * 4);
                    else
                        std::memset(out, 0, n * 4);
                    break;
                case HLM_FIELD_SHADOW:
                    for (size_t i = 0; i < n; ++i) out[i] = hlm::f32_from_bf16_bits(t.shadow()[i]);
                    break;
                default: throw std::invalid_argument("unknown store field");
            }
            out += n;
        }
    });
}

int hlm_store_import_master(HlmStore* s, const float* w) {
    return guarded([&] {
        hlm::MasterStore& st = *s->s;
        st.quiesce();
        for (hlm::i64 p = 0; p < st.physical_tiles(); ++p) {
            hlm::LayerTile& t = st.physical(p);
            std::memcpy(t.master(), w, static_cast<size_t>(t.n_params()) * 4);
            w += t.n_params();
        }
        st.repack_shadow();
        st.bump_epoch();
    });
}

const char* hlm_host_isa(void) { return hlm::host_isa(); }

int hlm_store_bitwise_equal(const HlmStore* a, const HlmStore* b) { return a->s->bitwise_equal(*b->s) ? 1 : 0; }

int hlm_store_adam_embed_rows(HlmStore* s, const int32_t* rows, int64_t n_rows, const float* compact,
                              const HlmHyper* hp, int64_t t) {
    return guarded([&] {
        hlm::MasterStore& st = *s->s;
        const hlm::ModelConfig& m = st.config();
        std::vector<int32_t> map(static_cast<size_t>(m.vocab), -1);
        for (int64_t c = 0; c < n_rows; ++c) {
            if (rows[c] < 0 || rows[c] >= m.vocab || (c && rows[c] <= rows[c - 1]))
                throw std::invalid_argument("embedding rows must be ascending ids in [0, vocab)");
            map[static_cast<size_t>(rows[c])] = static_cast<int32_t>(c);
        }
        hlm::adam_step_rows_sparse(st.tile(m.embed_tile_id()), m.vocab, m.hidden, map.data(), compact,
                                   to_hyper(hp), t);
    });
}

int hlm_rank_cpu_slice(int rank, const int* gpu_nodes, int world, const int* allowed, int n_allowed, int online,
                       const int* node_of_cpu, int n_cpus, int* out, int out_cap) {
    if (world < 1 || rank < 0 || rank >= world || n_allowed < 0 || n_cpus < 0 || out_cap < 0) return -1;
    std::vector<std::vector<int>> of_node;
    for (int c = 0; c < n_cpus; ++c) {
        const int n = node_of_cpu[c];
        if (n < 0) continue;
        if (static_cast<size_t>(n) >= of_node.size()) of_node.resize(static_cast<size_t>(n) + 1);
        of_node[static_cast<size_t>(n)].push_back(c);
    }
    const std::vector<int> cpus = hlm::rank_cpu_slice(rank, std::vector<int>(gpu_nodes, gpu_nodes + world),
                                                      std::vector<int>(allowed, allowed + n_allowed), online, of_node);
    const int n = static_cast<int>(std::min<size_t>(cpus.size(), static_cast<size_t>(out_cap)));
    std::copy(cpus.begin(), cpus.begin() + n, out);
    return static_cast<int>(cpus.size());
}

int hlm_store_adam_step(HlmStore* s, const float* grads, const HlmHyper* hp, int64_t t) {
    return guarded([&] {
        hlm::MasterStore& st = *s->s;
        const hlm::HyperParams h = to_hyper(hp);
        for (hlm::i64 p = 0; p < st.physical_tiles(); ++p) {
            hlm::LayerTile& tile = st.physical(p);
            hlm::adam_step_tile_from(tile, grads, h, t);
            grads += tile.n_params();
        }
        st.set_adam_steps(t);
    });
}

int hlm_arena_create(const HlmModelConfig* cfg, int64_t budget_cap, int device, HlmArena** out) {
    return guarded([&] {
        auto a = std::make_unique<HlmArena>();
        std::optional<hlm::i64> cap;
        if (budget_cap > 0) cap = budget_cap;
        a->a = std::make_unique<hlm::DeviceArena>(to_model(cfg), cap, device);
        *out = a.release();
    });
}

int hlm_arena_create_ex(const HlmModelConfig* cfg, int64_t budget_cap, int device, int64_t weight_cache_bytes,
                        HlmArena** out) {
    return guarded([&] {
        auto a = std::make_unique<HlmArena>();
        std::optional<hlm::i64> cap;
        if (budget_cap > 0) cap = budget_cap;
        a->a = std::make_unique<hlm::DeviceArena>(to_model(cfg), cap, device, weight_cache_bytes);
        *out = a.release();
    });
}

void hlm_arena_destroy(HlmArena* a) { delete a; }

int hlm_arena_footprint(const HlmModelConfig* cfg, int64_t* out) {
    return guarded([&] {
        const hlm::ArenaFootprint fp = hlm::arena_footprint(to_model(cfg));
        out[0] = fp.stream_buf;
        out[1] = fp.anchor_slot;
        out[2] = fp.anchor_slots;
        out[3] = fp.stack;
        out[4] = fp.workspace;
    });
}

int hlm_engine_create(HlmStore* s, HlmArena* a, const HlmHyper* hp, const HlmEngineOptions* o, HlmEngine** out) {
    return guarded([&] {
        auto e = std::make_unique<HlmEngine>();
        e->e = std::make_unique<hlm::Engine>(*s->s, *a->a, to_hyper(hp), to_opts(o));
        *out = e.release();
    });
}

void hlm_engine_destroy(HlmEngine* e) { delete e; }

int hlm_engine_train_step(HlmEngine* e, const int32_t* tokens, const int32_t* targets, HlmStepResult* out) {
    return guarded([&] {
        const hlm::StepResult r = e->e->train_step(to_batch(e->e->store().config(), tokens, targets));
        e->last_trace = hlm::trace_to_jsonl(r.trace);
        fill_result(r, *e->e, out);
    });
}

int hlm_engine_sync(HlmEngine* e) {
    return guarded([&] { e->e->sync(); });
}

int hlm_engine_wait_optimizer(HlmEngine* e) {
    return guarded([&] { e->e->wait_optimizer(); });
}

int hlm_engine_begin_step(HlmEngine* e, const int32_t* tokens, const int32_t* targets) {
    return guarded([&] { e->e->begin_step(to_batch(e->e->store().config(), tokens, targets)); });
}
int hlm_engine_forward(HlmEngine* e) {
    return guarded([&] { e->e->forward_streaming(); });
}
int hlm_engine_anchor_loss(HlmEngine* e, double* loss) {
    return guarded([&] {
        const double l = e->e->anchor_loss();
        if (loss) *loss = l;
    });
}
int hlm_engine_backward(HlmEngine* e) {
    return guarded([&] { e->e->backward_blockwise(); });
}
int hlm_engine_finish_step(HlmEngine* e, HlmStepResult* out) {
    return guarded([&] {
        const hlm::StepResult r = e->e->finish_step();
        e->last_trace = hlm::trace_to_jsonl(r.trace);
        fill_result(r, *e->e, out);
    });
}
int hlm_engine_debug_hidden(HlmEngine* e, float* out) {
    return guarded([&] {
        const std::vector<float> h = e->e->debug_hidden();
        std::memcpy(out, h.data(), h.size() * 4);
    });
}

int hlm_engine_last_trace(HlmEngine* e, char* buf, size_t cap, size_t* needed) {
    const size_t n = e->last_trace.size() + 1;
    if (needed) *needed = n;
    if (buf && cap >= n) std::memcpy(buf, e->last_trace.c_str(), n);
    return HLM_OK;
}

int hlm_make_copy_task_batch(const HlmModelConfig* cfg, uint64_t data_seed, int64_t skip, int32_t* tokens) {
    return guarded([&] {
        const hlm::ModelConfig m = to_model(cfg);
        hlm::Rng rng(data_seed);
        for (int64_t s = 0; s < skip; ++s) (void)hlm::make_copy_task_batch(m, rng);
        const hlm::Batch b = hlm::make_copy_task_batch(m, rng);
        std::memcpy(tokens, b.tokens.data(), b.tokens.size() * 4);
    });
}

int hlm_run_training(const HlmModelConfig* cfg, const HlmHyper* hp, uint64_t seed, int dtype, int64_t steps,
                     const HlmEngineOptions* o, double* losses, HlmStepResult* last) {
    return guarded([&] {
        hlm::RunConfig rc;
        rc.model = to_model(cfg);
        rc.hyper = to_hyper(hp);
        rc.run.steps = steps;
        rc.run.seed = seed;
        rc.run.dtype = dtype == 1 ? hlm::Dtype::FP32 : hlm::Dtype::BF16;
        const hlm::EngineOptions eo = to_opts(o);
        rc.run.eager_optim = eo.eager_optim;
        rc.run.n_slab = eo.n_slab;
        rc.run.threaded_accum = eo.threaded_accum;
        auto store = hlm::build_store(rc.model, seed, rc.run.dtype);
        hlm::DeviceArena arena(rc.model);
        const hlm::TrainOutput out = hlm::run_training(rc, *store, arena, {}, eo);
        for (size_t i = 0; i < out.steps.size(); ++i) losses[i] = out.steps[i].loss;
        if (last && !out.steps.empty()) {
            last->loss = out.steps.back().loss;
            last->h2d_bytes = out.steps.back().h2d_bytes;
            last->d2h_bytes = out.steps.back().d2h_bytes;
            last->gpu_ms = out.steps.back().gpu_ms;
            last->arena_committed = out.final_arena.committed_total;
            last->arena_peak = out.final_arena.step_peak_total;
            last->host_total = out.final_host.total;
        }
    });
}

}  // extern "C"
