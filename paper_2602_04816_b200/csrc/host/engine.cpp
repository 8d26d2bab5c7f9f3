// The B200 streaming engine (see include/hlm/engine.hpp). Control flow
// follows reference proj/src/engine.cpp (begin_step :150-174, forward_impl
// :176-216, anchor_loss_impl :227-269, backward_impl :279-368, finish_step
// :379-424); the memcpy "transfers" and CPU kernels become async copies and
// sm_100a kernels on three streams ordered by events.
#include "hlm/engine.hpp"
#include "hlm/numa_place.hpp"

#include <unistd.h>

#include <cuda_runtime.h>
#include <omp.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "hlm/flop_model.hpp"
#include "hlm_cuda.h"
#include "nccl_dyn.h"

namespace hlm {
inline namespace b200 {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
void ck_hlm(int rc, const char* what) {
    if (rc != HLM_OK) throw CudaError(std::string(what) + ": " + hlm_cuda_last_error());
}
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
cudaEvent_t E(void* e) { return static_cast<cudaEvent_t>(e); }
void* new_event(bool timing) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "cudaEventCreate");
    return e;
}
double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

Engine::Engine(MasterStore& store, DeviceArena& arena, const HyperParams& hyper, EngineOptions opts)
    : store_(store), arena_(arena), hyper_(hyper), opts_(opts) {
    const ModelConfig& m = store.config();
    const ModelConfig& a = arena.config();
    if (m.layers != a.layers || m.hidden != a.hidden || m.ffn != a.ffn || m.vocab != a.vocab || m.seq != a.seq ||
        m.batch != a.batch || m.k_ckpt != a.k_ckpt || m.n_heads != a.n_heads)
        throw ConfigError("engine: store and arena configs differ");
    ck(cudaSetDevice(arena_.device()), "cudaSetDevice");
    if (opts_.world < 1 || opts_.rank < 0 || opts_.rank >= opts_.world) throw ConfigError("engine: bad rank/world");
    if (opts_.world > 1 && !opts_.comm_grad) throw ConfigError("engine: world > 1 needs a gradient communicator");
    if (opts_.comm_grad) {
        if (store_.shared() && store_.world() != opts_.world) throw ConfigError("engine: store world mismatch");
        (void)nccl();
        ck(cudaMalloc(&loss_dev_, sizeof(double)), "cudaMalloc loss");
    }
    // data parallel: slabs hold a 1/world gradient shard, in the DRAM of this GPU's socket
    {
        const ScopedPreferNode local(opts_.world > 1 ? gpu_numa_node(arena_.device()) : -1);
        // two widest-tile slabs (embedding / head gradients), the rest block-sized
        auto round = [](i64 b) { return (b + 255) / 256 * 256; };
        const i64 widest = round(grad_buf_bytes(m) / opts_.world);
        const i64 block = round(4 * m.block_params() / opts_.world);
        std::vector<i64> caps(static_cast<size_t>(std::max<i64>(opts_.n_slab, 1)), widest);
        if (opts_.n_slab >= 4 && block < widest)
            for (size_t i = 2; i < caps.size(); ++i) caps[i] = block;
        pool_ = std::make_unique<SlabPool>(caps, true);
    }
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    h2d_ = s;
    // The critical path gets the block scheduler first: the finiteness scans (D2H stream)
    // and the resident tiles' device Adam (optimizer stream) fill the SMs it leaves idle
    // instead of stealing them from the next layer's GEMMs and attention waves.
    int prio_least = 0, prio_greatest = 0;
    ck(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest), "stream priority range");
    const bool flat = std::getenv("HLM_FLAT_STREAM_PRIORITY") != nullptr;   // A/B switch
    ck(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, flat ? prio_least : prio_greatest), "stream");
    compute_ = s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    d2h_ = s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    opt_ = s;
    if (opts_.comm_grad) {
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        comm_ = s;
    }
    ev_res_grad_ = new_event(false);
    for (int i = 0; i < 2; ++i) {
        ev_w_ready_[i] = new_event(false);
        ev_buf_free_[i] = new_event(false);
        ck(cudaEventRecord(E(ev_buf_free_[i]), S(compute_)), "record");
    }
    {
        const i64 n_gb = std::max<i64>(2, opts_.grad_buffers);
        gbuf_ = {arena_.grad_out(0), arena_.grad_out(1)};
        if (n_gb > 2) {
            const size_t each = static_cast<size_t>((grad_buf_bytes(m) + 255) / 256 * 256);
            ck(cudaMalloc(&gbuf_mem_, each * static_cast<size_t>(n_gb - 2)), "cudaMalloc gradient buffers");
            for (i64 i = 0; i < n_gb - 2; ++i)
                gbuf_.push_back(reinterpret_cast<float*>(static_cast<char*>(gbuf_mem_) + each * static_cast<size_t>(i)));
        }
        for (i64 i = 0; i < n_gb; ++i) {
            ev_grad_ready_.push_back(new_event(false));
            ev_rs_done_.push_back(new_event(false));
            ev_gradbuf_free_.push_back(new_event(false));
            ck(cudaEventRecord(E(ev_gradbuf_free_.back()), S(compute_)), "record");
        }
    }
    for (i64 i = 0; i < pool_->size(); ++i) ev_slab_done_.push_back(new_event(false));
    if (opts_.piece_elems > 0) piece_elems_ = opts_.piece_elems;
    max_pieces_ = std::max<i64>(1, (pool_->slab_capacity() / 4 + piece_elems_ - 1) / piece_elems_);
    // vocab-chunked head (untied): pieces of head_vc_ vocab rows. One rank only: the pieces
    // go D2H without a reduce-scatter (at world 1 the reduction is the identity; at world > 1
    // the head gradient takes the per-tile reduce-scatter of evacuate)
    if ((!opts_.comm_grad || opts_.world == 1) && !m.tie_embeddings && opts_.head_piece_vocab >= 0) {
        i64 vc = opts_.head_piece_vocab;
        if (vc == 0 && m.embed_params() >= 2 * piece_elems_)
            vc = std::max<i64>(128, piece_elems_ / m.hidden / 128 * 128);
        if (vc > 0) vc = std::min<i64>(vc, hlm_cuda_head_chunk_vocab(m.rows(), m.vocab));
        if (vc > 0 && vc < m.vocab) head_vc_ = vc;
    }
    if (head_vc_ > 0) {
        const i64 chunks = (m.vocab + head_vc_ - 1) / head_vc_;
        max_pieces_ = std::max(max_pieces_, chunks);
        for (i64 k = 0; k < chunks; ++k) ev_head_chunk_.push_back(new_event(false));
        ev_head_cert_ = new_event(false);
        ck(cudaMalloc(&head_cert_dev_, 8), "cudaMalloc head certificate");
    }
    ck(cudaMalloc(&nf2_dev_, static_cast<size_t>(pool_->size()) * 8), "cudaMalloc nf2");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&nf2_host_), static_cast<size_t>(pool_->size()) * 8,
                     cudaHostAllocPortable),
       "cudaHostAlloc nf2");
    for (i64 i = 0; i < pool_->size(); ++i) {
        ev_slab_flag_.push_back(new_event(false));
        for (i64 k = 0; k < max_pieces_; ++k) ev_piece_.push_back(new_event(false));
    }
    ck(cudaMalloc(&nf_dev_, static_cast<size_t>(pool_->size()) * 8), "cudaMalloc nf");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&nf_host_), static_cast<size_t>(pool_->size()) * 8,
                     cudaHostAllocPortable),
       "cudaHostAlloc nf");
    ev_step_start_ = new_event(true);
    ev_step_end_ = new_event(true);
    const i64 T = m.rows();
    void* p = nullptr;
    ck(cudaHostAlloc(&p, static_cast<size_t>(4 * (4 * T + m.vocab + 1 + 64)), cudaHostAllocPortable),
       "cudaHostAlloc staging");
    loss_host_ = static_cast<int32_t*>(p);
    if (m.rope_theta > 0)
        ck_hlm(hlm_cuda_rope_table(arena_.rope_cos(), arena_.rope_sin(), m.seq, m.head_dim(), m.rope_theta),
               "rope table");
    // weight cache: the last `slots` blocks stay resident between forward and backward
    cache_slot_of_.assign(static_cast<size_t>(m.tile_count()), -1);
    const i64 slots = arena_.cache_slots();
    for (i64 s = 0; s < slots; ++s) {
        cache_slot_of_[static_cast<size_t>(m.layers - slots + 1 + s)] = s;
        ev_cache_ready_.push_back(new_event(false));
    }
    cache_xfer_op_.assign(static_cast<size_t>(slots), -1);
    if (!(opts_.threaded_accum && opts_.eager_optim && !opts_.skip_optimizer)) opts_.overlap_optimizer_tail = false;
    deferred_.assign(static_cast<size_t>(m.tile_count()), 0);
    // deferred tiles hold their slabs until the tail opens: keep two slabs for the rest
    if (opts_.overlap_optimizer_tail) opts_.tail_blocks = std::min(opts_.tail_blocks, pool_->size() - 3);
    if (opts_.overlap_optimizer_tail && opts_.tail_blocks < 0) opts_.overlap_optimizer_tail = false;
    if (opts_.overlap_optimizer_tail) {
        // a tied head shares the embedding's tile (two consumers): nothing to defer
        if (!m.tie_embeddings) deferred_[static_cast<size_t>(m.head_tile_id())] = 1;
        for (i64 l = std::max<i64>(1, m.layers - opts_.tail_blocks + 1); l <= m.layers; ++l)
            deferred_[static_cast<size_t>(l)] = 1;
    }
    for (i64 p = 0; p < store_.physical_tiles(); ++p)
        target_version_.push_back(store_.physical(p).min_version());
    progress_.assign(static_cast<size_t>(store_.physical_tiles()), 0);
    // HBM-resident optimizer tiles
    resident_of_.assign(static_cast<size_t>(m.tile_count()), -1);
    const bool resident_ok = opts_.eager_optim && !opts_.skip_optimizer && opts_.world == 1 && !opts_.comm_grad &&
                             !m.tie_embeddings && m.k_ckpt == 1 && opts_.fused_recompute;
    if (resident_ok && (opts_.resident_embed || opts_.resident_blocks > 0)) {
        std::vector<i64> ids;
        if (opts_.resident_embed) ids.push_back(m.embed_tile_id());
        for (i64 l = 1; l <= std::min(opts_.resident_blocks, m.layers); ++l) ids.push_back(l);
        size_t bytes = 0;
        for (i64 id : ids) bytes += static_cast<size_t>((store_.tile(id).n_params() * 14 + 255) / 256 * 256);
        ck(cudaMalloc(&resident_mem_, bytes), "cudaMalloc resident optimizer tiles");
        ck(cudaMalloc(&resident_bad_, ids.size() * 8), "cudaMalloc resident flags");
        ck(cudaHostAlloc(reinterpret_cast<void**>(&resident_bad_host_), ids.size() * 8, cudaHostAllocPortable),
           "cudaHostAlloc resident flags");
        char* q = static_cast<char*>(resident_mem_);
        for (i64 id : ids) {
            LayerTile& t = store_.tile(id);
            Resident r{id, t.n_params(), reinterpret_cast<float*>(q),
                       reinterpret_cast<uint16_t*>(q + 12 * t.n_params())};
            resident_of_[static_cast<size_t>(id)] = static_cast<i64>(residents_.size());
            residents_.push_back(r);
            q += (t.n_params() * 14 + 255) / 256 * 256;
        }
        upload_resident();
    }
    // saved activations: the top blocks' forward activations stay in HBM for their backward
    saved_acts_.assign(static_cast<size_t>(m.tile_count()), nullptr);
    if (opts_.saved_act_layers > 0 && m.k_ckpt == 1 && opts_.fused_recompute) {
        const i64 n = std::min(opts_.saved_act_layers, m.layers);
        const size_t bytes = static_cast<size_t>(align256(block_act_bytes(m)));
        ck(cudaMalloc(&saved_mem_, static_cast<size_t>(n) * bytes), "cudaMalloc saved activations");
        for (i64 k = 0; k < n; ++k)
            saved_acts_[static_cast<size_t>(m.layers - k)] = static_cast<char*>(saved_mem_) + static_cast<size_t>(k) * bytes;
    }
    // row-sparse embedding gradient: one rank (at world > 1 the ranks' token rows differ and
    // the dense table takes the per-tile reduce-scatter)
    sparse_embed_ = opts_.sparse_embed_grad && !m.tie_embeddings && resident_of_[0] < 0 && opts_.world == 1 &&
                    opts_.eager_optim && !opts_.skip_optimizer;
    if (sparse_embed_) {
        ck(cudaHostAlloc(reinterpret_cast<void**>(&embed_rows_host_), static_cast<size_t>(m.vocab) * 4,
                         cudaHostAllocPortable),
           "cudaHostAlloc embed rows");
        ck(cudaMalloc(&embed_rows_dev_, static_cast<size_t>(m.vocab) * 4), "cudaMalloc embed rows");
        embed_row_map_.assign(static_cast<size_t>(m.vocab), -1);
    }
    // (data parallel too: each rank gathers its own rows of the shared host shadow)
    if (opts_.embed_gather_host && !m.tie_embeddings && resident_of_[0] < 0 && store_.shadow_pinned()) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, const_cast<uint16_t*>(store_.tile(m.embed_tile_id()).shadow()), 0) ==
            cudaSuccess)
            embed_host_dev_ = dp;
        else
            (void)cudaGetLastError();   // not mapped: stream the table as usual
    }
    // head prefetch: as early as possible, such that no block after the prefetch point
    // uses a stream buffer (cached or HBM-resident), and at the latest before block L - 1
    if (opts_.overlap_optimizer_tail && !m.tie_embeddings && m.k_ckpt == 1 && opts_.fused_recompute &&
        m.layers >= 2) {
        i64 at = m.layers + 1;
        while (at > 1 && (cache_slot_of_[static_cast<size_t>(at - 1)] >= 0 ||
                          resident_of_[static_cast<size_t>(at - 1)] >= 0))
            --at;
        if (at <= m.layers - 1) {
            head_prefetch_ = true;
            head_prefetch_at_ = at;
        }
    }
    if (opts_.threaded_accum) worker_ = std::thread([this] { worker_loop(); });
    store_.set_quiesce(
        [this](bool strict) {
            if (phase_ != Phase::Idle) {
                if (strict) throw ProtocolError("the store was saved / loaded while its engine is inside a step");
                return;
            }
            sync();
        },
        this);
}

// Order in which the next forward needs the tiles (embedding, blocks, head); with
// the head prefetch the head is needed right after block L - 2.
i64 Engine::tail_key(i64 layer) const {
    const ModelConfig& m = store_.config();
    if (layer == m.head_tile_id() && head_prefetch_) return 2 * (head_prefetch_at_ - 1) + 1;
    return 2 * layer;
}

Engine::~Engine() {
    store_.clear_quiesce(this);
    try {
        sync();
    } catch (...) {
    }
    if (resident_mem_) cudaFree(resident_mem_);
    if (resident_bad_) cudaFree(resident_bad_);
    if (resident_bad_host_) cudaFreeHost(resident_bad_host_);
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
        tail_open_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    cudaStreamSynchronize(S(compute_));
    cudaStreamSynchronize(S(h2d_));
    cudaStreamSynchronize(S(d2h_));
    cudaStreamSynchronize(S(opt_));
    cudaEventDestroy(E(ev_res_grad_));
    cudaEventDestroy(E(ev_step_start_));
    cudaEventDestroy(E(ev_step_end_));
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(E(ev_w_ready_[i]));
        cudaEventDestroy(E(ev_buf_free_[i]));
    }
    for (void* e : ev_slab_done_) cudaEventDestroy(E(e));
    for (void* e : ev_slab_flag_) cudaEventDestroy(E(e));
    for (void* e : ev_grad_ready_) cudaEventDestroy(E(e));
    for (void* e : ev_rs_done_) cudaEventDestroy(E(e));
    for (void* e : ev_gradbuf_free_) cudaEventDestroy(E(e));
    if (gbuf_mem_) cudaFree(gbuf_mem_);
    if (embed_rows_host_) cudaFreeHost(embed_rows_host_);
    if (embed_rows_dev_) cudaFree(embed_rows_dev_);
    for (void* e : ev_piece_) cudaEventDestroy(E(e));
    for (void* e : ev_head_chunk_) cudaEventDestroy(E(e));
    if (ev_head_cert_) cudaEventDestroy(E(ev_head_cert_));
    if (head_cert_dev_) cudaFree(head_cert_dev_);
    if (nf2_dev_) cudaFree(nf2_dev_);
    if (nf2_host_) cudaFreeHost(nf2_host_);
    for (void* e : ev_cache_ready_) cudaEventDestroy(E(e));
    for (void* e : timing_events_) cudaEventDestroy(E(e));
    cudaStreamDestroy(S(h2d_));
    cudaStreamDestroy(S(compute_));
    cudaStreamDestroy(S(d2h_));
    cudaStreamDestroy(S(opt_));
    if (comm_) cudaStreamDestroy(S(comm_));
    if (saved_mem_) cudaFree(saved_mem_);
    if (loss_host_) cudaFreeHost(loss_host_);
    if (loss_dev_) cudaFree(loss_dev_);
    if (nf_dev_) cudaFree(nf_dev_);
    if (nf_host_) cudaFreeHost(nf_host_);
}

i64 Engine::shard_elems(i64 n) const {
    if (n % opts_.world) throw ConfigError("data parallel: tile size not divisible by world size");
    return n / opts_.world;
}

// H2D of a tile's bf16 shadow: full copy, or this rank's shard + NVLink all-gather.
void Engine::h2d_tile(void* dst, const LayerTile& tile, i64 bytes) {
    if (opts_.comm_weights && tile.n_params() % opts_.world == 0) {
        const i64 cnt = tile.n_params() / opts_.world;
        const i64 off = opts_.rank * cnt;
        uint16_t* d = static_cast<uint16_t*>(dst);
        ck(cudaMemcpyAsync(d + off, tile.shadow() + off, static_cast<size_t>(cnt) * 2, cudaMemcpyHostToDevice, S(h2d_)),
           "H2D weight shard");
        nccl_check(nccl().AllGather(d + off, d, static_cast<size_t>(cnt), ncclBfloat16,
                                    static_cast<ncclComm_t>(opts_.comm_weights), S(h2d_)),
                   "all-gather weights");
        arena_.add_h2d(cnt * 2);
        return;
    }
    ck(cudaMemcpyAsync(dst, tile.shadow(), static_cast<size_t>(bytes), cudaMemcpyHostToDevice, S(h2d_)), "H2D weights");
    arena_.add_h2d(bytes);
}

// ------------------------------------------------------------------ trace helpers
i64 Engine::op_begin(StreamOp op, void* stream) {
    if (op.kind == OpKind::LocalBackward && gbuf_dep_ >= 0) {   // waits for its gradient buffer
        op.deps.push_back(gbuf_dep_);
        gbuf_dep_ = -1;
    }
    const i64 id = trace_.add(std::move(op));
    if (opts_.record_trace && stream) {
        if (timing_used_ + 2 > timing_events_.size()) {
            timing_events_.push_back(new_event(true));
            timing_events_.push_back(new_event(true));
        }
        ck(cudaEventRecord(E(timing_events_[timing_used_]), S(stream)), "record");
        op_events_.push_back({id, static_cast<int>(timing_used_)});
        timing_used_ += 2;
    }
    return id;
}

void Engine::op_end(i64 id, void* stream) {
    if (!opts_.record_trace || !stream) return;
    for (auto it = op_events_.rbegin(); it != op_events_.rend(); ++it)
        if (it->first == id) {
            ck(cudaEventRecord(E(timing_events_[static_cast<size_t>(it->second + 1)]), S(stream)), "record");
            return;
        }
}

// ------------------------------------------------------------------ streaming
// reference engine.cpp:55-71: alternate buffers, release the old occupant,
// H2D (here straight from the pinned bf16 shadow: no staging copy), with a
// buffer-free dependency on the buffer's last reader.
void* Engine::weights_ptr(int buf) const {
    return buf >= 2 ? arena_.cache_slot(buf - 2) : arena_.buffer(buf);
}

void Engine::wait_tile_current(i64 tile_id, bool all_ranks) {
    if (!opts_.overlap_optimizer_tail) return;
    const i64 p = store_.physical_index(tile_id);
    const LayerTile& tile = store_.physical(p);
    const i64 target = target_version_[static_cast<size_t>(p)];
    const bool others = all_ranks && opts_.world > 1;
    auto ready = [&] {
        return (others ? tile.min_version() : tile.rank_version(opts_.rank)) >= target || worker_error_ != nullptr;
    };
    std::unique_lock<std::mutex> lk(mu_);
    if (others) {
        // other ranks bump their counters in the shared mapping from other processes, which
        // never signal this process's condition variable: poll
        while (!ready()) cv_.wait_for(lk, std::chrono::microseconds(100));
    } else {
        cv_.wait(lk, ready);
    }
    lk.unlock();
    rethrow_worker_error();
}

// Wait until elements [0, end) of the tile hold the update the next H2D needs;
// returns false when the whole tile is current (the rest need not be waited for).
bool Engine::wait_elems_current(i64 tile_id, i64 end) {
    const i64 p = store_.physical_index(tile_id);
    const LayerTile& tile = store_.physical(p);
    bool whole = false;
    std::unique_lock<std::mutex> lk(mu_);
    // this rank's updates only: the piecewise H2D copies this rank's shard (all of the
    // tile at world 1); progress_ counts elements of that shard
    cv_.wait(lk, [&] {
        whole = tile.rank_version(opts_.rank) >= target_version_[static_cast<size_t>(p)];
        return whole || progress_[static_cast<size_t>(p)] >= end || worker_error_ != nullptr;
    });
    lk.unlock();
    rethrow_worker_error();
    return !whole;
}

int Engine::stream_tile(i64 tile_id, i64* op_id, bool forward_pass) {
    const i64 slot = cache_slot_of_[static_cast<size_t>(tile_id)];
    // forward into a cache slot: copy piece by piece behind the optimizer — the whole tile
    // (single GPU) or this rank's shard, then the NVLink all-gather (data parallel with
    // sharded weight H2D; every rank's optimizer publishes progress over its own shard)
    const LayerTile& stile = store_.tile(tile_id);
    const bool piecewise = slot >= 0 && forward_pass && cache_xfer_op_[static_cast<size_t>(slot)] < 0 &&
                           opts_.overlap_optimizer_tail && (opts_.world == 1 || sharded_h2d(stile));
    if (!piecewise && !(slot >= 0 && cache_xfer_op_[static_cast<size_t>(slot)] >= 0))
        wait_tile_current(tile_id, !sharded_h2d(stile));
    if (piecewise) {
        const LayerTile& tile = stile;
        const bool shard = sharded_h2d(tile);
        const i64 n = shard ? tile.n_params() / opts_.world : tile.n_params();
        const i64 base = shard ? opts_.rank * n : 0;
        arena_.claim_cache_slot(slot);
        uint16_t* dst = static_cast<uint16_t*>(arena_.cache_slot(slot)) + base;
        bool waiting = true;
        i64 id = -1;
        const i64 hp = std::min(piece_elems_, kPublishElems);
        for (i64 off = 0; off < n; off += hp) {
            const i64 len = std::min(hp, n - off);
            if (waiting) waiting = wait_elems_current(tile_id, off + len);
            StreamOp op;
            op.stream = StreamId::H2D;
            op.kind = OpKind::WeightXfer;
            op.layer = tile_id;
            op.buf = 2 + slot;
            op.bytes = 2 * len;
            op.pinned = store_.shadow_pinned();
            id = op_begin(std::move(op), h2d_);
            ck(cudaMemcpyAsync(dst + off, tile.shadow() + base + off, static_cast<size_t>(len) * 2,
                               cudaMemcpyHostToDevice, S(h2d_)),
               "H2D weight piece");
            arena_.add_h2d(2 * len);
            op_end(id, h2d_);
        }
        if (shard)
            nccl_check(nccl().AllGather(dst, static_cast<uint16_t*>(arena_.cache_slot(slot)), static_cast<size_t>(n),
                                        ncclBfloat16, static_cast<ncclComm_t>(opts_.comm_weights), S(h2d_)),
                       "all-gather weights");
        ck(cudaEventRecord(E(ev_cache_ready_[static_cast<size_t>(slot)]), S(h2d_)), "record cache ready");
        cache_xfer_op_[static_cast<size_t>(slot)] = id;
        *op_id = id;
        return 2 + static_cast<int>(slot);
    }
    if (slot >= 0) {
        if (cache_xfer_op_[static_cast<size_t>(slot)] >= 0) {   // resident since this step's forward
            *op_id = cache_xfer_op_[static_cast<size_t>(slot)];
            return 2 + static_cast<int>(slot);
        }
        if (forward_pass) {
            const LayerTile& tile = store_.tile(tile_id);
            const i64 bytes = tile.weight_bytes();
            arena_.claim_cache_slot(slot);
            StreamOp op;
            op.stream = StreamId::H2D;
            op.kind = OpKind::WeightXfer;
            op.layer = tile_id;
            op.buf = 2 + slot;
            op.bytes = bytes;
            op.pinned = store_.shadow_pinned();
            const i64 id = op_begin(std::move(op), h2d_);
            h2d_tile(arena_.cache_slot(slot), tile, bytes);
            op_end(id, h2d_);
            ck(cudaEventRecord(E(ev_cache_ready_[static_cast<size_t>(slot)]), S(h2d_)), "record cache ready");
            cache_xfer_op_[static_cast<size_t>(slot)] = id;
            *op_id = id;
            return 2 + static_cast<int>(slot);
        }
    }
    const int buf = next_buf_;
    next_buf_ ^= 1;
    if (arena_.buffer_occupant(buf) != -1) arena_.release_buffer(buf);
    const LayerTile& tile = store_.tile(tile_id);
    const i64 bytes = tile.weight_bytes();
    void* dst = arena_.claim_buffer(buf, tile_id, bytes);
    StreamOp op;
    op.stream = StreamId::H2D;
    op.kind = OpKind::WeightXfer;
    op.layer = tile_id;
    op.buf = buf;
    op.bytes = bytes;
    op.pinned = store_.shadow_pinned();
    if (last_reader_[buf] >= 0) op.deps.push_back(last_reader_[buf]);
    ck(cudaStreamWaitEvent(S(h2d_), E(ev_buf_free_[buf]), 0), "wait buf free");
    const i64 id = op_begin(std::move(op), h2d_);
    h2d_tile(dst, tile, bytes);
    op_end(id, h2d_);
    ck(cudaEventRecord(E(ev_w_ready_[buf]), S(h2d_)), "record w ready");
    *op_id = id;
    return buf;
}

void Engine::compute_wait_weights(int buf) {
    void* ev = buf >= 2 ? ev_cache_ready_[static_cast<size_t>(buf - 2)] : ev_w_ready_[buf];
    ck(cudaStreamWaitEvent(S(compute_), E(ev), 0), "wait weights");
}

void Engine::compute_done_with(int buf, i64 op_id) {
    if (buf >= 2) return;   // cache slots are rewritten only by the next step's forward
    ck(cudaEventRecord(E(ev_buf_free_[buf]), S(compute_)), "record buf free");
    last_reader_[buf] = op_id;
}

int Engine::next_grad_buf() {
    const int gb = next_gbuf_;
    next_gbuf_ = (next_gbuf_ + 1) % static_cast<int>(gbuf_.size());
    ck(cudaStreamWaitEvent(S(compute_), E(ev_gradbuf_free_[gb]), 0), "wait grad buf");
    gbuf_dep_ = static_cast<size_t>(gb) < gbuf_free_op_.size() ? gbuf_free_op_[static_cast<size_t>(gb)] : -1;
    return gb;
}

// A FREE slab of at least `bytes` (reference SlabPool::acquire,
// host_store.cpp:197-218): blocks on the worker, or consumes the oldest READY
// slab inline.
i64 Engine::acquire_slab(i64 bytes) {
    i64 slab = pool_->try_acquire(bytes);
    while (slab < 0) {
        if (opts_.threaded_accum) {
            rethrow_worker_error();
            {
                std::lock_guard<std::mutex> lk(mu_);
                bool any = in_process_ > 0;
                for (const auto& q : pending_) any = any || eligible(q);
                if (!any && !pending_.empty()) tail_open_ = true;   // never wedge on deferred slabs
            }
            cv_.notify_all();
            slab = pool_->acquire_blocking(bytes);
        } else {
            process_oldest_inline();
            slab = pool_->try_acquire(bytes);
        }
    }
    return slab;
}

// reference engine.cpp:103-121: acquire a slab (inline back-pressure
// consumes the oldest READY slab), D2H the fp32 gradient, emit GradXfer.
void Engine::evacuate(i64 tile_id, int gbuf, i64 n_params, i64 lb_op, bool sparse_rows) {
    const i64 cnt = opts_.comm_grad ? shard_elems(n_params) : n_params;
    const i64 bytes = 4 * cnt;
    const i64 slab = acquire_slab(bytes);
    pool_->mark_in_flight(slab, tile_id, bytes);
    // the reference's "all gradients finite before any mutation" check, on the GPU, in
    // stream order behind the kernels that wrote the gradient (single GPU: the compute
    // stream; data parallel: the communicator's stream, behind the reduce-scatter, since a
    // sum of finite shards can overflow). A scan on a side stream would take SMs from the
    // persistent GEMM that follows on the compute stream and stall its static tile schedule.
    if (!opts_.comm_grad) ck_hlm(hlm_cuda_nonfinite(grad_buf(gbuf), cnt, nf_dev_ + slab, compute_), "nonfinite scan");
    ck(cudaEventRecord(E(ev_grad_ready_[gbuf]), S(compute_)), "record grad ready");
    StreamOp op;
    op.stream = StreamId::D2H;
    op.kind = OpKind::GradXfer;
    op.layer = tile_id;
    op.slab = slab;
    op.bytes = bytes;
    op.deps.push_back(lb_op);
    if (last_accum_op_[static_cast<size_t>(slab)] >= 0) op.deps.push_back(last_accum_op_[static_cast<size_t>(slab)]);
    float* src = grad_buf(gbuf);
    if (opts_.comm_grad) {
        // in-place reduce-scatter over NVLink on its own stream, so layer i's shard D2H
        // (d2h_) runs beside layer i-1's reduce-scatter (comm_); then D2H of this rank's shard
        src += opts_.rank * cnt;
        ck(cudaStreamWaitEvent(S(comm_), E(ev_grad_ready_[gbuf]), 0), "wait grad ready (comm)");
        nccl_check(nccl().ReduceScatter(grad_buf(gbuf), src, static_cast<size_t>(cnt), ncclFloat32, ncclSum,
                                        static_cast<ncclComm_t>(opts_.comm_grad), S(comm_)),
                   "reduce-scatter grads");
        ck_hlm(hlm_cuda_nonfinite(src, cnt, nf_dev_ + slab, comm_), "nonfinite scan");
        ck(cudaEventRecord(E(ev_rs_done_[static_cast<size_t>(gbuf)]), S(comm_)), "record rs done");
        ck(cudaStreamWaitEvent(S(d2h_), E(ev_rs_done_[static_cast<size_t>(gbuf)]), 0), "wait rs done");
    } else {
        ck(cudaStreamWaitEvent(S(d2h_), E(ev_grad_ready_[gbuf]), 0), "wait grad ready");
    }
    const i64 id = op_begin(std::move(op), d2h_);
    gbuf_free_op_[static_cast<size_t>(gbuf)] = id;
    // the finiteness flag lands first, then the gradient in pieces (the optimizer starts on piece 0)
    ck(cudaMemcpyAsync(nf_host_ + slab, nf_dev_ + slab, 8, cudaMemcpyDeviceToHost, S(d2h_)), "D2H nf flag");
    ck(cudaEventRecord(E(ev_slab_flag_[static_cast<size_t>(slab)]), S(d2h_)), "record slab flag");
    const i64 pieces = (cnt + piece_elems_ - 1) / piece_elems_;
    for (i64 k = 0; k < pieces; ++k) {
        const i64 off = k * piece_elems_, len = std::min(piece_elems_, cnt - off);
        ck(cudaMemcpyAsync(pool_->data(slab) + off, src + off, static_cast<size_t>(len) * 4, cudaMemcpyDeviceToHost,
                           S(d2h_)),
           "D2H grads");
        ck(cudaEventRecord(E(ev_piece_[static_cast<size_t>(slab * max_pieces_ + k)]), S(d2h_)), "record piece");
    }
    op_end(id, d2h_);
    ck(cudaEventRecord(E(ev_slab_done_[static_cast<size_t>(slab)]), S(d2h_)), "record slab done");
    ck(cudaEventRecord(E(ev_gradbuf_free_[gbuf]), S(d2h_)), "record grad buf free");
    {
        std::lock_guard<std::mutex> lk(mu_);
        pending_.push_back({slab, tile_id, id, step_index_, step_t_, cnt, pieces, piece_elems_, sparse_rows});
    }
    cv_.notify_all();
}

// One slab: wait for its D2H, then accumulate / optimise (reference
// host_store.cpp:254-284 and the eager hook engine.cpp:136-148). Numerics do
// not depend on inline vs threaded consumption nor on the slab count.
void Engine::consume(const Pending& p) {
    LayerTile& tile = store_.tile(p.layer);
    const i64 phys = store_.physical_index(p.layer);
    const bool optimise = opts_.eager_optim && !opts_.skip_optimizer;
    // fused (slab IS the gradient, one consumer): wait for the finiteness flag, then
    // optimise piece by piece as the D2H lands; otherwise wait for the whole slab
    const bool piecewise = optimise && store_.consumer_count(phys) == 1 && !p.sparse_rows;
    ck(cudaEventSynchronize(E(piecewise ? ev_slab_flag_[static_cast<size_t>(p.slab)]
                                        : ev_slab_done_[static_cast<size_t>(p.slab)])),
       "slab sync");
    pool_->mark_ready(p.slab);
    bool stop = false;
    const i64 id = pool_->pop_ready_blocking(&stop);
    if (id != p.slab) throw ProtocolError("slab FIFO order violated");
    if (opts_.accum_delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(opts_.accum_delay_us));
    HostOpRecord rec{p.slab, p.layer, p.grad_op, p.step, now_us(), 0.0, false, 0.0, 0.0};
    unsigned long long bad = nf_host_[p.slab];
    if (bad == HLM_HEAD_UNCERTIFIED) {   // vocab-chunked head without a certificate: the full scan
        ck(cudaEventSynchronize(E(ev_slab_done_[static_cast<size_t>(p.slab)])), "slab sync");
        bad = nf2_host_[p.slab];
    }
    if (bad != ~0ull && optimise && p.sparse_rows) {   // compact index -> table element
        const i64 h = store_.config().hidden;
        const i64 c = static_cast<i64>(bad) / h, j = static_cast<i64>(bad) % h;
        throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + " at element " +
                            std::to_string(static_cast<i64>(embed_rows_host_[c]) * h + j) + "; step aborted");
    }
    if (bad != ~0ull && optimise) {
        const i64 base = opts_.comm_grad ? opts_.rank * shard_elems(tile.n_params()) : 0;
        throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + " at element " +
                            std::to_string(base + static_cast<i64>(bad)) + "; step aborted");
    }
    // fused piecewise Adam over [base, base + count): the tile, or this rank's shard
    auto adam_pieces = [&](i64 base) {
        rec.t1 = now_us();
        rec.opt = true;
        rec.topt0 = rec.t1;
        const float* g = pool_->data(p.slab);
        const size_t pi = static_cast<size_t>(phys);
        for (i64 k = 0; k < p.pieces; ++k) {
            const i64 off = k * p.piece, len = std::min(p.piece, p.count - off);
            ck(cudaEventSynchronize(E(ev_piece_[static_cast<size_t>(p.slab * max_pieces_ + k)])), "piece sync");
            // optimise in sub-pieces and publish each: a forward H2D copies right behind
            for (i64 so = 0; so < len; so += kPublishElems) {
                const i64 sl = std::min(kPublishElems, len - so);
                adam_step_range(tile, g + off + so, base + off + so, sl, hyper_, p.t, /*prechecked=*/true);
                {   // elements of this rank's range done (the piecewise forward H2D follows)
                    std::lock_guard<std::mutex> lk(mu_);
                    progress_[pi] = off + so + sl;
                }
                cv_.notify_all();
            }
        }
        {   // the version now covers the whole tile; progress counts the next update
            std::lock_guard<std::mutex> lk(mu_);
            tile.bump_version(opts_.rank);
            progress_[pi] = 0;
        }
        cv_.notify_all();
        rec.topt1 = now_us();
    };
    if (opts_.comm_grad && !p.sparse_rows) {   // this rank's shard [begin, begin + cnt)
        const i64 cnt = shard_elems(tile.n_params()), begin = opts_.rank * cnt;
        const float* g = pool_->data(p.slab);
        if (piecewise) {
            adam_pieces(begin);
        } else {
            float* dst = tile.grads() + begin;
            for (i64 i = 0; i < cnt; ++i) dst[i] = dst[i] + g[i];
            rec.t1 = now_us();
            bool last = false;
            {
                std::lock_guard<std::mutex> lk(mu_);
                last = --consumers_left_[static_cast<size_t>(phys)] == 0;
            }
            if (optimise && last) {
                rec.opt = true;
                rec.topt0 = now_us();
                adam_step_range(tile, dst, begin, cnt, hyper_, p.t);
                std::fill(dst, dst + cnt, 0.0f);
                tile.bump_version(opts_.rank);
                rec.topt1 = now_us();
            }
        }
    } else if (p.sparse_rows) {
        // row-compact embedding gradient: untouched rows optimised with a zero gradient
        rec.t1 = now_us();
        rec.opt = true;
        rec.topt0 = rec.t1;
        const ModelConfig& m = store_.config();
        adam_step_rows_sparse(tile, m.vocab, m.hidden, embed_row_map_.data(), pool_->data(p.slab), hyper_, p.t);
        rec.topt1 = now_us();
    } else if (piecewise) {
        // fused: the pinned slab IS the gradient; no store gradient region touched
        adam_pieces(0);
    } else {
        accumulate_grads(tile, pool_->data(p.slab));
        rec.t1 = now_us();
        bool last = false;
        {
            std::lock_guard<std::mutex> lk(mu_);
            last = --consumers_left_[static_cast<size_t>(phys)] == 0;
        }
        if (optimise && last) {
            rec.opt = true;
            rec.topt0 = now_us();
            adam_step_tile(store_, phys, hyper_, p.t);
            rec.topt1 = now_us();
        }
    }
    pool_->release(p.slab);
    std::lock_guard<std::mutex> lk(mu_);
    host_ops_.push_back(rec);
    if (p.step == step_index_ && !deferred_[static_cast<size_t>(p.layer)] && --regular_left_ == 0) tail_open_ = true;
}

bool Engine::eligible(const Pending&) const { return true; }

// Gradient of a resident tile: GPU finiteness scan, then the device Adam (no-op
// on a flagged gradient; finish_step raises NumericsError). HBM-bound, so it runs on
// its own stream beside the compute-bound backward of the layers below; nothing in
// this step reads the tile's weights again, the next step starts after finish_step
// synchronised that stream, and the gradient buffer is released when the Adam is done.
void Engine::resident_update(i64 tile, int gbuf, i64 dep_op) {
    const i64 ri = resident_of_[static_cast<size_t>(tile)];
    const Resident& r = residents_[static_cast<size_t>(ri)];
    ck(cudaEventRecord(E(ev_res_grad_), S(compute_)), "record resident grad");
    ck(cudaStreamWaitEvent(S(opt_), E(ev_res_grad_), 0), "wait resident grad");
    StreamOp op;
    op.stream = StreamId::Compute;   // trace schema: a GPU op of the step (on the optimizer stream)
    op.kind = OpKind::OptStep;
    op.layer = tile;
    op.params = r.n;
    op.deps.push_back(dep_op);
    const i64 id = op_begin(op, opt_);
    ck_hlm(hlm_cuda_nonfinite(grad_buf(gbuf), r.n, resident_bad_ + ri, opt_), "nonfinite (resident)");
    HlmHyper hp{hyper_.lr, hyper_.beta1, hyper_.beta2, hyper_.eps, hyper_.weight_decay};
    ck_hlm(hlm_cuda_adam(r.state, r.state + r.n, r.state + 2 * r.n, r.w16, grad_buf(gbuf), r.n,
                         resident_bad_ + ri, &hp, step_t_, opt_),
           "device adam");
    op_end(id, opt_);
    gbuf_free_op_[static_cast<size_t>(gbuf)] = id;
    ck(cudaEventRecord(E(ev_gradbuf_free_[gbuf]), S(opt_)), "record grad buf free (resident)");
    if (!resident_dirty_) store_.add_device_newer(1);
    resident_dirty_ = true;
}

void Engine::process_oldest_inline() {
    Pending p;
    {
        std::lock_guard<std::mutex> lk(mu_);
        if (pending_.empty()) throw ProtocolError("slab pool exhausted with nothing to accumulate");
        p = pending_.front();
        pending_.pop_front();
    }
    consume(p);
}

// Pin the optimizer's OpenMP team one thread per CPU. Unpinned, the team's threads
// migrate and collide with the issue / CUDA threads: measured at C2, 8.2-8.6 k tok/s
// unpinned vs 8.7-9.3 k pinned on the same boxes. One rank: every allowed CPU; data
// parallel: the rank's slice of its GPU's NUMA node, shared evenly with the other ranks
// on that node, so N ranks on one host never stack N pinned teams on the same cores.
// Without an explicit thread count the team leaves one CPU of a slice of 8 or more to
// the thread issuing the GPU work (15 of 16: 9.1-9.2 k, steadier than 16).
// Scheduling only; results unchanged.
void pin_optimizer_team(int rank, int world, bool default_team) {
    const std::vector<int> allowed = allowed_cpus();
    if (allowed.empty()) return;
    std::vector<int> cpus = allowed;
    if (world > 1) {
        std::vector<std::vector<int>> of_node(static_cast<size_t>(numa_node_count()));
        for (size_t n = 0; n < of_node.size(); ++n) of_node[n] = node_cpus(static_cast<int>(n));
        cpus = rank_cpu_slice(rank, rank_gpu_nodes(world), allowed, static_cast<int>(sysconf(_SC_NPROCESSORS_ONLN)),
                              of_node);
    }
    if (default_team) {
        const int n = static_cast<int>(cpus.size());
        omp_set_num_threads(n >= 8 ? n - 1 : std::max(1, n));
    }
#pragma omp parallel
    {
        cpu_set_t one;
        CPU_ZERO(&one);
        CPU_SET(cpus[static_cast<size_t>(omp_get_thread_num()) % cpus.size()], &one);
        pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
    }
}

void Engine::worker_loop() {
    if (opts_.host_threads > 0) omp_set_num_threads(opts_.host_threads);
    if (opts_.pin_threads) pin_optimizer_team(opts_.rank, opts_.world, opts_.host_threads <= 0);
    for (;;) {
        Pending p;
        {
            std::unique_lock<std::mutex> lk(mu_);
            // Never idle while a gradient is available. Among slabs whose D2H has
            // landed: the previous step's tail first (the running forward needs
            // it, in tile order), then this step's regular tiles in arrival order,
            // then this step's tail tiles in the order the next forward consumes
            // them (ascending id, head last). With none landed, the oldest entry
            // (the D2H stream completes in issue order).
            auto pick = [&]() -> bool {
                if (pending_.empty()) return false;
                auto best = pending_.end();
                std::pair<int, i64> best_rank{3, 0};
                i64 pos = 0;
                for (auto it = pending_.begin(); it != pending_.end(); ++it, ++pos) {
                    const cudaError_t q = cudaEventQuery(E(ev_slab_flag_[static_cast<size_t>(it->slab)]));
                    if (q == cudaErrorNotReady) continue;
                    if (q != cudaSuccess) (void)cudaGetLastError();   // surfaced by consume's synchronize
                    std::pair<int, i64> rank;
                    if (it->step < step_index_)
                        rank = {0, tail_key(it->layer)};
                    else if (!deferred_[static_cast<size_t>(it->layer)])
                        rank = {1, pos};
                    else
                        rank = {2, tail_key(it->layer)};
                    if (rank < best_rank) {
                        best_rank = rank;
                        best = it;
                    }
                }
                if (best == pending_.end()) best = pending_.begin();
                p = *best;
                pending_.erase(best);
                return true;
            };
            bool got = false;
            cv_.wait(lk, [&] {
                got = pick();
                return got || (stop_ && pending_.empty());
            });
            if (!got) return;
            ++in_process_;
        }
        try {
            consume(p);
        } catch (...) {
            std::lock_guard<std::mutex> lk(mu_);
            if (!worker_error_) worker_error_ = std::current_exception();
            // a failed slab must not wedge back-pressure
            try {
                pool_->release(p.slab);
            } catch (...) {
            }
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            --in_process_;
        }
        cv_.notify_all();
    }
}

void Engine::rethrow_worker_error() {
    std::exception_ptr e;
    {
        std::lock_guard<std::mutex> lk(mu_);
        e = worker_error_;
        worker_error_ = nullptr;
    }
    if (e) std::rethrow_exception(e);
}

void Engine::sync_resident() {
    if (!resident_dirty_) return;
    ck(cudaStreamSynchronize(S(compute_)), "sync compute");
    ck(cudaStreamSynchronize(S(opt_)), "sync optimizer stream");
    for (const auto& r : residents_) {
        LayerTile& t = store_.tile(r.tile);
        ck(cudaMemcpy(t.master(), r.state, static_cast<size_t>(12 * r.n), cudaMemcpyDeviceToHost), "download state");
        ck(cudaMemcpy(t.shadow(), r.w16, static_cast<size_t>(2 * r.n), cudaMemcpyDeviceToHost), "download weights");
    }
    resident_dirty_ = false;
    store_.add_device_newer(-1);
}

void Engine::sync() {
    wait_optimizer();
    sync_resident();
}

// FP32 state and BF16 weights of the HBM-resident tiles from the store (construction,
// and again when load_checkpoint / import_master replaced the store: epoch changed).
void Engine::upload_resident() {
    for (const auto& r : residents_) {
        const LayerTile& t = store_.tile(r.tile);
        ck(cudaMemcpy(r.state, t.master(), static_cast<size_t>(12 * r.n), cudaMemcpyHostToDevice),
           "upload resident state");
        ck(cudaMemcpy(r.w16, t.shadow(), static_cast<size_t>(2 * r.n), cudaMemcpyHostToDevice),
           "upload resident weights");
    }
    resident_epoch_ = store_.epoch();
}

void Engine::wait_optimizer() {
    if (!opts_.threaded_accum) return;
    {
        std::unique_lock<std::mutex> lk(mu_);
        tail_open_ = true;
        cv_.notify_all();
        cv_.wait(lk, [&] { return pending_.empty() && in_process_ == 0; });
    }
    rethrow_worker_error();
}

void Engine::drain() {
    if (opts_.threaded_accum && opts_.overlap_optimizer_tail) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return tail_open_ || worker_error_ != nullptr; });
    } else if (opts_.threaded_accum) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return pending_.empty() && in_process_ == 0; });
    } else {
        for (;;) {
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (pending_.empty()) break;
            }
            process_oldest_inline();
        }
    }
    rethrow_worker_error();
}

// ------------------------------------------------------------------ phases
void Engine::begin_step(const Batch& batch) {
    if (phase_ != Phase::Idle) throw ProtocolError("begin_step outside Idle phase");
    const ModelConfig& m = store_.config();
    const i64 T = m.rows();
    if (static_cast<i64>(batch.tokens.size()) != T || static_cast<i64>(batch.targets.size()) != T)
        throw ConfigError("batch size does not match model config");
    batch_ = batch;
    if (!residents_.empty() && store_.epoch() != resident_epoch_) {
        // the store was replaced (sync() ran first through the quiesce hook, so nothing
        // newer lives on the device): train on the loaded state
        if (resident_dirty_) {
            resident_dirty_ = false;
            store_.add_device_newer(-1);
        }
        upload_resident();
    }
    arena_.begin_step();
    arena_.claim_workspace();
    trace_ = EventTrace{};
    gbuf_free_op_.assign(gbuf_.size(), -1);   // op ids are per step
    gbuf_dep_ = -1;
    trace_.meta = TraceMeta{m.layers, 2, pool_->size(), m.embed_tile_id(), m.head_tile_id()};
    op_events_.clear();
    timing_used_ = 0;
    next_buf_ = 0;
    next_gbuf_ = 0;
    head_buf_ = -1;
    g_cur_ = 0;
    last_reader_[0] = last_reader_[1] = -1;
    last_accum_op_.assign(static_cast<size_t>(pool_->size()), -1);
    rethrow_worker_error();
    {
        std::lock_guard<std::mutex> lk(mu_);
        ++step_index_;
        regular_left_ = 0;
        for (i64 t = 0; t < m.tile_count(); ++t)
            if (!deferred_[static_cast<size_t>(t)] && resident_of_[static_cast<size_t>(t)] < 0) ++regular_left_;
        tail_open_ = !opts_.overlap_optimizer_tail || regular_left_ == 0;
        if (!opts_.overlap_optimizer_tail) pending_.clear();
        consumers_left_.assign(static_cast<size_t>(store_.physical_tiles()), 0);
        for (i64 p = 0; p < store_.physical_tiles(); ++p)
            consumers_left_[static_cast<size_t>(p)] = store_.consumer_count(p);
    }
    std::fill(cache_xfer_op_.begin(), cache_xfer_op_.end(), -1);
    step_t_ = store_.adam_steps() + 1;
    d2h_base_ = pool_->d2h_bytes();
    recompute_forwards_ = 0;
    host_t0_us_ = now_us();
    ck(cudaEventRecord(E(ev_step_start_), S(compute_)), "record step start");
    ck(cudaStreamWaitEvent(S(h2d_), E(ev_step_start_), 0), "wait");
    ck(cudaStreamWaitEvent(S(d2h_), E(ev_step_start_), 0), "wait");
    // batch -> device (pinned staging, compute stream orders it before use)
    int32_t* st = loss_host_;
    std::memcpy(st, batch.tokens.data(), static_cast<size_t>(T) * 4);
    std::memcpy(st + T, batch.targets.data(), static_cast<size_t>(T) * 4);
    ck(cudaMemcpyAsync(arena_.tokens(), st, static_cast<size_t>(T) * 4, cudaMemcpyHostToDevice, S(compute_)), "H2D tok");
    ck(cudaMemcpyAsync(arena_.targets(), st + T, static_cast<size_t>(T) * 4, cudaMemcpyHostToDevice, S(compute_)),
       "H2D tgt");
    ck(cudaMemsetAsync(arena_.err_flag(), 0, 4, S(compute_)), "memset err");
    phase_ = Phase::Forward;
}

// reference engine.cpp:176-216
void Engine::forward_streaming() {
    if (phase_ != Phase::Forward) throw ProtocolError("forward_streaming out of order");
    const ModelConfig& m = store_.config();
    const i64 T = m.rows();
    for (i64 t = 0; t < T; ++t)
        if (batch_.tokens[static_cast<size_t>(t)] < 0 || batch_.tokens[static_cast<size_t>(t)] >= m.vocab)
            throw std::out_of_range("embed_fwd: token id out of range");
    const HlmBlockDims dims = block_dims(m, opts_.block_flags);
    const float* rc = m.rope_theta > 0 ? arena_.rope_cos() : nullptr;
    const float* rs = m.rope_theta > 0 ? arena_.rope_sin() : nullptr;

    i64 w_op = -1;
    const bool embed_res = is_resident(m.embed_tile_id());
    const bool embed_zc = !embed_res && embed_host_dev_ != nullptr;
    if (embed_zc) {   // zero-copy gather: only the table version must be current (every shard)
        wait_tile_current(m.embed_tile_id(), true);
        arena_.add_h2d(T * m.hidden * 2);
    }
    const int ebuf = embed_res ? -2 : embed_zc ? -3 : stream_tile(m.embed_tile_id(), &w_op);
    if (!embed_res && !embed_zc) compute_wait_weights(ebuf);
    float* h0 = arena_.anchor_checkpoint(0);
    StreamOp op;
    op.stream = StreamId::Compute;
    op.kind = OpKind::Forward;
    op.layer = m.embed_tile_id();
    op.buf = ebuf;   // -2: HBM-resident weights, -3: rows gathered zero-copy from the host shadow
    op.flops = fwd_flops(m.embed_params(), T);
    if (w_op >= 0) op.deps.push_back(w_op);
    i64 id = op_begin(op, compute_);
    const void* etab = embed_res  ? static_cast<const void*>(residents_[static_cast<size_t>(resident_of_[0])].w16)
                       : embed_zc ? embed_host_dev_
                                  : weights_ptr(ebuf);
    ck_hlm(hlm_cuda_embed_fwd(arena_.tokens(), etab, h0, T, m.hidden, m.vocab, arena_.err_flag(), compute_),
           "embed_fwd");
    op_end(id, compute_);
    if (!embed_res && !embed_zc) compute_done_with(ebuf, id);
    h_cur_ = h0;
    int roll = 0;
    for (i64 i = 1; i <= m.layers; ++i) {
        if (head_prefetch_ && i == head_prefetch_at_) head_buf_ = stream_tile(m.head_tile_id(), &head_wop_);
        const bool res = is_resident(i);
        w_op = -1;
        const int buf = res ? -2 : stream_tile(i, &w_op, true);
        if (!res) compute_wait_weights(buf);
        const void* wptr = res ? static_cast<const void*>(residents_[static_cast<size_t>(resident_of_[static_cast<size_t>(i)])].w16)
                               : weights_ptr(buf);
        float* out = (i % m.k_ckpt == 0) ? arena_.anchor_checkpoint(i) : arena_.h_roll(roll);
        if (i % m.k_ckpt != 0) roll ^= 1;
        StreamOp bo;
        bo.stream = StreamId::Compute;
        bo.kind = OpKind::Forward;
        bo.layer = i;
        bo.buf = buf;
        bo.flops = fwd_flops(m.block_params(), T);
        if (w_op >= 0) bo.deps.push_back(w_op);
        id = op_begin(bo, compute_);
        void* acts = saved_acts_[static_cast<size_t>(i)] ? saved_acts_[static_cast<size_t>(i)] : arena_.discard_acts();
        ck_hlm(hlm_cuda_block_fwd(&dims, wptr, h_cur_, out, acts, arena_.block_ws(), rc, rs, compute_), "block_fwd");
        op_end(id, compute_);
        if (!res) compute_done_with(buf, id);
        h_cur_ = out;
    }
    phase_ = Phase::Anchor;
}

// reference engine.cpp:227-269: head fwd + CE + head bwd; g_L into the carry,
// the head gradient straight to the outbound buffer and a slab.
double Engine::anchor_loss() {
    anchor_loss_async();
    ck(cudaStreamSynchronize(S(compute_)), "sync loss");
    const i64 T = store_.config().rows();
    double loss = 0.0;
    const float* lr = reinterpret_cast<const float*>(loss_host_ + 2 * T);
    for (i64 r = 0; r < T; ++r) loss += static_cast<double>(lr[r]);
    return loss;
}

void Engine::anchor_loss_async() {
    if (phase_ != Phase::Anchor) throw ProtocolError("anchor_loss out of order");
    const ModelConfig& m = store_.config();
    const i64 T = m.rows();
    for (i64 t = 0; t < T; ++t)
        if (batch_.targets[static_cast<size_t>(t)] < 0 || batch_.targets[static_cast<size_t>(t)] >= m.vocab)
            throw std::out_of_range("ce_loss_and_grad: target id out of range");
    i64 w_op = 0;
    int buf = head_buf_;
    if (buf >= 0) {   // prefetched during the forward
        w_op = head_wop_;
        head_buf_ = -1;
    } else {
        buf = stream_tile(m.head_tile_id(), &w_op);
    }
    compute_wait_weights(buf);
    if (head_vc_ > 0) {
        anchor_loss_pieces(buf, w_op);
        if (m.layers % m.k_ckpt == 0) arena_.release_checkpoint(m.layers);
        phase_ = Phase::Backward;
        return;
    }
    const int gb = next_grad_buf();
    StreamOp op;
    op.stream = StreamId::Compute;
    op.kind = OpKind::Forward;
    op.layer = m.head_tile_id();
    op.buf = buf;
    op.flops = fwd_flops(m.embed_params(), T);
    op.deps.push_back(w_op);
    const i64 fid = op_begin(op, compute_);
    ck_hlm(hlm_cuda_head_loss(T, m.hidden, m.vocab, weights_ptr(buf), h_cur_, arena_.targets(),
                              1.0f / static_cast<float>(T * opts_.world), arena_.g_roll(g_cur_), grad_buf(gb), 0,
                              arena_.loss_rows(), arena_.head_ws(), compute_),
           "head_loss");
    op_end(fid, compute_);
    // the logical trace keeps the reference's separate Forward / LocalBackward ops
    StreamOp lb;
    lb.stream = StreamId::Compute;
    lb.kind = OpKind::LocalBackward;
    lb.layer = m.head_tile_id();
    lb.buf = buf;
    lb.flops = bwd_flops(m.embed_params(), T);
    lb.deps.push_back(w_op);
    const i64 lb_op = trace_.add(lb);
    trace_.ops[static_cast<size_t>(lb_op)].t_start_us = -2.0;   // shares the fused launch's timing
    compute_done_with(buf, lb_op);
    ck(cudaMemcpyAsync(loss_host_ + 2 * T, arena_.loss_rows(), static_cast<size_t>(T) * 4, cudaMemcpyDeviceToHost,
                       S(compute_)),
       "D2H loss");
    ck(cudaMemcpyAsync(loss_host_ + 3 * T, arena_.err_flag(), 4, cudaMemcpyDeviceToHost, S(compute_)), "D2H err");
    evacuate(m.head_tile_id(), gb, m.embed_params(), lb_op);
    if (m.layers % m.k_ckpt == 0) arena_.release_checkpoint(m.layers);
    phase_ = Phase::Backward;
}

// Vocab-chunked head (same numbers as hlm_cuda_head_loss, in pieces): pass 1
// (row statistics, loss, finiteness certificate) as the head Forward, then per
// piece of head_vc_ vocab rows a LocalBackward (logits, d_logits, d_head rows,
// d_x accumulation) whose d_head rows go to the slab at once, so the host Adam of
// the head starts one piece after the statistics instead of after the whole head.
void Engine::anchor_loss_pieces(int buf, i64 w_op) {
    const ModelConfig& m = store_.config();
    const i64 T = m.rows(), V = m.vocab, h = m.hidden, n = m.embed_params();
    const i64 head = m.head_tile_id();
    const float inv = 1.0f / static_cast<float>(T * opts_.world);
    const void* W = weights_ptr(buf);
    const int gb = next_grad_buf();
    StreamOp op;
    op.stream = StreamId::Compute;
    op.kind = OpKind::Forward;
    op.layer = head;
    op.buf = buf;
    op.flops = fwd_flops(n, T);
    op.deps.push_back(w_op);
    const i64 fid = op_begin(op, compute_);
    ck_hlm(hlm_cuda_head_stats(T, h, V, W, h_cur_, arena_.targets(), inv, arena_.loss_rows(), head_cert_dev_,
                               arena_.head_ws(), compute_),
           "head_stats");
    op_end(fid, compute_);
    ck(cudaEventRecord(E(ev_head_cert_), S(compute_)), "record head certificate");
    ck(cudaMemcpyAsync(loss_host_ + 2 * T, arena_.loss_rows(), static_cast<size_t>(T) * 4, cudaMemcpyDeviceToHost,
                       S(compute_)),
       "D2H loss");
    ck(cudaMemcpyAsync(loss_host_ + 3 * T, arena_.err_flag(), 4, cudaMemcpyDeviceToHost, S(compute_)), "D2H err");

    const i64 bytes = 4 * n;
    const i64 slab = acquire_slab(bytes);
    pool_->mark_in_flight(slab, head, bytes);
    ck(cudaStreamWaitEvent(S(d2h_), E(ev_head_cert_), 0), "wait head certificate");
    ck(cudaMemcpyAsync(nf_host_ + slab, head_cert_dev_, 8, cudaMemcpyDeviceToHost, S(d2h_)), "D2H certificate");
    ck(cudaEventRecord(E(ev_slab_flag_[static_cast<size_t>(slab)]), S(d2h_)), "record slab flag");
    const i64 pieces = (V + head_vc_ - 1) / head_vc_;
    i64 first_gx = -1, last_lb = -1;
    float* g = grad_buf(gb);
    for (i64 k = 0; k < pieces; ++k) {
        const i64 v0 = k * head_vc_, vc = std::min(head_vc_, V - v0);
        StreamOp lb;
        lb.stream = StreamId::Compute;
        lb.kind = OpKind::LocalBackward;
        lb.layer = head;
        lb.buf = buf;
        lb.flops = bwd_flops(n, T) * vc / V;
        lb.deps.push_back(w_op);
        const i64 lbid = op_begin(lb, compute_);
        ck_hlm(hlm_cuda_head_grad_chunk(T, h, V, W, arena_.targets(), inv, v0, vc, arena_.g_roll(g_cur_), k > 0, g, 0,
                                        arena_.head_ws(), compute_),
               "head_grad_chunk");
        op_end(lbid, compute_);
        ck(cudaEventRecord(E(ev_head_chunk_[static_cast<size_t>(k)]), S(compute_)), "record head chunk");
        StreamOp gx;
        gx.stream = StreamId::D2H;
        gx.kind = OpKind::GradXfer;
        gx.layer = head;
        gx.slab = slab;
        gx.bytes = 4 * vc * h;
        gx.deps.push_back(lbid);
        if (k == 0 && last_accum_op_[static_cast<size_t>(slab)] >= 0)
            gx.deps.push_back(last_accum_op_[static_cast<size_t>(slab)]);
        ck(cudaStreamWaitEvent(S(d2h_), E(ev_head_chunk_[static_cast<size_t>(k)]), 0), "wait head chunk");
        const i64 gxid = op_begin(std::move(gx), d2h_);
        ck(cudaMemcpyAsync(pool_->data(slab) + v0 * h, g + v0 * h, static_cast<size_t>(vc * h) * 4,
                           cudaMemcpyDeviceToHost, S(d2h_)),
           "D2H head piece");
        op_end(gxid, d2h_);
        ck(cudaEventRecord(E(ev_piece_[static_cast<size_t>(slab * max_pieces_ + k)]), S(d2h_)), "record piece");
        if (k == 0) first_gx = gxid;
        last_lb = lbid;
        gbuf_free_op_[static_cast<size_t>(gb)] = gxid;
    }
    compute_done_with(buf, last_lb);
    // the certificate's fallback: the full scan of the head gradient
    ck_hlm(hlm_cuda_nonfinite_if_uncertified(g, n, nf2_dev_ + slab, head_cert_dev_, d2h_), "nonfinite scan (head)");
    ck(cudaMemcpyAsync(nf2_host_ + slab, nf2_dev_ + slab, 8, cudaMemcpyDeviceToHost, S(d2h_)), "D2H nf2 flag");
    ck(cudaEventRecord(E(ev_slab_done_[static_cast<size_t>(slab)]), S(d2h_)), "record slab done");
    ck(cudaEventRecord(E(ev_gradbuf_free_[gb]), S(d2h_)), "record grad buf free");
    {
        std::lock_guard<std::mutex> lk(mu_);
        pending_.push_back({slab, head, first_gx, step_index_, step_t_, n, pieces, head_vc_ * h});
    }
    cv_.notify_all();
}

// reference engine.cpp:279-368 (K-block recompute onto the LIFO stack, then
// reverse backward with immediate evacuation). With K == 1 and
// fused_recompute, recompute and backward of a layer share one weight H2D.
void Engine::backward_blockwise() {
    if (phase_ != Phase::Backward) throw ProtocolError("backward_blockwise out of order");
    const ModelConfig& m = store_.config();
    const i64 T = m.rows(), K = m.k_ckpt, h = m.hidden;
    const HlmBlockDims dims = block_dims(m, opts_.block_flags);
    const float* rc = m.rope_theta > 0 ? arena_.rope_cos() : nullptr;
    const float* rs = m.rope_theta > 0 ? arena_.rope_sin() : nullptr;
    const i64 n_block = m.block_params();
    const bool fused = opts_.fused_recompute && K == 1;
    const size_t act_bytes = static_cast<size_t>(block_act_bytes(m));
    (void)act_bytes;

    for (i64 b = m.layers / K; b >= 0; --b) {
        const i64 lo = b * K + 1, hi = std::min((b + 1) * K, m.layers);
        if (lo > hi) continue;
        const float* anchor = arena_.load_checkpoint(b * K);
        std::vector<const float*> inputs(static_cast<size_t>(hi - lo + 1));
        std::vector<void*> acts(static_cast<size_t>(hi - lo + 1));
        if (fused) {
            i64 w_op = -1;
            const bool res = is_resident(lo);
            const int buf = res ? -2 : stream_tile(lo, &w_op);
            if (!res) compute_wait_weights(buf);
            const void* wptr = res ? static_cast<const void*>(residents_[static_cast<size_t>(resident_of_[static_cast<size_t>(lo)])].w16)
                                   : weights_ptr(buf);
            void* saved = saved_acts_[static_cast<size_t>(lo)];
            void* a = saved ? saved : arena_.push_acts();
            StreamOp rop;
            rop.stream = StreamId::Compute;
            rop.kind = OpKind::Recompute;
            rop.layer = lo;
            rop.buf = buf;   // -2: HBM-resident weights
            rop.flops = saved ? 0 : fwd_flops(n_block, T);   // saved: the forward's activations, no kernel
            if (w_op >= 0) rop.deps.push_back(w_op);
            i64 id = op_begin(rop, compute_);
            if (!saved) {
                ck_hlm(hlm_cuda_block_fwd(&dims, wptr, anchor, arena_.h_roll(0), a, arena_.block_ws(), rc, rs,
                                          compute_),
                       "block_fwd (recompute)");
                ++recompute_forwards_;
            }
            op_end(id, compute_);
            const int gb = next_grad_buf();
            StreamOp bop;
            bop.stream = StreamId::Compute;
            bop.kind = OpKind::LocalBackward;
            bop.layer = lo;
            bop.buf = buf;
            bop.flops = bwd_flops(n_block, T);
            if (w_op >= 0) bop.deps.push_back(w_op);
            const i64 lb = op_begin(bop, compute_);
            ck_hlm(hlm_cuda_block_bwd(&dims, wptr, anchor, a, arena_.g_roll(g_cur_), arena_.g_roll(g_cur_ ^ 1),
                                      grad_buf(gb), arena_.block_ws(), rc, rs, compute_),
                   "block_bwd");
            op_end(lb, compute_);
            if (res) {
                resident_update(lo, gb, lb);
            } else {
                compute_done_with(buf, lb);
                evacuate(lo, gb, n_block, lb);
            }
            if (!saved) arena_.pop_acts();
            g_cur_ ^= 1;
        } else {
            // recompute lo..hi; each stack slab holds the layer's acts, inputs live
            // in the anchor / rolling buffers (copied into h_roll pairs per layer)
            const float* x = anchor;
            std::vector<float*> saved(static_cast<size_t>(hi - lo + 1), nullptr);
            for (i64 i = lo; i <= hi; ++i) {
                i64 w_op = 0;
                const int buf = stream_tile(i, &w_op);
                compute_wait_weights(buf);
                void* a = arena_.push_acts();
                acts[static_cast<size_t>(i - lo)] = a;
                inputs[static_cast<size_t>(i - lo)] = x;
                // the block output becomes the next layer's input; keep one fp32 copy
                // per layer inside the stack slab's tail (see footprint: stack slab
                // = acts + (rows,h) fp32 input when K > 1)
                float* out = reinterpret_cast<float*>(static_cast<char*>(a) + align256(block_act_bytes(m)));
                StreamOp rop;
                rop.stream = StreamId::Compute;
                rop.kind = OpKind::Recompute;
                rop.layer = i;
                rop.buf = buf;
                rop.flops = fwd_flops(n_block, T);
                rop.deps.push_back(w_op);
                const i64 id = op_begin(rop, compute_);
                ck_hlm(hlm_cuda_block_fwd(&dims, weights_ptr(buf), x, out, a, arena_.block_ws(), rc, rs, compute_),
                       "block_fwd (recompute)");
                op_end(id, compute_);
                compute_done_with(buf, id);
                ++recompute_forwards_;
                saved[static_cast<size_t>(i - lo)] = out;
                x = out;
            }
            for (i64 i = hi; i >= lo; --i) {
                i64 w_op = 0;
                const int buf = stream_tile(i, &w_op);
                compute_wait_weights(buf);
                const int gb = next_grad_buf();
                StreamOp bop;
                bop.stream = StreamId::Compute;
                bop.kind = OpKind::LocalBackward;
                bop.layer = i;
                bop.buf = buf;
                bop.flops = bwd_flops(n_block, T);
                bop.deps.push_back(w_op);
                const i64 lb = op_begin(bop, compute_);
                ck_hlm(hlm_cuda_block_bwd(&dims, weights_ptr(buf), inputs[static_cast<size_t>(i - lo)],
                                          acts[static_cast<size_t>(i - lo)], arena_.g_roll(g_cur_),
                                          arena_.g_roll(g_cur_ ^ 1), grad_buf(gb), arena_.block_ws(), rc, rs,
                                          compute_),
                       "block_bwd");
                op_end(lb, compute_);
                compute_done_with(buf, lb);
                evacuate(i, gb, n_block, lb);
                arena_.pop_acts();
                g_cur_ ^= 1;
            }
        }
        arena_.release_checkpoint(b * K);
    }
    (void)h;
    // embedding backward: deterministic scatter of g_0 by token id (kernels.hpp:396-408)
    const i64 n_embed = m.embed_params();
    int32_t* rp = loss_host_ + 3 * T + 16;
    int32_t* pos = rp + m.vocab + 1;
    // pos lives after row_ptr in the pinned staging (sized 4T + V + 1 + 64 ints)
    if (hlm_embed_csr(batch_.tokens.data(), T, m.vocab, rp, pos) != HLM_OK)
        throw std::out_of_range("embed_bwd: token id out of range");
    ck(cudaMemcpyAsync(arena_.csr_row_ptr(), rp, static_cast<size_t>(m.vocab + 1) * 4, cudaMemcpyHostToDevice,
                       S(compute_)),
       "H2D csr");
    ck(cudaMemcpyAsync(arena_.csr_pos(), pos, static_cast<size_t>(T) * 4, cudaMemcpyHostToDevice, S(compute_)),
       "H2D csr pos");
    const int gb = next_grad_buf();
    StreamOp eop;
    eop.stream = StreamId::Compute;
    eop.kind = OpKind::LocalBackward;
    eop.layer = m.embed_tile_id();
    eop.flops = bwd_flops(n_embed, T);
    if (sparse_embed_) {   // the batch's distinct tokens, ascending (CSR order)
        i64 n = 0;
        for (i64 v = 0; v < m.vocab; ++v) {
            const bool touched = rp[v + 1] > rp[v];
            embed_row_map_[static_cast<size_t>(v)] = touched ? static_cast<int32_t>(n) : -1;
            if (touched) embed_rows_host_[n++] = static_cast<int32_t>(v);
        }
        embed_rows_n_ = n;
        ck(cudaMemcpyAsync(embed_rows_dev_, embed_rows_host_, static_cast<size_t>(std::max<i64>(n, 1)) * 4,
                           cudaMemcpyHostToDevice, S(compute_)),
           "H2D embed rows");
    }
    const i64 lb = op_begin(eop, compute_);
    if (sparse_embed_)
        ck_hlm(hlm_cuda_embed_bwd_compact(arena_.csr_row_ptr(), arena_.csr_pos(), embed_rows_dev_, embed_rows_n_,
                                          arena_.g_roll(g_cur_), grad_buf(gb), m.hidden, compute_),
               "embed_bwd_compact");
    else
        ck_hlm(hlm_cuda_embed_bwd(arena_.csr_row_ptr(), arena_.csr_pos(), arena_.g_roll(g_cur_), grad_buf(gb),
                                  m.vocab, m.hidden, 0, compute_),
               "embed_bwd");
    op_end(lb, compute_);
    if (is_resident(m.embed_tile_id()))
        resident_update(m.embed_tile_id(), gb, lb);
    else if (sparse_embed_)
        evacuate(m.embed_tile_id(), gb, std::max<i64>(embed_rows_n_, 1) * m.hidden, lb, true);
    else
        evacuate(m.embed_tile_id(), gb, n_embed, lb);
    phase_ = Phase::Optimize;
}

// reference engine.cpp:379-424
StepResult Engine::finish_step() {
    if (phase_ != Phase::Optimize) throw ProtocolError("finish_step out of order");
    const ModelConfig& m = store_.config();
    const i64 T = m.rows();
    if (resident_dirty_) {   // the step's GPU span includes the device Adam
        ck(cudaEventRecord(E(ev_res_grad_), S(opt_)), "record optimizer stream done");
        ck(cudaStreamWaitEvent(S(compute_), E(ev_res_grad_), 0), "wait optimizer stream");
    }
    ck(cudaEventRecord(E(ev_step_end_), S(compute_)), "record step end");
    drain();
    ck(cudaStreamSynchronize(S(compute_)), "sync compute");
    ck(cudaStreamSynchronize(S(d2h_)), "sync d2h");
    ck(cudaStreamSynchronize(S(h2d_)), "sync h2d");
    ck(cudaStreamSynchronize(S(opt_)), "sync optimizer stream");
    if (!residents_.empty()) {
        ck(cudaMemcpy(resident_bad_host_, resident_bad_, residents_.size() * 8, cudaMemcpyDeviceToHost),
           "D2H resident flags");
        for (size_t i = 0; i < residents_.size(); ++i)
            if (resident_bad_host_[i] != ~0ull)
                throw NumericsError("non-finite gradient in layer " + std::to_string(residents_[i].tile) +
                                    " at element " + std::to_string(resident_bad_host_[i]) + "; step aborted");
    }
    const int err = loss_host_[3 * T];
    if (err & 1) throw std::out_of_range("embed_fwd: token id out of range (device)");
    if (err & 2) throw std::out_of_range("ce_loss_and_grad: target id out of range (device)");
    double loss = 0.0;
    const float* lr = reinterpret_cast<const float*>(loss_host_ + 2 * T);
    for (i64 r = 0; r < T; ++r) loss += static_cast<double>(lr[r]);
    if (opts_.comm_grad) {   // sum of every rank's (1/global_rows)-scaled partial loss
        // on the communicator's own stream, behind this step's reduce-scatters: one stream
        // per communicator keeps the collectives in the same order on every rank
        ck(cudaMemcpyAsync(loss_dev_, &loss, sizeof(double), cudaMemcpyHostToDevice, S(comm_)), "H2D loss");
        nccl_check(nccl().AllReduce(loss_dev_, loss_dev_, 1, ncclFloat64, ncclSum,
                                    static_cast<ncclComm_t>(opts_.comm_grad), S(comm_)),
                   "all-reduce loss");
        ck(cudaMemcpyAsync(&loss, loss_dev_, sizeof(double), cudaMemcpyDeviceToHost, S(comm_)), "D2H loss");
        ck(cudaStreamSynchronize(S(comm_)), "sync loss");
    }

    // host ops into the trace, in consumption order
    std::vector<i64> accum_ids;
    std::vector<HostOpRecord> recs;
    {   // records completing after this point land in the next step's trace
        std::lock_guard<std::mutex> lk(mu_);
        recs.swap(host_ops_);
    }
    for (const auto& rec : recs) {
        StreamOp op;
        op.stream = StreamId::Host;
        op.kind = OpKind::Accum;
        op.layer = rec.layer;
        op.slab = rec.slab;
        op.params = store_.tile(rec.layer).n_params();
        if (rec.step == step_index_) op.deps.push_back(rec.grad_op);   // earlier step: op ids of another trace
        op.t_start_us = rec.t0 - host_t0_us_;
        op.t_end_us = rec.t1 - host_t0_us_;
        const i64 id = trace_.add(op);
        last_accum_op_[static_cast<size_t>(rec.slab)] = id;
        accum_ids.push_back(id);
        if (rec.opt) {
            StreamOp o;
            o.stream = StreamId::Host;
            o.kind = OpKind::OptStep;
            o.layer = rec.layer;
            o.params = store_.tile(rec.layer).n_params();
            o.deps.push_back(id);
            o.t_start_us = rec.topt0 - host_t0_us_;
            o.t_end_us = rec.topt1 - host_t0_us_;
            trace_.add(o);
        }
    }
    if (!opts_.eager_optim && !opts_.skip_optimizer && opts_.comm_grad) {
        const double t0 = now_us();
        for (i64 p = 0; p < store_.physical_tiles(); ++p) {   // validate every shard first
            LayerTile& tile = store_.physical(p);
            const i64 cnt = shard_elems(tile.n_params());
            if (!all_finite(tile.grads() + opts_.rank * cnt, cnt))
                throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + "; step aborted");
        }
        for (i64 p = 0; p < store_.physical_tiles(); ++p) {
            LayerTile& tile = store_.physical(p);
            const i64 cnt = shard_elems(tile.n_params()), begin = opts_.rank * cnt;
            adam_step_range(tile, tile.grads() + begin, begin, cnt, hyper_, step_t_);
            std::fill(tile.grads() + begin, tile.grads() + begin + cnt, 0.0f);
            tile.bump_version(opts_.rank);
        }
        StreamOp op;
        op.stream = StreamId::Host;
        op.kind = OpKind::OptStep;
        op.params = store_.total_params() / opts_.world;
        op.deps = accum_ids;
        op.t_start_us = t0 - host_t0_us_;
        op.t_end_us = now_us() - host_t0_us_;
        trace_.add(op);
    } else if (!opts_.eager_optim && !opts_.skip_optimizer) {
        const double t0 = now_us();
        adam_step(store_, hyper_, step_t_);
        StreamOp op;
        op.stream = StreamId::Host;
        op.kind = OpKind::OptStep;
        op.params = store_.total_params();
        op.deps = accum_ids;
        op.t_start_us = t0 - host_t0_us_;
        op.t_end_us = now_us() - host_t0_us_;
        trace_.add(op);
    }
    if (!opts_.skip_optimizer) store_.set_adam_steps(step_t_);
    if (opts_.overlap_optimizer_tail)
        for (auto& tv : target_version_) ++tv;

    // resolve GPU timestamps
    float ms = 0.f;
    for (const auto& oe : op_events_) {
        StreamOp& op = trace_.ops[static_cast<size_t>(oe.first)];
        float a = 0.f, b = 0.f;
        if (cudaEventElapsedTime(&a, E(ev_step_start_), E(timing_events_[static_cast<size_t>(oe.second)])) ==
                cudaSuccess &&
            cudaEventElapsedTime(&b, E(ev_step_start_), E(timing_events_[static_cast<size_t>(oe.second + 1)])) ==
                cudaSuccess) {
            op.t_start_us = 1e3 * a;
            op.t_end_us = 1e3 * b;
        }
    }
    for (auto& op : trace_.ops)
        if (op.t_start_us == -2.0) {   // fused head fwd/bwd: same launch as the preceding Forward
            for (const auto& o2 : trace_.ops)
                if (o2.layer == op.layer && o2.kind == OpKind::Forward) {
                    op.t_start_us = o2.t_start_us;
                    op.t_end_us = o2.t_end_us;
                }
        }
    cudaEventElapsedTime(&ms, E(ev_step_start_), E(ev_step_end_));

    for (int b = 0; b < 2; ++b)
        if (arena_.buffer_occupant(b) != -1) arena_.release_buffer(b);
    arena_.release_cache_slots();
    arena_.release_workspace();

    StepResult r;
    r.loss = loss;
    r.trace = std::move(trace_);
    r.arena = arena_.snapshot();
    r.host.persistent = store_.persistent_bytes();
    r.host.slabs = pool_->pool_bytes();
    r.host.total = r.host.persistent + r.host.slabs;
    r.h2d_bytes = arena_.h2d_bytes();
    r.d2h_bytes = pool_->d2h_bytes() - d2h_base_;
    r.recompute_forwards = recompute_forwards_;
    r.gpu_ms = ms;
    phase_ = Phase::Idle;
    return r;
}

StepResult Engine::train_step(const Batch& batch) {
    try {
        begin_step(batch);
        forward_streaming();
        anchor_loss_async();
        backward_blockwise();
        return finish_step();
    } catch (...) {
        // leave the engine reusable: wait for in-flight work, reset protocol state
        cudaStreamSynchronize(S(compute_));
        cudaStreamSynchronize(S(h2d_));
        cudaStreamSynchronize(S(d2h_));
        cudaStreamSynchronize(S(opt_));
        try {
            drain();
        } catch (...) {
        }
        for (int b = 0; b < 2; ++b)
            if (arena_.buffer_occupant(b) != -1) arena_.release_buffer(b);
        arena_.release_cache_slots();
        std::fill(cache_xfer_op_.begin(), cache_xfer_op_.end(), -1);
        head_buf_ = -1;
        while (arena_.stack_depth() > 0) arena_.pop_acts();
        for (i64 i = 0; i <= store_.config().layers; i += store_.config().k_ckpt) {
            try {
                arena_.release_checkpoint(i);
            } catch (...) {
            }
        }
        try {
            arena_.release_workspace();
        } catch (...) {
        }
        phase_ = Phase::Idle;
        throw;
    }
}

std::vector<float> Engine::debug_hidden() {
    const ModelConfig& m = store_.config();
    std::vector<float> out(static_cast<size_t>(m.rows() * m.hidden));
    ck(cudaStreamSynchronize(S(compute_)), "sync");
    ck(cudaMemcpy(out.data(), h_cur_, out.size() * 4, cudaMemcpyDeviceToHost), "D2H hidden");
    return out;
}

// reference engine.cpp:434-441
Batch make_copy_task_batch(const ModelConfig& m, Rng& rng) {
    Batch b;
    const i64 n = m.rows();
    b.tokens.resize(static_cast<size_t>(n));
    for (auto& t : b.tokens) t = rng.uniform_int(static_cast<std::int32_t>(m.vocab));
    b.targets = b.tokens;
    return b;
}

}  // inline namespace b200
}  // namespace hlm
