// The B200 training engine: CPU-master / GPU-template layer streaming
// (reference proj/include/hlm/engine.hpp:21-119, same public surface).
//
// Three CUDA streams — H2D weights, compute, D2H gradients — ordered only by
// events (PAPER.md:326-342 protocol):
//   weights-ready  : H2D of tile i into buffer b  ->  compute reading b
//   buffer-free    : last compute reading b       ->  next H2D into b
//   grad-ready     : backward of tile i           ->  D2H of its fp32 gradient
//   grad-buf-free  : D2H of a gradient buffer     ->  next backward writing it
// so layer i+1's weights stream in while layer i computes, and layer i's
// gradient drains while layer i-1 computes. A host worker thread consumes
// gradient slabs as their D2H completes and runs the fused host Adam per
// tile (eager optimizer), overlapping the GPU backward.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "hlm/device_arena.hpp"
#include "hlm/host_store.hpp"
#include "hlm/trace.hpp"

namespace hlm {
inline namespace b200 {

struct Batch {
    std::vector<std::int32_t> tokens;    // batch * seq
    std::vector<std::int32_t> targets;   // batch * seq
};

struct EngineOptions {
    bool eager_optim = false;      // per-tile Adam as gradients land
    i64 n_slab = 12;
    bool threaded_accum = false;   // consume slabs on a host worker thread
    i64 accum_delay_us = 0;        // test hook, forces slab back-pressure
    bool skip_optimizer = false;   // verification runs: leave gradients in the store
    // B200 additions
    bool fused_recompute = true;   // K == 1: recompute + backward share one weight H2D
    bool record_trace = true;      // CUDA-event timestamps per op
    int block_flags = 0;           // HLM_BLOCK_* (e.g. force the generic attention)
    // Cross-step overlap (eager + threaded only): the head and the top `tail_blocks`
    // blocks are optimised after the embedding (the order the next forward needs
    // them), train_step returns once every other tile is updated, and the next
    // step's H2D of each tile waits for that tile's update. Numerics unchanged.
    bool overlap_optimizer_tail = false;
    i64 tail_blocks = 2;
    // Data parallel (one process per GPU over a shared host store): this rank
    // trains on its rows of the global micro-batch (loss scaled by
    // 1/global_rows); every layer gradient is reduce-scattered (comm_grad, D2H
    // stream) and only this rank's 1/world shard is copied to the host and
    // optimised here. With comm_weights, each rank H2Ds 1/world of a layer and
    // the full layer is all-gathered over NVLink (h2d stream).
    int rank = 0;
    int world = 1;
    void* comm_grad = nullptr;      // ncclComm_t
    void* comm_weights = nullptr;   // ncclComm_t, optional
    // OpenMP threads of the host optimizer worker (0 = OpenMP default). Ranks sharing
    // a host split its cores; initialisation elsewhere keeps every core.
    int host_threads = 0;
    // HBM-resident optimizer tiles (eager, K == 1, single process, untied): the
    // embedding (resident_embed) and blocks 1..resident_blocks keep FP32 master, m, v
    // and their BF16 weights in device memory for the engine's lifetime. Their
    // weights are never streamed and their gradients never leave the GPU (finiteness
    // scan + device Adam, bit-identical to the host Adam, right after the backward).
    // These are the tiles the next forward needs first and the host Adam would
    // finish last. sync() (and the destructor) copies them back into the store.
    i64 resident_blocks = 0;
    // Vocab-chunked head: the head weight gradient is computed, copied and optimised
    // in pieces of head_piece_vocab vocab rows (0 = auto, ~kPieceElems elements per
    // piece when the head spans two or more; -1 = off). Eager untied single-GPU only.
    i64 head_piece_vocab = 0;
    // Elements per D2H / optimizer / forward-H2D piece (0 = 64 Mi = 256 MB of fp32).
    i64 piece_elems = 0;
    // Outbound fp32 gradient buffers on the device (>= 2; the arena holds two, the engine
    // allocates the rest, each the widest tile).
    i64 grad_buffers = 2;
    // Row-sparse embedding gradient: only the rows of the batch's tokens are computed,
    // copied and read by the host Adam (the other rows' gradient is exactly zero; their
    // Adam update runs without reading one). Single GPU, untied, eager optimizer.
    bool sparse_embed_grad = false;
    // Forward embedding lookup reads the batch's rows straight from the pinned host BF16
    // shadow (zero-copy over PCIe: T x h x 2 bytes) instead of streaming the (V, h) table.
    // Single GPU, untied, host-resident embedding.
    bool embed_gather_host = false;
    // Pin the host optimizer's OpenMP team to cores (scheduling only).
    bool pin_threads = true;
    bool resident_embed = false;
    // Blocks L - saved_act_layers + 1 .. L (K == 1, fused recompute) keep the activations
    // their forward computed in HBM until their backward, which then skips the recompute
    // (the same kernels on the same inputs and weights would reproduce them bit for bit).
    // Trades HBM (one block's activations each) for GPU time where the GPU is the bound.
    i64 saved_act_layers = 0;
};

struct StepResult {
    double loss = 0.0;
    EventTrace trace;
    ArenaSnapshot arena;
    HostBytesReport host;
    i64 h2d_bytes = 0;
    i64 d2h_bytes = 0;
    i64 recompute_forwards = 0;
    double gpu_ms = 0.0;           // step-start to last GPU op, CUDA events
};

enum class Phase { Idle, Forward, Anchor, Backward, Optimize };

class Engine {
public:
    Engine(MasterStore& store, DeviceArena& arena, const HyperParams& hyper, EngineOptions opts = {});
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    StepResult train_step(const Batch& batch);
    // Waits until every pending host optimizer update has been applied and copies
    // HBM-resident optimizer tiles back into the store: the store is consistent.
    void sync();
    // Waits for the host optimizer only (no resident write-back): the end of a
    // training step's work when timing.
    void wait_optimizer();

    void begin_step(const Batch& batch);
    void forward_streaming();
    double anchor_loss();          // synchronises to return the loss (phase API, tests)
    void backward_blockwise();
    StepResult finish_step();

    Phase phase() const { return phase_; }
    // Rolling hidden state on the device; after forward_streaming it is h_L.
    const float* debug_hidden_device() const { return h_cur_; }
    std::vector<float> debug_hidden();   // copies h_L to the host
    SlabPool& pool() { return *pool_; }
    MasterStore& store() { return store_; }
    DeviceArena& arena() { return arena_; }
    const HyperParams& hyper() const { return hyper_; }
    const EngineOptions& options() const { return opts_; }
    void* compute_stream() const { return compute_; }

private:
    struct Pending {
        i64 slab;
        i64 layer;
        i64 grad_op;
        i64 step = 0;   // engine step index (tail eligibility)
        i64 t = 0;      // Adam step index of the gradient (bias correction)
        i64 count = 0;  // fp32 elements copied into the slab (the tile, or this rank's shard)
        i64 pieces = 1; // D2H pieces, each with its own event (the optimizer starts on piece 0)
        i64 piece = 0;  // elements per piece
        bool sparse_rows = false;   // row-compact embedding gradient (embed_row_map_)
    };
    struct HostOpRecord {   // host-side Accum / OptStep, appended to the trace in finish_step
        i64 slab, layer, grad_op, step;   // step: the gradient's step (an earlier one for a tail tile)
        double t0, t1;
        bool opt;
        double topt0, topt1;
    };

    void anchor_loss_async();
    // Returns a weight "buffer" id: 0/1 = stream buffers, 2+s = weight-cache slot s.
    // forward_pass: a cacheable block streams into its cache slot; later passes
    // of the same step reuse the resident copy without any H2D.
    int stream_tile(i64 tile_id, i64* op_id, bool forward_pass = false);
    void* weights_ptr(int buf) const;
    void compute_wait_weights(int buf);
    void compute_done_with(int buf, i64 op_id);
    int next_grad_buf();
    void evacuate(i64 tile_id, int gbuf, i64 n_params, i64 lb_op, bool sparse_rows = false);
    void consume(const Pending& p);          // READY -> ACCUMULATING -> FREE (+ Adam)
    void process_oldest_inline();
    void worker_loop();
    void drain();
    bool eligible(const Pending& p) const;   // mu_ held
    // all_ranks: every rank's shard of the tile must be current (a full H2D or a zero-copy
    // read of the host shadow); otherwise only this rank's shard (sharded H2D + all-gather:
    // the other shards arrive over NVLink from ranks that waited on their own versions)
    void wait_tile_current(i64 tile_id, bool all_ranks);
    bool sharded_h2d(const LayerTile& tile) const {
        return opts_.comm_weights && tile.n_params() % opts_.world == 0;
    }
    i64 op_begin(StreamOp op, void* stream);
    void op_end(i64 id, void* stream);
    void rethrow_worker_error();

    MasterStore& store_;
    DeviceArena& arena_;
    HyperParams hyper_;
    EngineOptions opts_;
    std::unique_ptr<SlabPool> pool_;

    void* h2d_ = nullptr;
    void* compute_ = nullptr;
    void* d2h_ = nullptr;
    void* comm_ = nullptr;           // data parallel: per-layer gradient reduce-scatter
    std::vector<void*> ev_rs_done_;  // per gradient buffer: reduce-scatter finished (comm_ -> d2h_)
    void* opt_ = nullptr;            // device Adam of HBM-resident tiles, beside the backward
    void* ev_res_grad_ = nullptr;    // a resident tile's gradient is complete (compute -> opt_)
    void* ev_w_ready_[2] = {};
    void* ev_buf_free_[2] = {};
    // outbound fp32 gradient buffers: the arena's two (reference footprint) plus
    // EngineOptions.grad_buffers - 2 engine-owned ones, so the backward runs ahead of a
    // slow D2H instead of waiting for the buffer two layers back
    std::vector<float*> gbuf_;
    void* gbuf_mem_ = nullptr;
    std::vector<void*> ev_grad_ready_;
    std::vector<void*> ev_gradbuf_free_;
    // trace: the op after which each gradient buffer is free (its D2H, or the device Adam of
    // a resident tile), attached as a dependency of the next backward writing that buffer
    std::vector<i64> gbuf_free_op_;
    i64 gbuf_dep_ = -1;
    float* grad_buf(int i) const { return gbuf_[static_cast<size_t>(i)]; }
    std::vector<void*> ev_slab_done_;
    // Large gradients land in pieces of kPieceElems: per slab, an event after the
    // finiteness flag and one per piece, so the host Adam starts on the first piece
    // instead of waiting for the whole tile (the head gradient is 2.2 GB at C2).
    static constexpr i64 kPieceElems = i64(64) << 20;
    // the host Adam publishes progress (and a forward H2D copies) in 16 Mi-element steps
    static constexpr i64 kPublishElems = i64(16) << 20;
    i64 piece_elems_ = kPieceElems;     // EngineOptions::piece_elems (tests use small pieces)
    i64 max_pieces_ = 1;
    std::vector<void*> ev_slab_flag_;    // per slab
    std::vector<void*> ev_piece_;        // per slab x max_pieces_
    // The head tile is prefetched into a stream buffer during the forward, before
    // block head_prefetch_at_ is issued: the first block from which every block is
    // cached or HBM-resident (never touches a stream buffer). The optimizer worker
    // orders the previous step's head right before that block, so the last tile the
    // forward waits for is block L, not the 2 GB head.
    bool head_prefetch_ = false;
    i64 head_prefetch_at_ = 0;
    int head_buf_ = -1;
    i64 head_wop_ = -1;
    i64 tail_key(i64 layer) const;      // forward-need order of a tile (optimizer priority)
    // Per physical tile: leading elements whose running Adam update is done (mu_).
    // A forward H2D into a cache slot copies piece by piece behind the optimizer.
    std::vector<i64> progress_;
    bool wait_elems_current(i64 tile_id, i64 end);   // false: whole tile current
    // vocab-chunked head: vocab rows per piece (0 = off), certificate word, per-piece
    // compute events, full-scan fallback flag per slab (device + pinned mirror)
    i64 head_vc_ = 0;
    unsigned long long* head_cert_dev_ = nullptr;
    void* ev_head_cert_ = nullptr;
    std::vector<void*> ev_head_chunk_;
    unsigned long long* nf2_dev_ = nullptr;
    unsigned long long* nf2_host_ = nullptr;
    i64 acquire_slab(i64 bytes);        // back-pressure: blocks (worker) or consumes inline
    // row-sparse embedding gradient state of the running step
    bool sparse_embed_ = false;
    int32_t* embed_rows_host_ = nullptr;   // pinned: touched rows, ascending
    int32_t* embed_rows_dev_ = nullptr;
    std::vector<int32_t> embed_row_map_;   // row -> compact index or -1
    i64 embed_rows_n_ = 0;
    const void* embed_host_dev_ = nullptr;   // device alias of the embedding's pinned shadow (zero-copy)
    void anchor_loss_pieces(int buf, i64 w_op);
    void* ev_step_start_ = nullptr;
    void* ev_step_end_ = nullptr;
    std::vector<void*> timing_events_;   // pairs per traced GPU op
    std::vector<std::pair<i64, int>> op_events_;   // op id -> first timing event index
    size_t timing_used_ = 0;
    int32_t* loss_host_ = nullptr;       // pinned: loss rows (float bits) + error flag

    Phase phase_ = Phase::Idle;
    Batch batch_;
    EventTrace trace_;
    double host_t0_us_ = 0.0;
    int next_buf_ = 0;
    int next_gbuf_ = 0;
    i64 last_reader_[2] = {-1, -1};
    std::vector<i64> last_accum_op_;
    const float* h_cur_ = nullptr;
    int g_cur_ = 0;
    i64 step_t_ = 0;
    i64 d2h_base_ = 0;
    i64 recompute_forwards_ = 0;
    std::vector<i64> consumers_left_;
    std::vector<HostOpRecord> host_ops_;   // guarded by mu_
    std::vector<i64> cache_slot_of_;       // per logical tile, -1 when not cached
    std::vector<i64> cache_xfer_op_;       // per slot: this step's WeightXfer op, -1 if not resident
    std::vector<void*> ev_cache_ready_;
    struct Resident {
        i64 tile;          // logical tile id
        i64 n;
        float* state;      // device [master | m | v]
        uint16_t* w16;     // device bf16 weights
    };
    std::vector<i64> resident_of_;         // per logical tile: index into residents_ or -1
    std::vector<Resident> residents_;
    void* resident_mem_ = nullptr;
    unsigned long long* resident_bad_ = nullptr;   // device: per resident tile, first non-finite index
    unsigned long long* resident_bad_host_ = nullptr;
    bool resident_dirty_ = false;
    bool is_resident(i64 tile) const { return resident_of_[static_cast<size_t>(tile)] >= 0; }
    void resident_update(i64 tile, int gbuf, i64 dep_op);   // device finiteness scan + Adam
    void sync_resident();
    void upload_resident();
    i64 resident_epoch_ = 0;
    std::vector<void*> saved_acts_;        // per logical tile: HBM activations kept from the forward
    void* saved_mem_ = nullptr;
    i64 shard_elems(i64 n) const;          // n / world (throws unless divisible)
    void h2d_tile(void* dst, const LayerTile& tile, i64 bytes);
    double* loss_dev_ = nullptr;
    unsigned long long* nf_dev_ = nullptr;    // per slab: first non-finite index (device)
    unsigned long long* nf_host_ = nullptr;   // pinned mirror
    std::vector<char> deferred_;           // per logical tile: optimised in the tail
    std::vector<i64> target_version_;      // per physical tile: version the next H2D needs
    bool tail_open_ = true;                // every regular tile of this step processed (mu_)
    i64 regular_left_ = 0;                 // host (non-deferred, non-resident) tiles still to consume (mu_)
    i64 step_index_ = 0;

    // worker
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Pending> pending_;
    i64 in_process_ = 0;
    bool stop_ = false;
    std::exception_ptr worker_error_;
    std::thread worker_;
};

// Deterministic synthetic data: random tokens echoed as their own targets
// (reference proj/src/engine.cpp:434-441).
Batch make_copy_task_batch(const ModelConfig& m, Rng& rng);

}  // inline namespace b200
}  // namespace hlm
