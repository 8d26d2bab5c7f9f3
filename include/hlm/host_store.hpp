// The authoritative host-side parameter store of the B200 engine.
//
// Re-design of reference proj/include/hlm/host_store.hpp:42-235 for a real
// GPU: per physical tile the store keeps
//   * FP32 master weights, FP32 Adam moments m and v — one huge-page backed,
//     first-touch-initialised host allocation (12 B/param), never transferred;
//   * a BF16 shadow of the master, packed per layer in ONE pinned allocation
//     (2 B/param) — the H2D source, so "pack_layer" is a zero-copy view;
//   * an FP32 gradient region (4 B/param), allocated only when gradients must
//     persist in the store (skip_optimizer, tied tables, lazy optimizer).
// Gradients return from the GPU in FP32 through a pool of pinned slabs
// (SlabPool); the fused Adam reads the slab directly, updates master/m/v and
// re-packs the shadow in one pass (reference adam_update_tile,
// host_store.cpp:334-362, bit-identical math, AVX-512 + all host cores).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hlm/errors.hpp"
#include "hlm/model_config.hpp"
#include "hlm/tensor.hpp"

namespace hlm {
inline namespace b200 {

struct NamedRegion {
    std::string name;
    i64 offset = 0;   // elements from the tile base
    std::vector<i64> shape;
    i64 numel() const {
        i64 n = 1;
        for (i64 d : shape) n *= d;
        return n;
    }
};

// Canonical packed orders (host_store.cpp:70-92).
std::vector<NamedRegion> block_offset_table(i64 h, i64 f);
std::vector<NamedRegion> table_offset_table(const std::string& name, i64 vocab, i64 h);

class MasterStore;

class LayerTile {
public:
    LayerTile(i64 layer_id, i64 n_params, std::vector<NamedRegion> offsets, float* state,
              std::uint16_t* shadow);

    i64 layer_id() const { return layer_id_; }
    i64 n_params() const { return n_params_; }
    const std::vector<NamedRegion>& offset_table() const { return offsets_; }
    const NamedRegion& region(const std::string& name) const;

    float* master() { return state_; }
    const float* master() const { return state_; }
    float* moment_m() { return state_ + n_params_; }
    const float* moment_m() const { return state_ + n_params_; }
    float* moment_v() { return state_ + 2 * n_params_; }
    const float* moment_v() const { return state_ + 2 * n_params_; }
    std::uint16_t* shadow() { return shadow_; }
    const std::uint16_t* shadow() const { return shadow_; }
    i64 weight_bytes() const { return 2 * n_params_; }   // streamed bytes (bf16 shadow)

    bool has_grads() const { return grads_ != nullptr; }
    float* grads();               // allocates (zeroed) on first use
    const float* grads_or_null() const { return grads_.get(); }
    void drop_grads() { grads_.reset(); }

    float load_weight(i64 i) const { return state_[i]; }
    void store_weight(i64 i, float v);   // master = v, shadow = RNE(v)
    float load_grad(i64 i) const { return grads_ ? grads_[i] : 0.0f; }
    void store_grad(i64 i, float v) { grads()[i] = v; }

    // Completed optimizer updates of this tile (cross-step H2D gating). In a
    // shared (multi-process) store every rank owns one counter per tile in the
    // shared mapping: bump_version(rank) after updating its shard, and a tile is
    // current for the next H2D when min_version() reached the target.
    std::atomic<i64> version{0};
    void attach_shared_versions(std::atomic<i64>* v, int world) {
        shared_versions_ = v;
        world_ = world;
    }
    void bump_version(int rank) {
        if (shared_versions_)
            shared_versions_[rank].fetch_add(1, std::memory_order_acq_rel);
        else
            version.fetch_add(1, std::memory_order_acq_rel);
    }
    // this rank's own counter (its shard's completed updates)
    i64 rank_version(int rank) const {
        if (!shared_versions_) return version.load(std::memory_order_acquire);
        return shared_versions_[rank].load(std::memory_order_acquire);
    }
    i64 min_version() const {
        if (!shared_versions_) return version.load(std::memory_order_acquire);
        i64 v = shared_versions_[0].load(std::memory_order_acquire);
        for (int r = 1; r < world_; ++r) {
            const i64 x = shared_versions_[r].load(std::memory_order_acquire);
            if (x < v) v = x;
        }
        return v;
    }

private:
    std::atomic<i64>* shared_versions_ = nullptr;
    int world_ = 1;
    i64 layer_id_;
    i64 n_params_;
    std::vector<NamedRegion> offsets_;
    float* state_;                // [master n][m n][v n]
    std::uint16_t* shadow_;       // pinned
    std::unique_ptr<float[]> grads_;
};

enum class InitMode : std::uint8_t {
    Reference = 0,   // one sequential mt19937 over all tiles: bit-identical to reference build_store
    Parallel = 1     // counter-seeded per 64Ki-element chunk: same distribution, any thread count
};

// Multi-process (one process per GPU) store: every rank maps the same POSIX
// shared-memory object (/dev/shm/<name>); rank 0 creates and initialises it,
// the others attach once it is marked ready. Each process pins the shared BF16
// shadow for its own DMA (cudaHostRegister).
struct SharedStoreSpec {
    std::string name;
    int rank = 0;
    int world = 1;
    // Per-run token every rank agrees on (e.g. derived from the NCCL unique id). Rank 0
    // writes it into the segment header; an attaching rank accepts only a segment that
    // carries it, so a stale segment of a crashed run under the same name is never used.
    // 0 = no token (the dims are still checked).
    std::uint64_t nonce = 0;
};

class MasterStore {
public:
    // Allocates host memory (master/moments: huge-page anonymous mapping;
    // shadow: pinned through the CUDA runtime, or plain memory when
    // pin_shadow is false, e.g. on CPU-only machines).
    MasterStore(const ModelConfig& config, Dtype dtype, bool pin_shadow = true,
                const SharedStoreSpec* shared = nullptr);
    ~MasterStore();
    MasterStore(const MasterStore&) = delete;
    MasterStore& operator=(const MasterStore&) = delete;

    const ModelConfig& config() const { return config_; }
    Dtype dtype() const { return dtype_; }
    i64 logical_tiles() const { return config_.tile_count(); }
    i64 physical_tiles() const { return static_cast<i64>(tiles_.size()); }
    LayerTile& tile(i64 logical_id) { return *tiles_[static_cast<size_t>(physical_of_[static_cast<size_t>(logical_id)])]; }
    const LayerTile& tile(i64 logical_id) const {
        return *tiles_[static_cast<size_t>(physical_of_[static_cast<size_t>(logical_id)])];
    }
    LayerTile& physical(i64 idx) { return *tiles_[static_cast<size_t>(idx)]; }
    const LayerTile& physical(i64 idx) const { return *tiles_[static_cast<size_t>(idx)]; }
    i64 physical_index(i64 logical_id) const { return physical_of_[static_cast<size_t>(logical_id)]; }
    bool is_aliased(i64 logical_id) const {
        return config_.tie_embeddings && logical_id == config_.head_tile_id();
    }
    i64 consumer_count(i64 physical_idx) const;

    i64 total_params() const { return total_params_; }
    i64 persistent_bytes() const;   // master + m + v + shadow (+ grad regions present)
    bool shadow_pinned() const { return pinned_; }

    i64 adam_steps() const { return adam_steps_; }
    void set_adam_steps(i64 t) { adam_steps_ = t; }
    // Engines holding HBM-resident tiles whose optimizer state is newer than this
    // store's (between a resident Adam and Engine::sync()). save_checkpoint refuses
    // while the count is non-zero: the file would silently hold stale tiles.
    void add_device_newer(int d) { device_newer_.fetch_add(d); }
    int device_newer() const { return device_newer_.load(); }
    // An attached Engine registers a hook that brings the store up to date: it waits for
    // the optimizer tail it may still be running on a worker thread (train_step returns
    // before the head / top blocks of an overlapped tail are optimised) and copies
    // HBM-resident tiles back. save_checkpoint / load_checkpoint / export / import call
    // quiesce() first, so a file never mixes tiles from two steps and a load is never
    // overwritten by a late tail update.
    // strict: mid-step calls are a ProtocolError (save / load / import); a non-strict read
    // (export) during a step just sees the store as it is.
    void set_quiesce(std::function<void(bool strict)> hook, const void* owner) {
        std::lock_guard<std::mutex> lk(quiesce_mu_);
        quiesce_ = std::move(hook);
        quiesce_owner_ = owner;
    }
    void clear_quiesce(const void* owner) {
        std::lock_guard<std::mutex> lk(quiesce_mu_);
        if (quiesce_owner_ == owner) {
            quiesce_ = nullptr;
            quiesce_owner_ = nullptr;
        }
    }
    void quiesce(bool strict = true) const {
        std::function<void(bool)> f;
        {
            std::lock_guard<std::mutex> lk(quiesce_mu_);
            f = quiesce_;
        }
        if (f) f(strict);
    }
    // Bumped whenever the store's state is replaced from outside (load_checkpoint,
    // import_master): an engine holding HBM-resident tiles re-uploads them.
    i64 epoch() const { return epoch_.load(); }
    void bump_epoch() { epoch_.fetch_add(1); }

    bool bitwise_equal(const MasterStore& other) const;   // master, moments, shadow

    // Re-packs the BF16 shadow of every tile from the master (after external edits).
    void repack_shadow();

    bool shared() const { return shm_fd_ >= 0; }
    int rank() const { return rank_; }
    int world() const { return world_; }
    bool owner() const { return rank_ == 0; }
    void mark_ready();            // rank 0, after initialisation
    void wait_ready() const;      // other ranks

private:
    void attach_shared(std::uint64_t nonce);
    ModelConfig config_;
    Dtype dtype_;
    std::vector<std::unique_ptr<LayerTile>> tiles_;
    std::vector<i64> physical_of_;
    i64 total_params_ = 0;
    i64 adam_steps_ = 0;
    float* state_base_ = nullptr;
    size_t state_bytes_ = 0;
    std::uint16_t* shadow_base_ = nullptr;
    size_t shadow_bytes_ = 0;
    bool pinned_ = false;
    // shared mapping: [header 2 MiB][state][shadow][versions]
    int shm_fd_ = -1;
    std::string shm_name_;
    void* map_base_ = nullptr;
    size_t map_bytes_ = 0;
    int rank_ = 0, world_ = 1;
    bool registered_ = false;
    std::atomic<int> device_newer_{0};
    std::atomic<i64> epoch_{0};
    mutable std::mutex quiesce_mu_;
    std::function<void(bool)> quiesce_;
    const void* quiesce_owner_ = nullptr;
};

// Allocates and initialises a store: trunc_normal(0.02) matrices, unit norm
// scales, zero moments (reference host_store.cpp:141-156).
std::unique_ptr<MasterStore> build_store(const ModelConfig& config, std::uint64_t seed,
                                         Dtype dtype = Dtype::BF16, InitMode mode = InitMode::Reference,
                                         bool pin_shadow = true, const SharedStoreSpec* shared = nullptr);

// ------------------------------------------------------------------ gradient slabs
enum class SlabState : std::uint8_t { FREE = 0, IN_FLIGHT = 1, READY = 2, ACCUMULATING = 3 };
const char* slab_state_name(SlabState s);

// Fixed pool of pinned FP32 gradient slabs with the reference state machine
// FREE -> IN_FLIGHT -> READY -> ACCUMULATING -> FREE (host_store.hpp:162-235).
// IN_FLIGHT = D2H enqueued; READY = copy complete; consumed in READY order.
class SlabPool {
public:
    SlabPool(i64 n_slabs, i64 slab_capacity_bytes, bool pinned = true);
    // Mixed capacities: acquire(bytes) takes the smallest FREE slab that fits
    // (two widest-tile slabs for the embedding/head, the rest block-sized).
    explicit SlabPool(const std::vector<i64>& capacities, bool pinned = true);
    ~SlabPool();
    SlabPool(const SlabPool&) = delete;
    SlabPool& operator=(const SlabPool&) = delete;

    i64 size() const { return static_cast<i64>(slabs_.size()); }
    i64 slab_capacity() const { return capacity_; }   // the largest slab
    i64 capacity_of(i64 id) const { return slabs_[static_cast<size_t>(id)].capacity; }
    i64 pool_bytes() const { return pool_bytes_; }
    SlabState state(i64 id) const;
    float* data(i64 id) { return slabs_[static_cast<size_t>(id)].data; }
    i64 layer_of(i64 id) const { return slabs_[static_cast<size_t>(id)].layer_id; }
    i64 d2h_bytes() const { return d2h_bytes_; }
    i64 max_in_use() const { return max_in_use_; }

    i64 try_acquire(i64 bytes = 0);          // FREE -> IN_FLIGHT, -1 if none fits
    i64 acquire_blocking(i64 bytes = 0);     // waits for a FREE slab that fits
    void mark_in_flight(i64 id, i64 layer_id, i64 bytes);
    void mark_ready(i64 id);                 // IN_FLIGHT -> READY (+ FIFO)
    i64 pop_ready_blocking(bool* stop);      // oldest READY -> ACCUMULATING, -1 when stopped
    void release(i64 id);                    // ACCUMULATING -> FREE
    void wait_all_free();

private:
    struct Slab {
        float* data = nullptr;
        i64 capacity = 0;
        bool pinned = false;
        bool registered = false;   // huge-page mapping pinned with cudaHostRegister
        SlabState state = SlabState::FREE;
        i64 layer_id = -1;
        i64 bytes = 0;
    };
    i64 pick_free_locked(i64 bytes);
    i64 capacity_ = 0, pool_bytes_ = 0;
    std::vector<Slab> slabs_;
    std::deque<i64> ready_;
    mutable std::mutex mu_;
    std::condition_variable cv_;
    i64 in_use_ = 0, max_in_use_ = 0;
    i64 d2h_bytes_ = 0;
};

// ------------------------------------------------------------------ optimizer
// Decoupled-weight-decay Adam, bias-corrected with powf(beta, t), FP32 math in
// the reference operation order (no FMA contraction) so results are
// bit-identical to reference adam_update_tile; master updated, shadow re-packed.
// All host cores (OpenMP), AVX-512.
//   adam_step_tile: gradients from the tile's grad region (zeroed after).
//   adam_step:      validates every gradient is finite first (no mutation on failure).
//   adam_step_tile_from: gradients from an external FP32 buffer (a slab).
void adam_step(MasterStore& store, const HyperParams& hyper, i64 t);
void adam_step_tile(MasterStore& store, i64 physical_idx, const HyperParams& hyper, i64 t);
// prechecked: the caller already verified every gradient is finite (the engine
// does it on the GPU before the D2H), so the host skips its validation read.
void adam_step_tile_from(LayerTile& tile, const float* grad, const HyperParams& hyper, i64 t,
                         bool prechecked = false);
// Shard version (data parallel): elements [begin, begin + count) of the tile,
// grad points at the shard's first element. Does not bump the version.
void adam_step_range(LayerTile& tile, const float* grad, i64 begin, i64 count, const HyperParams& hyper,
                     i64 t, bool prechecked = false);

// grads(tile) += g  (slab accumulation, host_store.cpp:254-284, FP32).
void accumulate_grads(LayerTile& tile, const float* g);
// Adam over a (rows x width) tile whose gradient is zero except on the rows with
// row_map[r] >= 0, whose gradient row is compact[row_map[r] * width ...]: the zero
// rows are optimised without reading a gradient. Bit-identical to adam_step_tile_from
// on the dense gradient (same per-element IEEE operations).
void adam_step_rows_sparse(LayerTile& tile, i64 rows, i64 width, const std::int32_t* row_map, const float* compact,
                           const HyperParams& hyper, i64 t);

// Anonymous huge-page-advised mapping (throws on failure).
void* map_huge_public(size_t bytes);

// True when every element is finite (parallel scan).
bool all_finite(const float* g, i64 n);
// "avx512" or "generic": the host loop bodies this process selected at load time.
const char* host_isa();

struct HostBytesReport {
    i64 persistent = 0;
    i64 slabs = 0;
    i64 staging = 0;   // always 0: the pinned shadow is the staging buffer
    i64 total = 0;
};

}  // inline namespace b200
}  // namespace hlm
