// Device memory of the B200 engine: ONE cudaMalloc sized by the footprint
// formulas (footprint.hpp), carved into the reference's regions
// (proj/include/hlm/device_arena.hpp:25-185): two weight stream buffers, a
// LIFO activation stack (K block-activation slabs), checkpoint anchors and a
// fixed workspace. Nothing is allocated after construction; every claim and
// release goes through the exact ledger and over-claims throw ArenaOomError
// naming the region.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "hlm/errors.hpp"
#include "hlm/footprint.hpp"
#include "hlm/model_config.hpp"

namespace hlm {
inline namespace b200 {

enum class Region : int { Stream0 = 0, Stream1 = 1, Stack = 2, Anchors = 3, Workspace = 4, WeightCache = 5 };
inline constexpr int kRegionCount = 6;
const char* region_name(Region r);

struct LedgerEvent {
    int region;
    i64 delta;
};

// Byte accounting per region (the reference ArenaLedger's contract: per-region and
// whole-arena step peaks, a peak excluding the checkpoint anchors, an event log, the
// region named in the ArenaOomError of an over-claim).
class ArenaLedger {
public:
    void init_region(Region r, i64 capacity) { slot(r).cap = capacity; }
    void claim(Region r, i64 bytes);
    void release(Region r, i64 bytes);
    void begin_step();
    i64 capacity(Region r) const { return slot(r).cap; }
    i64 current(Region r) const { return slot(r).cur; }
    i64 step_peak(Region r) const { return slot(r).peak; }
    i64 total_capacity() const;
    i64 total_current() const { return all_.cur; }
    i64 step_peak_total() const { return all_.peak; }
    i64 step_peak_non_anchor() const { return non_anchor_.peak; }
    const std::vector<LedgerEvent>& events() const { return events_; }

private:
    struct Level {   // a running byte count and its high-water mark since begin_step()
        i64 cap = 0, cur = 0, peak = 0;
        void add(i64 b) { cur += b; peak = cur > peak ? cur : peak; }
    };
    Level& slot(Region r) { return regions_[static_cast<size_t>(r)]; }
    const Level& slot(Region r) const { return regions_[static_cast<size_t>(r)]; }
    std::array<Level, kRegionCount> regions_{};
    Level all_, non_anchor_;
    std::vector<LedgerEvent> events_;
};

struct ArenaSnapshot {
    struct RegionStat {
        std::string name;
        i64 capacity, current, step_peak;
    };
    std::vector<RegionStat> regions;
    i64 committed_total = 0;
    i64 committed_core = 0;
    i64 step_peak_total = 0;
    i64 step_peak_non_anchor = 0;
};

class DeviceArena {
public:
    // budget_cap: hard limit the footprint must fit (first region that does
    // not fit is named in the ArenaOomError). device: CUDA ordinal.
    // weight_cache_bytes: optional HBM region that keeps forward-streamed block
    // weights resident for the backward turnaround (one H2D pass per cached layer).
    DeviceArena(const ModelConfig& config, std::optional<i64> budget_cap = std::nullopt, int device = -1,
                i64 weight_cache_bytes = 0);
    ~DeviceArena();
    DeviceArena(const DeviceArena&) = delete;
    DeviceArena& operator=(const DeviceArena&) = delete;

    const ModelConfig& config() const { return cfg_; }
    const ArenaFootprint& footprint() const { return fp_; }
    int device() const { return device_; }
    void begin_step();
    ArenaSnapshot snapshot() const;
    const ArenaLedger& ledger() const { return ledger_; }

    // stream buffers: claim on H2D issue, release when its last reader finished
    void* claim_buffer(int i, i64 layer_id, i64 bytes);
    void release_buffer(int i);
    i64 buffer_occupant(int i) const { return occupant_[i]; }
    void* buffer(int i) const { return stream_[i]; }
    i64 h2d_bytes() const { return h2d_bytes_; }
    void add_h2d(i64 bytes) { h2d_bytes_ += bytes; }

    // weight cache: `cache_slots()` block-sized slots
    i64 cache_slots() const { return cache_slots_; }
    void* cache_slot(i64 s) const { return cache_base_ + s * fp_.stream_buf_block; }
    void claim_cache_slot(i64 s);
    void release_cache_slots();

    // activation stack (LIFO, K slabs of A_max)
    void* push_acts();
    void pop_acts();
    void* acts_at(i64 depth) const;
    i64 stack_depth() const { return depth_; }

    // anchors at multiples of K
    float* anchor_checkpoint(i64 layer_index);     // claims the slot, returns it for writing
    const float* load_checkpoint(i64 layer_index) const;
    void release_checkpoint(i64 layer_index);

    // workspace
    void claim_workspace();
    void release_workspace();
    float* g_roll(int i) const { return g_roll_[i]; }
    float* h_roll(int i) const { return h_roll_[i]; }
    void* block_ws() const { return block_ws_; }
    void* head_ws() const { return head_ws_; }
    float* grad_out(int i) const { return grad_out_[i]; }
    void* discard_acts() const { return discard_acts_; }
    int32_t* tokens() const { return tokens_; }
    int32_t* targets() const { return targets_; }
    int32_t* csr_row_ptr() const { return row_ptr_; }
    int32_t* csr_pos() const { return pos_; }
    float* loss_rows() const { return loss_rows_; }
    float* rope_cos() const { return rope_cos_; }
    float* rope_sin() const { return rope_sin_; }
    int* err_flag() const { return err_; }

private:
    float* anchor_slot(i64 layer_index) const;

    ModelConfig cfg_;
    ArenaFootprint fp_;
    ArenaLedger ledger_;
    int device_ = 0;
    char* base_ = nullptr;
    void* stream_[2] = {nullptr, nullptr};
    i64 occupant_[2] = {-1, -1};
    i64 occupant_bytes_[2] = {0, 0};
    char* stack_base_ = nullptr;
    char* cache_base_ = nullptr;
    i64 cache_slots_ = 0;
    std::vector<bool> cache_live_;
    i64 depth_ = 0;
    char* anchors_base_ = nullptr;
    std::vector<bool> anchor_live_;
    bool ws_claimed_ = false;
    float* g_roll_[2] = {nullptr, nullptr};
    float* h_roll_[2] = {nullptr, nullptr};
    void* block_ws_ = nullptr;
    void* head_ws_ = nullptr;
    float* grad_out_[2] = {nullptr, nullptr};
    void* discard_acts_ = nullptr;
    int32_t *tokens_ = nullptr, *targets_ = nullptr, *row_ptr_ = nullptr, *pos_ = nullptr;
    float *loss_rows_ = nullptr, *rope_cos_ = nullptr, *rope_sin_ = nullptr;
    int* err_ = nullptr;
    i64 h2d_bytes_ = 0;
};

}  // inline namespace b200
}  // namespace hlm
