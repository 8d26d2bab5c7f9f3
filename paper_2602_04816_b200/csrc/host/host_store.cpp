// Host parameter store, gradient slabs and the fused host Adam.
// See include/hlm/host_store.hpp for the design; reference counterparts in
// proj/src/host_store.cpp are cited per function.
#include "hlm/host_store.hpp"
#include "hlm/numa_place.hpp"

#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>
#include <sched.h>
#include <pthread.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/statvfs.h>
#include <unistd.h>

#include <chrono>
#include <thread>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "hlm/bf16.hpp"

namespace hlm {
inline namespace b200 {

namespace {

constexpr i64 kAlignElems = 1024;   // 4 KiB of fp32 / 2 KiB of bf16 per tile boundary

i64 round_up(i64 x, i64 a) { return (x + a - 1) / a * a; }

void* map_huge(size_t bytes) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw ConfigError("host store: cannot map " + std::to_string(bytes) + " bytes");
    madvise(p, bytes, MADV_HUGEPAGE);
    return p;
}

// Parallel first-touch zero fill (places pages and avoids faults inside Adam).
void parallel_zero(void* p, size_t bytes) {
    char* c = static_cast<char*>(p);
    const i64 chunk = 1 << 24;
    const i64 n = static_cast<i64>((bytes + chunk - 1) / chunk);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        const size_t off = static_cast<size_t>(i) * chunk;
        std::memset(c + off, 0, std::min<size_t>(chunk, bytes - off));
    }
}

// Host ISA: the library is compiled for x86-64-v3 (any AVX2 host); the hot host loops
// (Adam, BF16 packing, finiteness) have AVX-512 bodies selected at run time when the CPU
// has AVX-512F/BW/VL/DQ, else portable scalar bodies. Both do the same IEEE single ops
// in the same order (no FMA contraction), so results are bit-identical either way.
// HLM_HOST_ISA=generic forces the portable bodies (tests).
#define HLM_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512dq")))

bool detect_avx512() {
    const char* force = std::getenv("HLM_HOST_ISA");
    if (force && std::strcmp(force, "generic") == 0) return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
           __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
}
const bool g_avx512 = detect_avx512();

// RNE float -> bf16 for 16 lanes (bf16.hpp semantics incl. NaN quieting).
HLM_AVX512 inline __m256i bf16x16(__m512 x) {
    const __m512i b = _mm512_castps_si512(x);
    const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(b, 16), _mm512_set1_epi32(1));
    const __m512i rounded = _mm512_srli_epi32(_mm512_add_epi32(_mm512_add_epi32(b, _mm512_set1_epi32(0x7FFF)), lsb), 16);
    const __m512i hi = _mm512_srli_epi32(b, 16);
    const __mmask16 special =
        _mm512_cmpeq_epi32_mask(_mm512_and_si512(b, _mm512_set1_epi32(0x7F800000)), _mm512_set1_epi32(0x7F800000));
    const __mmask16 nan = _mm512_mask_test_epi32_mask(special, b, _mm512_set1_epi32(0x7FFFFF));
    __m512i r = _mm512_mask_mov_epi32(rounded, special, hi);
    r = _mm512_mask_or_epi32(r, nan, r, _mm512_set1_epi32(0x40));
    return _mm512_cvtepi32_epi16(r);
}

HLM_AVX512 void pack_range_avx512(const float* src, std::uint16_t* dst, i64 b, i64 e) {
    i64 i = b;
    for (; i + 16 <= e; i += 16)
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), bf16x16(_mm512_loadu_ps(src + i)));
    for (; i < e; ++i) dst[i] = bf16_bits_from_f32(src[i]);
}

void pack_range_generic(const float* src, std::uint16_t* dst, i64 b, i64 e) {
    for (i64 i = b; i < e; ++i) dst[i] = bf16_bits_from_f32(src[i]);
}

void pack_shadow(const float* src, std::uint16_t* dst, i64 n) {
    const i64 chunk = 1 << 16;
    const i64 nc = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < nc; ++c) {
        const i64 b = c * chunk, e = std::min(n, b + chunk);
        if (g_avx512)
            pack_range_avx512(src, dst, b, e);
        else
            pack_range_generic(src, dst, b, e);
    }
}

std::uint64_t mix64(std::uint64_t x) {   // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

void* map_huge_public(size_t bytes) { return map_huge(bytes); }

namespace {
size_t align_2m(size_t x) { return (x + (2u << 20) - 1) & ~size_t((2u << 20) - 1); }
}  // namespace

// Pinned host memory on transparent huge pages: a 2 MiB-aligned anonymous mapping,
// touched in parallel (huge pages fault in), then page-locked with cudaHostRegister.
// The host Adam streams gradients and shadows through these buffers; 2 MiB pages
// keep its page walks short. Opt-in (HLM_PIN_HUGE=1): measured at C2 on the pool's box
// it changes the step by less than the box's run-to-run noise (8.85 vs 9.0 k tok/s over
// 2 + 2 runs) while cutting store + slab setup from ~31 s to ~12 s.
bool pin_huge_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("HLM_PIN_HUGE");
        on = (e && *e == '1') ? 1 : 0;
    }
    return on == 1;
}
void* alloc_pinned_huge(size_t bytes) {
    const size_t b = align_2m(bytes);
    void* p = map_huge(b);
    parallel_zero(p, b);
    if (cudaHostRegister(p, b, cudaHostRegisterPortable) != cudaSuccess) {
        (void)cudaGetLastError();
        munmap(p, b);
        return nullptr;
    }
    return p;
}
void free_pinned_huge(void* p, size_t bytes) {
    cudaHostUnregister(p);
    munmap(p, align_2m(bytes));
}

// ------------------------------------------------------------------ offset tables
std::vector<NamedRegion> block_offset_table(i64 h, i64 f) {
    std::vector<NamedRegion> t;
    i64 off = 0;
    auto add = [&](const char* name, std::vector<i64> shape) {
        NamedRegion r{name, off, std::move(shape)};
        off += r.numel();
        t.push_back(std::move(r));
    };
    add("w_q", {h, h});
    add("w_k", {h, h});
    add("w_v", {h, h});
    add("w_o", {h, h});
    add("w_up", {h, f});
    add("w_gate", {h, f});
    add("w_down", {f, h});
    add("norm1", {h});
    add("norm2", {h});
    return t;
}

std::vector<NamedRegion> table_offset_table(const std::string& name, i64 vocab, i64 h) {
    return {NamedRegion{name, 0, {vocab, h}}};
}

// ------------------------------------------------------------------ LayerTile
LayerTile::LayerTile(i64 layer_id, i64 n_params, std::vector<NamedRegion> offsets, float* state,
                     std::uint16_t* shadow)
    : layer_id_(layer_id), n_params_(n_params), offsets_(std::move(offsets)), state_(state), shadow_(shadow) {
    i64 covered = 0;
    for (const auto& r : offsets_) {
        if (r.offset != covered) throw ProtocolError("tile offset table has a gap or overlap at '" + r.name + "'");
        covered += r.numel();
    }
    if (covered != n_params) throw ProtocolError("tile offset table does not cover the tile");
}

const NamedRegion& LayerTile::region(const std::string& name) const {
    for (const auto& r : offsets_)
        if (r.name == name) return r;
    throw ProtocolError("tile has no tensor named " + name);
}

float* LayerTile::grads() {
    if (!grads_) {
        grads_.reset(new float[static_cast<size_t>(n_params_)]);
        parallel_zero(grads_.get(), static_cast<size_t>(n_params_) * 4);
    }
    return grads_.get();
}

void LayerTile::store_weight(i64 i, float v) {
    state_[i] = v;
    shadow_[i] = bf16_bits_from_f32(v);
}

// ------------------------------------------------------------------ MasterStore
namespace {
constexpr size_t kShmHeader = 2u << 20;
constexpr std::uint64_t kShmMagic = 0x484C4D53484D3031ull;   // "HLMSHM01"
struct ShmHeader {
    std::uint64_t magic;
    std::atomic<std::uint64_t> ready;
    std::int64_t dims[8];
    std::uint64_t nonce;
};
size_t align2m(size_t x) { return (x + (2u << 20) - 1) & ~size_t((2u << 20) - 1); }
}  // namespace

MasterStore::MasterStore(const ModelConfig& config, Dtype dtype, bool pin_shadow, const SharedStoreSpec* shared)
    : config_(config), dtype_(dtype) {
    config_.validate();
    const i64 h = config_.hidden, f = config_.ffn, V = config_.vocab;
    struct Spec {
        i64 id, n;
        std::vector<NamedRegion> off;
    };
    std::vector<Spec> specs;
    specs.push_back({config_.embed_tile_id(), V * h, table_offset_table("embed", V, h)});
    for (i64 l = 1; l <= config_.layers; ++l) specs.push_back({l, config_.block_params(), block_offset_table(h, f)});
    if (!config_.tie_embeddings) specs.push_back({config_.head_tile_id(), V * h, table_offset_table("head", V, h)});

    i64 state_elems = 0, shadow_elems = 0;
    for (const auto& s : specs) {
        state_elems += 3 * round_up(s.n, kAlignElems);
        shadow_elems += round_up(s.n, kAlignElems);
    }
    state_bytes_ = static_cast<size_t>(state_elems) * 4;
    shadow_bytes_ = static_cast<size_t>(shadow_elems) * 2;
    std::atomic<i64>* versions = nullptr;
    if (shared && shared->world >= 1 && !shared->name.empty()) {
        rank_ = shared->rank;
        world_ = shared->world;
        shm_name_ = "/" + shared->name;
        const size_t ver_bytes = align2m(specs.size() * static_cast<size_t>(world_) * sizeof(i64));
        map_bytes_ = kShmHeader + align2m(state_bytes_) + align2m(shadow_bytes_) + ver_bytes;
        if (rank_ == 0) {
            // tmpfs pages are allocated on first touch: a store larger than the free space of
            // /dev/shm would die of SIGBUS mid-initialisation, so refuse it up front
            struct statvfs vs {};
            if (statvfs("/dev/shm", &vs) == 0) {
                const double avail = static_cast<double>(vs.f_bavail) * static_cast<double>(vs.f_frsize);
                if (avail < static_cast<double>(map_bytes_))
                    throw ConfigError("shared store: " + std::to_string(map_bytes_ >> 20) + " MiB needed but /dev/shm has " +
                                      std::to_string(static_cast<long long>(avail) >> 20) +
                                      " MiB free (remount /dev/shm larger or use fewer / smaller tiles)");
            }
            shm_unlink(shm_name_.c_str());
            shm_fd_ = shm_open(shm_name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
            if (shm_fd_ < 0) throw ConfigError("shared store: shm_open(create) failed for " + shm_name_);
            if (ftruncate(shm_fd_, static_cast<off_t>(map_bytes_)) != 0)
                throw ConfigError("shared store: ftruncate failed");
            map_base_ = mmap(nullptr, map_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, shm_fd_, 0);
            if (map_base_ == MAP_FAILED) throw ConfigError("shared store: mmap failed");
        } else {
            attach_shared(shared->nonce);
        }
        char* b = static_cast<char*>(map_base_);
        auto* hdr = reinterpret_cast<ShmHeader*>(b);
        state_base_ = reinterpret_cast<float*>(b + kShmHeader);
        shadow_base_ = reinterpret_cast<std::uint16_t*>(b + kShmHeader + align2m(state_bytes_));
        versions = reinterpret_cast<std::atomic<i64>*>(b + kShmHeader + align2m(state_bytes_) + align2m(shadow_bytes_));
        const std::int64_t dims[8] = {config_.layers, config_.hidden, config_.ffn, config_.vocab,
                                      config_.tie_embeddings ? 1 : 0, static_cast<std::int64_t>(world_), 0, 0};
        if (rank_ == 0) {
            hdr->magic = kShmMagic;
            hdr->nonce = shared->nonce;
            std::memcpy(hdr->dims, dims, sizeof dims);
        } else if (std::memcmp(hdr->dims, dims, sizeof dims) != 0) {
            throw ConfigError("shared store: " + shm_name_ + " was created for another model / world size");
        }
        if (rank_ == 0) {
            if (world_ > 1 && numa_node_count() > 1) {
                // multi-socket host: each rank's shard of every tile (master, m, v, shadow)
                // in the DRAM of its GPU's socket, where its Adam team and its DMA run
                const std::vector<int> nodes = rank_gpu_nodes(world_);
                i64 so = 0, sh = 0;
                for (const auto& sp : specs) {
                    const i64 cnt = sp.n / world_;
                    for (int r = 0; r < world_; ++r)
                        for (int a = 0; a < 4; ++a) {
                            if (a < 3)
                                prefer_node(state_base_ + so + a * sp.n + r * cnt, static_cast<size_t>(cnt) * 4,
                                            nodes[static_cast<size_t>(r)]);
                            else
                                prefer_node(shadow_base_ + sh + r * cnt, static_cast<size_t>(cnt) * 2,
                                            nodes[static_cast<size_t>(r)]);
                        }
                    so += 3 * round_up(sp.n, kAlignElems);
                    sh += round_up(sp.n, kAlignElems);
                }
            }
            parallel_zero(state_base_, state_bytes_);
            parallel_zero(shadow_base_, shadow_bytes_);
            parallel_zero(versions, specs.size() * static_cast<size_t>(world_) * sizeof(i64));
        }
        if (pin_shadow) {
            if (cudaHostRegister(shadow_base_, align2m(shadow_bytes_), cudaHostRegisterPortable) == cudaSuccess)
                registered_ = pinned_ = true;
            else
                (void)cudaGetLastError();
        }
    } else {
    state_base_ = static_cast<float*>(map_huge(state_bytes_));
    parallel_zero(state_base_, state_bytes_);
    }
    if (shm_fd_ < 0 && pin_shadow && pin_huge_enabled()) {
        if (void* p = alloc_pinned_huge(static_cast<size_t>(shadow_bytes_))) {
            shadow_base_ = static_cast<std::uint16_t*>(p);
            pinned_ = registered_ = true;
        }
    }
    if (shm_fd_ < 0 && pin_shadow && !shadow_base_) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, shadow_bytes_, cudaHostAllocPortable) == cudaSuccess) {
            shadow_base_ = static_cast<std::uint16_t*>(p);
            pinned_ = true;
        } else {
            (void)cudaGetLastError();
        }
    }
    if (!shadow_base_) {
        shadow_base_ = static_cast<std::uint16_t*>(map_huge(shadow_bytes_));
        parallel_zero(shadow_base_, shadow_bytes_);
    }

    i64 so = 0, sh = 0;
    for (auto& s : specs) {
        const i64 padded = round_up(s.n, kAlignElems);
        tiles_.push_back(std::make_unique<LayerTile>(s.id, s.n, std::move(s.off), state_base_ + so, shadow_base_ + sh));
        if (versions) tiles_.back()->attach_shared_versions(versions + (tiles_.size() - 1) * world_, world_);
        so += 3 * padded;
        sh += padded;
    }
    // master, m, v are contiguous inside each tile's slot; the padding sits after v.
    physical_of_.push_back(0);
    for (i64 l = 1; l <= config_.layers; ++l) physical_of_.push_back(l);
    physical_of_.push_back(config_.tie_embeddings ? 0 : config_.layers + 1);
    for (const auto& t : tiles_) total_params_ += t->n_params();
}

MasterStore::~MasterStore() {
    for (auto& t : tiles_) t.reset();
    if (shm_fd_ >= 0) {
        if (registered_) cudaHostUnregister(shadow_base_);
        munmap(map_base_, map_bytes_);
        close(shm_fd_);
        if (rank_ == 0) shm_unlink(shm_name_.c_str());
        return;
    }
    if (state_base_) munmap(state_base_, state_bytes_);
    if (shadow_base_) {
        if (registered_)
            free_pinned_huge(shadow_base_, static_cast<size_t>(shadow_bytes_));
        else if (pinned_)
            cudaFreeHost(shadow_base_);
        else
            munmap(shadow_base_, shadow_bytes_);
    }
}

i64 MasterStore::consumer_count(i64 physical_idx) const {
    i64 n = 0;
    for (i64 l = 0; l < logical_tiles(); ++l)
        if (physical_of_[static_cast<size_t>(l)] == physical_idx) ++n;
    return n;
}

i64 MasterStore::persistent_bytes() const {
    i64 total = 0;
    for (const auto& t : tiles_) {
        total += t->n_params() * (12 + 2);
        if (t->has_grads()) total += t->n_params() * 4;
    }
    return total;
}

bool MasterStore::bitwise_equal(const MasterStore& o) const {
    if (physical_tiles() != o.physical_tiles()) return false;
    for (i64 p = 0; p < physical_tiles(); ++p) {
        const LayerTile& a = physical(p);
        const LayerTile& b = o.physical(p);
        if (a.n_params() != b.n_params()) return false;
        const size_t n = static_cast<size_t>(a.n_params());
        if (std::memcmp(a.master(), b.master(), 3 * n * 4) != 0) return false;
        if (std::memcmp(a.shadow(), b.shadow(), n * 2) != 0) return false;
    }
    return true;
}

void MasterStore::mark_ready() {
    if (shm_fd_ < 0) return;
    reinterpret_cast<ShmHeader*>(map_base_)->ready.store(1, std::memory_order_release);
}

// Attaching rank: open the segment under the name, wait for its full size, map it and
// accept it only once it carries this run's nonce. A segment left by a crashed run
// (same name, magic, even ready == 1) has another nonce: drop the mapping and re-open
// by name, which yields rank 0's fresh segment once rank 0 unlinked and recreated it.
void MasterStore::attach_shared(std::uint64_t nonce) {
    for (int attempt = 0; attempt < 120000; ++attempt) {
        if (attempt) std::this_thread::sleep_for(std::chrono::milliseconds(5));
        if (shm_fd_ < 0) shm_fd_ = shm_open(shm_name_.c_str(), O_RDWR, 0600);
        if (shm_fd_ < 0) continue;
        if (lseek(shm_fd_, 0, SEEK_END) < static_cast<off_t>(map_bytes_)) {
            // too small: still being sized by rank 0, or a stale segment of another model
            struct stat by_fd {}, by_name {};
            const int nfd = shm_open(shm_name_.c_str(), O_RDONLY, 0600);
            const bool replaced = nfd >= 0 && fstat(shm_fd_, &by_fd) == 0 && fstat(nfd, &by_name) == 0 &&
                                  by_fd.st_ino != by_name.st_ino;
            if (nfd >= 0) close(nfd);
            if (replaced) {
                close(shm_fd_);
                shm_fd_ = -1;
            }
            continue;
        }
        void* base = mmap(nullptr, map_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, shm_fd_, 0);
        if (base == MAP_FAILED) throw ConfigError("shared store: mmap failed");
        auto* hdr = reinterpret_cast<volatile ShmHeader*>(base);
        if (hdr->magic == kShmMagic && hdr->nonce == nonce) {
            map_base_ = base;
            return;
        }
        munmap(base, map_bytes_);
        close(shm_fd_);   // stale or not yet stamped: look the name up again
        shm_fd_ = -1;
    }
    throw ConfigError("shared store: no segment " + shm_name_ + " with this run's nonce appeared (rank 0 never "
                      "created it, or a stale segment is in the way)");
}

void MasterStore::wait_ready() const {
    if (shm_fd_ < 0) return;
    auto* hdr = reinterpret_cast<ShmHeader*>(map_base_);
    for (;;) {
        if (hdr->magic == kShmMagic && hdr->ready.load(std::memory_order_acquire) == 1) return;
        std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
}

void MasterStore::repack_shadow() {
    for (auto& t : tiles_) pack_shadow(t->master(), t->shadow(), t->n_params());
}

// reference host_store.cpp:141-156 (InitMode::Reference is bit-identical).
std::unique_ptr<MasterStore> build_store(const ModelConfig& config, std::uint64_t seed, Dtype dtype, InitMode mode,
                                         bool pin_shadow, const SharedStoreSpec* shared) {
    auto store = std::make_unique<MasterStore>(config, dtype, pin_shadow, shared);
    if (store->shared() && !store->owner()) {   // attach: rank 0 initialises
        store->wait_ready();
        return store;
    }
    const bool bf = dtype == Dtype::BF16;
    if (mode == InitMode::Reference) {
        Rng rng(seed);
        for (i64 p = 0; p < store->physical_tiles(); ++p) {
            LayerTile& t = store->physical(p);
            float* w = t.master();
            for (const auto& r : t.offset_table()) {
                const bool norm = r.name == "norm1" || r.name == "norm2";
                for (i64 i = 0; i < r.numel(); ++i) {
                    const float v = norm ? 1.0f : rng.trunc_normal(0.02f);
                    w[r.offset + i] = bf ? bf16_round(v) : v;
                }
            }
        }
    } else {
        const i64 chunk = 1 << 16;
        for (i64 p = 0; p < store->physical_tiles(); ++p) {
            LayerTile& t = store->physical(p);
            float* w = t.master();
            const i64 n = t.n_params();
            const i64 norm_begin = config.is_block_tile(t.layer_id()) ? config.block_matmul_params() : n;
            const i64 nc = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 16)
            for (i64 c = 0; c < nc; ++c) {
                Rng rng(mix64(seed ^ mix64(static_cast<std::uint64_t>(p) * 0x100000001B3ull + static_cast<std::uint64_t>(c))));
                const i64 b = c * chunk, e = std::min(n, b + chunk);
                for (i64 i = b; i < e; ++i) {
                    const float v = i >= norm_begin ? 1.0f : rng.trunc_normal(0.02f);
                    w[i] = bf ? bf16_round(v) : v;
                }
            }
        }
    }
    store->repack_shadow();
    store->mark_ready();
    return store;
}

// ------------------------------------------------------------------ SlabPool
const char* slab_state_name(SlabState s) {
    switch (s) {
        case SlabState::FREE: return "FREE";
        case SlabState::IN_FLIGHT: return "IN_FLIGHT";
        case SlabState::READY: return "READY";
        case SlabState::ACCUMULATING: return "ACCUMULATING";
    }
    return "?";
}

SlabPool::SlabPool(i64 n_slabs, i64 capacity_bytes, bool pinned)
    : SlabPool(std::vector<i64>(static_cast<size_t>(std::max<i64>(n_slabs, 0)), capacity_bytes), pinned) {}

SlabPool::SlabPool(const std::vector<i64>& capacities, bool pinned) {
    if (capacities.empty()) throw ConfigError("slab pool needs at least one slab");
    slabs_.resize(capacities.size());
    for (size_t i = 0; i < capacities.size(); ++i) {
        Slab& s = slabs_[i];
        s.capacity = capacities[i];
        capacity_ = std::max(capacity_, s.capacity);
        pool_bytes_ += s.capacity;
        void* p = nullptr;
        if (pinned && pin_huge_enabled() && (p = alloc_pinned_huge(static_cast<size_t>(s.capacity))) != nullptr) {
            s.pinned = s.registered = true;
        } else if (pinned && cudaHostAlloc(&p, static_cast<size_t>(s.capacity), cudaHostAllocPortable) == cudaSuccess) {
            s.pinned = true;
        } else {
            (void)cudaGetLastError();
            p = map_huge(static_cast<size_t>(s.capacity));
        }
        s.data = static_cast<float*>(p);
    }
}

SlabPool::~SlabPool() {
    for (auto& s : slabs_) {
        if (!s.data) continue;
        if (s.registered)
            free_pinned_huge(s.data, static_cast<size_t>(s.capacity));
        else if (s.pinned)
            cudaFreeHost(s.data);
        else
            munmap(s.data, static_cast<size_t>(s.capacity));
    }
}

SlabState SlabPool::state(i64 id) const {
    std::lock_guard<std::mutex> lk(mu_);
    return slabs_[static_cast<size_t>(id)].state;
}

// smallest FREE slab with capacity >= bytes (first such in index order on ties)
i64 SlabPool::pick_free_locked(i64 bytes) {
    i64 best = -1;
    for (size_t i = 0; i < slabs_.size(); ++i) {
        const Slab& s = slabs_[i];
        if (s.state != SlabState::FREE || s.capacity < bytes) continue;
        if (best < 0 || s.capacity < slabs_[static_cast<size_t>(best)].capacity) best = static_cast<i64>(i);
    }
    if (best >= 0) {
        slabs_[static_cast<size_t>(best)].state = SlabState::IN_FLIGHT;
        if (++in_use_ > max_in_use_) max_in_use_ = in_use_;
    }
    return best;
}

i64 SlabPool::try_acquire(i64 bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    if (bytes > capacity_) throw ProtocolError("slab request exceeds the largest slab");
    return pick_free_locked(bytes);
}

i64 SlabPool::acquire_blocking(i64 bytes) {
    std::unique_lock<std::mutex> lk(mu_);
    if (bytes > capacity_) throw ProtocolError("slab request exceeds the largest slab");
    for (;;) {
        const i64 id = pick_free_locked(bytes);
        if (id >= 0) return id;
        cv_.wait(lk);
    }
}

void SlabPool::mark_in_flight(i64 id, i64 layer_id, i64 bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    Slab& s = slabs_[static_cast<size_t>(id)];
    if (s.state != SlabState::IN_FLIGHT) throw ProtocolError(std::string("slab fill in state ") + slab_state_name(s.state));
    if (bytes > s.capacity) throw ProtocolError("slab payload exceeds slab capacity");
    s.layer_id = layer_id;
    s.bytes = bytes;
    d2h_bytes_ += bytes;   // counted when the copy is issued
}

void SlabPool::mark_ready(i64 id) {
    std::lock_guard<std::mutex> lk(mu_);
    Slab& s = slabs_[static_cast<size_t>(id)];
    if (s.state != SlabState::IN_FLIGHT) throw ProtocolError(std::string("slab ready in state ") + slab_state_name(s.state));
    s.state = SlabState::READY;
    ready_.push_back(id);
    cv_.notify_all();
}

i64 SlabPool::pop_ready_blocking(bool* stop) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !ready_.empty() || *stop; });
    if (ready_.empty()) return -1;
    const i64 id = ready_.front();
    ready_.pop_front();
    slabs_[static_cast<size_t>(id)].state = SlabState::ACCUMULATING;
    return id;
}

void SlabPool::release(i64 id) {
    std::lock_guard<std::mutex> lk(mu_);
    Slab& s = slabs_[static_cast<size_t>(id)];
    if (s.state != SlabState::ACCUMULATING && s.state != SlabState::IN_FLIGHT)
        throw ProtocolError(std::string("slab release in state ") + slab_state_name(s.state));
    s.state = SlabState::FREE;
    s.layer_id = -1;
    s.bytes = 0;
    --in_use_;
    cv_.notify_all();
}

void SlabPool::wait_all_free() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return in_use_ == 0; });
}

// ------------------------------------------------------------------ Adam
namespace {
HLM_AVX512 bool finite_range_avx512(const float* g, i64 b, i64 e) {
    i64 i = b;
    __mmask16 acc = 0;
    for (; i + 16 <= e; i += 16) {
        const __m512i x = _mm512_castps_si512(_mm512_loadu_ps(g + i));
        acc |= _mm512_cmpeq_epi32_mask(_mm512_and_si512(x, _mm512_set1_epi32(0x7F800000)),
                                       _mm512_set1_epi32(0x7F800000));
    }
    for (; i < e; ++i)
        if (!std::isfinite(g[i])) acc = 1;
    return acc == 0;
}

bool finite_range_generic(const float* g, i64 b, i64 e) {
    std::uint32_t acc = 0;   // branch-free: exponent all ones = Inf / NaN
    for (i64 i = b; i < e; ++i) {
        std::uint32_t bits;
        std::memcpy(&bits, g + i, 4);
        acc |= static_cast<std::uint32_t>((bits & 0x7F800000u) == 0x7F800000u);
    }
    return acc == 0;
}
}  // namespace

bool all_finite(const float* g, i64 n) {
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (i64 c = 0; c < (n + 65535) / 65536; ++c) {
        const i64 b = c * 65536, e = std::min(n, b + 65536);
        const bool ok = g_avx512 ? finite_range_avx512(g, b, e) : finite_range_generic(g, b, e);
        if (!ok) bad = 1;
    }
    return bad == 0;
}

const char* host_isa() { return g_avx512 ? "avx512" : "generic"; }

namespace {

i64 first_non_finite(const float* g, i64 n) {
    for (i64 i = 0; i < n; ++i)
        if (!std::isfinite(g[i])) return i;
    return -1;
}

// Reference host_store.cpp:342-361. Every operation is an IEEE single op in the
// reference's order (this TU is compiled with -ffp-contract=off), so the 16-wide lanes
// and the scalar bodies equal the scalar reference bit for bit. `g == nullptr` is an
// all-zero gradient that is never read (row-sparse embedding update).
struct AdamScalars {
    float lr, b1, b2, eps, wd, bc1, bc2;
};

inline void adam_scalar(float* w, float* m, float* v, std::uint16_t* shadow, const float* g, i64 i,
                        const AdamScalars& a) {
    const float gv = g ? g[i] : 0.0f;
    m[i] = a.b1 * m[i] + (1.0f - a.b1) * gv;
    v[i] = a.b2 * v[i] + (1.0f - a.b2) * gv * gv;
    const float mhat = m[i] / a.bc1;
    const float vhat = v[i] / a.bc2;
    float th = w[i];
    th -= a.lr * (mhat / (std::sqrt(vhat) + a.eps) + a.wd * th);
    w[i] = th;
    shadow[i] = bf16_bits_from_f32(th);
}

// stream_shadow: the shadow is only read by the next H2D DMA, so full 32-byte groups
// are stored non-temporally (no read-for-ownership of the destination lines).
HLM_AVX512 void adam_range_avx512(float* __restrict w, float* __restrict m, float* __restrict v,
                                  std::uint16_t* __restrict shadow, const float* __restrict g, i64 b, i64 e,
                                  const AdamScalars& a, float* zero_after, bool stream_shadow) {
    const __m512 vb1 = _mm512_set1_ps(a.b1), vb2 = _mm512_set1_ps(a.b2), vo1 = _mm512_set1_ps(1.0f - a.b1),
                 vo2 = _mm512_set1_ps(1.0f - a.b2), vbc1 = _mm512_set1_ps(a.bc1), vbc2 = _mm512_set1_ps(a.bc2),
                 veps = _mm512_set1_ps(a.eps), vwd = _mm512_set1_ps(a.wd), vlr = _mm512_set1_ps(a.lr);
    i64 i = b;
    for (; i + 16 <= e; i += 16) {
        const __m512 gg = g ? _mm512_loadu_ps(g + i) : _mm512_setzero_ps();
        __m512 mm = _mm512_loadu_ps(m + i);
        __m512 vv = _mm512_loadu_ps(v + i);
        __m512 th = _mm512_loadu_ps(w + i);
        mm = _mm512_add_ps(_mm512_mul_ps(vb1, mm), _mm512_mul_ps(vo1, gg));
        vv = _mm512_add_ps(_mm512_mul_ps(vb2, vv), _mm512_mul_ps(_mm512_mul_ps(vo2, gg), gg));
        const __m512 mhat = _mm512_div_ps(mm, vbc1);
        const __m512 vhat = _mm512_div_ps(vv, vbc2);
        const __m512 upd = _mm512_add_ps(_mm512_div_ps(mhat, _mm512_add_ps(_mm512_sqrt_ps(vhat), veps)),
                                         _mm512_mul_ps(vwd, th));
        th = _mm512_sub_ps(th, _mm512_mul_ps(vlr, upd));
        _mm512_storeu_ps(m + i, mm);
        _mm512_storeu_ps(v + i, vv);
        _mm512_storeu_ps(w + i, th);
        if (stream_shadow && (reinterpret_cast<uintptr_t>(shadow + i) & 31) == 0)
            _mm256_stream_si256(reinterpret_cast<__m256i*>(shadow + i), bf16x16(th));
        else
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(shadow + i), bf16x16(th));
        if (zero_after) _mm512_storeu_ps(zero_after + i, _mm512_setzero_ps());
    }
    for (; i < e; ++i) {
        adam_scalar(w, m, v, shadow, g, i, a);
        if (zero_after) zero_after[i] = 0.0f;
    }
}

void adam_range_generic(float* __restrict w, float* __restrict m, float* __restrict v,
                        std::uint16_t* __restrict shadow, const float* __restrict g, i64 b, i64 e,
                        const AdamScalars& a, float* zero_after) {
    for (i64 i = b; i < e; ++i) {
        adam_scalar(w, m, v, shadow, g, i, a);
        if (zero_after) zero_after[i] = 0.0f;
    }
}

void adam_kernel(float* __restrict w, float* __restrict m, float* __restrict v, std::uint16_t* __restrict shadow,
                 const float* __restrict g, i64 n, float lr, float b1, float b2, float eps, float wd, float bc1,
                 float bc2, float* zero_after) {
    const i64 chunk = 1 << 15;
    const i64 nc = (n + chunk - 1) / chunk;
    const AdamScalars a{lr, b1, b2, eps, wd, bc1, bc2};
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < nc; ++c) {
        const i64 b = c * chunk, e = std::min(n, b + chunk);
        if (g_avx512) {
            adam_range_avx512(w, m, v, shadow, g, b, e, a, zero_after, true);
            _mm_sfence();   // order this thread's non-temporal shadow stores
        } else {
            adam_range_generic(w, m, v, shadow, g, b, e, a, zero_after);
        }
    }
}

void adam_apply(LayerTile& tile, const float* grad, const HyperParams& hyper, i64 t, float* zero_after,
                bool prechecked = false) {
    if (t < 1) throw ProtocolError("adam step index must be >= 1");
    if (!prechecked && !all_finite(grad, tile.n_params()))
        throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + " at element " +
                            std::to_string(first_non_finite(grad, tile.n_params())) + "; step aborted");
    const float lr = static_cast<float>(hyper.lr), b1 = static_cast<float>(hyper.beta1),
                b2 = static_cast<float>(hyper.beta2), eps = static_cast<float>(hyper.eps),
                wd = static_cast<float>(hyper.weight_decay);
    const float bc1 = 1.0f - std::pow(b1, static_cast<float>(t));
    const float bc2 = 1.0f - std::pow(b2, static_cast<float>(t));
    adam_kernel(tile.master(), tile.moment_m(), tile.moment_v(), tile.shadow(), grad, tile.n_params(), lr, b1, b2,
                eps, wd, bc1, bc2, zero_after);
    tile.bump_version(0);
}

}  // namespace

void adam_step_range(LayerTile& tile, const float* grad, i64 begin, i64 count, const HyperParams& hyper, i64 t,
                     bool prechecked) {
    if (t < 1) throw ProtocolError("adam step index must be >= 1");
    if (begin < 0 || begin + count > tile.n_params()) throw ProtocolError("adam shard out of range");
    if (!prechecked && !all_finite(grad, count))
        throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + " at element " +
                            std::to_string(begin + first_non_finite(grad, count)) + "; step aborted");
    const float lr = static_cast<float>(hyper.lr), b1 = static_cast<float>(hyper.beta1),
                b2 = static_cast<float>(hyper.beta2), eps = static_cast<float>(hyper.eps),
                wd = static_cast<float>(hyper.weight_decay);
    const float bc1 = 1.0f - std::pow(b1, static_cast<float>(t));
    const float bc2 = 1.0f - std::pow(b2, static_cast<float>(t));
    adam_kernel(tile.master() + begin, tile.moment_m() + begin, tile.moment_v() + begin, tile.shadow() + begin, grad,
                count, lr, b1, b2, eps, wd, bc1, bc2, nullptr);
}

void adam_step_rows_sparse(LayerTile& tile, i64 rows, i64 width, const std::int32_t* row_map, const float* compact,
                           const HyperParams& hyper, i64 t) {
    if (t < 1) throw ProtocolError("adam step index must be >= 1");
    if (rows * width != tile.n_params()) throw ProtocolError("sparse adam: geometry mismatch");
    const float lr = static_cast<float>(hyper.lr), b1 = static_cast<float>(hyper.beta1),
                b2 = static_cast<float>(hyper.beta2), eps = static_cast<float>(hyper.eps),
                wd = static_cast<float>(hyper.weight_decay);
    const float bc1 = 1.0f - std::pow(b1, static_cast<float>(t));
    const float bc2 = 1.0f - std::pow(b2, static_cast<float>(t));
    const AdamScalars a{lr, b1, b2, eps, wd, bc1, bc2};
    float* W = tile.master();
    float* M = tile.moment_m();
    float* Vv = tile.moment_v();
    std::uint16_t* SH = tile.shadow();
#pragma omp parallel for schedule(static, 16)
    for (i64 r = 0; r < rows; ++r) {
        const i64 b = r * width, e = b + width;
        // adam_kernel's lane sequence; an untouched row's zero gradient is not read
        const float* g = row_map[r] >= 0 ? compact + static_cast<i64>(row_map[r]) * width - b : nullptr;
        if (g_avx512)
            adam_range_avx512(W, M, Vv, SH, g, b, e, a, nullptr, false);
        else
            adam_range_generic(W, M, Vv, SH, g, b, e, a, nullptr);
    }
    tile.bump_version(0);
}

void adam_step_tile_from(LayerTile& tile, const float* grad, const HyperParams& hyper, i64 t, bool prechecked) {
    adam_apply(tile, grad, hyper, t, nullptr, prechecked);
}

void adam_step_tile(MasterStore& store, i64 physical_idx, const HyperParams& hyper, i64 t) {
    LayerTile& tile = store.physical(physical_idx);
    float* g = tile.grads();
    adam_apply(tile, g, hyper, t, g);
}

// reference host_store.cpp:371-385: validate everything before any mutation.
void adam_step(MasterStore& store, const HyperParams& hyper, i64 t) {
    if (t < 1) throw ProtocolError("adam step index must be >= 1");
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        LayerTile& tile = store.physical(p);
        const float* g = tile.grads();
        if (!all_finite(g, tile.n_params()))
            throw NumericsError("non-finite gradient in layer " + std::to_string(tile.layer_id()) + " at element " +
                                std::to_string(first_non_finite(g, tile.n_params())) + "; step aborted");
    }
    for (i64 p = 0; p < store.physical_tiles(); ++p) adam_step_tile(store, p, hyper, t);
}

void accumulate_grads(LayerTile& tile, const float* g) {
    float* dst = tile.grads();
    const i64 n = tile.n_params();
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < (n + 65535) / 65536; ++c) {
        const i64 b = c * 65536, e = std::min(n, b + 65536);
        for (i64 i = b; i < e; ++i) dst[i] = dst[i] + g[i];
    }
}

}  // inline namespace b200
}  // namespace hlm

namespace hlm {
inline namespace b200 {
double triad_gbs_impl(int64_t bytes_per_array, int reps);
}  // inline namespace b200
}  // namespace hlm

// STREAM triad on a thread of its own with a team pinned like the optimizer's (one
// thread per allowed CPU), so the roofline denominator sees the same placement.
extern "C" double hlm_host_triad_gbs(int64_t bytes_per_array, int reps) {
    double best = 0.0;
    std::thread th([&] {
        cpu_set_t allowed;
        CPU_ZERO(&allowed);
        std::vector<int> cpus;
        if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0)
            for (int c = 0; c < CPU_SETSIZE; ++c)
                if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
        if (!cpus.empty()) {
            omp_set_num_threads(static_cast<int>(cpus.size()));
#pragma omp parallel
            {
                cpu_set_t one;
                CPU_ZERO(&one);
                CPU_SET(cpus[static_cast<size_t>(omp_get_thread_num()) % cpus.size()], &one);
                pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
            }
        }
        best = hlm::triad_gbs_impl(bytes_per_array, reps);
    });
    th.join();
    return best;
}

namespace hlm {
inline namespace b200 {
double triad_gbs_impl(int64_t bytes_per_array, int reps) {
    const hlm::i64 n = bytes_per_array / 4;
    float* a = static_cast<float*>(hlm::map_huge_public(static_cast<size_t>(n) * 4));
    float* b = static_cast<float*>(hlm::map_huge_public(static_cast<size_t>(n) * 4));
    float* c = static_cast<float*>(hlm::map_huge_public(static_cast<size_t>(n) * 4));
#pragma omp parallel for schedule(static)
    for (hlm::i64 i = 0; i < n; ++i) {
        a[i] = 0.f;
        b[i] = 1.f;
        c[i] = 2.f;
    }
    double best = 0;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
        for (hlm::i64 i = 0; i < n; ++i) a[i] = b[i] + 0.5f * c[i];
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::max(best, 3.0 * static_cast<double>(n) * 4 / dt / 1e9);
    }
    munmap(a, static_cast<size_t>(n) * 4);
    munmap(b, static_cast<size_t>(n) * 4);
    munmap(c, static_cast<size_t>(n) * 4);
    return best;
}
}  // inline namespace b200
}  // namespace hlm
