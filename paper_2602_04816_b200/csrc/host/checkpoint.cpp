// HLM2 checkpoint (see include/hlm/checkpoint.hpp), plus the reference's HLM1
// container read by load_checkpoint and written by save_checkpoint_hlm1.
#include "hlm/checkpoint.hpp"

#include <cstdint>
#include <cstring>
#include <fstream>
#include <vector>

#include "hlm/bf16.hpp"

namespace hlm {
inline namespace b200 {

namespace {

constexpr char kMagic[4] = {'H', 'L', 'M', '2'};
constexpr std::uint32_t kVersion = 1;
constexpr std::int64_t kAlign = 4096;

struct Header {
    char magic[4];
    std::uint32_t version;
    std::uint32_t physical_tiles;
    std::uint32_t logical_tiles;
    std::int64_t dims[8];   // layers, hidden, ffn, vocab, tie, n_heads, 0, 0
    std::uint64_t total_params;
    std::uint64_t adam_steps;
};

void fill_dims(const ModelConfig& m, std::int64_t* d) {
    const std::int64_t v[8] = {m.layers, m.hidden, m.ffn, m.vocab, m.tie_embeddings ? 1 : 0, m.n_heads, 0, 0};
    std::memcpy(d, v, sizeof v);
}

}  // namespace

void save_checkpoint(const MasterStore& store, const std::string& path) {
    store.quiesce();   // an attached engine's optimizer tail and resident tiles land first
    if (store.device_newer() > 0)
        throw ProtocolError("save_checkpoint: an engine holds HBM-resident tiles newer than the store; "
                            "call Engine::sync() first");
    Header h{};
    std::memcpy(h.magic, kMagic, 4);
    h.version = kVersion;
    h.physical_tiles = static_cast<std::uint32_t>(store.physical_tiles());
    h.logical_tiles = static_cast<std::uint32_t>(store.logical_tiles());
    fill_dims(store.config(), h.dims);
    h.total_params = static_cast<std::uint64_t>(store.total_params());
    h.adam_steps = static_cast<std::uint64_t>(store.adam_steps());
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw ConfigError("cannot open checkpoint file for writing: " + path);
    f.write(reinterpret_cast<const char*>(&h), sizeof h);
    std::int64_t written = sizeof h;
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        const std::uint64_t n = static_cast<std::uint64_t>(store.physical(p).n_params());
        f.write(reinterpret_cast<const char*>(&n), sizeof n);
        written += sizeof n;
    }
    const std::vector<char> pad(kAlign, 0);
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        const std::int64_t aligned = (written + kAlign - 1) / kAlign * kAlign;
        if (aligned > written) f.write(pad.data(), aligned - written);
        written = aligned;
        const LayerTile& t = store.physical(p);
        const std::int64_t bytes = 12 * t.n_params();   // master, m, v (contiguous)
        f.write(reinterpret_cast<const char*>(t.master()), bytes);
        written += bytes;
    }
    if (!f) throw ConfigError("checkpoint write failed: " + path);
}

namespace {

// ---------------------------------------------------------------- HLM1 (reference)
// The reference container (proj/src/checkpoint.cpp:15-120): "HLM1", u32 version 1,
// u32 physical tiles, u32 dtype code, u64 total params, u64 Adam steps, u64 params per
// physical tile, u32 logical tiles + u32 physical index per logical tile; then each
// physical tile's raw LayerTile image at a 4096-aligned file offset, laid out as the
// reference tile (proj/include/hlm/host_store.hpp:40-66): [weights | grads] in the store
// dtype, then FP32 m, FP32 v.
constexpr char kMagic1[4] = {'H', 'L', 'M', '1'};

struct Reader {
    std::ifstream f;
    std::int64_t pos = 0;
    template <typename T>
    T take() {
        T v{};
        f.read(reinterpret_cast<char*>(&v), sizeof v);
        if (!f) throw ConfigError("checkpoint truncated");
        pos += sizeof v;
        return v;
    }
    void bytes(void* dst, std::int64_t n) {
        f.read(static_cast<char*>(dst), n);
        if (!f) throw ConfigError("checkpoint truncated");
        pos += n;
    }
    void seek(std::int64_t to) {
        f.seekg(to);
        pos = to;
    }
};

void load_hlm1(MasterStore& store, Reader& r) {
    if (r.take<std::uint32_t>() != 1u) throw ConfigError("unsupported HLM1 version");
    const auto n_physical = r.take<std::uint32_t>();
    const auto dtype_code = r.take<std::uint32_t>();
    const auto total = r.take<std::uint64_t>();
    const auto adam_steps = r.take<std::uint64_t>();
    // the reference's checks, in its order and with its messages
    if (static_cast<i64>(n_physical) != store.physical_tiles())
        throw ConfigError("checkpoint tile count does not match the model");
    if (dtype_code != static_cast<std::uint32_t>(store.dtype()))
        throw ConfigError("checkpoint dtype does not match the store");
    if (static_cast<i64>(total) != store.total_params())
        throw ConfigError("checkpoint parameter count does not match the model");
    std::vector<std::uint64_t> n(n_physical);
    for (auto& x : n) x = r.take<std::uint64_t>();
    const auto n_logical = r.take<std::uint32_t>();
    if (static_cast<i64>(n_logical) != store.logical_tiles())
        throw ConfigError("checkpoint alias table does not match the model");
    for (std::uint32_t l = 0; l < n_logical; ++l)
        if (static_cast<i64>(r.take<std::uint32_t>()) != store.physical_index(static_cast<i64>(l)))
            throw ConfigError("checkpoint alias table does not match the model");
    const bool bf16 = store.dtype() == Dtype::BF16;
    const std::int64_t e = bf16 ? 2 : 4;
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        LayerTile& t = store.physical(p);
        const i64 np = t.n_params();
        if (static_cast<i64>(n[static_cast<size_t>(p)]) != np)
            throw ConfigError("checkpoint tile geometry does not match the model");
        r.seek((r.pos + kAlign - 1) / kAlign * kAlign);
        if (bf16) {
            // the reference BF16 tile holds the rounded weights: master = that value exactly
            std::vector<std::uint16_t> w(static_cast<size_t>(np));
            r.bytes(w.data(), 2 * np);
            for (i64 i = 0; i < np; ++i) t.master()[i] = f32_from_bf16_bits(w[static_cast<size_t>(i)]);
        } else {
            r.bytes(t.master(), 4 * np);
        }
        // grads: the reference's last-step scratch; a resumed step rewrites them first
        r.seek(r.pos + e * np);
        r.bytes(t.moment_m(), 4 * np);
        r.bytes(t.moment_v(), 4 * np);
        if (t.has_grads()) std::memset(t.grads(), 0, static_cast<size_t>(np) * 4);
    }
    store.repack_shadow();
    store.set_adam_steps(static_cast<i64>(adam_steps));
    store.bump_epoch();
}

}  // namespace

void save_checkpoint_hlm1(const MasterStore& store, const std::string& path) {
    store.quiesce();
    if (store.device_newer() > 0)
        throw ProtocolError("save_checkpoint_hlm1: an engine holds HBM-resident tiles newer than the store; "
                            "call Engine::sync() first");
    std::vector<char> header;
    auto put = [&](const void* p, size_t n) {
        header.insert(header.end(), static_cast<const char*>(p), static_cast<const char*>(p) + n);
    };
    auto u32 = [&](std::uint32_t v) { put(&v, 4); };
    auto u64 = [&](std::uint64_t v) { put(&v, 8); };
    put(kMagic1, 4);
    u32(1u);
    u32(static_cast<std::uint32_t>(store.physical_tiles()));
    u32(static_cast<std::uint32_t>(store.dtype()));
    u64(static_cast<std::uint64_t>(store.total_params()));
    u64(static_cast<std::uint64_t>(store.adam_steps()));
    for (i64 p = 0; p < store.physical_tiles(); ++p) u64(static_cast<std::uint64_t>(store.physical(p).n_params()));
    u32(static_cast<std::uint32_t>(store.logical_tiles()));
    for (i64 l = 0; l < store.logical_tiles(); ++l) u32(static_cast<std::uint32_t>(store.physical_index(l)));
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw ConfigError("cannot open checkpoint file for writing: " + path);
    f.write(header.data(), static_cast<std::streamsize>(header.size()));
    std::int64_t written = static_cast<std::int64_t>(header.size());
    const std::vector<char> pad(kAlign, 0);
    const bool bf16 = store.dtype() == Dtype::BF16;
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        const std::int64_t aligned = (written + kAlign - 1) / kAlign * kAlign;
        if (aligned > written) f.write(pad.data(), aligned - written);
        written = aligned;
        const LayerTile& t = store.physical(p);
        const i64 np = t.n_params();
        const float* g = t.grads_or_null();
        if (bf16) {
            // weights as the reference BF16 store holds them: RNE(master) = the shadow
            f.write(reinterpret_cast<const char*>(t.shadow()), 2 * np);
            std::vector<std::uint16_t> gb(static_cast<size_t>(np), 0);
            if (g)
                for (i64 i = 0; i < np; ++i) gb[static_cast<size_t>(i)] = bf16_bits_from_f32(g[i]);
            f.write(reinterpret_cast<const char*>(gb.data()), 2 * np);
            written += 4 * np;
        } else {
            f.write(reinterpret_cast<const char*>(t.master()), 4 * np);
            if (g) {
                f.write(reinterpret_cast<const char*>(g), 4 * np);
            } else {
                const std::vector<float> z(static_cast<size_t>(np), 0.0f);
                f.write(reinterpret_cast<const char*>(z.data()), 4 * np);
            }
            written += 8 * np;
        }
        f.write(reinterpret_cast<const char*>(t.moment_m()), 8 * np);   // m, v contiguous
        written += 8 * np;
    }
    if (!f) throw ConfigError("checkpoint write failed: " + path);
}

void load_checkpoint(MasterStore& store, const std::string& path) {
    store.quiesce();   // no late tail update of an attached engine may overwrite the load
    {
        Reader r;
        r.f.open(path, std::ios::binary);
        if (!r.f) throw ConfigError("cannot open checkpoint file: " + path);
        char magic[4] = {};
        r.f.read(magic, 4);
        r.pos = 4;
        if (r.f && std::memcmp(magic, kMagic1, 4) == 0) return load_hlm1(store, r);
    }
    std::ifstream f(path, std::ios::binary);
    if (!f) throw ConfigError("cannot open checkpoint file: " + path);
    Header h{};
    f.read(reinterpret_cast<char*>(&h), sizeof h);
    if (!f || std::memcmp(h.magic, kMagic, 4) != 0) throw ConfigError("not an HLM2 or HLM1 checkpoint: " + path);
    if (h.version != kVersion) throw ConfigError("unsupported HLM2 version " + std::to_string(h.version));
    std::int64_t dims[8];
    fill_dims(store.config(), dims);
    if (std::memcmp(dims, h.dims, sizeof dims) != 0 ||
        h.physical_tiles != static_cast<std::uint32_t>(store.physical_tiles()) ||
        h.logical_tiles != static_cast<std::uint32_t>(store.logical_tiles()) ||
        h.total_params != static_cast<std::uint64_t>(store.total_params()))
        throw ConfigError("checkpoint geometry does not match the store");
    std::int64_t read = sizeof h;
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        std::uint64_t n = 0;
        f.read(reinterpret_cast<char*>(&n), sizeof n);
        read += sizeof n;
        if (!f || n != static_cast<std::uint64_t>(store.physical(p).n_params()))
            throw ConfigError("checkpoint tile " + std::to_string(p) + " size mismatch");
    }
    for (i64 p = 0; p < store.physical_tiles(); ++p) {
        const std::int64_t aligned = (read + kAlign - 1) / kAlign * kAlign;
        f.seekg(aligned);
        read = aligned;
        LayerTile& t = store.physical(p);
        const std::int64_t bytes = 12 * t.n_params();
        f.read(reinterpret_cast<char*>(t.master()), bytes);
        if (!f) throw ConfigError("checkpoint truncated in tile " + std::to_string(p));
        read += bytes;
        if (t.has_grads()) std::memset(t.grads(), 0, static_cast<size_t>(t.n_params()) * 4);
    }
    store.repack_shadow();
    store.set_adam_steps(static_cast<i64>(h.adam_steps));
    store.bump_epoch();   // engines holding HBM-resident tiles re-upload them
}

}  // inline namespace b200
}  // namespace hlm
