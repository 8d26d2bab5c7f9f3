// HLM2 checkpoint (see include/hlm/checkpoint.hpp).
#include "hlm/checkpoint.hpp"

#include <cstdint>
#include <cstring>
#include <fstream>
#include <vector>

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

void load_checkpoint(MasterStore& store, const std::string& path) {
    store.quiesce();   // no late tail update of an attached engine may overwrite the load
    std::ifstream f(path, std::ios::binary);
    if (!f) throw ConfigError("cannot open checkpoint file: " + path);
    Header h{};
    f.read(reinterpret_cast<char*>(&h), sizeof h);
    if (!f || std::memcmp(h.magic, kMagic, 4) != 0) throw ConfigError("not an HLM2 checkpoint: " + path);
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
